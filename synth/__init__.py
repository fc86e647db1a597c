"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no products, no normalisation,
no pruning): it only draws graphs and sparse matrices from seeded numpy
``default_rng`` streams and lays them out as CSC arrays.  Both sides of every
parity check receive the arrays produced here; the oracle (``oracle/``) and the
CUDA path (``paper_2002_10083_b200``) each turn them into the column-stochastic
A_0 of Alg. 1 line 1 themselves.

Recipes follow SURVEY.md §8(d) d.2 (configs C1..C5, BASELINE.json ``configs``).
Every graph is symmetric, weighted, without self-loops, without duplicate
edges (the first draw of an unordered pair wins), and its vertex ids are
randomly permuted with the config's seed so file order carries no locality.
Weights are drawn as float32 so that the fp32 GPU path and the fp64 oracle see
bit-identical inputs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "Csc",
    "pairs_to_symmetric_csc",
    "planted_partition",
    "cliques_noise",
    "protein_like",
    "rmat",
    "random_sparse",
    "config_graph",
    "CONFIGS",
]


@dataclass
class Csc:
    """A CSC matrix: ``colptr`` int64[ncols+1], ``rows`` int32[nnz] (strictly
    increasing inside each column), ``vals`` float32[nnz]."""

    nrows: int
    ncols: int
    colptr: np.ndarray
    rows: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.colptr[-1])

    def col(self, j: int):
        a, b = int(self.colptr[j]), int(self.colptr[j + 1])
        return self.rows[a:b], self.vals[a:b]

    def slice_cols(self, b: int, e: int) -> "Csc":
        a0, a1 = int(self.colptr[b]), int(self.colptr[e])
        return Csc(self.nrows, e - b, (self.colptr[b:e + 1] - a0).astype(np.int64),
                   self.rows[a0:a1].copy(), self.vals[a0:a1].copy())


def _coo_to_csc(nrows: int, ncols: int, r: np.ndarray, c: np.ndarray, v: np.ndarray) -> Csc:
    """Sort (row, col, val) triples into CSC.  Triples must be unique (no summation here)."""
    key = c.astype(np.int64) * np.int64(nrows) + r.astype(np.int64)
    order = np.argsort(key, kind="stable")
    r = r[order].astype(np.int32)
    c = c[order].astype(np.int64)
    v = v[order].astype(np.float32)
    counts = np.bincount(c, minlength=ncols).astype(np.int64)
    colptr = np.zeros(ncols + 1, dtype=np.int64)
    np.cumsum(counts, out=colptr[1:])
    return Csc(nrows, ncols, colptr, r, v)


def pairs_to_symmetric_csc(n: int, i: np.ndarray, j: np.ndarray, w: np.ndarray,
                           perm: np.ndarray | None = None) -> Csc:
    """Unordered pairs -> symmetric CSC.  Self pairs dropped; for a repeated
    unordered pair the FIRST occurrence (in array order) is kept, its weight
    mirrored to both triangles.  ``perm`` (old id -> new id) relabels vertices."""
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    w = np.asarray(w, dtype=np.float32)
    keep = i != j
    i, j, w = i[keep], j[keep], w[keep]
    lo = np.minimum(i, j)
    hi = np.maximum(i, j)
    key = lo * np.int64(n) + hi
    _, first = np.unique(key, return_index=True)
    lo, hi, w = lo[first], hi[first], w[first]
    if perm is not None:
        lo, hi = perm[lo], perm[hi]
    r = np.concatenate([lo, hi])
    c = np.concatenate([hi, lo])
    v = np.concatenate([w, w])
    return _coo_to_csc(n, n, r, c, v)


def _u(rng, lo, hi, size):
    return rng.uniform(lo, hi, size=size).astype(np.float32)


def planted_partition(n: int = 1000, blocks: int = 20, p_in: float = 18 / 49,
                      p_out: float = 2 / 950, seed: int = 1, return_truth: bool = False):
    """C1: ``blocks`` equal blocks; each unordered pair is an edge
    with probability p_in inside a block and p_out across; weights U[0.5,1.0)
    intra, U[0.05,0.30) inter; ids randomly permuted."""
    rng = np.random.default_rng(seed)
    bs = n // blocks
    iu, ju = np.triu_indices(n, k=1)
    same = (iu // bs) == (ju // bs)
    p = np.where(same, p_in, p_out)
    hit = rng.random(iu.shape[0]) < p
    iu, ju, same = iu[hit], ju[hit], same[hit]
    w = np.where(same, _u(rng, 0.5, 1.0, iu.shape[0]), _u(rng, 0.05, 0.30, iu.shape[0]))
    perm = rng.permutation(n)
    g = pairs_to_symmetric_csc(n, iu, ju, w, perm)
    if not return_truth:
        return g
    truth = np.empty(n, dtype=np.int64)
    truth[perm] = np.arange(n) // bs
    return g, truth


def cliques_noise(n: int = 20000, clique: int = 190, noise_per_vertex: float = 10.0,
                  seed: int = 2, return_truth: bool = False):
    """C2: consecutive cliques of ``clique`` vertices (the last one shorter), clique
    weights U[0.5,1.0); Poisson(noise_per_vertex*n/2) uniform random pairs with
    weights U[0.01,0.25); ids randomly permuted."""
    rng = np.random.default_rng(seed)
    starts = np.arange(0, n, clique)
    sizes = np.minimum(clique, n - starts)
    ii, jj = [], []
    for s in np.unique(sizes):
        st = starts[sizes == s]
        a, b = np.triu_indices(int(s), k=1)
        ii.append((st[:, None] + a[None, :]).ravel())
        jj.append((st[:, None] + b[None, :]).ravel())
    ci = np.concatenate(ii)
    cj = np.concatenate(jj)
    cw = _u(rng, 0.5, 1.0, ci.shape[0])
    m = rng.poisson(noise_per_vertex * n / 2)
    ni = rng.integers(0, n, size=m)
    nj = rng.integers(0, n, size=m)
    nw = _u(rng, 0.01, 0.25, m)
    perm = rng.permutation(n)
    g = pairs_to_symmetric_csc(n, np.concatenate([ci, ni]), np.concatenate([cj, nj]),
                               np.concatenate([cw, nw]), perm)
    if not return_truth:
        return g
    truth = np.empty(n, dtype=np.int64)
    truth[perm] = np.arange(n) // clique
    return g, truth


def protein_like(n: int = 500_000, zipf_a: float = 2.1, fam_cap: int = 2000,
                 complete_max: int = 257, draw_k: int = 128, super_size: int = 10,
                 super_mean: float = 10.0, uniform_mean: float = 2.0, seed: int = 3,
                 permute: bool = True) -> Csc:
    """C3/C5 protein-similarity-like graph.

    Family sizes ~ Zipf(zipf_a) capped at ``fam_cap``.  Intra-family: complete if
    size <= complete_max, else every vertex draws ``draw_k`` in-family partners;
    weights U[0.3,1.0).  Superfamilies of ``super_size`` consecutive families:
    Poisson(super_mean) partners per vertex inside the superfamily, U[0.05,0.4).
    Plus Poisson(uniform_mean) uniform partners per vertex, U[0.01,0.2).
    ``permute=False`` keeps vertices numbered family by family (labels with locality)."""
    rng = np.random.default_rng(seed)
    sizes = []
    tot = 0
    while tot < n:
        s = np.minimum(rng.zipf(zipf_a, size=max(1024, (n - tot) // 4)), fam_cap)
        cs = np.cumsum(s)
        k = int(np.searchsorted(cs, n - tot, side="left"))
        if k < s.shape[0]:
            s = s[:k + 1].copy()
            s[-1] -= int(cs[k] - (n - tot))
            s = s[s > 0]
        sizes.append(s)
        tot += int(s.sum())
    sizes = np.concatenate(sizes).astype(np.int64)
    starts = np.zeros_like(sizes)
    np.cumsum(sizes[:-1], out=starts[1:])
    fam_of = np.repeat(np.arange(sizes.shape[0]), sizes)

    ii, jj = [], []
    small = sizes <= complete_max
    for s in np.unique(sizes[small]):
        if s < 2:
            continue
        st = starts[small & (sizes == s)]
        a, b = np.triu_indices(int(s), k=1)
        ii.append((st[:, None] + a[None, :]).ravel())
        jj.append((st[:, None] + b[None, :]).ravel())
    big = np.nonzero(~small)[0]
    for f in big:
        st, s = int(starts[f]), int(sizes[f])
        v = np.repeat(np.arange(st, st + s), draw_k)
        ii.append(v)
        jj.append(st + rng.integers(0, s, size=v.shape[0]))
    fi = np.concatenate(ii) if ii else np.zeros(0, np.int64)
    fj = np.concatenate(jj) if jj else np.zeros(0, np.int64)
    fw = _u(rng, 0.3, 1.0, fi.shape[0])

    sf = np.arange(sizes.shape[0]) // super_size
    nsf = int(sf[-1]) + 1
    sf_start = np.full(nsf, np.iinfo(np.int64).max)
    np.minimum.at(sf_start, sf, starts)
    sf_size = np.bincount(sf, weights=sizes, minlength=nsf).astype(np.int64)
    cnt = rng.poisson(super_mean, size=n)
    sv = np.repeat(np.arange(n), cnt)
    ssf = sf[fam_of[sv]]
    sj = sf_start[ssf] + (rng.random(sv.shape[0]) * sf_size[ssf]).astype(np.int64)
    sw = _u(rng, 0.05, 0.4, sv.shape[0])

    cnt = rng.poisson(uniform_mean, size=n)
    uv = np.repeat(np.arange(n), cnt)
    uj = rng.integers(0, n, size=uv.shape[0])
    uw = _u(rng, 0.01, 0.2, uv.shape[0])

    perm = rng.permutation(n)
    return pairs_to_symmetric_csc(n, np.concatenate([fi, sv, uv]), np.concatenate([fj, sj, uj]),
                                  np.concatenate([fw, sw, uw]), perm if permute else None)


def rmat(scale: int = 22, edge_factor: int = 32, a: float = 0.57, b: float = 0.19,
         c: float = 0.19, seed: int = 4, chunk: int = 1 << 24) -> Csc:
    """C4: Graph500-style R-MAT (a,b,c,d = 0.57,0.19,0.19,0.05), edge_factor*2^scale
    draws, symmetrised, deduplicated, loops dropped, ids permuted; weights U[0.05,1.0)."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edge_factor * n
    I, J = [], []
    done = 0
    while done < m:
        k = min(chunk, m - done)
        i = np.zeros(k, dtype=np.int64)
        j = np.zeros(k, dtype=np.int64)
        for _ in range(scale):
            u = rng.random(k)
            bi = (u >= a + b).astype(np.int64)          # quadrants c,d -> row bit
            bj = (((u >= a) & (u < a + b)) | (u >= a + b + c)).astype(np.int64)
            i = (i << 1) | bi
            j = (j << 1) | bj
        I.append(i)
        J.append(j)
        done += k
    i = np.concatenate(I)
    j = np.concatenate(J)
    w = _u(rng, 0.05, 1.0, i.shape[0])
    perm = rng.permutation(n)
    return pairs_to_symmetric_csc(n, i, j, w, perm)


def random_sparse(nrows: int, ncols: int, density: float, seed: int,
                  empty_cols: float = 0.0, lo: float = 0.01, hi: float = 1.0,
                  degree_skew: bool = False) -> Csc:
    """A general (non-symmetric) sparse matrix with positive float32 values, for
    kernel parity on ragged shapes.  ``empty_cols`` is the fraction of forced-empty
    columns; ``degree_skew`` draws per-column counts from a heavy tail."""
    rng = np.random.default_rng(seed)
    if degree_skew:
        cnt = np.minimum(rng.zipf(1.8, size=ncols) * max(1, int(density * nrows) // 4), nrows)
    else:
        cnt = rng.binomial(nrows, density, size=ncols)
    if empty_cols > 0:
        cnt[rng.random(ncols) < empty_cols] = 0
    cols = np.repeat(np.arange(ncols, dtype=np.int64), cnt)
    rows = np.concatenate([rng.choice(nrows, size=int(k), replace=False) for k in cnt]) \
        if cnt.sum() else np.zeros(0, np.int64)
    vals = _u(rng, lo, hi, rows.shape[0])
    return _coo_to_csc(nrows, ncols, rows.astype(np.int64), cols, vals)


CONFIGS = {
    "C1": dict(kind="planted_partition", seed=1, theta=1e-4, S=1100, R=1400, pct=0.9),
    "C2": dict(kind="cliques_noise", seed=2, theta=1e-4, S=100, R=100, pct=0.9),
    "C3": dict(kind="protein_like", seed=3, theta=1e-4, S=1100, R=1400, pct=0.9),
    "C4": dict(kind="rmat", seed=4, theta=1e-4, S=1100, R=1400, pct=0.9),
    "C5": dict(kind="protein_like_c5", seed=5, theta=1e-4, S=1100, R=1400, pct=0.9),
}


def config_graph(name: str, scale: float = 1.0) -> Csc:
    """The graph of config ``name`` (C1..C5).  ``scale`` < 1 shrinks C3..C5 for tests."""
    cfg = CONFIGS[name]
    if name == "C1":
        return planted_partition(seed=cfg["seed"])
    if name == "C2":
        return cliques_noise(seed=cfg["seed"])
    if name == "C3":
        return protein_like(n=int(500_000 * scale), seed=cfg["seed"])
    if name == "C4":
        s = 22 + int(round(np.log2(scale))) if scale != 1.0 else 22
        return rmat(scale=s, seed=cfg["seed"])
    if name == "C5":
        return protein_like(n=int(3_243_106 * scale), zipf_a=2.05, fam_cap=4000,
                            complete_max=261, draw_k=130, seed=cfg["seed"])
    raise KeyError(name)
