"""Pins for the oracle's prune/inflate, MCL loop and cluster extraction.

O2/O3 pins: the hand examples of tests/golden/prune_examples.json (SPEC examples
and the reading-derived SURVEY §8(c) c.3 examples), invariants (|kept| <= max(S,R),
argmax kept, columns sum to 1, values in (0,1]), and an independent top-K check by
numpy lexsort.  O4/O5 pins: identity and disjoint-clique fixed points, the planted
partition (C1) and the clique graph (C2) recovered exactly, idempotence at
convergence, scipy's connected_components.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

import oracle as O
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "prune_examples.json")))


def _col(vals):
    v = np.asarray(vals, np.float64)
    return O.Mat(len(v), 1, np.array([0, len(v)], np.int64), np.arange(len(v), dtype=np.int32), v)


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_prune_golden(case):
    A, info = O.prune_inflate(_col(case["col"]), case["theta"], case["S"], case["R"],
                              case["pct"], case["r"])
    assert A.rows.tolist() == case["rows"]
    np.testing.assert_allclose(A.vals, case["vals"], rtol=1e-12)
    assert int(info.branch[0]) == case["branch"]
    if "chaos" in case:
        assert abs(info.chaos[0] - case["chaos"]) <= case.get("chaos_tol", 1e-12)


def _random_columns(seed, ncols=200):
    rng = np.random.default_rng(seed)
    cnt = rng.integers(0, 60, size=ncols)
    cnt[::17] = 0
    cp = np.zeros(ncols + 1, np.int64)
    np.cumsum(cnt, out=cp[1:])
    rows, vals = [], []
    for c in cnt:
        rows.append(np.sort(rng.choice(500, size=int(c), replace=False)))
        v = rng.exponential(1.0, size=int(c)) ** 3
        if c and rng.random() < 0.3:       # plant exact ties
            v[: c // 2] = v[0]
        vals.append(v / max(v.sum(), 1e-300))
    return O.Mat(500, ncols, cp, np.concatenate(rows).astype(np.int32), np.concatenate(vals))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("params", [(1e-2, 5, 8, 0.9), (1e-3, 20, 0, 0.9), (0.05, 3, 30, 0.5),
                                    (0.0, 1000, 0, 0.9)])
def test_prune_invariants_and_topk(seed, params):
    theta, S, R, pct = params
    Cm = _random_columns(seed)
    A, info = O.prune_inflate(Cm, theta, S, R, pct, 2.0)
    for j in range(Cm.ncols):
        r = Cm.rows[Cm.colptr[j]:Cm.colptr[j + 1]]
        v = Cm.vals[Cm.colptr[j]:Cm.colptr[j + 1]]
        kr = A.rows[A.colptr[j]:A.colptr[j + 1]]
        kv = A.vals[A.colptr[j]:A.colptr[j + 1]]
        if len(v) == 0:
            assert len(kr) == 0
            continue
        assert len(kr) <= max(S, R, 1)
        assert r[np.argmax(v)] in kr or np.sum(v == v.max()) > 1
        np.testing.assert_allclose(kv.sum(), 1.0, atol=1e-12)
        assert np.all(kv > 0) and np.all(kv <= 1.0)
        assert np.all(np.diff(kr) > 0)
        # independent top-K: order by (value desc, row asc) with numpy lexsort
        order = np.lexsort((r, -v))
        m = int((v >= theta).sum())
        s = float(v[v >= theta].sum())
        if m > S:
            K = S
        elif R > 0 and m < R and s < pct and len(v) > m:
            K = min(R, len(v))
        elif m > 0:
            K = m
        else:
            K = 1
        assert sorted(r[order[:K]].tolist()) == kr.tolist()
        w = v[order[:K]] / v[order[:K]].sum()
        np.testing.assert_allclose(np.sort(kv), np.sort(w ** 2 / (w ** 2).sum()), rtol=1e-12)


def _cols(A):
    return [(A.rows[A.colptr[j]:A.colptr[j + 1]], A.vals[A.colptr[j]:A.colptr[j + 1]])
            for j in range(A.ncols)]


@pytest.mark.parametrize("seed", range(4))
def test_prune_branch_properties(seed):
    """Properties of the prune branches (readings Q5-Q8) that do not restate the branch rule:
    each would catch a flipped comparison, a swapped S / R, or a dropped branch."""
    Cm = _random_columns(seed)
    cols = _cols(Cm)
    # threshold only (S large, no recovery): kept = exactly the entries >= theta, or the
    # single largest entry when none reaches theta (Q8)
    A, _ = O.prune_inflate(Cm, 1e-2, 10 ** 6, 0, 0.9, 2.0)
    for (r, v), (kr, _) in zip(cols, _cols(A)):
        if len(v) == 0:
            continue
        if (v >= 1e-2).any():
            assert kr.tolist() == r[v >= 1e-2].tolist()
        else:
            assert len(kr) == 1 and v[np.searchsorted(r, kr[0])] == v.max()
    # select: growing S only ever adds entries (nested kept sets), and never more than S
    prev = None
    for S in (1, 3, 7, 15):
        A, _ = O.prune_inflate(Cm, 0.0, S, 0, 0.9, 2.0)
        ks = [set(kr.tolist()) for kr, _ in _cols(A)]
        for (r, v), k in zip(cols, ks):
            assert len(k) == min(S, len(v))
        if prev is not None:
            assert all(a <= b for a, b in zip(prev, ks))
        prev = ks
    # every kept entry is >= every dropped one (a top set, whatever the branch)
    for params in [(1e-2, 5, 8, 0.9), (0.05, 3, 30, 0.5), (1e-3, 2, 0, 0.9)]:
        A, _ = O.prune_inflate(Cm, *params, 2.0)
        for (r, v), (kr, _) in zip(cols, _cols(A)):
            keep = np.isin(r, kr)
            if keep.any() and (~keep).any():
                assert v[keep].min() >= v[~keep].max()
    # recovery: with a threshold above every entry and mass below pct, recovery keeps
    # min(R, nnz) entries; with R = 0 the same columns keep one entry
    A, _ = O.prune_inflate(Cm, 2.0, 10, 4, 1.0, 2.0)
    B, _ = O.prune_inflate(Cm, 2.0, 10, 0, 1.0, 2.0)
    for (r, v), (ka, _), (kb, _) in zip(cols, _cols(A), _cols(B)):
        if len(v):
            assert len(ka) == min(4, len(v)) and len(kb) == 1
    # scale invariance: multiplying a column by c and theta, pct by c leaves A' unchanged
    c = 8.0
    Cs = O.Mat(Cm.nrows, Cm.ncols, Cm.colptr, Cm.rows, Cm.vals * c)
    A1, _ = O.prune_inflate(Cm, 1e-2, 5, 8, 0.6, 2.0)
    A2, _ = O.prune_inflate(Cs, 1e-2 * c, 5, 8, 0.6 * c, 2.0)
    assert np.array_equal(A1.colptr, A2.colptr) and np.array_equal(A1.rows, A2.rows)
    np.testing.assert_allclose(A1.vals, A2.vals, rtol=1e-12)


def test_max_abs_change_dense():
    """O.max_abs_change (SPEC S:484's alternative convergence measure, a logging helper)
    against dense arrays: max |A - B| with absent entries = 0."""
    for seed in range(3):
        a = synth.random_sparse(40, 30, 0.1, seed=seed)
        b = synth.random_sparse(40, 30, 0.1, seed=seed + 10)
        da, db = np.zeros((40, 30)), np.zeros((40, 30))
        for d, m in ((da, a), (db, b)):
            for j in range(30):
                for q in range(m.colptr[j], m.colptr[j + 1]):
                    d[m.rows[q], j] = m.vals[q]
        assert O.max_abs_change(O.as_mat(a), O.as_mat(b)) == pytest.approx(np.abs(da - db).max(), abs=0)


def test_identity_fixed_point():
    n = 50
    I = synth.Csc(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32),
                  np.ones(n, np.float32))
    res = O.mcl(I, A0=O.as_mat(I))
    assert res.iterations == 1 and res.chaos[0] == 0.0
    assert res.nclusters == n and res.labels.tolist() == list(range(n))


def test_disjoint_cliques_fixed_point():
    # unit-weight cliques with loops: A = blockdiag(J/m); A.A = A, prune keeps all,
    # inflation keeps the uniform column -> A' = A, chaos 0, clusters = cliques
    sizes = [3, 5, 1, 8, 2]
    ii, jj = [], []
    st = 0
    for s in sizes:
        a, b = np.triu_indices(s, 1)
        ii.append(a + st)
        jj.append(b + st)
        st += s
    n = st
    G = synth.pairs_to_symmetric_csc(n, np.concatenate(ii), np.concatenate(jj),
                                     np.ones(sum(len(x) for x in ii)))
    A0 = O.preprocess(G)
    res = O.mcl(G)
    assert res.iterations == 1 and res.chaos[0] < 1e-15
    np.testing.assert_allclose(res.A.dense(), A0.dense(), atol=1e-15)
    expect = np.repeat(np.arange(len(sizes)), sizes)
    assert res.labels.tolist() == expect.tolist()


def test_block_diagonal_preserved():
    g1 = synth.random_sparse(20, 20, 0.3, seed=1)
    g2 = synth.random_sparse(15, 15, 0.3, seed=2)
    D = sp.block_diag([sp.csc_matrix((g.vals, g.rows, g.colptr), shape=(g.nrows, g.ncols))
                       for g in (g1, g2)]).tocsc()
    D = D + D.T
    D = sp.csc_matrix(D)
    D.sort_indices()
    G = synth.Csc(35, 35, D.indptr.astype(np.int64), D.indices.astype(np.int32),
                  D.data.astype(np.float32))
    A = O.preprocess(G)
    for _ in range(3):
        Cm, _ = O.expand(A)
        A, _ = O.prune_inflate(Cm, 1e-4, 1100, 1400, 0.9)
        d = A.dense()
        assert np.all(d[:20, 20:] == 0) and np.all(d[20:, :20] == 0)


def test_c1_planted_partition_recovered():
    G, truth = synth.planted_partition(return_truth=True)
    res = O.mcl(G, theta=1e-4, S=1100, R=1400, pct=0.9, eps=1e-3)
    assert res.nclusters == 20
    # the partition equals the planted blocks
    assert len(set(zip(res.labels.tolist(), truth.tolist()))) == 20
    # idempotence at convergence (SURVEY c.3 O4): one more step moves A_f by <= 1e-6
    Cm, _ = O.expand(res.A)
    A2, _ = O.prune_inflate(Cm, 1e-4, 1100, 1400, 0.9)
    assert O.max_abs_change(res.A, A2) <= 1e-6
    assert O.clusters(A2)[0].tolist() == res.labels.tolist()
    # column sums after every normalisation
    np.testing.assert_allclose(np.add.reduceat(res.A.vals, res.A.colptr[:-1]), 1.0, atol=1e-12)


@pytest.mark.slow
def test_c2_cliques_recovered():
    G, truth = synth.cliques_noise(return_truth=True)
    res = O.mcl(G, theta=1e-4, S=100, R=100, pct=0.9, eps=1e-3)
    assert res.nclusters == 106
    assert len(set(zip(res.labels.tolist(), truth.tolist()))) == 106


@pytest.mark.parametrize("seed", range(5))
def test_clusters_match_scipy(seed):
    M = synth.random_sparse(300, 300, 0.004, seed=seed, empty_cols=0.2)
    labels, ncl = O.clusters(M)
    S = sp.csc_matrix((np.ones(M.nnz), M.rows, M.colptr), shape=(300, 300))
    k, lab = connected_components(S, directed=True, connection="weak")
    assert k == ncl
    # same partition
    assert len(set(zip(labels.tolist(), lab.tolist()))) == k
    # canonical: labels appear in order of each component's smallest vertex
    first = [int(np.nonzero(labels == c)[0][0]) for c in range(ncl)]
    assert first == sorted(first)


def test_clusters_spec_examples():
    n = 4
    I = O.Mat(n, n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n))
    lab, k = O.clusters(I)
    assert k == 4 and lab.tolist() == [0, 1, 2, 3]
    P = O.Mat(n, n, np.arange(n + 1, dtype=np.int64), np.array([1, 2, 3, 0], np.int32), np.ones(n))
    assert O.clusters(P)[1] == 1


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("nblocks", [2, 3, 7])
def test_kept_set_within_row_block_candidates(seed, nblocks):
    """The reading behind the split parts' candidates and the fused 2D SUMMA:
    cut a column's rows into blocks and keep each block's top-max(S, R) entries by (value
    desc, row asc); the oracle's kept set lies in their union for every branch.  Random
    columns with planted ties; block boundaries random."""
    rng = np.random.default_rng(100 + seed)
    Cm = _random_columns(seed)
    for theta, S, R, pct in [(1e-2, 5, 8, 0.9), (0.05, 3, 30, 0.5), (1e-3, 2, 0, 0.9),
                             (0.0, 1, 0, 0.9), (0.2, 4, 4, 0.99)]:
        A, _ = O.prune_inflate(Cm, theta, S, R, pct, 2.0)
        kmax = max(S, R, 1)
        cuts = np.sort(rng.choice(np.arange(1, Cm.nrows), size=nblocks - 1, replace=False))
        bounds = np.concatenate([[0], cuts, [Cm.nrows]])
        for (r, v), (kr, _) in zip(_cols(Cm), _cols(A)):
            cand = set()
            for b0, b1 in zip(bounds[:-1], bounds[1:]):
                sel = (r >= b0) & (r < b1)
                rb, vb = r[sel], v[sel]
                cand |= set(rb[np.lexsort((rb, -vb))[:kmax]].tolist())
            assert set(kr.tolist()) <= cand
