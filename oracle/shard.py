"""Column-sharded runs of the oracle over host cores (TEST INFRASTRUCTURE ONLY, like the
rest of oracle/).

SURVEY.md §8(c) c.5 / §8(d) d.5: O1-O3 are column-local given A_t, so an iteration's output
columns may be split into [b, e) ranges, each computed by an independent single-threaded
oracle process (forked workers calling the same C functions on the same inputs), and
concatenated in order (chaos = max).  The result is identical, entry for entry, to one
single-threaded run; only the wall time changes.  Nothing here does arithmetic of the
method: it only cuts ranges, forks and concatenates.
"""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

from . import Mat, expand, prune_inflate, spgemm

_A = None       # the iterate the workers read (inherited through fork, never written)
_PRM = None


def _ranges(n: int, flops: np.ndarray, pieces: int):
    """Column ranges of near-equal oracle work (flops + nnz proxy)."""
    w = flops.astype(np.float64) + 1.0
    cum = np.cumsum(w)
    cuts = np.searchsorted(cum, np.linspace(0, cum[-1], pieces + 1)[1:-1])
    b = np.unique(np.concatenate([[0], cuts, [n]]))
    return [(int(b[i]), int(b[i + 1])) for i in range(len(b) - 1) if b[i + 1] > b[i]]


def _flops(A) -> np.ndarray:
    """flops_j = sum_{k in A_*j} nnz(A_*k): integer counting, no method arithmetic
    beyond the definition (used only to balance the shards)."""
    deg = np.diff(A.colptr)
    return np.add.reduceat(np.concatenate([deg[A.rows].astype(np.int64), [0]]),
                           np.minimum(A.colptr[:-1], A.rows.size)) * (deg > 0)


def _w_step(rng):
    b, e = rng
    C, fl = expand(_A, b, e)
    An, info = prune_inflate(C, *_PRM, 2.0)
    return b, np.diff(An.colptr), An.rows, An.vals, float(info.chaos.max()) if info.chaos.size else 0.0


def _w_nnz(rng):
    b, e = rng
    out = []
    fl = []
    step = max(1, min(e - b, 4096))
    for s in range(b, e, step):
        C, f = expand(_A, s, min(e, s + step))
        out.append(np.diff(C.colptr))
        fl.append(f)
        del C
    return b, np.concatenate(out), np.concatenate(fl)


def _pool(nproc):
    return mp.get_context("fork").Pool(nproc)


def sharded_step(A, prm, nproc):
    """One MCL iteration (expand + prune/inflate) of the oracle, sharded by columns."""
    global _A, _PRM
    _A, _PRM = A, prm
    rng = _ranges(A.ncols, _flops(A), nproc * 24)
    parts = {}
    with _pool(nproc) as p:
        for b, cnt, rows, vals, ch in p.imap_unordered(_w_step, rng):
            parts[b] = (cnt, rows, vals, ch)
    keys = sorted(parts)
    cnt = np.concatenate([parts[k][0] for k in keys])
    cp = np.zeros(A.ncols + 1, np.int64)
    np.cumsum(cnt, out=cp[1:])
    rows = np.concatenate([parts[k][1] for k in keys])
    vals = np.concatenate([parts[k][2] for k in keys])
    chaos = max(parts[k][3] for k in keys) if keys else 0.0
    _A = None
    return Mat(A.nrows, A.ncols, cp, rows, vals), chaos


def sharded_nnz(A, nproc):
    global _A
    _A = A
    rng = _ranges(A.ncols, _flops(A), nproc * 32)
    parts = {}
    with _pool(nproc) as p:
        for b, cnt, fl in p.imap_unordered(_w_nnz, rng):
            parts[b] = (cnt, fl)
    keys = sorted(parts)
    _A = None
    return (np.concatenate([parts[k][0] for k in keys]).astype(np.int64),
            np.concatenate([parts[k][1] for k in keys]).astype(np.int64))




def _w_cols(rng):
    b, e = rng
    B = _PRM
    C, fl = spgemm(_A, B, b, e)
    return b, C.colptr, C.rows, C.vals, fl


def sharded_spgemm(A, B, nproc=None):
    """C = A * B by column shards of B (O1); returns (Mat, flops per column)."""
    global _A, _PRM
    nproc = nproc or os.cpu_count() or 1
    _A, _PRM = A, B
    deg = np.diff(A.colptr)
    w = np.zeros(B.ncols, np.float64)
    cols = np.repeat(np.arange(B.ncols), np.diff(B.colptr))
    np.add.at(w, cols, deg[B.rows])
    rng = _ranges(B.ncols, w, nproc * 8)
    parts = {}
    with _pool(nproc) as p:
        for b, cp, rows, vals, fl in p.imap_unordered(_w_cols, rng):
            parts[b] = (np.diff(cp), rows, vals, fl)
    keys = sorted(parts)
    _A = _PRM = None
    cnt = np.concatenate([parts[k][0] for k in keys]) if keys else np.zeros(0, np.int64)
    cp = np.zeros(B.ncols + 1, np.int64)
    np.cumsum(cnt, out=cp[1:])
    rows = np.concatenate([parts[k][1] for k in keys]) if keys else np.zeros(0, np.int32)
    vals = np.concatenate([parts[k][2] for k in keys]) if keys else np.zeros(0)
    fl = np.concatenate([parts[k][3] for k in keys]) if keys else np.zeros(0, np.int64)
    return Mat(A.nrows, B.ncols, cp, rows, vals), fl


def sharded_mcl_iterates(A, prm, its, nproc=None):
    """`its` oracle MCL iterations of A (expand + prune/inflate), column-sharded."""
    nproc = nproc or os.cpu_count() or 1
    for _ in range(its):
        A, _ = sharded_step(A, prm, nproc)
    return A
