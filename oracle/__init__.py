"""The CPU oracle for the HipMCL expansion hot path (arxiv 2002.10083).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2002_10083_b200`` never imports it and
shares no code with it.

The arithmetic lives in ``mcl_oracle.c`` (plain C99, fp64, single-threaded; see
its header for the PAPER.md passage each function writes out).  This file only
marshals numpy arrays through ctypes and holds the Alg. 1 driver loop and the
Alg. 2 stack (pure control flow).

Parity status:
  spgemm / expand          pinned (dense brute force, closed forms, invariants)
  prune_inflate            pinned for threshold/select/argmax by SPEC examples and
                           hand examples; RECOVERY (R, pct) and CHAOS are
                           "parity unpinned" by the paper (readings Q7, Q9).
  preprocess, clusters     pinned (closed forms, scipy connected_components)
  cohen                    pinned (Philox known-answer vectors, unbiasedness)
  merge / binary_merge     pinned (sum-of-blocks identity, Alg. 2 trace)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mcl_oracle.c")
_LIB = os.path.join(_HERE, "liborc.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no fast-math, no OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i64, i32, f64 = C.c_int64, C.c_int32, C.c_double
        L.orc_spgemm.argtypes = [i64, i64, i64, P, P, P, P, P, P, i64, i64, P, P, P, P]
        L.orc_prune_inflate.argtypes = [i64, P, P, P, f64, i64, i64, f64, f64, P, P, P,
                                        P, P, P, P, P]
        L.orc_preprocess.argtypes = [i64, P, P, P, C.c_int, P, P, P]
        L.orc_clusters.argtypes = [i64, P, P, P, P]
        L.orc_philox.argtypes = [P, P, P]
        L.orc_philox.restype = None
        L.orc_cohen_key.argtypes = [C.c_uint64, i64, i64]
        L.orc_cohen_key.restype = C.c_float
        L.orc_cohen.argtypes = [i64, i64, i64, P, P, P, P, i32, C.c_uint64, P, P, P]
        L.orc_merge.argtypes = [i32, i64, i64, P, P, P, P, P, P]
        L.orc_free.argtypes = [P]
        L.orc_free.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class Mat:
    """An fp64 CSC matrix (the oracle's own type)."""
    nrows: int
    ncols: int
    colptr: np.ndarray  # int64
    rows: np.ndarray    # int32
    vals: np.ndarray    # float64

    @property
    def nnz(self) -> int:
        return int(self.colptr[-1])

    def dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        for j in range(self.ncols):
            a, b = self.colptr[j], self.colptr[j + 1]
            d[self.rows[a:b], j] = self.vals[a:b]
        return d


def as_mat(m) -> Mat:
    """Any object with nrows/ncols/colptr/rows/vals -> Mat (values promoted to fp64)."""
    return Mat(int(m.nrows), int(m.ncols), np.ascontiguousarray(m.colptr, np.int64),
               np.ascontiguousarray(m.rows, np.int32), np.ascontiguousarray(m.vals, np.float64))


def _take(ncols: int, nrows: int, pcp, prow, pval) -> Mat:
    L = lib()
    cp = np.ctypeslib.as_array(C.cast(pcp, C.POINTER(C.c_int64)), shape=(ncols + 1,)).copy()
    nnz = int(cp[-1])
    if nnz:
        rows = np.ctypeslib.as_array(C.cast(prow, C.POINTER(C.c_int32)), shape=(nnz,)).copy()
        vals = np.ctypeslib.as_array(C.cast(pval, C.POINTER(C.c_double)), shape=(nnz,)).copy()
    else:
        rows = np.zeros(0, np.int32)
        vals = np.zeros(0, np.float64)
    for p in (pcp, prow, pval):
        L.orc_free(p)
    return Mat(nrows, ncols, cp, rows, vals)


def spgemm(A, B, col_begin: int = 0, col_end: int | None = None):
    """C[:, b:e) = A·B[:, b:e) and per-column flops. Returns (Mat, flops)."""
    A, B = as_mat(A), as_mat(B)
    assert A.ncols == B.nrows, "dimension mismatch"
    e = B.ncols if col_end is None else col_end
    flops = np.zeros(max(e - col_begin, 0), np.int64)
    pcp, prow, pval = C.c_void_p(), C.c_void_p(), C.c_void_p()
    rc = lib().orc_spgemm(A.nrows, A.ncols, B.ncols, _p(A.colptr), _p(A.rows), _p(A.vals),
                          _p(B.colptr), _p(B.rows), _p(B.vals), col_begin, e,
                          C.byref(pcp), C.byref(prow), C.byref(pval), _p(flops))
    if rc:
        raise ValueError("orc_spgemm failed")
    return _take(e - col_begin, A.nrows, pcp, prow, pval), flops


def expand(A, col_begin: int = 0, col_end: int | None = None):
    """The MCL expansion B = A·A (Alg. 1 l.3) on a column range."""
    return spgemm(A, A, col_begin, col_end)


@dataclass
class PruneInfo:
    chaos: np.ndarray   # per column, Q9
    tau: np.ndarray     # effective cut, Q19
    branch: np.ndarray  # 0 thresh, 1 select, 2 recover, 3 argmax, 4 empty
    m: np.ndarray       # entries >= theta
    s: np.ndarray       # their mass


def prune_inflate(Cm, theta=1e-4, S=1100, R=1400, pct=0.9, r=2.0):
    """Alg. 1 l.4-5 under readings Q1-Q9.  Returns (A_next Mat, PruneInfo)."""
    Cm = as_mat(Cm)
    n = Cm.ncols
    chaos = np.zeros(n)
    tau = np.zeros(n)
    br = np.zeros(n, np.int32)
    m = np.zeros(n, np.int64)
    s = np.zeros(n)
    pcp, prow, pval = C.c_void_p(), C.c_void_p(), C.c_void_p()
    rc = lib().orc_prune_inflate(n, _p(Cm.colptr), _p(Cm.rows), _p(Cm.vals), float(theta),
                                 int(S), int(R), float(pct), float(r),
                                 C.byref(pcp), C.byref(prow), C.byref(pval),
                                 _p(chaos), _p(tau), _p(br), _p(m), _p(s))
    if rc:
        raise ValueError("orc_prune_inflate failed")
    return _take(n, Cm.nrows, pcp, prow, pval), PruneInfo(chaos, tau, br, m, s)


def preprocess(G, add_loops: bool = True) -> Mat:
    """Alg. 1 l.1: self-loops of weight 1 (Q10) then column normalisation."""
    n = int(G.ncols)
    cp = np.ascontiguousarray(G.colptr, np.int64)
    rows = np.ascontiguousarray(G.rows, np.int32)
    w = np.ascontiguousarray(G.vals, np.float32)
    pcp, prow, pval = C.c_void_p(), C.c_void_p(), C.c_void_p()
    rc = lib().orc_preprocess(n, _p(cp), _p(rows), _p(w), int(add_loops),
                              C.byref(pcp), C.byref(prow), C.byref(pval))
    if rc:
        raise ValueError("orc_preprocess failed")
    return _take(n, int(G.nrows), pcp, prow, pval)


def clusters(A):
    """Alg. 1 l.6: weak components of the symmetrised pattern, canonical labels (Q11)."""
    A = as_mat(A)
    labels = np.zeros(A.ncols, np.int32)
    ncl = C.c_int64()
    rc = lib().orc_clusters(A.ncols, _p(A.colptr), _p(A.rows), _p(labels), C.byref(ncl))
    if rc:
        raise ValueError("orc_clusters failed")
    return labels, int(ncl.value)


def philox(ctr, key):
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    o = np.zeros(4, np.uint32)
    lib().orc_philox(_p(c), _p(k), _p(o))
    return o


def cohen_key(seed: int, s: int, i: int) -> np.float32:
    return np.float32(lib().orc_cohen_key(seed, s, i))


def cohen(A, B, r: int = 10, seed: int = 0, return_keys: bool = False):
    """Cohen's estimate of nnz(C_*j) for C = A·B (lambda = 1)."""
    A, B = as_mat(A), as_mat(B)
    est = np.zeros(B.ncols)
    keys = np.zeros(r * A.nrows, np.float32)
    mid = np.zeros(r * A.ncols, np.float32)
    rc = lib().orc_cohen(A.nrows, A.ncols, B.ncols, _p(A.colptr), _p(A.rows),
                         _p(B.colptr), _p(B.rows), int(r), int(seed), _p(keys), _p(mid), _p(est))
    if rc:
        raise ValueError("orc_cohen failed")
    if return_keys:
        return est, keys.reshape(r, A.nrows), mid.reshape(r, A.ncols)
    return est


def merge(mats) -> Mat:
    """Sum of equally shaped CSC blocks by merging their lists."""
    mats = [as_mat(m) for m in mats]
    L = len(mats)
    nr, nc = mats[0].nrows, mats[0].ncols
    cps = (C.c_void_p * L)(*[m.colptr.ctypes.data for m in mats])
    rws = (C.c_void_p * L)(*[m.rows.ctypes.data for m in mats])
    vls = (C.c_void_p * L)(*[m.vals.ctypes.data for m in mats])
    pcp, prow, pval = C.c_void_p(), C.c_void_p(), C.c_void_p()
    rc = lib().orc_merge(L, nr, nc, cps, rws, vls, C.byref(pcp), C.byref(prow), C.byref(pval))
    if rc:
        raise ValueError("orc_merge failed")
    return _take(nc, nr, pcp, prow, pval)


def binary_merge(lists, trace: list | None = None) -> Mat:
    """Alg. 2 verbatim: push l_i; nmerges = number of times i halves
    while even; pop nmerges+1 lists, merge, push.  Returns S.pop() (Q16: exact
    when nstages is a power of two).  ``trace`` receives the stack depth after
    each stage."""
    S = []
    for i, li in enumerate(lists, start=1):
        S.append(li)
        j, nmerges = i, 0
        while j % 2 == 0 and j != 0:
            nmerges += 1
            j //= 2
        if nmerges > 0:
            Lst = [S.pop() for _ in range(nmerges + 1)]
            S.append(merge(Lst[::-1]))
        if trace is not None:
            trace.append(len(S))
    return S.pop()


def max_abs_change(A: Mat, B: Mat) -> float:
    """SPEC's alternative convergence measure: max |A-B| with absent = 0."""
    d = 0.0
    for j in range(A.ncols):
        ra, va = A.rows[A.colptr[j]:A.colptr[j + 1]], A.vals[A.colptr[j]:A.colptr[j + 1]]
        rb, vb = B.rows[B.colptr[j]:B.colptr[j + 1]], B.vals[B.colptr[j]:B.colptr[j + 1]]
        da = dict(zip(ra.tolist(), va.tolist()))
        for r_, v_ in zip(rb.tolist(), vb.tolist()):
            d = max(d, abs(da.pop(r_, 0.0) - v_))
        for v_ in da.values():
            d = max(d, abs(v_))
    return d


@dataclass
class RunResult:
    A: Mat
    labels: np.ndarray
    nclusters: int
    iterations: int
    chaos: list
    iterates: list | None


def mcl(G, theta=1e-4, S=1100, R=1400, pct=0.9, r=2.0, eps=1e-3, max_iter=100,
        keep_iterates=False, A0: Mat | None = None) -> RunResult:
    """Alg. 1: A <- column-stochastic(G); repeat expand, prune, inflate
    while chaos >= eps (Q9, at most max_iter iterations); return the components."""
    A = preprocess(G) if A0 is None else as_mat(A0)
    its = [A] if keep_iterates else None
    chaos_hist = []
    it = 0
    while it < max_iter:
        Cm, _ = expand(A)
        A, info = prune_inflate(Cm, theta, S, R, pct, r)
        it += 1
        c = float(info.chaos.max()) if info.chaos.size else 0.0
        chaos_hist.append(c)
        if keep_iterates:
            its.append(A)
        if c < eps:
            break
    labels, ncl = clusters(A)
    return RunResult(A, labels, ncl, it, chaos_hist, its)
