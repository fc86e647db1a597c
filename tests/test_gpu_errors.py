"""C-ABI error paths (include/mclx.h "Every call returns MCL_OK (0) or a negative MCL_ERR_*
code.  On error, out matrices are zeroed (nnz 0, NULL pointers), nothing leaks").

Calls go straight through ctypes to libmclx.so so the raw status and the out struct
can be inspected; SURVEY §8(b) lists the conventions (dimension mismatch -> rejection
S:79/129/138/305, negative value -> rejection S:70, non-square -> error S:494).
"""
import ctypes as C

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2002_10083_b200 as M
    from paper_2002_10083_b200 import _lib, CscT, ParamsT, StatsT


def _zeroed(m) -> bool:
    return (m.nnz == 0 and not m.col_ptr and not m.row_idx and not m.val and m.ncols == 0
            and m.nrows == 0)


def _dirty():
    """An out struct pre-filled with garbage: the library must zero it on error."""
    o = CscT()
    o.nrows, o.ncols, o.nnz = 7, 7, 7
    o.col_ptr, o.row_idx, o.val = 8, 16, 24
    return o


def _sq(n=50, seed=0):
    return M.CSC.from_host(synth.random_sparse(n, n, 0.1, seed=seed))


def _err(ctx):
    return (_lib.mcl_last_error(ctx.h) or b"").decode()


def _live(ctx):
    torch.cuda.synchronize()
    return len(ctx._live)


def test_expand_rejects_non_square_and_bad_ranges():
    ctx = M.Context()
    R = M.CSC.from_host(synth.random_sparse(40, 30, 0.1, seed=1))
    p = M.Params().c()
    for A, b, e, code in [(R, 0, 30, -2), (_sq(), -1, 10, -2), (_sq(), 0, 51, -2), (_sq(), 9, 3, -2)]:
        out, st = _dirty(), StatsT()
        before = _live(ctx)
        rc = _lib.mcl_expand(ctx.h, C.byref(A.c()), b, e, C.byref(p), C.byref(out), C.byref(st))
        assert rc == code, (rc, _err(ctx))
        assert _zeroed(out)
        assert _live(ctx) == before
    # rectangular spgemm with mismatched inner dimension
    A = M.CSC.from_host(synth.random_sparse(40, 30, 0.1, seed=1))
    B = M.CSC.from_host(synth.random_sparse(31, 20, 0.1, seed=2))
    out = _dirty()
    rc = _lib.mcl_spgemm(ctx.h, C.byref(A.c()), C.byref(B.c()), 0, 20, C.byref(p), C.byref(out),
                         None)
    assert rc == -2 and _zeroed(out) and "A.ncols" in _err(ctx)
    ctx.close()


@pytest.mark.parametrize("field,value", [("inflation", 1.0), ("inflation", 0.5),
                                         ("prune_threshold", -1e-4), ("select_k", 0),
                                         ("recover_k", -1), ("recover_pct", 1.5),
                                         ("est_keys", 1), ("est_keys", 17)])
def test_iterate_rejects_bad_params(field, value):
    ctx = M.Context()
    A = _sq()
    p = M.Params()
    setattr(p, field, value)
    for fn in ("mcl_iterate", "mcl_prune_inflate"):
        out = _dirty()
        before = _live(ctx)
        if fn == "mcl_iterate":
            rc = _lib.mcl_iterate(ctx.h, C.byref(A.c()), C.byref(p.c()), C.byref(out), None)
        else:
            rc = _lib.mcl_prune_inflate(ctx.h, C.byref(A.c()), C.byref(p.c()), C.byref(out), None,
                                        None)
        assert rc == -1, (fn, rc, _err(ctx))
        assert _zeroed(out)
        assert _live(ctx) == before
    ctx.close()


def test_null_pointers():
    ctx = M.Context()
    A = _sq()
    p = M.Params().c()
    out = _dirty()
    assert _lib.mcl_iterate(ctx.h, None, C.byref(p), C.byref(out), None) == -1
    assert _lib.mcl_iterate(ctx.h, C.byref(A.c()), None, C.byref(out), None) == -1
    assert _lib.mcl_iterate(ctx.h, C.byref(A.c()), C.byref(p), None, None) == -1
    assert _lib.mcl_expand(ctx.h, None, 0, 1, C.byref(p), C.byref(out), None) == -1
    assert _zeroed(out)
    assert _lib.mcl_expand(None, C.byref(A.c()), 0, 1, C.byref(p), C.byref(out), None) == -1
    assert _lib.mcl_clusters(ctx.h, C.byref(A.c()), None, None) == -1
    bad = A.c()
    bad.col_ptr = None
    out = _dirty()
    assert _lib.mcl_expand(ctx.h, C.byref(bad), 0, 1, C.byref(p), C.byref(out), None) == -1
    assert _zeroed(out)
    bad = A.c()
    bad.row_idx = None
    assert _lib.mcl_iterate(ctx.h, C.byref(bad), C.byref(p), C.byref(out), None) == -1
    assert _lib.mcl_merge(ctx.h, 0, None, C.byref(out)) == -1
    assert _lib.mcl_csc_release(ctx.h, None) == -1
    z = CscT()
    assert _lib.mcl_csc_release(ctx.h, C.byref(z)) == 0  # no-op on an all-zero struct
    assert _lib.mcl_summa_iterate(ctx.h, C.byref(A.c()), C.byref(p), C.byref(out), None) == -1
    assert "set_grid" in _err(ctx)
    ctx.close()


def _broken(kind):
    """A 4x4 CSC that breaks one header invariant."""
    cp = np.array([0, 2, 3, 5, 6], np.int64)
    rows = np.array([0, 2, 1, 0, 3, 2], np.int32)
    vals = np.array([0.5, 0.5, 1.0, 0.3, 0.7, 1.0], np.float32)
    if kind == "unsorted":
        rows[3], rows[4] = 3, 0
    elif kind == "duplicate":
        rows[1] = 0
    elif kind == "range":
        rows[5] = 4
    elif kind == "negative":
        vals[2] = -1.0
    elif kind == "nan":
        vals[0] = np.nan
    elif kind == "colptr":
        cp[2], cp[3] = 4, 3
    elif kind == "nnz":
        cp[4] = 5
    return synth.Csc(4, 4, cp, rows, vals)


@pytest.mark.parametrize("kind,bit", [("unsorted", "strictly increasing"),
                                      ("duplicate", "strictly increasing"),
                                      ("range", "out of range"), ("negative", "negative"),
                                      ("nan", "not finite"), ("colptr", "col_ptr"),
                                      ("nnz", "col_ptr")])
def test_validate_format(monkeypatch, kind, bit):
    """MCLX_VALIDATE=1: malformed CSC inputs are rejected with MCL_ERR_FORMAT (-3) before
    any kernel of the path runs; without it the caller's promise is trusted."""
    monkeypatch.setenv("MCLX_VALIDATE", "1")
    ctx = M.Context()
    A = M.CSC.from_host(_broken(kind))
    p = M.Params().c()
    for call in ("iterate", "expand", "prune_inflate", "clusters"):
        out = _dirty()
        if call == "iterate":
            rc = _lib.mcl_iterate(ctx.h, C.byref(A.c()), C.byref(p), C.byref(out), None)
        elif call == "expand":
            rc = _lib.mcl_expand(ctx.h, C.byref(A.c()), 0, 4, C.byref(p), C.byref(out), None)
        elif call == "prune_inflate":
            rc = _lib.mcl_prune_inflate(ctx.h, C.byref(A.c()), C.byref(p), C.byref(out), None, None)
        else:
            lab = torch.empty(4, dtype=torch.int32, device="cuda")
            rc = _lib.mcl_clusters(ctx.h, C.byref(A.c()), lab.data_ptr(), None)
            out = CscT()
        assert rc == -3, (call, rc, _err(ctx))
        assert bit in _err(ctx), _err(ctx)
        assert _zeroed(out)
    # a valid matrix passes validation and gives the ordinary result
    good = M.CSC.from_host(_broken("none"))
    out, st = ctx.iterate(good, M.Params())
    assert out.ncols == 4
    ctx.close()


def test_validate_accepts_underflowed_product():
    """An unpruned product may hold 0.0 entries (an fp32 product that underflowed stays in
    the structure, Q13); validation of mcl_prune_inflate's input accepts them."""
    import os
    os.environ["MCLX_VALIDATE"] = "1"
    try:
        ctx = M.Context()
    finally:
        del os.environ["MCLX_VALIDATE"]
    Cm = synth.Csc(3, 2, np.array([0, 2, 3], np.int64), np.array([0, 2, 1], np.int32),
                   np.array([0.0, 0.5, 1.0], np.float32))
    out, st = ctx.prune_inflate(M.CSC.from_host(Cm), M.Params(recover_k=0))
    cp, rw, vl = out.to_host()
    assert cp.tolist() == [0, 1, 2] and rw.tolist() == [2, 1]
    ctx.close()
