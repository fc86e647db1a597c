"""paper_2002_10083_b200 -- B200-native (sm_100a) MCL expansion hot path of HipMCL
(arXiv:2002.10083), exposed through the C ABI of ``libmclx.so`` (include/mclx.h).

This module is a THIN binding: it marshals torch CUDA tensors into ``mcl_csc_t``
structs, hands the library torch's caching allocator and the current stream, and
raises on error codes.  Every step of the path runs in the library's own kernels;
there is no CPU fallback.  If ``libmclx.so`` is missing or cannot load, importing
this package raises ``ImportError``.

Entry points (same names as the C ABI, ``mcl_`` prefix dropped):
    preprocess(G, add_loops=True)       Alg. 1 l.1
    flops(A, B)
    estimate(A, B, r, seed)             Cohen
    symbolic(A, B)
    spgemm(A, B, cols, params)          P:159, P:239-246 (rectangular blocks)
    expand(A, cols, params)             Alg. 1 l.3
    prune_inflate(C, params)            Alg. 1 l.4-5
    iterate(A, params)                  Alg. 1 l.3-5 fused
    clusters(A)                         Alg. 1 l.6
    run(G, params)                      the Alg. 1 loop driven from Python
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.path.join(_PKG, "libmclx.so")

if not os.path.exists(_LIBPATH):
    raise ImportError(f"libmclx.so not built at {_LIBPATH}; run __graft_entry__.build() "
                      "(there is no CPU fallback)")
try:
    _lib = C.CDLL(_LIBPATH)
except OSError as e:  # pragma: no cover
    raise ImportError(f"cannot load {_LIBPATH}: {e}") from e

MCL_OK = 0
ERRORS = {-1: "MCL_ERR_INVALID_ARG", -2: "MCL_ERR_DIM", -3: "MCL_ERR_FORMAT", -4: "MCL_ERR_OOM",
          -5: "MCL_ERR_CUDA", -6: "MCL_ERR_NCCL", -7: "MCL_ERR_UNSUPPORTED_DEVICE",
          -8: "MCL_ERR_NOT_IMPLEMENTED", -9: "MCL_ERR_INTERNAL"}
NUM_BINS = 6


class CscT(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("row0", C.c_int64), ("col0", C.c_int64), ("n_global", C.c_int64),
                ("col_ptr", C.c_void_p), ("row_idx", C.c_void_p), ("val", C.c_void_p)]


class ParamsT(C.Structure):
    _fields_ = [("inflation", C.c_double), ("prune_threshold", C.c_double),
                ("select_k", C.c_int32), ("recover_k", C.c_int32), ("recover_pct", C.c_double),
                ("chaos_eps", C.c_double), ("est_keys", C.c_int32),
                ("est_cf_threshold", C.c_double), ("seed", C.c_uint64), ("mem_safety", C.c_double),
                ("estimator", C.c_int32), ("force_bin", C.c_int32)]


class StatsT(C.Structure):
    _fields_ = [("flops", C.c_int64), ("nnz_in", C.c_int64), ("nnz_unpruned", C.c_int64),
                ("nnz_out", C.c_int64), ("est_nnz", C.c_double), ("cf", C.c_double),
                ("chaos", C.c_float), ("phases", C.c_int32), ("retries", C.c_int32),
                ("estimator_used", C.c_int32), ("bin_cols", C.c_int64 * (NUM_BINS + 1)),
                ("bin_flops", C.c_int64 * (NUM_BINS + 1)), ("ms", C.c_float * 8),
                ("peak_bytes", C.c_int64), ("launches", C.c_int64),
                ("bin_ms", C.c_float * (NUM_BINS + 1)), ("bin_nnzb", C.c_int64 * (NUM_BINS + 1)),
                ("bin_out", C.c_int64 * (NUM_BINS + 1)), ("comm_bytes", C.c_int64),
                ("peak_partial", C.c_int64), ("split_cols", C.c_int64),
                ("split_items", C.c_int64), ("split_ms", C.c_float),
                ("split_vcols", C.c_int64 * 3), ("split_vms", C.c_float * 3),
                ("stages", C.c_int32), ("esc_cols", C.c_int64), ("esc_flops", C.c_int64),
                ("esc_out", C.c_int64), ("esc_ms", C.c_float)]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        for k in ("bin_cols", "bin_flops", "ms", "bin_ms", "bin_nnzb", "bin_out", "split_vcols",
                  "split_vms"):
            d[k] = list(d[k])
        return d


class GraphT(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("col_ptr", C.POINTER(C.c_int64)),
                ("row_idx", C.POINTER(C.c_int32)), ("val", C.POINTER(C.c_float)),
                ("labels", C.POINTER(C.c_char_p))]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

_P = C.c_void_p
_i64 = C.c_int64
_sig = {
    "mcl_version": ([], C.c_int),
    "mcl_params_default": ([C.POINTER(ParamsT)], None),
    "mcl_ctx_create": ([C.POINTER(_P), C.c_int, _P, ALLOC_FN, FREE_FN, _P], C.c_int),
    "mcl_ctx_set_stream": ([_P, _P], C.c_int),
    "mcl_ctx_destroy": ([_P], C.c_int),
    "mcl_last_error": ([_P], C.c_char_p),
    "mcl_csc_release": ([_P, C.POINTER(CscT)], C.c_int),
    "mcl_preprocess": ([_P, C.POINTER(CscT), C.c_int, C.POINTER(CscT)], C.c_int),
    "mcl_flops": ([_P, C.POINTER(CscT), C.POINTER(CscT), _P, C.POINTER(_i64)], C.c_int),
    "mcl_estimate": ([_P, C.POINTER(CscT), C.POINTER(CscT), C.c_int32, C.c_uint64, _P, _P,
                      C.POINTER(C.c_double)], C.c_int),
    "mcl_symbolic": ([_P, C.POINTER(CscT), C.POINTER(CscT), _P, C.POINTER(_i64)], C.c_int),
    "mcl_spgemm": ([_P, C.POINTER(CscT), C.POINTER(CscT), _i64, _i64, C.POINTER(ParamsT),
                    C.POINTER(CscT), C.POINTER(StatsT)], C.c_int),
    "mcl_expand": ([_P, C.POINTER(CscT), _i64, _i64, C.POINTER(ParamsT), C.POINTER(CscT),
                    C.POINTER(StatsT)], C.c_int),
    "mcl_prune_inflate": ([_P, C.POINTER(CscT), C.POINTER(ParamsT), C.POINTER(CscT), _P,
                           C.POINTER(StatsT)], C.c_int),
    "mcl_iterate": ([_P, C.POINTER(CscT), C.POINTER(ParamsT), C.POINTER(CscT),
                     C.POINTER(StatsT)], C.c_int),
    "mcl_iterate_range": ([_P, C.POINTER(CscT), _i64, _i64, C.POINTER(ParamsT), C.POINTER(CscT),
                           C.POINTER(StatsT)], C.c_int),
    "mcl_clusters": ([_P, C.POINTER(CscT), _P, C.POINTER(_i64)], C.c_int),
    "mcl_merge": ([_P, C.c_int32, C.POINTER(CscT), C.POINTER(CscT)], C.c_int),
    "mcl_block": ([_P, C.POINTER(CscT), _i64, _i64, _i64, _i64, C.POINTER(CscT)], C.c_int),
    "mcl_prof_read": ([C.POINTER(C.c_uint64 * 12), C.c_int], C.c_int),
    "mcl_nccl_unique_id": ([C.c_char * 128], C.c_int),
    "mcl_ctx_set_grid": ([_P, C.c_int, C.c_int, C.c_int, C.c_char * 128], C.c_int),
    "mcl_summa_iterate": ([_P, C.POINTER(CscT), C.POINTER(ParamsT), C.POINTER(CscT),
                           C.POINTER(StatsT)], C.c_int),
    "mcl_iterate_hostmem": ([_P, C.POINTER(CscT), C.POINTER(ParamsT), C.c_int32, C.c_int32,
                             C.POINTER(CscT), C.POINTER(StatsT)], C.c_int),
    "mcl_host_csc_release": ([C.POINTER(CscT)], C.c_int),
    "mcl_summa_schedule": ([C.c_int, C.c_int, C.c_int, _i64, C.c_int, _P, _i64], C.c_int),
    "mcl_graph_read": ([C.c_char_p, C.c_int, C.POINTER(GraphT), C.c_char_p, C.c_size_t], C.c_int),
    "mcl_graph_free": ([C.POINTER(GraphT)], None),
    "mcl_clusters_write": ([C.c_char_p, _P, _i64, C.POINTER(GraphT)], C.c_int),
}
for _name, (_args, _res) in _sig.items():
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_sig)


class MclError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


@dataclass
class Params:
    """Python mirror of mcl_params_t (defaults = mcl_params_default)."""
    inflation: float = 2.0
    prune_threshold: float = 1e-4
    select_k: int = 1100
    recover_k: int = 1400
    recover_pct: float = 0.9
    chaos_eps: float = 1e-3
    est_keys: int = 10
    est_cf_threshold: float = 2.0
    seed: int = 0x5EED
    mem_safety: float = 0.9
    estimator: int = 0
    force_bin: int = -1

    def c(self) -> ParamsT:
        p = ParamsT()
        for k in self.__dataclass_fields__:
            setattr(p, k, getattr(self, k))
        return p


@dataclass
class CSC:
    """A device CSC matrix: three CUDA tensors plus shape and block offsets."""
    nrows: int
    ncols: int
    colptr: torch.Tensor  # int64 [ncols+1]
    rows: torch.Tensor    # int32 [nnz]
    vals: torch.Tensor    # float32 [nnz]
    row0: int = 0
    col0: int = 0
    n_global: int = 0
    _keep: list = field(default_factory=list, repr=False)

    @property
    def nnz(self) -> int:
        return int(self.rows.numel())

    def c(self) -> CscT:
        return CscT(self.nrows, self.ncols, self.nnz, self.row0, self.col0,
                    self.n_global or self.nrows, self.colptr.data_ptr(),
                    self.rows.data_ptr() if self.nnz else None,
                    self.vals.data_ptr() if self.nnz else None)

    @staticmethod
    def from_host(m, device="cuda", row0: int = 0, col0: int = 0, n_global: int = 0) -> "CSC":
        """Copy an object with nrows/ncols/colptr/rows/vals (numpy) to the device.
        Values are cast to float32."""
        cp = torch.from_numpy(np.ascontiguousarray(m.colptr, np.int64)).to(device)
        rw = torch.from_numpy(np.ascontiguousarray(m.rows, np.int32)).to(device)
        vl = torch.from_numpy(np.ascontiguousarray(m.vals, np.float32)).to(device)
        return CSC(int(m.nrows), int(m.ncols), cp, rw, vl, row0, col0, n_global)

    def to_host(self):
        """(colptr int64, rows int32, vals float32) numpy arrays."""
        return (self.colptr.cpu().numpy(), self.rows.cpu().numpy(), self.vals.cpu().numpy())


class Context:
    """An mcl_ctx bound to one device; outputs are allocated from torch's caching
    allocator (so they are ordinary torch tensors) on the current stream."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise MclError(-7, "no CUDA device (the path has no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._live: dict[int, torch.Tensor] = {}

        def _alloc(state, nbytes, stream):
            t = torch.empty(int(nbytes), dtype=torch.uint8, device=f"cuda:{self.device}")
            p = t.data_ptr()
            self._live[p] = t
            return p

        def _free(state, ptr, nbytes, stream):
            self._live.pop(ptr, None)

        self._alloc_cb = ALLOC_FN(_alloc)
        self._free_cb = FREE_FN(_free)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            rc = _lib.mcl_ctx_create(C.byref(h), self.device,
                                     C.c_void_p(torch.cuda.current_stream().cuda_stream),
                                     self._alloc_cb, self._free_cb, None)
        if rc != MCL_OK:
            raise MclError(rc, "mcl_ctx_create failed")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            _lib.mcl_ctx_destroy(self.h)
            self.h = None
            self._live.clear()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # -- helpers
    def _sync_stream(self):
        _lib.mcl_ctx_set_stream(self.h, C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))

    def _check(self, rc: int):
        if rc != MCL_OK:
            raise MclError(rc, (_lib.mcl_last_error(self.h) or b"").decode())

    def _adopt(self, m: CscT) -> CSC:
        """Turn a library-allocated mcl_csc_t into a CSC of torch tensors (ownership moves
        from the allocator table to the tensors)."""
        def take(ptr, n, dtype):
            t = self._live.pop(ptr)
            return t[: n * dtype.itemsize].view(dtype) if n else t[:0].view(dtype)
        cp = take(m.col_ptr, m.ncols + 1, torch.int64)
        rw = take(m.row_idx, m.nnz, torch.int32)
        vl = take(m.val, m.nnz, torch.float32)
        return CSC(m.nrows, m.ncols, cp, rw, vl, m.row0, m.col0, m.n_global)

    # -- entry points
    def preprocess(self, G: CSC, add_loops: bool = True) -> CSC:
        self._sync_stream()
        out = CscT()
        self._check(_lib.mcl_preprocess(self.h, C.byref(G.c()), int(add_loops), C.byref(out)))
        return self._adopt(out)

    def flops(self, A: CSC, B: CSC | None = None):
        B = A if B is None else B
        self._sync_stream()
        f = torch.empty(B.ncols, dtype=torch.int64, device=A.colptr.device)
        tot = C.c_int64()
        self._check(_lib.mcl_flops(self.h, C.byref(A.c()), C.byref(B.c()), f.data_ptr(),
                                   C.byref(tot)))
        return f, int(tot.value)

    def estimate(self, A: CSC, B: CSC | None = None, r: int = 10, seed: int = 0x5EED,
                 return_keys: bool = False):
        B = A if B is None else B
        self._sync_stream()
        est = torch.empty(B.ncols, dtype=torch.float32, device=A.colptr.device)
        keys = torch.empty(r * A.nrows, dtype=torch.float32, device=A.colptr.device) \
            if return_keys else None
        tot = C.c_double()
        self._check(_lib.mcl_estimate(self.h, C.byref(A.c()), C.byref(B.c()), r, seed,
                                      est.data_ptr(), keys.data_ptr() if keys is not None else None,
                                      C.byref(tot)))
        if return_keys:
            return est, float(tot.value), keys.view(r, A.nrows)
        return est, float(tot.value)

    def symbolic(self, A: CSC, B: CSC | None = None):
        B = A if B is None else B
        self._sync_stream()
        nnz = torch.empty(B.ncols, dtype=torch.int64, device=A.colptr.device)
        tot = C.c_int64()
        self._check(_lib.mcl_symbolic(self.h, C.byref(A.c()), C.byref(B.c()), nnz.data_ptr(),
                                      C.byref(tot)))
        return nnz, int(tot.value)

    def spgemm(self, A: CSC, B: CSC, cols=None, params: Params | None = None):
        b, e = (0, B.ncols) if cols is None else cols
        self._sync_stream()
        out, st = CscT(), StatsT()
        self._check(_lib.mcl_spgemm(self.h, C.byref(A.c()), C.byref(B.c()), b, e,
                                    C.byref((params or Params()).c()), C.byref(out), C.byref(st)))
        return self._adopt(out), st.as_dict()

    def expand(self, A: CSC, cols=None, params: Params | None = None):
        b, e = (0, A.ncols) if cols is None else cols
        self._sync_stream()
        out, st = CscT(), StatsT()
        self._check(_lib.mcl_expand(self.h, C.byref(A.c()), b, e,
                                    C.byref((params or Params()).c()), C.byref(out), C.byref(st)))
        return self._adopt(out), st.as_dict()

    def prune_inflate(self, Cm: CSC, params: Params | None = None, return_chaos: bool = False):
        self._sync_stream()
        out, st = CscT(), StatsT()
        chaos = torch.empty(Cm.ncols, dtype=torch.float32, device=Cm.colptr.device) \
            if return_chaos else None
        self._check(_lib.mcl_prune_inflate(self.h, C.byref(Cm.c()),
                                           C.byref((params or Params()).c()), C.byref(out),
                                           chaos.data_ptr() if chaos is not None else None,
                                           C.byref(st)))
        res = self._adopt(out), st.as_dict()
        return (*res, chaos) if return_chaos else res

    def iterate(self, A: CSC, params: Params | None = None, cols=None):
        self._sync_stream()
        out, st = CscT(), StatsT()
        if cols is None:
            rc = _lib.mcl_iterate(self.h, C.byref(A.c()), C.byref((params or Params()).c()),
                                  C.byref(out), C.byref(st))
        else:
            rc = _lib.mcl_iterate_range(self.h, C.byref(A.c()), int(cols[0]), int(cols[1]),
                                        C.byref((params or Params()).c()), C.byref(out),
                                        C.byref(st))
        self._check(rc)
        return self._adopt(out), st.as_dict()

    def iterate_hostmem(self, A_host, params: Params | None = None, stages: int = 0,
                        phases: int = 0):
        """One MCL iteration of an iterate held in HOST memory (mcl_iterate_hostmem: column
        panels streamed to the device, Alg. 2 on the device, pruned phases back to host).
        A_host: any object with nrows/ncols/colptr/rows/vals (numpy); it is pinned here.
        Returns (HostGraph of numpy arrays, stats)."""
        self._sync_stream()
        cp = torch.from_numpy(np.ascontiguousarray(A_host.colptr, np.int64)).pin_memory()
        rw = torch.from_numpy(np.ascontiguousarray(A_host.rows, np.int32)).pin_memory()
        vl = torch.from_numpy(np.ascontiguousarray(A_host.vals, np.float32)).pin_memory()
        n = int(A_host.ncols)
        a = CscT(int(A_host.nrows), n, int(rw.numel()), 0, 0, n, cp.data_ptr(),
                 rw.data_ptr() if rw.numel() else None, vl.data_ptr() if vl.numel() else None)
        out, st = CscT(), StatsT()
        self._check(_lib.mcl_iterate_hostmem(self.h, C.byref(a), C.byref((params or Params()).c()),
                                             int(stages), int(phases), C.byref(out), C.byref(st)))
        try:
            nnz = int(out.nnz)
            ocp = np.ctypeslib.as_array(C.cast(out.col_ptr, C.POINTER(C.c_int64)), shape=(n + 1,)).copy()
            orw = np.ctypeslib.as_array(C.cast(out.row_idx, C.POINTER(C.c_int32)), shape=(max(nnz, 1),))[:nnz].copy()
            ovl = np.ctypeslib.as_array(C.cast(out.val, C.POINTER(C.c_float)), shape=(max(nnz, 1),))[:nnz].copy()
        finally:
            _lib.mcl_host_csc_release(C.byref(out))
        return HostGraph(n, n, ocp, orw, ovl), st.as_dict()

    def clusters(self, A: CSC):
        self._sync_stream()
        labels = torch.empty(A.ncols, dtype=torch.int32, device=A.colptr.device)
        k = C.c_int64()
        self._check(_lib.mcl_clusters(self.h, C.byref(A.c()), labels.data_ptr(), C.byref(k)))
        return labels, int(k.value)

    def merge(self, lists):
        """Sum of equally shaped CSC blocks (the merge of Alg. 2 / P:246) on the device."""
        self._sync_stream()
        arr = (CscT * len(lists))(*[m.c() for m in lists])
        out = CscT()
        self._check(_lib.mcl_merge(self.h, len(lists), arr, C.byref(out)))
        return self._adopt(out)

    def block(self, A: CSC, rows, cols) -> CSC:
        """A[r0:r1, c0:c1] as a block (row ids rebased, row0/col0 advanced)."""
        self._sync_stream()
        out = CscT()
        self._check(_lib.mcl_block(self.h, C.byref(A.c()), int(rows[0]), int(rows[1]),
                                   int(cols[0]), int(cols[1]), C.byref(out)))
        return self._adopt(out)

    def set_grid(self, pr: int, pc: int, rank: int, uid: bytes):
        """Collective over pr*pc ranks: NCCL world / row / column communicators."""
        buf = (C.c_char * 128).from_buffer_copy(uid)
        with torch.cuda.device(self.device):
            self._check(_lib.mcl_ctx_set_grid(self.h, pr, pc, rank, buf))
        self.grid = (pr, pc, rank)

    def summa_iterate(self, A_blk: CSC, params: Params | None = None):
        """One MCL iteration on the 2D-distributed iterate (collective)."""
        self._sync_stream()
        out, st = CscT(), StatsT()
        self._check(_lib.mcl_summa_iterate(self.h, C.byref(A_blk.c()),
                                           C.byref((params or Params()).c()), C.byref(out),
                                           C.byref(st)))
        return self._adopt(out), st.as_dict()

    def run(self, G: CSC, params: Params | None = None, max_iter: int = 100, callback=None):
        """Alg. 1 driven from Python: preprocess, iterate until chaos <
        chaos_eps (Q9) or max_iter, then the components.  Returns (labels, ncl, stats list)."""
        params = params or Params()
        A = self.preprocess(G)
        hist = []
        for it in range(max_iter):
            A, st = self.iterate(A, params)
            hist.append(st)
            if callback:
                callback(it, A, st)
            if st["chaos"] < params.chaos_eps:
                break
        labels, k = self.clusters(A)
        return labels, k, hist, A


_default: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    d = torch.cuda.current_device() if device is None else device
    if d not in _default:
        _default[d] = Context(d)
    return _default[d]


def version() -> int:
    return int(_lib.mcl_version())


def params_default() -> Params:
    p = ParamsT()
    _lib.mcl_params_default(C.byref(p))
    return Params(**{k: getattr(p, k) for k, _ in ParamsT._fields_})


def preprocess(G, add_loops=True):
    return context().preprocess(G, add_loops)


def flops(A, B=None):
    return context().flops(A, B)


def estimate(A, B=None, r=10, seed=0x5EED, return_keys=False):
    return context().estimate(A, B, r, seed, return_keys)


def symbolic(A, B=None):
    return context().symbolic(A, B)


def spgemm(A, B, cols=None, params=None):
    return context().spgemm(A, B, cols, params)


def expand(A, cols=None, params=None):
    return context().expand(A, cols, params)


def prune_inflate(Cm, params=None, return_chaos=False):
    return context().prune_inflate(Cm, params, return_chaos)


def iterate(A, params=None, cols=None):
    return context().iterate(A, params, cols)


def clusters(A):
    return context().clusters(A)


def merge(lists):
    return context().merge(lists)


def prof_read(reset: bool = True):
    """Development counters of the SpGEMM kernel (zeros unless built with -DMCLX_PROF)."""
    v = (C.c_uint64 * 12)()
    _lib.mcl_prof_read(C.byref(v), int(reset))
    return list(v)


def summa_schedule(pr: int, pc: int, rank: int, n: int, stage_mult: int = 1) -> dict:
    """The 2D Sparse-SUMMA schedule of mcl_summa_iterate, from the library (host arithmetic):
    block ranges, and per stage the inner panel, the two panel owners and Alg. 2's nmerges."""
    cap = 4 + 5 * pr * pc * stage_mult
    buf = (C.c_int64 * cap)()
    s = _lib.mcl_summa_schedule(pr, pc, rank, n, stage_mult, C.cast(buf, C.c_void_p), cap)
    if s < 0:
        raise MclError(s, "mcl_summa_schedule")
    v = list(buf)
    return {"rows": (v[0], v[1]), "cols": (v[2], v[3]), "s": s,
            "stages": [dict(k0=v[4 + 5 * q], k1=v[5 + 5 * q], a_owner_col=v[6 + 5 * q],
                            b_owner_row=v[7 + 5 * q], nmerges=v[8 + 5 * q]) for q in range(s)]}


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    rc = _lib.mcl_nccl_unique_id(buf)
    if rc != MCL_OK:
        raise MclError(rc, "ncclGetUniqueId failed")
    return bytes(buf.raw)


def run(G, params=None, max_iter=100, callback=None):
    return context().run(G, params, max_iter, callback)


@dataclass
class HostGraph:
    """A graph read by mcl_graph_read: host CSC arrays (numpy) and optional vertex labels."""
    nrows: int
    ncols: int
    colptr: np.ndarray
    rows: np.ndarray
    vals: np.ndarray
    labels: list | None = None

    @property
    def nnz(self) -> int:
        return int(self.rows.size)


def read_graph(path: str, symmetrize: bool = True) -> HostGraph:
    """MatrixMarket coordinate or a labelled 'src dst [weight]' edge list -> HostGraph
    (host-side native parser in libmclx.so; no GPU needed).  Raises MclError on bad input."""
    g = GraphT()
    err = C.create_string_buffer(512)
    rc = _lib.mcl_graph_read(os.fsencode(path), int(symmetrize), C.byref(g), err, 512)
    if rc != MCL_OK:
        raise MclError(rc, err.value.decode())
    try:
        n, nnz = int(g.n), int(g.nnz)
        cp = np.ctypeslib.as_array(g.col_ptr, shape=(n + 1,)).copy()
        rows = np.ctypeslib.as_array(g.row_idx, shape=(max(nnz, 1),))[:nnz].copy()
        vals = np.ctypeslib.as_array(g.val, shape=(max(nnz, 1),))[:nnz].copy()
        labels = [g.labels[i].decode() for i in range(n)] if g.labels else None
    finally:
        _lib.mcl_graph_free(C.byref(g))
    return HostGraph(n, n, cp, rows, vals, labels)


def write_clusters(path: str, labels, graph: HostGraph | None = None) -> None:
    """One line per cluster (members by ascending vertex, space-separated graph labels or
    1-based ids), clusters in label order (mcl_clusters numbers them by smallest member)."""
    lab = labels.cpu().numpy() if isinstance(labels, torch.Tensor) else np.asarray(labels)
    lab = np.ascontiguousarray(lab, np.int32)
    g = None
    keep = None
    if graph is not None and graph.labels is not None:
        g = GraphT()
        g.n = len(graph.labels)
        keep = (C.c_char_p * len(graph.labels))(*[x.encode() for x in graph.labels])
        g.labels = C.cast(keep, C.POINTER(C.c_char_p))
    rc = _lib.mcl_clusters_write(os.fsencode(path), lab.ctypes.data_as(C.c_void_p), lab.size,
                                 C.byref(g) if g is not None else None)
    if rc != MCL_OK:
        raise MclError(rc, f"cannot write clusters to {path}")
