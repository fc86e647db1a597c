"""CPU-side checks of the C ABI boundary: libmclx.so loads, exports every entry
point include/mclx.h declares, reports its defaults, and refuses to run without a
B200 instead of falling back to the CPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "mclx.h")
LIB = os.path.join(ROOT, "paper_2002_10083_b200", "libmclx.so")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char \*)\s*(mcl_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return C.CDLL(LIB)


def test_header_declares_the_four_calls():
    names = _declared()
    for n in ("mcl_expand", "mcl_prune_inflate", "mcl_iterate", "mcl_clusters"):
        assert n in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_symbol():
    import paper_2002_10083_b200 as M
    assert sorted(M.EXPORTED) == _declared()


def test_defaults(lib):
    import paper_2002_10083_b200 as M
    p = M.params_default()
    assert p.inflation == 2.0 and p.select_k == 1100 and p.recover_k == 1400
    assert p.prune_threshold == 1e-4 and p.recover_pct == 0.9 and p.est_keys == 10
    assert M.version() == 1


def test_no_cpu_fallback(lib):
    """Without a GPU the library refuses to create a context (no CPU path exists)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    AL = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
    FR = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)
    lib.mcl_ctx_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, AL, FR, C.c_void_p]
    rc = lib.mcl_ctx_create(C.byref(h), 0, None, AL(), FR(), None)
    assert rc in (-5, -7)
    import paper_2002_10083_b200 as M
    with pytest.raises(M.MclError):
        M.Context()


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2002_10083_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liborc" not in txt and "mcl_oracle" not in txt, f
