"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same
seeded inputs.

  P1 unpruned structure bit-exact (col_ptr, row_idx);
  P2 unpruned values |v32 - v64| <= 1e-5 v64 for v64 >= 1e-30;
  P3 pruned/inflated output: kept sets equal except entries within 1e-6 of the
     column's cut tau_j; values 1e-5 relative (re-inflated over the GPU's kept set);
  P4 cluster labels identical;
  P5 Cohen keys identical (<= 1 ulp, rare), estimates 1e-6 relative.
Inputs handed to both sides are the SAME fp32 numbers (the oracle promotes them).
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2002_10083_b200 as M


def dev(m, **kw):
    return M.CSC.from_host(m, **kw)


_ORC = {}


def _key(m):
    import hashlib
    h = hashlib.sha1()
    for a in (m.colptr, m.rows, m.vals):
        h.update(np.ascontiguousarray(a).tobytes())
    return (m.nrows, m.ncols, h.hexdigest())


def oexp(A):
    """O.expand(A), memoised for the session: the same oracle products (C2, R-MAT scale 14,
    C1's first iterate) recur across many tests; the oracle is deterministic."""
    k = ("expand",) + _key(A)
    if k not in _ORC:
        _ORC[k] = O.expand(A)
    return _ORC[k]


def opi(Cr, theta, S, R, pct, r=2.0):
    """O.prune_inflate memoised like oexp."""
    k = ("prune", id(Cr), theta, S, R, pct, r)
    if k not in _ORC:
        _ORC[k] = (O.prune_inflate(Cr, theta, S, R, pct, r), Cr)  # keep Cr alive with its id
    return _ORC[k][0]


def host_mat(g):
    cp, rw, vl = g.to_host()
    return O.Mat(g.nrows, g.ncols, cp.astype(np.int64), rw.astype(np.int32), vl.astype(np.float64))


def f32(m):
    """fp32 copy of an oracle Mat (the GPU input); the oracle is then run on the same numbers."""
    return O.Mat(m.nrows, m.ncols, m.colptr.copy(), m.rows.copy(),
                 m.vals.astype(np.float32).astype(np.float64))


def assert_unpruned_parity(G, Ref, rtol=1e-5):
    assert G.nrows == Ref.nrows and G.ncols == Ref.ncols
    assert np.array_equal(G.colptr, Ref.colptr), "P1 col_ptr"
    assert np.array_equal(G.rows, Ref.rows), "P1 row_idx"
    big = Ref.vals >= 1e-30
    rel = np.abs(G.vals[big] - Ref.vals[big]) / Ref.vals[big]
    assert rel.size == 0 or rel.max() <= rtol, f"P2 max rel err {rel.max()}"


def c1_it1():
    """C1's first iterate (the oracle's, cast to fp32): dense columns, every bin."""
    k = ("c1it1",)
    if k not in _ORC:
        A0 = O.preprocess(synth.planted_partition())
        A1, _ = O.prune_inflate(oexp(A0)[0], 1e-4, 1100, 1400, 0.9, 2.0)
        _ORC[k] = f32(A1)
    return _ORC[k]


def kept_parity(Gm, Cref, info, params, band=1e-6, rtol=1e-5):
    """P3 for a pruned output Gm (GPU) against oracle info on unpruned Cref (fp64)."""
    theta, S, R, pct = params
    stats = dict(band_excluded=0, band_flip_cols=0)
    Ao, _ = O.prune_inflate(Cref, theta, S, R, pct, 2.0)
    for j in range(Gm.ncols):
        gr = Gm.rows[Gm.colptr[j]:Gm.colptr[j + 1]]
        gv = Gm.vals[Gm.colptr[j]:Gm.colptr[j + 1]]
        orow = Ao.rows[Ao.colptr[j]:Ao.colptr[j + 1]]
        assert np.all(np.diff(gr) > 0)
        if np.array_equal(gr, orow):
            ov = Ao.vals[Ao.colptr[j]:Ao.colptr[j + 1]]
            rel = np.abs(gv - ov) / ov
            assert rel.max() <= rtol, (j, rel.max())
            continue
        cr = Cref.rows[Cref.colptr[j]:Cref.colptr[j + 1]]
        cv = Cref.vals[Cref.colptr[j]:Cref.colptr[j + 1]]
        diff = np.setxor1d(gr, orow)
        vals = cv[np.searchsorted(cr, diff)]
        assert np.all(np.abs(vals - info.tau[j]) <= band), (j, vals, info.tau[j])
        stats["band_excluded"] += len(diff)
        stats["band_flip_cols"] += 1
        # re-inflate the oracle values over the GPU's kept set
        w = cv[np.searchsorted(cr, gr)]
        w = w / w.sum()
        ref = w * w / (w * w).sum()
        assert np.max(np.abs(gv - ref) / ref) <= rtol
    return stats


# ---------------------------------------------------------------- preprocess
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_preprocess(name):
    G = synth.config_graph(name)
    A = host_mat(M.preprocess(dev(G)))
    R = O.preprocess(G)
    assert np.array_equal(A.colptr, R.colptr) and np.array_equal(A.rows, R.rows)
    np.testing.assert_allclose(A.vals, R.vals, rtol=1e-6)


def test_preprocess_empty_and_loops():
    G = synth.Csc(4, 4, np.array([0, 0, 1, 1, 3], np.int64), np.array([3, 0, 2], np.int32),
                  np.array([2.0, 1.0, 3.0], np.float32))
    A = host_mat(M.preprocess(dev(G)))
    R = O.preprocess(G)
    assert np.array_equal(A.colptr, R.colptr) and np.array_equal(A.rows, R.rows)
    np.testing.assert_allclose(A.vals, R.vals, rtol=1e-6)


# ---------------------------------------------------------------- expansion (P1, P2)
@pytest.mark.parametrize("seed", range(8))
def test_expand_random(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    A = synth.random_sparse(n, n, float(rng.uniform(0.001, 0.05)), seed=seed,
                            empty_cols=0.05, degree_skew=bool(seed % 2))
    Cg, st = M.expand(dev(A))
    Cr, fl = O.expand(A)
    assert_unpruned_parity(host_mat(Cg), Cr)
    assert st["flops"] == int(fl.sum())
    assert st["nnz_unpruned"] == Cr.nnz
    assert st["estimator_used"] == 3  # upper-bound slots, no symbolic pass


@pytest.mark.parametrize("sizing", ["exact_symbolic", "capacity_fallback"])
@pytest.mark.parametrize("seed", [1, 6])
def test_expand_sizing_paths(monkeypatch, sizing, seed):
    """Unfused products are sized by upper-bound slots min(f_j, m) + compaction by default;
    the exact symbolic pass runs when asked (MCLX_EXACT_SYMBOLIC) or when the slots would
    exceed the context's budget (MCLX_CAP_BUDGET_MB=0)."""
    if sizing == "exact_symbolic":
        monkeypatch.setenv("MCLX_EXACT_SYMBOLIC", "1")
    else:
        monkeypatch.setenv("MCLX_CAP_BUDGET_MB", "0")
    rng = np.random.default_rng(seed)
    n = int(rng.integers(500, 3000))
    A = synth.random_sparse(n, n, float(rng.uniform(0.001, 0.05)), seed=seed, empty_cols=0.05,
                            degree_skew=bool(seed % 2))
    ctx = M.Context()
    Cg, st = ctx.expand(dev(A))
    Cr, fl = O.expand(A)
    assert_unpruned_parity(host_mat(Cg), Cr)
    assert st["estimator_used"] == 1
    assert st["nnz_unpruned"] == Cr.nnz


@pytest.mark.parametrize("bin_", list(range(14)))
def test_expand_forced_bins(bin_):
    """Bin invariance (T2): every column forced into bin >= b (0-6: private row-range
    slices, 7-13: CTA-shared atomic table) gives the same product."""
    A = synth.random_sparse(700, 700, 0.02, seed=11, empty_cols=0.1)
    p = M.Params(force_bin=bin_)
    Cg, st = M.expand(dev(A), params=p)
    Cr, _ = O.expand(A)
    assert_unpruned_parity(host_mat(Cg), Cr)
    assert sum(st["bin_cols"][:bin_ % 7]) == 0


@pytest.mark.parametrize("seed", range(4))
def test_spgemm_rectangular_and_ranges(seed):
    rng = np.random.default_rng(40 + seed)
    m, p, n = (int(x) for x in rng.integers(1, 1500, size=3))
    A = synth.random_sparse(m, p, 0.01, seed=seed)
    B = synth.random_sparse(p, n, 0.01, seed=seed + 7, empty_cols=0.2)
    b = int(rng.integers(0, n))
    e = int(rng.integers(b, n + 1))
    Cg, _ = M.spgemm(dev(A), dev(B), (b, e))
    Cr, _ = O.spgemm(A, B, b, e)
    assert_unpruned_parity(host_mat(Cg), Cr)


def test_expand_empty_and_degenerate():
    Z = synth.Csc(5, 5, np.zeros(6, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    Cg, st = M.expand(dev(Z))
    assert Cg.nnz == 0 and st["flops"] == 0
    one = synth.Csc(1, 1, np.array([0, 1], np.int64), np.array([0], np.int32),
                    np.array([0.5], np.float32))
    Cg, _ = M.expand(dev(one))
    assert host_mat(Cg).vals.tolist() == [0.25]
    Cg, _ = M.expand(dev(one), cols=(0, 0))
    assert Cg.ncols == 0 and Cg.nnz == 0


def test_expand_hub_column_global_bin():
    """A dense hub (column with > 16384 terms -> fp64 global bin)."""
    n = 40000
    rng = np.random.default_rng(5)
    hub = np.sort(rng.choice(n, size=20000, replace=False))
    cols = [np.array([j]) for j in range(n)]
    cols[7] = np.union1d(hub, [7])
    cnt = np.array([len(c) for c in cols])
    cp = np.zeros(n + 1, np.int64)
    np.cumsum(cnt, out=cp[1:])
    rows = np.concatenate(cols).astype(np.int32)
    vals = rng.uniform(0.01, 1, size=rows.size).astype(np.float32)
    A = synth.Csc(n, n, cp, rows, vals)
    Cg, st = M.expand(dev(A))
    Cr, _ = O.expand(A)
    assert_unpruned_parity(host_mat(Cg), Cr)
    assert st["bin_cols"][6] >= 1


def test_symbolic_and_flops():
    A = synth.random_sparse(2000, 2000, 0.01, seed=3, degree_skew=True)
    nnz, tot = M.symbolic(dev(A))
    Cr, fl = O.expand(A)
    assert np.array_equal(nnz.cpu().numpy(), np.diff(Cr.colptr))
    assert tot == Cr.nnz
    f, ftot = M.flops(dev(A))
    assert np.array_equal(f.cpu().numpy(), fl) and ftot == int(fl.sum())


@pytest.mark.parametrize("L", [1, 2, 3, 5])
def test_merge_partials(L):
    """Device merge (Alg. 2's "merge all lists") equals the oracle's list merge."""
    mats = [synth.random_sparse(3000, 2500, 0.004, seed=50 + s, empty_cols=0.2) for s in range(L)]
    Mg = M.merge([dev(m) for m in mats])
    Mo = O.merge(mats)
    assert_unpruned_parity(host_mat(Mg), Mo, rtol=1e-6)


# ---------------------------------------------------------------- Cohen (P5)
@pytest.mark.parametrize("r,seed", [(3, 1), (10, 7), (16, 123456789)])
def test_cohen_keys_and_estimates(r, seed):
    A = synth.random_sparse(3000, 2500, 0.003, seed=seed % 1000, empty_cols=0.05)
    B = synth.random_sparse(2500, 2000, 0.003, seed=seed % 1000 + 1, empty_cols=0.05)
    est, tot, keys = M.estimate(dev(A), dev(B), r=r, seed=seed, return_keys=True)
    eo, ko, _ = O.cohen(A, B, r=r, seed=seed, return_keys=True)
    kg = keys.cpu().numpy()
    mism = kg != ko
    assert mism.mean() < 1e-4
    if mism.any():
        ulps = np.abs(kg.view(np.int32)[mism] - ko.view(np.int32)[mism])
        assert ulps.max() <= 1
    eg = est.cpu().numpy().astype(np.float64)
    np.testing.assert_allclose(eg, eo, rtol=1e-6)
    assert tot == pytest.approx(eo.sum(), rel=1e-6)


# ---------------------------------------------------------------- prune / inflate (P3)
PRUNE_CASES = [(1e-4, 1100, 1400, 0.9), (1e-4, 100, 100, 0.9), (1e-3, 20, 0, 0.9),
               (0.05, 3, 30, 0.5), (0.0, 7, 0, 0.9)]


@pytest.mark.parametrize("params", PRUNE_CASES)
def test_prune_inflate_identical_inputs(params):
    """Same fp32 C on both sides: selection is exact on both, so kept sets must be equal."""
    theta, S, R, pct = params
    A = O.preprocess(synth.planted_partition())
    Cr, _ = O.expand(A)
    # plant exact ties and a few empty columns
    idx = np.arange(0, Cr.vals.size - 1, 97)
    Cr.vals[idx] = Cr.vals[idx + 1]
    C32 = f32(Cr)
    Ag, st, chaos = M.prune_inflate(dev(C32), M.Params(prune_threshold=theta, select_k=S,
                                                       recover_k=R, recover_pct=pct),
                                    return_chaos=True)
    Ao, info = O.prune_inflate(C32, theta, S, R, pct, 2.0)
    G = host_mat(Ag)
    assert np.array_equal(G.colptr, Ao.colptr) and np.array_equal(G.rows, Ao.rows)
    np.testing.assert_allclose(G.vals, Ao.vals, rtol=1e-5)
    np.testing.assert_allclose(chaos.cpu().numpy(), info.chaos, rtol=1e-4, atol=1e-6)
    assert st["chaos"] == pytest.approx(info.chaos.max(), rel=1e-4, abs=1e-6)


def test_prune_big_columns():
    """Columns far larger than any shared-memory bin (standalone prune reads global)."""
    rng = np.random.default_rng(9)
    n, ncol = 200000, 6
    cols = [np.sort(rng.choice(n, size=s, replace=False)) for s in (1, 50, 5000, 60000, 150000, 0)]
    cnt = np.array([len(c) for c in cols])
    cp = np.zeros(ncol + 1, np.int64)
    np.cumsum(cnt, out=cp[1:])
    vals = (rng.exponential(size=cnt.sum()) ** 4).astype(np.float32)
    Cm = synth.Csc(n, ncol, cp, np.concatenate(cols).astype(np.int32), vals)
    for params in PRUNE_CASES:
        theta, S, R, pct = params
        Ag, _ = M.prune_inflate(dev(Cm), M.Params(prune_threshold=theta, select_k=S, recover_k=R,
                                                  recover_pct=pct))
        Ao, _ = O.prune_inflate(O.as_mat(Cm), theta, S, R, pct, 2.0)
        G = host_mat(Ag)
        assert np.array_equal(G.colptr, Ao.colptr) and np.array_equal(G.rows, Ao.rows)
        np.testing.assert_allclose(G.vals, Ao.vals, rtol=1e-5)


# ---------------------------------------------------------------- fused iterate (P1-P3)
@pytest.mark.parametrize("estimator", [1, 2])
@pytest.mark.parametrize("name,params", [("C1", (1e-4, 1100, 1400, 0.9)),
                                         ("C2", (1e-4, 100, 100, 0.9))])
def test_iterate_step_parity(name, params, estimator):
    theta, S, R, pct = params
    A = f32(O.preprocess(synth.config_graph(name)))
    Ag, st = M.iterate(dev(A), M.Params(prune_threshold=theta, select_k=S, recover_k=R,
                                        recover_pct=pct, estimator=estimator))
    Cr, fl = oexp(A)
    _, info = opi(Cr, theta, S, R, pct, 2.0)
    stats = kept_parity(host_mat(Ag), Cr, info, params)
    assert st["flops"] == int(fl.sum())
    assert st["chaos"] == pytest.approx(info.chaos.max(), rel=1e-3, abs=1e-5)
    assert stats["band_flip_cols"] <= max(2, A.ncols // 1000)


def test_iterate_c1_second_iteration_all_bins():
    """Iteration 1 of C1 expands to ~1e6 nnz (dense columns); force each bin."""
    A0 = O.preprocess(synth.planted_partition())
    Cr, _ = O.expand(A0)
    A1, _ = O.prune_inflate(Cr, 1e-4, 1100, 1400, 0.9, 2.0)
    A1 = f32(A1)
    Cr1, _ = O.expand(A1)
    _, info = O.prune_inflate(Cr1, 1e-4, 1100, 1400, 0.9, 2.0)
    for b in (-1, 3, 5, 6, 8, 10, 12, 13):
        Ag, st = M.iterate(dev(A1), M.Params(force_bin=b, estimator=2))
        kept_parity(host_mat(Ag), Cr1, info, (1e-4, 1100, 1400, 0.9))


def test_iterate_label_locality():
    """Vertices numbered family by family: a column's output rows crowd into one warp's
    row range, so private row-range slices overflow and the columns must be re-run in the
    CTA-shared-table family (regression: this used to fail after exact re-binning)."""
    A = f32(O.preprocess(synth.protein_like(n=30_000, seed=5, permute=False)))
    Ag, st = M.iterate(dev(A), M.Params())
    Cr, fl = oexp(A)
    _, info = opi(Cr, 1e-4, 1100, 1400, 0.9, 2.0)
    kept_parity(host_mat(Ag), Cr, info, (1e-4, 1100, 1400, 0.9))
    assert st["flops"] == int(fl.sum())
    assert st["retries"] > 0


@pytest.mark.parametrize("graph,min_need,part_need,budget_mb,fp64_terms", [
    ("C2", 600, 0, 0, 0), ("rmat14", 200, 0, 0, 0), ("C1it1", 100, 0, 0, 0),
    ("C2", 600, 64, 0, 0), ("rmat14", 200, 16, 2, 0), ("C1it1", 100, 16, 0, 0),
    ("C2", 600, 0, 0, 64), ("rmat14", 200, 0, 0, 32), ("C1it1", 100, 0, 0, -1)])
def test_iterate_split_columns(monkeypatch, graph, min_need, part_need, budget_mb, fp64_terms):
    """Row-range split columns (parts stitched, pruned by k_prune), forced onto every
    column with need > min_need.  part_need > 0 shrinks the parts' target size so the
    variants with 32 parts of 2x tables and of dense fp32 row tiles run; fp64_terms > 0
    lowers the long-sum threshold so columns run as dense fp64 tiles; budget_mb > 0
    forces many chunks."""
    monkeypatch.setenv("MCLX_SPLIT_MIN_NEED", str(min_need))
    if fp64_terms > 0:
        monkeypatch.setenv("MCLX_FP64_TERMS", str(fp64_terms))
    if fp64_terms < 0:  # parts of P <= 4 in the CTA-shared family instead of private slices
        monkeypatch.setenv("MCLX_SPLIT_PRIVATE", "0")
    if part_need:
        monkeypatch.setenv("MCLX_SPLIT_PART_NEED", str(part_need))
    if budget_mb:
        monkeypatch.setenv("MCLX_SPLIT_BUDGET_MB", str(budget_mb))
    if graph == "C2":
        A, params = f32(O.preprocess(synth.config_graph("C2"))), (1e-4, 100, 100, 0.9)
    elif graph == "rmat14":
        A, params = f32(O.preprocess(synth.rmat(scale=14, seed=4))), (1e-4, 1100, 1400, 0.9)
    else:
        A, params = c1_it1(), (1e-4, 1100, 1400, 0.9)
    theta, S, R, pct = params
    ctx = M.Context()  # fresh context: the env knobs are read at creation
    Ag, st = ctx.iterate(dev(A), M.Params(prune_threshold=theta, select_k=S, recover_k=R,
                                          recover_pct=pct))
    Cr, fl = oexp(A)
    _, info = opi(Cr, theta, S, R, pct, 2.0)
    kept_parity(host_mat(Ag), Cr, info, params)
    assert st["flops"] == int(fl.sum())
    assert st["chaos"] == pytest.approx(info.chaos.max(), rel=1e-3, abs=1e-5)
    assert st["bin_cols"][6] > 0


@pytest.mark.parametrize("scale", [12, 14])
def test_rmat_iterate_parity(scale):
    """R-MAT (C4 shape: skewed degrees, hub columns) -- one fused iteration vs the oracle."""
    A = f32(O.preprocess(synth.rmat(scale=scale, seed=4)))
    Ag, st = M.iterate(dev(A), M.Params())
    Cr, fl = oexp(A)
    _, info = opi(Cr, 1e-4, 1100, 1400, 0.9, 2.0)
    kept_parity(host_mat(Ag), Cr, info, (1e-4, 1100, 1400, 0.9))
    assert st["flops"] == int(fl.sum())


def test_global_bin_chunked(monkeypatch):
    """fp64 global-memory bin processed in memory-bounded chunks (R-MAT hubs)."""
    monkeypatch.setenv("MCLX_GBIN_BUDGET_MB", "1")
    ctx = M.Context()
    A0 = O.preprocess(synth.planted_partition())
    Cr, _ = O.expand(A0)
    A1, _ = O.prune_inflate(Cr, 1e-4, 1100, 1400, 0.9, 2.0)
    A1 = f32(A1)
    Cg, st = ctx.expand(dev(A1), params=M.Params(force_bin=6))
    Cr1, _ = O.expand(A1)
    assert_unpruned_parity(host_mat(Cg), Cr1)
    assert st["bin_cols"][6] == A1.ncols
    Ag, st = ctx.iterate(dev(A1), M.Params(force_bin=6))
    _, info = O.prune_inflate(Cr1, 1e-4, 1100, 1400, 0.9, 2.0)
    kept_parity(host_mat(Ag), Cr1, info, (1e-4, 1100, 1400, 0.9))
    ctx.close()


# ---------------------------------------------------------------- clusters (P4)
@pytest.mark.parametrize("seed", range(4))
def test_clusters_random(seed):
    Mx = synth.random_sparse(5000, 5000, 0.0003, seed=seed, empty_cols=0.3)
    lab, k = M.clusters(dev(Mx))
    lo, ko = O.clusters(Mx)
    assert k == ko and np.array_equal(lab.cpu().numpy(), lo)


@pytest.mark.parametrize("name,params", [("C1", (1e-4, 1100, 1400, 0.9)),
                                         ("C2", (1e-4, 100, 100, 0.9))])
def test_full_mcl_clusters_equal(name, params):
    theta, S, R, pct = params
    G = synth.config_graph(name)
    p = M.Params(prune_threshold=theta, select_k=S, recover_k=R, recover_pct=pct)
    labels, k, hist, _ = M.run(dev(G), p)
    ref = O.mcl(G, theta=theta, S=S, R=R, pct=pct, eps=1e-3)
    assert k == ref.nclusters
    assert np.array_equal(labels.cpu().numpy(), ref.labels)
    assert abs(len(hist) - ref.iterations) <= 1


@pytest.mark.slow
@pytest.mark.parametrize("shape", ["protein_n5000", "rmat_s12"])
def test_full_mcl_clusters_equal_small_c3_c4_shapes(shape):
    """P4 on the C3/C5 (protein-like) and C4 (R-MAT) generators at sizes where the
    single-threaded oracle runs MCL to convergence in seconds: identical clusters."""
    G = synth.protein_like(n=5000, seed=3) if shape == "protein_n5000" else synth.rmat(scale=12, seed=4)
    p = M.Params()
    labels, k, hist, _ = M.run(dev(G), p)
    ref = O.mcl(G, theta=1e-4, S=1100, R=1400, pct=0.9, eps=1e-3)
    assert k == ref.nclusters
    assert np.array_equal(labels.cpu().numpy(), ref.labels)
    assert abs(len(hist) - ref.iterations) <= 1


@pytest.mark.parametrize("graph", ["rmat14", "C1it1"])
def test_iterate_split_columns_all_entries(monkeypatch, graph):
    """Split parts that stage every entry (MCLX_SPLIT_CAND=0) instead of their top max(S, R)
    candidates plus statistics: the same kept sets as the oracle."""
    monkeypatch.setenv("MCLX_SPLIT_CAND", "0")
    monkeypatch.setenv("MCLX_SPLIT_MIN_NEED", "100")
    monkeypatch.setenv("MCLX_SPLIT_PART_NEED", "16")
    if graph == "rmat14":
        A = f32(O.preprocess(synth.rmat(scale=14, seed=4)))
    else:
        A0 = O.preprocess(synth.planted_partition())
        A, _ = O.prune_inflate(O.expand(A0)[0], 1e-4, 1100, 1400, 0.9, 2.0)
        A = f32(A)
    ctx = M.Context()
    Ag, st = ctx.iterate(dev(A), M.Params())
    Cr, fl = oexp(A)
    _, info = opi(Cr, 1e-4, 1100, 1400, 0.9, 2.0)
    kept_parity(host_mat(Ag), Cr, info, (1e-4, 1100, 1400, 0.9))
    assert st["split_cols"] > 0


@pytest.mark.parametrize("seed", range(3))
def test_esc_low_cf_columns(monkeypatch, seed):
    """Expand-sort-compress (kernels_esc.cu), forced onto every column with <= 1024 products
    (MCLX_ESC_CF huge, and the per-product gate MCLX_ESC_ITER_CF open): unpruned product
    bit-exact in structure, exact symbolic counts, and the fused iterate equal to the oracle's."""
    monkeypatch.setenv("MCLX_ESC_CF", "1e9")
    monkeypatch.setenv("MCLX_ESC_ITER_CF", "inf")
    rng = np.random.default_rng(70 + seed)
    n = int(rng.integers(200, 3000))
    A = synth.random_sparse(n, n, float(rng.uniform(0.002, 0.01)), seed=seed, empty_cols=0.05,
                            degree_skew=bool(seed % 2))
    ctx = M.Context()
    Cg, st = ctx.expand(dev(A))
    Cr, fl = O.expand(A)
    assert_unpruned_parity(host_mat(Cg), Cr)
    assert st["esc_cols"] > 0 and st["esc_flops"] <= int(fl.sum())
    nnz, tot = ctx.symbolic(dev(A))
    assert np.array_equal(nnz.cpu().numpy(), np.diff(Cr.colptr))
    A1 = O.preprocess(synth.protein_like(n=3000, seed=seed))
    for it in range(6):  # skip to the late, low-cf iterations ESC is for (the oracle's iterates)
        A1, _ = O.prune_inflate(O.expand(A1)[0], 1e-4, 1100, 1400, 0.9, 2.0)
    A1 = f32(A1)
    esc = 0
    for it in range(4):  # MCL iterations 6-9: cf falls towards 1, most columns take ESC
        C1, _ = O.expand(A1)
        Ag, st = ctx.iterate(dev(A1), M.Params())
        _, info = O.prune_inflate(C1, 1e-4, 1100, 1400, 0.9, 2.0)
        kept_parity(host_mat(Ag), C1, info, (1e-4, 1100, 1400, 0.9))
        esc += st["esc_cols"]
        A1, _ = O.prune_inflate(C1, 1e-4, 1100, 1400, 0.9, 2.0)
        A1 = f32(A1)
    assert esc > 0
    ctx.close()


@pytest.mark.parametrize("graph", ["rmat14", "C1it1"])
def test_iterate_dense_sweep_threshold(monkeypatch, graph):
    """Every split column swept with dense tiles (MCLX_DENSE_MIN_P=1), candidates on."""
    monkeypatch.setenv("MCLX_DENSE_MIN_P", "1")
    monkeypatch.setenv("MCLX_SPLIT_MIN_NEED", "100")
    A = f32(O.preprocess(synth.rmat(scale=14, seed=4))) if graph == "rmat14" else c1_it1()
    ctx = M.Context()
    Ag, st = ctx.iterate(dev(A), M.Params())
    Cr, fl = oexp(A)
    _, info = opi(Cr, 1e-4, 1100, 1400, 0.9, 2.0)
    kept_parity(host_mat(Ag), Cr, info, (1e-4, 1100, 1400, 0.9))
    assert st["split_vcols"][2] == st["split_cols"] > 0
