"""Phases (§II "Overview of HipMCL": the product is formed in phases of column
batches; P:575-579 / P:594-595 §V: the estimate sizes them; reading Q15) and the staged
2D Sparse-SUMMA path (Alg. 2, distributed prune P:209) on ONE GPU.

* mcl_iterate with h forced column batches (MCLX_PHASES) or a tiny memory budget
  (MCLX_PHASE_BUDGET_MB) gives the oracle's iterate (P3), and reports stats.phases = h.
* mcl_summa_iterate on a 1 x 1 grid with the staged path (MCLX_SUMMA_STAGED=1) and s = 4
  inner panels (MCLX_SUMMA_STAGES=4): four stage products per phase, Alg. 2's binary merges
  after stages 2 and 4, and the distributed prune (no communicator) -- against the oracle,
  with 1 and 3 phases.
"""
import numpy as np
import pytest
import torch

import oracle as O
import synth
from test_gpu_parity import c1_it1, dev, f32, host_mat, kept_parity, oexp, opi

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    import paper_2002_10083_b200 as M

CASES = {"C1": (1e-4, 1100, 1400, 0.9), "C2": (1e-4, 100, 100, 0.9)}


def _params(prm):
    theta, S, R, pct = prm
    return M.Params(prune_threshold=theta, select_k=S, recover_k=R, recover_pct=pct)


def _input(name):
    if name == "C1it1":  # C1's first iterate: dense columns, every bin
        return c1_it1(), CASES["C1"]
    return f32(O.preprocess(synth.config_graph(name))), CASES[name]


@pytest.mark.parametrize("name", ["C1it1", "C2"])
@pytest.mark.parametrize("h", [1, 2, 4])
def test_iterate_phase_invariance(monkeypatch, name, h):
    monkeypatch.setenv("MCLX_PHASES", str(h))
    A, prm = _input(name)
    ctx = M.Context()
    Ag, st = ctx.iterate(dev(A), _params(prm))
    Cr, fl = oexp(A)
    _, info = opi(Cr, *prm, 2.0)
    kept_parity(host_mat(Ag), Cr, info, prm)
    assert st["phases"] == h
    assert st["flops"] == int(fl.sum())
    assert st["chaos"] == pytest.approx(info.chaos.max(), rel=1e-3, abs=1e-5)
    ctx.close()


def test_iterate_phases_from_budget(monkeypatch):
    """The planner cuts by memory: 16 B x min(max(S,R), f_j, m) per column against a 1 MB
    budget gives several batches, and the result is unchanged."""
    monkeypatch.setenv("MCLX_PHASE_BUDGET_MB", "1")
    A, prm = _input("C2")
    ctx = M.Context()
    Ag, st = ctx.iterate(dev(A), _params(prm))
    f = np.zeros(A.ncols, np.int64)
    deg = np.diff(A.colptr)
    np.add.at(f, np.repeat(np.arange(A.ncols), deg), deg[A.rows])
    need = int((16 * np.minimum(np.minimum(f, A.nrows), max(prm[1], prm[2])) + 16).sum())
    assert st["phases"] == -(-need // (1 << 20))
    Cr, _ = oexp(A)
    _, info = opi(Cr, *prm, 2.0)
    kept_parity(host_mat(Ag), Cr, info, prm)
    ctx.close()


@pytest.mark.parametrize("name", ["C1it1", "C2"])
@pytest.mark.parametrize("phases", [1, 3])
@pytest.mark.parametrize("form", ["staged", "accumulating"])
def test_summa_staged_1x1(monkeypatch, name, phases, form):
    """form staged: one product per stage + Alg. 2 merges; accumulating (the pr > 1 default,
    forced on 1 x 1 by MCLX_SUMMA_ACCUM): the 4 A-panels side by side and the 4 B-panels
    stacked, one product, then the distributed prune."""
    monkeypatch.setenv("MCLX_SUMMA_STAGED" if form == "staged" else "MCLX_SUMMA_ACCUM", "1")
    monkeypatch.setenv("MCLX_SUMMA_STAGES", "4")
    monkeypatch.setenv("MCLX_PHASES", str(phases))
    A, prm = _input(name)
    ctx = M.Context()
    ctx.set_grid(1, 1, 0, M.nccl_unique_id())
    blk = ctx.block(dev(A), (0, A.nrows), (0, A.ncols))
    Ag, st = ctx.summa_iterate(blk, _params(prm))
    Cr, fl = oexp(A)
    _, info = opi(Cr, *prm, 2.0)
    kept_parity(host_mat(Ag), Cr, info, prm)
    assert st["stages"] == 4 and st["phases"] == phases
    assert st["flops"] == int(fl.sum())
    assert st["nnz_unpruned"] == Cr.nnz
    # Alg. 2 on 4 stages keeps at most 3 lists alive (m12, l3, l4 before the last merge);
    # the accumulating form holds one phase's unpruned block
    assert 0 < st["peak_partial"] <= (3 if form == "staged" else 1) * Cr.nnz
    assert st["chaos"] == pytest.approx(info.chaos.max(), rel=1e-3, abs=1e-5)
    ctx.close()


@pytest.mark.parametrize("name", ["C1it1", "C2"])
@pytest.mark.parametrize("stages,phases", [(1, 1), (3, 1), (4, 3), (0, 0)])
def test_iterate_hostmem(name, stages, phases):
    """Host-memory-backed iteration (the Pipelined Sparse SUMMA of
    P:337-363 on one GPU): A in pinned host memory, column panels streamed in, Alg. 2 merges
    and the prune on the device, pruned phases back to host -- the oracle's iterate."""
    A, prm = _input(name)
    ctx = M.Context()
    G, st = ctx.iterate_hostmem(A, _params(prm), stages=stages, phases=phases)
    Cr, fl = oexp(A)
    _, info = opi(Cr, *prm, 2.0)
    kept_parity(O.Mat(G.nrows, G.ncols, G.colptr, G.rows, G.vals.astype(np.float64)), Cr, info, prm)
    assert st["flops"] == int(fl.sum()) and st["nnz_unpruned"] == Cr.nnz
    if stages > 0:
        assert st["stages"] == stages and st["phases"] == phases
        assert 0 < st["peak_partial"] <= 3 * Cr.nnz
    assert st["chaos"] == pytest.approx(info.chaos.max(), rel=1e-3, abs=1e-5)
    assert st["comm_bytes"] >= 8 * A.nnz  # every column panel crossed the host link
    ctx.close()


@pytest.mark.parametrize("graph,min_need,part_need", [("C2", 600, 0), ("C1it1", 100, 0),
                                                      ("rmat14", 200, 0), ("rmat14", 200, 16)])
def test_summa_candidates_split_path(monkeypatch, graph, min_need, part_need):
    """The pr > 1 product's candidate mode through the split path -- row-range parts (private /
    shared tables, and with part_need 16 the dense tiles) stage their top-max(S, R) plus
    statistics, the stitched columns are cut by k_cand_select, and the distributed prune
    finishes them -- on a forced 1 x 1 accumulating SUMMA with 2 panels, every column with
    need > min_need split."""
    monkeypatch.setenv("MCLX_SUMMA_ACCUM", "1")
    monkeypatch.setenv("MCLX_SUMMA_STAGES", "2")
    monkeypatch.setenv("MCLX_SPLIT_MIN_NEED", str(min_need))
    if part_need:
        monkeypatch.setenv("MCLX_SPLIT_PART_NEED", str(part_need))
    if graph == "rmat14":
        A, prm = f32(O.preprocess(synth.rmat(scale=14, seed=4))), CASES["C1"]
    else:
        A, prm = _input(graph)
    ctx = M.Context()
    ctx.set_grid(1, 1, 0, M.nccl_unique_id())
    blk = ctx.block(dev(A), (0, A.nrows), (0, A.ncols))
    Ag, st = ctx.summa_iterate(blk, _params(prm))
    Cr, fl = oexp(A)
    _, info = opi(Cr, *prm, 2.0)
    kept_parity(host_mat(Ag), Cr, info, prm)
    assert st["flops"] == int(fl.sum()) and st["nnz_unpruned"] == Cr.nnz
    assert st["bin_cols"][6] > 0  # columns ran as split parts
    assert st["chaos"] == pytest.approx(info.chaos.max(), rel=1e-3, abs=1e-5)
    ctx.close()
