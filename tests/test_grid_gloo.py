"""Multi-process (gloo, world size 2, 4 and 8 on CPU) check of the Sparse-SUMMA schedule that
libmclx.so's mcl_summa_iterate runs (block ranges, inner panels, panel owners, Alg. 2 merge
points, read from the library's mcl_summa_schedule through paper_2002_10083_b200.grid): every
rank holds only its block, owners broadcast the panels the schedule names, each rank
multiplies them (oracle spgemm) and merges the stage partials where the schedule says; the
result must equal the oracle's A.A restricted to the block (C_ij = sum_k A_ik
B_kj).  The device products and NCCL broadcasts themselves are covered by the GPU tests and
the torchrun logs (profiles/r2_mgpu/)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth
from paper_2002_10083_b200.grid import Grid


def _sub(M, r0, r1, c0, c1):
    cp, rows, vals = [0], [], []
    for j in range(c0, c1):
        a, b = int(M.colptr[j]), int(M.colptr[j + 1])
        rr = M.rows[a:b]
        sel = (rr >= r0) & (rr < r1)
        rows.append(rr[sel] - r0)
        vals.append(M.vals[a:b][sel])
        cp.append(cp[-1] + int(sel.sum()))
    return O.Mat(r1 - r0, c1 - c0, np.array(cp, np.int64),
                 np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32),
                 np.concatenate(vals) if vals else np.zeros(0))


def _worker(rank, world, pr, pc, port, errq, mult=1):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        g = Grid(pr, pc, rank, mult)
        A = O.preprocess(synth.planted_partition())
        n = A.ncols
        r0, r1 = g.rows(n)
        c0, c1 = g.cols(n)
        mine = _sub(A, r0, r1, c0, c1)          # all this rank may read from now on
        row_groups = [dist.new_group([i * pc + j for j in range(pc)]) for i in range(pr)]
        col_groups = [dist.new_group([i * pc + j for i in range(pr)]) for j in range(pc)]
        stack = []
        for q in range(g.s):
            k0, k1 = g.panel(n, q)
            ca, rb = g.a_owner_col(q), g.b_owner_row(q)
            pa = [_sub(mine, 0, r1 - r0, k0 - c0, k1 - c0) if ca == g.j else None]
            pb = [_sub(mine, k0 - r0, k1 - r0, 0, c1 - c0) if rb == g.i else None]
            dist.broadcast_object_list(pa, src=g.i * pc + ca, group=row_groups[g.i])
            dist.broadcast_object_list(pb, src=rb * pc + g.j, group=col_groups[g.j])
            P, _ = O.spgemm(pa[0], pb[0])
            stack.append(P)
            nm = g.nmerges(q)
            if nm:
                L = [stack.pop() for _ in range(nm + 1)][::-1]
                stack.append(O.merge(L))
        Cb = stack.pop() if len(stack) == 1 else O.merge(stack)
        full, _ = O.expand(A)
        ref = _sub(full, r0, r1, c0, c1)
        assert np.array_equal(Cb.colptr, ref.colptr) and np.array_equal(Cb.rows, ref.rows)
        np.testing.assert_allclose(Cb.vals, ref.vals, rtol=1e-12)
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        errq.put(f"rank {rank}: {e!r}")
        raise


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("pr,pc,mult", [(1, 2, 1), (2, 1, 1), (2, 2, 1), (1, 4, 1), (1, 8, 1),
                                         (2, 4, 1), (2, 2, 2)])
def test_summa_schedule_gloo(pr, pc, mult):
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    world = pr * pc
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, pr, pc, port, errq, mult))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    codes = [p.exitcode for p in procs]
    msgs = []
    while not errq.empty():
        msgs.append(errq.get())
    assert codes == [0] * world, (codes, msgs)


def test_grid_arithmetic_matches_paper_square_case():
    # square grid, s = sqrt(P): stage k uses A_ik from p_ik and B_kj from p_kj
    for rank in range(4):
        g = Grid(2, 2, rank)
        assert g.s == 2
        for q in range(2):
            assert g.a_owner_col(q) == q and g.b_owner_row(q) == q
    g = Grid(2, 4, 5)
    assert g.s == 4 and (g.i, g.j) == (1, 1)
    assert [g.a_owner_col(q) for q in range(4)] == [0, 1, 2, 3]
    assert [g.b_owner_row(q) for q in range(4)] == [0, 0, 1, 1]
    assert [g.nmerges(q) for q in range(4)] == [0, 1, 0, 2]  # Alg. 2 trace
    # every inner panel lies inside one row stripe and one column stripe (Q17)
    for pr, pc, m in [(2, 4, 1), (4, 2, 1), (3, 2, 2)]:
        for r in range(pr * pc):
            g = Grid(pr, pc, r, m)
            n = 1000
            for q in range(g.s):
                k0, k1 = g.panel(n, q)
                c0, c1 = g.cols(n, g.a_owner_col(q))
                r0, r1 = g.rows(n, g.b_owner_row(q))
                assert c0 <= k0 < k1 <= c1 and r0 <= k0 < k1 <= r1


def test_bench_default_grids_are_the_north_stars():
    """bench.py --gpus N runs BASELINE.json's grids (1x1, 1x2, 2x2, 2x4); other N run 1xN."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location(
        "bench_mod", os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    saved = os.environ.get("PYTORCH_CUDA_ALLOC_CONF")
    spec.loader.exec_module(bench)  # (bench.py sets the allocator config; undo it here)
    if saved is None:
        os.environ.pop("PYTORCH_CUDA_ALLOC_CONF", None)
    else:
        os.environ["PYTORCH_CUDA_ALLOC_CONF"] = saved
    assert [bench.default_grid(n) for n in (1, 2, 4, 8)] == [(1, 1), (1, 2), (2, 2), (2, 4)]
    assert bench.default_grid(3) == (1, 3) and bench.default_grid(6) == (1, 6)
