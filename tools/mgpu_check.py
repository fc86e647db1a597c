#!/usr/bin/env python
"""Multi-GPU parity of the 2D Sparse-SUMMA iteration (mcl_summa_iterate) against the oracle.

Run under torchrun, one rank per GPU, e.g.
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
      --master-port 29512 tools/mgpu_check.py --grids 1x2,2x1

For each grid and config: every rank builds the full A_0 on its GPU, keeps its block,
runs SUMMA iterations; blocks are gathered to rank 0 and compared with the oracle
(one step: kept sets / values as in tests/test_gpu_parity.py; full MCL: identical
cluster labels).  Prints one PASS/FAIL line per case; exit code 1 on any failure.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2002_10083_b200 as M  # noqa: E402
import synth  # noqa: E402
from paper_2002_10083_b200.grid import Grid  # noqa: E402

PARAMS = {"C1": (1e-4, 1100, 1400, 0.9), "C2": (1e-4, 100, 100, 0.9)}


def gather_full(blk, g: Grid, n, world):
    """Stitch the grid's blocks into a full host CSC on every rank (small configs only)."""
    cp, rw, vl = blk.to_host()
    parts = [None] * world
    dist.all_gather_object(parts, (g.i, g.j, cp, rw, vl))
    cols = [[] for _ in range(n)]
    for (i, j, pcp, prw, pvl) in parts:
        r0, _ = g.rows(n, i)
        c0, _ = g.cols(n, j)
        for jj in range(len(pcp) - 1):
            a, b = pcp[jj], pcp[jj + 1]
            cols[c0 + jj].append((prw[a:b].astype(np.int64) + r0, pvl[a:b]))
    colptr = [0]
    rows, vals = [], []
    for lst in cols:
        if lst:
            r = np.concatenate([x[0] for x in lst])
            v = np.concatenate([x[1] for x in lst])
            o = np.argsort(r, kind="stable")
            rows.append(r[o])
            vals.append(v[o])
            colptr.append(colptr[-1] + len(r))
        else:
            colptr.append(colptr[-1])
    import oracle as O
    return O.Mat(n, n, np.array(colptr, np.int64),
                 np.concatenate(rows).astype(np.int32) if rows else np.zeros(0, np.int32),
                 np.concatenate(vals).astype(np.float64) if vals else np.zeros(0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grids", default="1x2,2x1")
    ap.add_argument("--configs", default="C1,C2")
    args = ap.parse_args()
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import oracle as O
    ctx = M.context()
    failures = 0
    for grid in args.grids.split(","):
        pr, pc = (int(x) for x in grid.split("x"))
        if pr * pc != world:
            continue
        uid = [M.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx.set_grid(pr, pc, rank, uid[0])
        g = Grid(pr, pc, rank)
        for cfg in args.configs.split(","):
            theta, S, R, pct = PARAMS[cfg]
            p = M.Params(prune_threshold=theta, select_k=S, recover_k=R, recover_pct=pct)
            G = synth.config_graph(cfg)
            A = ctx.preprocess(M.CSC.from_host(G))
            n = A.ncols
            blk = ctx.block(A, g.rows(n), g.cols(n))
            # ---- one step, same fp32 input on both sides
            A0 = gather_full(blk, g, n, world)
            nxt, st = ctx.summa_iterate(blk, p)
            G1 = gather_full(nxt, g, n, world)
            ok = True
            if rank == 0:
                Cr, _ = O.expand(A0)
                Ao, info = O.prune_inflate(Cr, theta, S, R, pct, 2.0)
                flips = 0
                for j in range(n):
                    gr = G1.rows[G1.colptr[j]:G1.colptr[j + 1]]
                    orow = Ao.rows[Ao.colptr[j]:Ao.colptr[j + 1]]
                    if np.array_equal(gr, orow):
                        gv = G1.vals[G1.colptr[j]:G1.colptr[j + 1]]
                        ov = Ao.vals[Ao.colptr[j]:Ao.colptr[j + 1]]
                        if np.max(np.abs(gv - ov) / ov) > 1e-5:
                            ok = False
                        continue
                    cr = Cr.rows[Cr.colptr[j]:Cr.colptr[j + 1]]
                    cv = Cr.vals[Cr.colptr[j]:Cr.colptr[j + 1]]
                    d = np.setxor1d(gr, orow)
                    if not np.all(np.abs(cv[np.searchsorted(cr, d)] - info.tau[j]) <= 1e-6):
                        ok = False
                    flips += 1
                chaos_ok = abs(st["chaos"] - info.chaos.max()) <= 1e-3 * max(1, info.chaos.max())
                ok = ok and chaos_ok
                print(f"{'PASS' if ok else 'FAIL'} step  grid={grid} {cfg}: nnz={G1.nnz} "
                      f"(oracle {Ao.nnz}) band_flip_cols={flips} chaos={st['chaos']:.4g} "
                      f"(oracle {info.chaos.max():.4g}) comm_bytes={st['comm_bytes']}", flush=True)
            # ---- full MCL to convergence; clusters on the gathered final iterate
            blk2 = blk
            iters = 0
            for it in range(100):
                blk2, st = ctx.summa_iterate(blk2, p)
                iters += 1
                if st["chaos"] < p.chaos_eps:
                    break
            Af = gather_full(blk2, g, n, world)
            if rank == 0:
                labels, k = O.clusters(Af)
                ref = O.mcl(G, theta=theta, S=S, R=R, pct=pct, eps=1e-3)
                same = k == ref.nclusters and np.array_equal(labels, ref.labels)
                ok = ok and same
                print(f"{'PASS' if same else 'FAIL'} mcl   grid={grid} {cfg}: clusters={k} "
                      f"(oracle {ref.nclusters}) iterations={iters} (oracle {ref.iterations})",
                      flush=True)
            failures += 0 if ok else 1
            dist.barrier()
    f = torch.tensor([failures], device="cuda")
    dist.all_reduce(f)
    dist.destroy_process_group()
    sys.exit(1 if int(f.item()) else 0)


if __name__ == "__main__":
    main()
