#!/usr/bin/env python
"""Time mcl_summa_iterate on a forced 1 x 1 grid (the accumulating form, MCLX_SUMMA_ACCUM=1 in
the environment) against the 1-GPU fused iteration on the same A: C3 iteration 0 by default."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2002_10083_b200 as M  # noqa: E402
import synth  # noqa: E402
from bench import CONFIG_PARAMS  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
G = synth.config_graph(cfg, 1.0)
ctx = M.context()
A = ctx.preprocess(M.CSC.from_host(G, device=torch.device("cuda", 0)))
params = M.Params(**CONFIG_PARAMS[cfg])
ctx.set_grid(1, 1, 0, M.nccl_unique_id())
blk = ctx.block(A, (0, A.nrows), (0, A.ncols))


def timeit(fn):
    for _ in range(2):
        out, st = fn()
        del out
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        out, st = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
        nnz = out.nnz
        del out
    return sorted(ts)[len(ts) // 2] * 1e3, st, nnz


ms_s, st_s, nnz_s = timeit(lambda: ctx.summa_iterate(blk, params))
ms_f, st_f, nnz_f = timeit(lambda: ctx.iterate(A, params))
print(f"{cfg} summa1x1 ms={ms_s:.1f} phases={st_s['phases']} nnz_out={nnz_s} unpruned={st_s['nnz_unpruned']}"
      f" peak_partial={st_s['peak_partial']}")
print(f"{cfg} fused    ms={ms_f:.1f} nnz_out={nnz_f} unpruned={st_f['nnz_unpruned']}")
