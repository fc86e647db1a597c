"""Development: run one fused iteration with the -DMCLX_PROF build and print the kernel
counters (insert calls, probe passes, products, cycles).  Usage on a GPU box:
  cp tools/libmclx_prof.so paper_2002_10083_b200/libmclx.so && python tools/prof_counters.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_10083_b200 as M  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
G = synth.config_graph(cfg)
ctx = M.context()
A = ctx.preprocess(M.CSC.from_host(G))
out, st = ctx.iterate(A, M.Params())
M.prof_read(reset=True)
for fb in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["-1", "2", "4"])]:
    out, st = ctx.iterate(A, M.Params(force_bin=fb))
    torch.cuda.synchronize()
    v = M.prof_read(reset=True)
    calls, passes, prods, acyc, ecyc, cols = v[:6]
    cc = max(cols, 1)
    print(f"force_bin={fb:2d} ms={st['ms'][3]:7.2f} calls={calls} passes/call={passes/max(calls,1):.2f} "
          f"products/call={prods/max(calls,1):.1f} acc_cycles/product/warp={acyc/max(prods,1):.1f} "
          f"epi_cycles/col={ecyc/cc:.0f} [compact {v[6]/cc:.0f} select {v[7]/cc:.0f} sums {v[8]/cc:.0f} "
          f"sort+write {v[9]/cc:.0f}] cols={cols} bins={st['bin_cols']}")
