"""Development: where does C4 (R-MAT) time go?  Per-bin times and the flops profile of
the columns that land in the global bin, at a reduced scale."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_10083_b200 as M  # noqa: E402
import synth  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 18
G = synth.rmat(scale=scale, seed=4)
ctx = M.context()
A = ctx.preprocess(M.CSC.from_host(G))
out, st = ctx.iterate(A, M.Params())
out, st = ctx.iterate(A, M.Params())
torch.cuda.synchronize()
print(f"scale {scale}: n={A.ncols} nnz={A.nnz} flops={st['flops']:.3e} fused ms={st['ms'][3]:.1f} "
      f"GF/s={2*st['flops']/st['ms'][3]/1e6:.1f}")
print("bin_cols ", st["bin_cols"])
print("bin_flops", [f"{x:.2e}" for x in st["bin_flops"]])
print("bin_ms   ", [round(x, 1) for x in st["bin_ms"]])
print(f"split: cols {st['split_cols']} items {st['split_items']} ms {st['split_ms']:.1f} retries {st['retries']}"
      f" per variant cols {st['split_vcols']} ms {[round(x, 1) for x in st['split_vms']]}")
# flops per column on the host (f_j = sum over k in A_*j of nnz(A_*k))
cp, rw, _ = A.to_host()
deg = np.diff(cp)
f = np.add.reduceat(deg[rw], cp[:-1]) if len(rw) else np.zeros(0)
f[deg == 0] = 0
fs = np.sort(f)[::-1]
print("top column flops", [f"{x:.2e}" for x in fs[:8]], "total", f"{f.sum():.3e}")
print("share of top 10/100/1000 columns", [round(fs[:k].sum() / f.sum(), 3) for k in (10, 100, 1000)])
