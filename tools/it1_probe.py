"""Development: C3 iteration 1 (the heaviest) -- split-path breakdown and part stats."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2002_10083_b200 as M  # noqa: E402
import synth  # noqa: E402

G = synth.config_graph("C3")
ctx = M.context()
A = ctx.preprocess(M.CSC.from_host(G))
p = M.Params()
A1, st0 = ctx.iterate(A, p)
for tag, env in (("default", {}), ("part_need 2048", {"MCLX_SPLIT_PART_NEED": "2048"})):
    for k, v in env.items():
        os.environ[k] = v
    c2 = M.Context()
    out, st = c2.iterate(A1, p)
    out, st = c2.iterate(A1, p)
    torch.cuda.synchronize()
    print(tag, f"flops={st['flops']:.3e} ms={st['ms'][3]:.1f} bin_cols={st['bin_cols']} "
          f"bin_ms={[round(x, 1) for x in st['bin_ms']]} split_cols={st['split_cols']} "
          f"items={st['split_items']} vcols={st['split_vcols']} vms={[round(x, 1) for x in st['split_vms']]} "
          f"retries={st['retries']} est={st['est_nnz']:.3e} nnz_out={st['nnz_out']}", flush=True)
    for k in env:
        del os.environ[k]
# flops per column of A1 products
cp, rw, _ = A1.to_host()
deg = np.diff(cp)
f = np.add.reduceat(deg[rw], cp[:-1]).astype(np.float64)
f[deg == 0] = 0
print("flops/col percentiles 50/90/99/max", np.percentile(f, [50, 90, 99]).round(), f.max())
