"""Time C4 (R-MAT scale 22) pieces on one GPU: fused iterate, symbolic, expand of a column range."""
import sys, time, json
sys.path.insert(0, ".")
import torch, synth
import paper_2002_10083_b200 as M
t = time.time(); G = synth.config_graph("C4"); print("gen", time.time() - t, G.nnz, flush=True)
ctx = M.context()
A = ctx.preprocess(M.CSC.from_host(G)); del G
def timed(f):
    torch.cuda.synchronize(); t = time.time(); r = f(); torch.cuda.synchronize(); return r, time.time() - t
(An, st), dt = timed(lambda: ctx.iterate(A, M.Params()))
print("iterate", dt, {k: st[k] for k in ("flops", "nnz_out", "retries", "split_cols", "split_ms", "bin_ms", "split_vcols", "split_vms", "ms", "peak_bytes")}, flush=True)
del An
(An, st), dt = timed(lambda: ctx.iterate(A, M.Params()))
print("iterate2", dt, st["ms"][6], flush=True)
del An
(r, dt) = timed(lambda: ctx.symbolic(A))
print("symbolic", dt, r[1], flush=True)
