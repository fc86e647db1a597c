"""C4 (R-MAT scale 22) iteration time for several dense-sweep thresholds (one generation)."""
import os, sys, time
sys.path.insert(0, ".")
import torch, synth
import paper_2002_10083_b200 as M
G = synth.config_graph("C4")
A = None
for p in sys.argv[1:] or ["64", "32"]:
    os.environ["MCLX_DENSE_MIN_P"] = p
    ctx = M.Context()
    if A is None:
        A = ctx.preprocess(M.CSC.from_host(G))
    ctx.iterate(A, M.Params())  # warm
    torch.cuda.synchronize(); t = time.time()
    An, st = ctx.iterate(A, M.Params())
    torch.cuda.synchronize()
    print(f"minP {p}: {time.time() - t:.2f} s", st["split_vcols"], [round(x / 1e3, 2) for x in st["split_vms"]], flush=True)
    del An
    ctx.close()
