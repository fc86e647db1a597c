"""One fused iteration of C3 iteration 1 (the heaviest) after an untimed iteration 0."""
import sys
sys.path.insert(0, ".")
import torch, synth
import paper_2002_10083_b200 as M
A = M.preprocess(M.CSC.from_host(synth.config_graph("C3")))
A, _ = M.iterate(A, M.Params())
torch.cuda.synchronize()
An, st = M.iterate(A, M.Params())
torch.cuda.synchronize()
print({k: st[k] for k in ("flops", "split_cols", "split_vcols", "split_vms", "bin_ms", "ms")})
