"""Host wall time vs device time of fused iterations (diagnoses host-side stalls)."""
import os, sys, time
sys.path.insert(0, ".")
import torch, synth
import paper_2002_10083_b200 as M
it = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ctx = M.context()
A = ctx.preprocess(M.CSC.from_host(synth.config_graph("C3")))
for _ in range(it):
    A, _ = ctx.iterate(A, M.Params())
for k in range(6):
    torch.cuda.synchronize(); t = time.perf_counter()
    An, st = ctx.iterate(A, M.Params())
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) * 1e3
    print(f"it{it} host {dt:.2f} ms  device total {st['ms'][6]:.2f} ms  ms={['%.2f' % x for x in st['ms']]} esc={st['esc_cols']} esc_ms={st['esc_ms']:.2f} phases={st['phases']} launches={st['launches']}", flush=True)
    del An
