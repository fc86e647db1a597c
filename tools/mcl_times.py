"""Per-iteration device times of full MCL on one GPU (Alg. 1 driven from Python):
python tools/mcl_times.py C3 [max_iter]  -> one JSON line per iteration + a summary."""
import json, sys, time
sys.path.insert(0, ".")
import torch, synth
import paper_2002_10083_b200 as M
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
mx = int(sys.argv[2]) if len(sys.argv) > 2 else 100
prm = {"C2": dict(select_k=100, recover_k=100)}.get(cfg, {})
p = M.Params(**prm)
rows = []
def cb(it, A, st):
    rows.append({"iter": it, "ms": round(st["ms"][6], 2), "flops": st["flops"], "nnz_out": st["nnz_out"],
                 "chaos": round(st["chaos"], 5), "gflops": round(2 * st["flops"] / (st["ms"][6] * 1e6), 1),
                 "split_cols": st["split_cols"], "esc_cols": st["esc_cols"], "phases": st["phases"]})
    print(json.dumps(rows[-1]), flush=True)
G = synth.config_graph(cfg)
torch.cuda.synchronize(); t = time.time()
labels, k, hist, _ = M.run(M.CSC.from_host(G), p, max_iter=mx, callback=cb)
torch.cuda.synchronize()
print(json.dumps({"config": cfg, "iterations": len(hist), "clusters": k,
                  "device_ms_total": round(sum(r["ms"] for r in rows), 1),
                  "wall_s_incl_upload_and_preprocess": round(time.time() - t, 2)}))
