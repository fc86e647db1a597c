"""python -m paper_2002_10083_b200 GRAPH OUT [--inflation R] [--select-k S] ...

End-to-end MCL (Alg. 1) on one GPU: read a MatrixMarket / labelled edge-list graph
(mcl_graph_read), iterate the fused expansion + prune + inflate until chaos < eps, extract
the clusters on the device and write one line per cluster (mcl_clusters_write)."""
import argparse
import json
import sys
import time

import torch

import paper_2002_10083_b200 as M


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2002_10083_b200")
    ap.add_argument("graph")
    ap.add_argument("out")
    ap.add_argument("--no-symmetrize", action="store_true")
    ap.add_argument("--inflation", type=float, default=2.0)
    ap.add_argument("--threshold", type=float, default=1e-4)
    ap.add_argument("--select-k", type=int, default=1100)
    ap.add_argument("--recover-k", type=int, default=1400)
    ap.add_argument("--recover-pct", type=float, default=0.9)
    ap.add_argument("--eps", type=float, default=1e-3)
    ap.add_argument("--max-iter", type=int, default=100)
    a = ap.parse_args(argv)
    t0 = time.time()
    g = M.read_graph(a.graph, symmetrize=not a.no_symmetrize)
    p = M.Params(inflation=a.inflation, prune_threshold=a.threshold, select_k=a.select_k,
                 recover_k=a.recover_k, recover_pct=a.recover_pct, chaos_eps=a.eps)
    labels, k, hist, _ = M.run(M.CSC.from_host(g), p, max_iter=a.max_iter)
    torch.cuda.synchronize()
    M.write_clusters(a.out, labels, g)
    print(json.dumps({"n": g.ncols, "nnz": g.nnz, "clusters": k, "iterations": len(hist),
                      "converged": bool(hist and hist[-1]["chaos"] < a.eps),
                      "wall_s": round(time.time() - t0, 3)}))
    return 0 if hist and hist[-1]["chaos"] < a.eps else 3


if __name__ == "__main__":
    sys.exit(main())
