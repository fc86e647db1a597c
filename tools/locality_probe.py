"""Development: how much does column locality matter?  Runs one fused C3 iteration on
the stock (randomly relabelled) graph and on the same graph without the relabelling
(vertices numbered family by family), printing per-bin kernel times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2002_10083_b200 as M  # noqa: E402
import synth  # noqa: E402


def run(G, tag):
    ctx = M.context()
    A = ctx.preprocess(M.CSC.from_host(G))
    for _ in range(2):
        out, st = ctx.iterate(A, M.Params())
    ts = []
    for _ in range(5):
        out, st = ctx.iterate(A, M.Params())
        torch.cuda.synchronize()
        ts.append(st["ms"][3])
    print(tag, "fused ms", round(min(ts), 2), "bin_ms", [round(x, 1) for x in st["bin_ms"]],
          "retries", st["retries"], "bin_cols", st["bin_cols"], flush=True)


G = synth.config_graph("C3")
run(G, "permuted  ")
orig = synth.pairs_to_symmetric_csc
synth.pairs_to_symmetric_csc = lambda n, i, j, w, perm=None: orig(n, i, j, w, None)
run(synth.config_graph("C3"), "family-order")
