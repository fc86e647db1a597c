"""Small invocations of every kernel family, for compute-sanitizer (memcheck / racecheck):
forced shared-memory bins of both families and the global bin (expand + fused iterate), the
split path (hashed parts, private parts, dense sweep with and without candidates), the
standalone prune, Cohen, the merge and the clusters.  Prints OK at the end."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2002_10083_b200 as M  # noqa: E402


def run(env=None, fn=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    try:
        ctx = M.Context()
        fn(ctx)
        torch.cuda.synchronize()
        ctx.close()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


A = M.CSC.from_host(synth.random_sparse(300, 300, 0.03, seed=11, empty_cols=0.1))
G1 = M.CSC.from_host(synth.planted_partition())


def forced(ctx):
    for b in range(14):
        ctx.expand(A, params=M.Params(force_bin=b))
        ctx.iterate(A, M.Params(force_bin=b, estimator=2))


def c1(ctx):
    A1 = ctx.preprocess(G1)
    for _ in range(2):
        A1, _ = ctx.iterate(A1, M.Params())
    ctx.clusters(A1)
    ctx.estimate(A1, r=10)
    ctx.merge([A1, A1])


def split(ctx):
    A1 = ctx.preprocess(G1)
    A1, _ = ctx.iterate(A1, M.Params())
    ctx.iterate(A1, M.Params())


run(None, forced)
run(None, c1)
run({"MCLX_SPLIT_MIN_NEED": "100"}, split)
run({"MCLX_SPLIT_MIN_NEED": "100", "MCLX_SPLIT_PART_NEED": "16"}, split)
run({"MCLX_SPLIT_MIN_NEED": "100", "MCLX_SPLIT_PART_NEED": "16", "MCLX_SPLIT_CAND": "0"}, split)
run({"MCLX_SPLIT_MIN_NEED": "100", "MCLX_FP64_TERMS": "32"}, split)
print("OK")
