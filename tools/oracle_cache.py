#!/usr/bin/env python
"""oracle_cache.py -- expected values for the full-size parity tests, computed by the
ORACLE ONLY (oracle/ + synth/; nothing here imports the CUDA package).

SURVEY.md §8(c) c.5 / §8(d) d.5: O1-O3 are column-local given A_t, so a harness may shard
an iteration's output columns over all host cores as independent single-threaded oracle
processes ([b, e) ranges, concatenated in order; chaos = max).  The result is identical
to one single-threaded oracle run -- every column is computed by the same C code on the
same inputs -- only the wall time changes.

Jobs (each writes tests/golden/<name>.npz and a line to tests/golden/oracle_cache.json):
  c3_mcl        full MCL on C3 (n = 500k) to convergence: canonical labels (P4),
                iteration count, chaos history
  nnz_<cfg>     per-column nnz(A_t * A_t) over ALL columns (P1 structure counts) for
                C2 it0, C3 it0, C3 it1, C5 it0 and C4 (R-MAT scale 22) it0, plus flops

Usage: python tools/oracle_cache.py [job ...]   (default: all; nice'd, all cores)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402
from oracle.shard import sharded_nnz, sharded_step  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
PARAMS = {c: (synth.CONFIGS[c]["theta"], synth.CONFIGS[c]["S"], synth.CONFIGS[c]["R"],
              synth.CONFIGS[c]["pct"]) for c in synth.CONFIGS}


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, file=sys.stderr, flush=True)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def record(name: str, meta: dict):
    p = os.path.join(GOLD, "oracle_cache.json")
    d = json.load(open(p)) if os.path.exists(p) else {}
    d[name] = meta
    json.dump(d, open(p, "w"), indent=1, sort_keys=True)


def iterate_oracle(A, prm, its, nproc):
    for _ in range(its):
        A, _ = sharded_step(A, prm, nproc)
    return A


def job_nnz(cfg: str, it: int, nproc: int, scale: float = 1.0):
    name = f"nnz_{cfg}_it{it}"
    t0 = time.time()
    A = O.preprocess(synth.config_graph(cfg, scale))
    log(name, "A0", A.ncols, A.nnz)
    A = iterate_oracle(A, PARAMS[cfg], it, nproc)
    # the GPU test squares the fp32 cast of this iterate (the oracle squares the same numbers)
    A = O.Mat(A.nrows, A.ncols, A.colptr, A.rows, A.vals.astype(np.float32).astype(np.float64))
    nnz, fl = sharded_nnz(A, nproc)
    np.savez_compressed(os.path.join(GOLD, name + ".npz"), nnz=nnz.astype(np.int32))
    meta = dict(config=cfg, iteration=it, scale=scale, n=int(A.ncols), nnz_in=int(A.nnz),
                flops=int(fl.sum()), nnz_unpruned=int(nnz.sum()), nnz_sha256=digest(nnz),
                flops_sha256=digest(fl), input_sha256=digest(A.rows) + ":" + digest(A.vals),
                cores=nproc, wall_s=round(time.time() - t0, 1),
                how="tools/oracle_cache.py: oracle expand over column shards (O1, fp64)")
    record(name, meta)
    log(name, meta)


def job_mcl(cfg: str, nproc: int, eps: float = 1e-3, max_iter: int = 100):
    name = f"{cfg.lower()}_mcl"
    t0 = time.time()
    A = O.preprocess(synth.config_graph(cfg))
    chaos_hist, it = [], 0
    while it < max_iter:
        A, ch = sharded_step(A, PARAMS[cfg], nproc)
        it += 1
        chaos_hist.append(ch)
        log(name, "iteration", it, "chaos", ch, "nnz", A.nnz, f"{time.time() - t0:.0f}s")
        if ch < eps:
            break
    labels, ncl = O.clusters(A)
    np.savez_compressed(os.path.join(GOLD, name + ".npz"), labels=labels)
    meta = dict(config=cfg, n=int(A.ncols), iterations=it, nclusters=int(ncl),
                chaos=chaos_hist, labels_sha256=digest(labels), final_nnz=int(A.nnz),
                cores=nproc, wall_s=round(time.time() - t0, 1),
                how="tools/oracle_cache.py: Alg. 1 loop, each iteration's columns sharded over "
                    "oracle processes (O1-O3), then O5 union-find clusters")
    record(name, meta)
    log(name, meta)


JOBS = {
    "nnz_C2_it0": lambda n: job_nnz("C2", 0, n),
    "nnz_C3_it0": lambda n: job_nnz("C3", 0, n),
    "c3_mcl": lambda n: job_mcl("C3", n),
    "nnz_C3_it1": lambda n: job_nnz("C3", 1, n),
    "nnz_C5_it0": lambda n: job_nnz("C5", 0, n),
    "nnz_C4_it0": lambda n: job_nnz("C4", 0, n),
}


def main():
    os.nice(10)
    nproc = int(os.environ.get("ORACLE_PROCS", os.cpu_count() or 1))
    jobs = sys.argv[1:] or list(JOBS)
    for j in jobs:
        log("job", j, "procs", nproc)
        JOBS[j](nproc)


if __name__ == "__main__":
    main()
