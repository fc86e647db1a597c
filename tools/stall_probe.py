#!/usr/bin/env python
"""Per-step anatomy of the 1-GPU C3 iteration: device time between events around the call,
the library's own total (ms[6]), the sum of bin kernel times, and host wall time -- to tell
host stalls (GPU idle while the host waits) from device-side variance."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2002_10083_b200 as M  # noqa: E402
import synth  # noqa: E402
from bench import CONFIG_PARAMS  # noqa: E402

import gc  # noqa: E402
if os.environ.get("PROBE_GC") == "off":
    gc.disable()
elif os.environ.get("PROBE_GC") == "freeze":
    gc.collect()
    gc.freeze()
print("gc", os.environ.get("PROBE_GC", "default"), gc.get_threshold(), gc.get_count())
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)), "load", open("/proc/loadavg").read().strip())
G = synth.config_graph("C3", 1.0)
ctx = M.context()
A = ctx.preprocess(M.CSC.from_host(G, device=torch.device("cuda", 0)))
params = M.Params(**CONFIG_PARAMS["C3"])
s = torch.cuda.current_stream()
for _ in range(3):
    out, st = ctx.iterate(A, params)
    del out
torch.cuda.synchronize()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s)
    out, st = ctx.iterate(A, params)
    e1.record(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    del out
    print(f"step {i:2d} dev {e0.elapsed_time(e1):7.2f} lib {st['ms'][6]:7.2f} bins {sum(st['bin_ms']):6.2f} "
          f"fused {st['ms'][3]:6.2f} host {1e3 * (t1 - t0):7.2f} retries {st['retries']} "
          f"split {st['split_ms']:.2f} gc {gc.get_count()}", flush=True)
