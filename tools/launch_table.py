"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel.
Usage: python tools/launch_table.py launches.csv [N]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", "ns"), 1e-6)
    k = d["Kernel Name"]
    agg[k][0] += 1
    agg[k][1] += v
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} ms over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:N]:
    print(f"{v[1]:10.2f} ms {v[1] / tot * 100:5.1f}% {v[0]:6d}  {k[:90]}")
