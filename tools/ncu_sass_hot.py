"""Hot SASS instructions of an .ncu-rep source page (development aid).
Usage: python tools/ncu_sass_hot.py REP [N]  -- prints instruction-count-weighted SASS
with stall samples, plus an opcode histogram."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 60
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ie, sm, th = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Avg. Threads Executed")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((i, int(r[ie]), int(r[sm]), float(r[th]), r[1].strip()))
    except Exception:
        pass
tot = sum(d[1] for d in data); ts = sum(d[2] for d in data)
print("total warp-inst", tot, "stall samples", ts)
op = collections.Counter(); ops = collections.Counter()
for d in data:
    o = d[4].split()[0] if d[4] else "?"
    if o.startswith("@"):
        o = d[4].split()[1]
    o = o.split(".")[0]
    op[o] += d[1]; ops[o] += d[2]
print("opcode share (inst%, stall%):")
for o, c in op.most_common(25):
    print(f"  {o:10s} {c/tot*100:5.1f} {ops[o]/ts*100:5.1f}")
if N:
    print("hot region (index, inst%, stall%, threads, sass):")
    for d in data:
        if d[1] / tot > 0.002 or d[2] / ts > 0.004:
            print(f"{d[0]:5d} {d[1]/tot*100:5.2f} {d[2]/ts*100:5.2f} {d[3]:5.1f}  {d[4][:90]}")
if len(sys.argv) > 3:
    B = int(sys.argv[3])
    print(f"per {B}-instruction region: inst%, stall%")
    for b0 in range(0, len(data), B):
        seg = data[b0:b0 + B]
        ii = sum(d[1] for d in seg) / tot * 100; ss = sum(d[2] for d in seg) / ts * 100
        if ii > 0.5 or ss > 0.5:
            print(f"  [{b0:5d},{b0+B:5d}) {ii:5.1f} {ss:5.1f}   first: {seg[0][4][:60]}")
