"""Summarise one kernel of an .ncu-rep into profiles/*.json (the metrics the round summary
quotes: duration, DRAM bytes, L2 hit rate, issue activity, occupancy, stall reasons,
shared-memory bank conflicts).  Usage: python tools/ncu_summary.py REP OUT.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.per_cycle_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def main(rep, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    m = {}
    for i, h in enumerate(hdr):
        if h in KEYS or h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            m[h] = [vals[i], units[i]]
    stalls = {h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]: float(v[0])
              for h, v in m.items() if h.startswith("smsp__average_warps_issue_stalled_")
              and v[0].replace(".", "", 1).isdigit()}
    top = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    m = {k: v for k, v in m.items() if not k.startswith("smsp__average_warps_issue_stalled_")}
    json.dump({"metrics": m, "top_stalls_per_issue": top, "source": rep}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
