#!/usr/bin/env python
"""Brief per-kernel summary of an ncu report: time, stall reasons, pipe use."""
import csv
import subprocess
import sys


def raw_page(path):
    """Raw-page CSV text of a report; a ready-made *.raw.csv (scripts/ncu_export.sh) is read as is."""
    if path.endswith(".csv"):
        return open(path).read()
    return subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                          text=True).stdout


rep = sys.argv[1]
out = raw_page(rep)
rows = list(csv.reader(out.splitlines()))
h = rows[0]
KEYS = ["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:90], "time", d.get("gpu__time_duration.sum"))
    keys = [k for k in h if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("_per_issue_active.ratio")]
    st = sorted(((float(d[k] or 0), k) for k in keys), reverse=True)[:7]
    print("   stalls:", ", ".join("%s %.2f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v) for v, k in st))
    for k in KEYS:
        if k in d:
            print("   %-70s %s" % (k, d[k]))
