#!/usr/bin/env python
"""Summarise an ncu launch list + full-set capture into profiles/<name>.md.

    python scripts/summarize_profile.py gpurun_out/launches.csv \
        gpurun_out/prof_full.ncu-rep profiles/r01_step.md [bench.json]

The launch list is `ncu --metrics gpu__time_duration.sum --clock-control none`
over `bench.py --steps 1 --warmup 1` (cold, serialised launches: compare
shares, not absolute times); the full capture is `ncu --set full` of the
dominant kernels (B200_PROFILING.md).
"""

from __future__ import annotations

import collections
import csv
import json
import subprocess
import sys


def raw_page(path):
    """Raw-page CSV text of a report; a ready-made *.raw.csv (scripts/ncu_export.sh) is read as is."""
    if path.endswith(".csv"):
        return open(path).read()
    return subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                          text=True).stdout



def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:60]
        key = f"{name} grid={d['Grid Size']} block={d['Block Size']}"
        v = float(d["Metric Value"].replace(",", ""))
        agg.setdefault(key, [0.0, 0])
        agg[key][0] += v
        agg[key][1] += 1
    return agg


RAW = {
    "gpu__time_duration.sum": "time",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma%",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_cyc%",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu%",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu%",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1%",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2%",
    "launch__registers_per_thread": "regs",
}


def full(path):
    out = raw_page(path)
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        rec = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")[:60]}
        for k, short in RAW.items():
            if k in hdr:
                rec[short] = r[hdr.index(k)] + (" " + units[hdr.index(k)] if short in
                                                 ("time", "dram_rd", "dram_wr") else "")
        res.append(rec)
    return res


def main():
    lpath, fpath, out = sys.argv[1:4]
    bench = json.load(open(sys.argv[4])) if len(sys.argv) > 4 else None
    agg = launches(lpath)
    tot = sum(v[0] for v in agg.values())
    lines = ["# ncu evidence", "", f"Launch list: `{lpath}` (every step of `bench.py "
             "--steps 1 --warmup 1`: warm-up, timed, the serial stage-timing pass and the "
             "launch-count step; cold and serialised under ncu: compare shares).", "",
             "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:25]:
        lines.append(f"| `{k}` | {v[1]} | {v[0] / 1e3:.1f} | {v[0] / 1e3 / v[1]:.1f} | "
                     f"{100 * v[0] / tot:.1f}% |")
    lines += ["", f"Total {tot / 1e6:.2f} ms.", ""]
    recs = full(fpath)
    if recs:
        keys = ["kernel"] + list(RAW.values())
        lines += [f"Full-set capture: `{fpath}`.", "", "| " + " | ".join(keys) + " |",
                  "|" + "---|" * len(keys)]
        for r in recs:
            lines.append("| " + " | ".join(str(r.get(k, "")) for k in keys) + " |")
    if bench:
        lines += ["", "Bench line of the same build:", "", "```json",
                  json.dumps(bench, indent=1)[:6000], "```"]
    open(out, "w").write("\n".join(lines) + "\n")
    print("wrote", out)


if __name__ == "__main__":
    main()
