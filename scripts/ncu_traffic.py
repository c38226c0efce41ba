#!/usr/bin/env python
"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of
every kernel in ncu full-set captures -> profiles/ncu_traffic_cfgN.json, which
bench.py reads for the `traffic` field of its roofline blocks.

    python scripts/ncu_traffic.py CONFIG gpurun_out/prof_full.ncu-rep [more.ncu-rep ...]

writes profiles/ncu_traffic_cfgCONFIG.json (the captures of one bench config).
"""
import csv
import json
import os
import subprocess
import sys


def raw_page(path):
    """Raw-page CSV text of a report; a ready-made *.raw.csv (scripts/ncu_export.sh) is read as is."""
    if path.endswith(".csv"):
        return open(path).read()
    return subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                          text=True).stdout


UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        f"ncu_traffic_cfg{sys.argv[1]}.json")
res = {}
for rep in sys.argv[2:]:
    txt = raw_page(rep)
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").strip()
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(m)
            b += float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
        res.setdefault(name, []).append(b)
out = {k: {"bytes_per_launch": sum(v) / len(v), "launches_captured": len(v)} for k, v in res.items()}
json.dump(out, open(out_path, "w"), indent=1, sort_keys=True)
print(json.dumps(out, indent=1))
