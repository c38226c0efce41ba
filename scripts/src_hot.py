#!/usr/bin/env python
"""Per-CUDA-source-line stall samples from `ncu --page source --print-source cuda,sass --csv`.

    ncu -i rep --page source --csv -k regex:NAME --print-source cuda,sass > x.csv
    python scripts/src_hot.py x.csv [top]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
res, fname = [], ""
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if len(r) > 8 and r[0] not in ("", "Line No") and r[4] not in ("-", ""):
        try:
            res.append((float(r[4]), float(r[7] or 0), fname, r[0], r[1]))
        except ValueError:
            pass
tot = sum(x[0] for x in res) or 1
for s, ins, f, ln, src in sorted(res, key=lambda x: -x[0])[:top]:
    print(f"{100 * s / tot:5.1f}%  inst={int(ins):>9}  {f}:{ln}  {src.strip()[:100]}")
