#!/bin/bash
# Run on the GPU box after the ncu captures: every gpurun_out/*.ncu-rep gets a
# raw-page CSV beside it, then the largest reports are dropped until
# gpurun_out/ fits the 64 MiB that gpurun copies back.
cd gpurun_out || exit 0
for r in *.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  ncu -i "$r" --page source --csv > "${r%.ncu-rep}.source.csv" 2>/dev/null
  gzip -f "${r%.ncu-rep}.source.csv"
done
LIMIT_KB=${1:-56000}
while [ "$(du -sk . | cut -f1)" -gt "$LIMIT_KB" ]; do
  big=$(ls -S *.ncu-rep 2>/dev/null | head -1)
  [ -n "$big" ] || break
  echo "dropping $big ($(du -k "$big" | cut -f1) KB)" >> dropped.txt
  rm -f "$big"
done
du -sk . >> dropped.txt
