#!/bin/bash
for np in 9 18 27 36 45; do
  timeout 300 python bench.py --config 4 --pairs $np --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/scan_$np.json 2>gpurun_out/scan_$np.err
done
