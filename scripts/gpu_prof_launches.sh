#!/bin/bash
# ncu launch lists (cold, serialised) of one bench step for the given configs
for C in "$@"; do
  CMD="python bench.py --config $C --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
  $CMD > gpurun_out/pl_${C}_plain.json 2> gpurun_out/pl_${C}_plain.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_cfg${C}.csv $CMD > gpurun_out/ncu_launches_cfg${C}.log 2>&1
  echo "cfg$C exit $?"
done
