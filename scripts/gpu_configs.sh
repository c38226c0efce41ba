#!/bin/bash
# bench lines of the non-headline configs (device stages + e2e, no CPU leg)
set -x
for c in 4 2 5 1; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  echo "cfg$c exit $?" >> gpurun_out/bench_cfg$c.err
done
