#!/bin/bash
# quick loop: GPU tests + the IPF-heavy configs
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for c in 4 2; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
done
