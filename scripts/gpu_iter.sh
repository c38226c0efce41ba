#!/bin/bash
# iteration loop: all GPU tests, then the headline bench (device + e2e, no CPU baseline)
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
grep -q "pytest exit 0" gpurun_out/pytest_gpu.log || exit 1
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo "bench exit $?" >> gpurun_out/bench_iter.err
