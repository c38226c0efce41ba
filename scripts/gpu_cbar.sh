#!/bin/bash
# C-bar iteration loop: fast-path tests + device bench of the headline config
timeout 600 python -m pytest tests/test_gpu_fast_paths.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fast.log
timeout 240 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench3.json 2> gpurun_out/bench3.err
