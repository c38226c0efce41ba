#!/bin/bash
# full check: GPU tests, smoke, default bench line, launch list of the bench
bash scripts/gpu_check.sh
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench exit $?" >> gpurun_out/bench_default.err
