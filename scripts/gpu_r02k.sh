#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for C in 5 1; do
  timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e >> gpurun_out/bench_cfg$C.json 2>> gpurun_out/bench_cfg$C.err; echo "exit $?" >> gpurun_out/bench_cfg$C.err
done
timeout 600 python bench.py --config 3 --precision fp64 --no-cpu-baseline --no-e2e >> gpurun_out/bench_cfg3_fp64.json 2>> gpurun_out/bench_cfg3_fp64.err
for C in 1 5; do
  GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so timeout 300 python scripts/ipf_trace.py $C >> gpurun_out/ipf_trace.txt 2>&1
done
