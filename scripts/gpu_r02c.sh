#!/bin/bash
# GPU tests, device bench lines of all configs (no e2e), ncu of the primal kernels
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for C in 3 4 2 5 1; do
  timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg$C.json 2> gpurun_out/bench_cfg$C.err; echo "exit $?" >> gpurun_out/bench_cfg$C.err
done
timeout 600 bash scripts/gpu_prof_k.sh 5 "ipf_kernel" cfg5_ipf 1 > gpurun_out/prof_cfg5.log 2>&1
timeout 600 bash scripts/gpu_prof_k.sh 3 "primal_coarse" cfg3_coarse 2 > gpurun_out/prof_cfg3c.log 2>&1
timeout 600 bash scripts/gpu_prof_k.sh 4 "primal_coarse" cfg4_coarse 1 > gpurun_out/prof_cfg4c.log 2>&1
