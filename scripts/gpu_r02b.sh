#!/bin/bash
# GPU tests (full), device bench lines of all configs, ncu captures of the
# exact fp64 IPF (cfg5, cfg1) and of the coarse-level primal stage (cfg3).
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "exit $?" >> gpurun_out/bench_cfg3.err
for C in 4 2 5 1; do
  timeout 600 python bench.py --config $C --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_cfg$C.json 2> gpurun_out/bench_cfg$C.err; echo "exit $?" >> gpurun_out/bench_cfg$C.err
done
timeout 600 bash scripts/gpu_prof_k.sh 5 "ipf_kernel" cfg5_ipf 1 > gpurun_out/prof_cfg5.log 2>&1
timeout 600 bash scripts/gpu_prof_k.sh 1 "ipf_kernel" cfg1_ipf 1 > gpurun_out/prof_cfg1.log 2>&1
timeout 600 bash scripts/gpu_prof_k.sh 3 "primal_coarse" cfg3_coarse 2 > gpurun_out/prof_cfg3c.log 2>&1
