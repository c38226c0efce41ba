#!/bin/bash
# Round measurement: GPU tests, smoke, the headline bench line (with CPU
# baseline), the reference arm, the other configs, and ncu evidence for cfg3
# (launch list + full capture of the dominant kernels) and cfg4 (fast IPF).
bash scripts/gpu_check.sh
timeout 900 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 exit $?" >> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?" >> gpurun_out/bench_ref.err
bash scripts/gpu_configs.sh
timeout 900 bash scripts/gpu_prof.sh > gpurun_out/prof.log 2>&1
timeout 900 bash scripts/gpu_prof_cfg.sh 4 ipf_fast cfg4 > gpurun_out/prof_cfg4.log 2>&1
