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
# entropic sweeps: throughput line per grid, then an ncu capture of one sweep's kernels at 128^2
timeout 600 python scripts/bench_entropic.py > gpurun_out/bench_entropic.jsonl 2> gpurun_out/bench_entropic.err
timeout 600 ncu --set full --clock-control none -k regex:"en_(row|col|colfold)_kernel" -s 30 -c 3 \
    -o gpurun_out/prof_entropic python scripts/bench_entropic.py --sides 128 > gpurun_out/ncu_entropic.log 2>&1
