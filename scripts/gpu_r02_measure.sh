#!/bin/bash
# Round-2 measurement: GPU tests, smoke, the headline bench line (stock-reference
# CPU baseline), the reference arm, fp64 mode, the other configs, ncu evidence
# (cfg3 launch list + full capture of the dominant kernels; exact IPF cfg5/cfg1;
# exact C-bar in fp64 mode; cfg4 coarse primal) and the trace-build counters.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; lscpu > gpurun_out/lscpu.txt; nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench_cfg3.json 2> gpurun_out/r02_bench_cfg3.err; echo "exit $?" >> gpurun_out/r02_bench_cfg3.err
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo "exit $?" >> gpurun_out/r02_bench_ref.err
timeout 900 python bench.py --precision fp64 --no-cpu-baseline > gpurun_out/r02_bench_cfg3_fp64.json 2> gpurun_out/r02_bench_cfg3_fp64.err
for C in 4 2 5 1; do
  timeout 900 python bench.py --config $C --no-cpu-baseline --e2e-steps 5 > gpurun_out/r02_bench_cfg$C.json 2> gpurun_out/r02_bench_cfg$C.err; echo "exit $?" >> gpurun_out/r02_bench_cfg$C.err
done
GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so timeout 300 python scripts/ct_trace.py > gpurun_out/ct_trace.json 2>&1
GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so timeout 300 python scripts/ipf_trace.py 1 2>&1 | tail -1 >> gpurun_out/ipf_trace.txt
for A in "5 64" "5 64 1" "3 45" "3 45 1"; do
  GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so timeout 300 python scripts/ipf_cl_trace.py $A 2>&1 | tail -2 >> gpurun_out/ipf_trace.txt
done
for A in "4 45" "3 45" "2 45"; do
  GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so timeout 300 python scripts/coarse_trace.py $A 2>&1 | tail -1 >> gpurun_out/ipf_trace.txt
done
timeout 120 python scripts/probe_dadd.py >> gpurun_out/ipf_trace.txt 2>&1
# ncu: each capture after the identical plain command exited 0
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches exit $?" >> gpurun_out/ncu_launches.log
timeout 1200 ncu --set full --clock-control none --import-source on \
    -k regex:"cbar_diag|pruned_ct_tab|primal_coarse|tv_pass|sep_tile|cbar_moments|interpolate_tab|cbar_pool" -c 16 \
    -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full exit $?" >> gpurun_out/ncu_full.log
timeout 600 bash scripts/gpu_prof_k.sh 5 "ipf_cluster|moments_tv|run_list_par|sep_tile" cfg5_ipf 4 > gpurun_out/prof_cfg5.log 2>&1
timeout 600 bash scripts/gpu_prof_k.sh 1 "ipf_kernel" cfg1_ipf 1 > gpurun_out/prof_cfg1.log 2>&1
timeout 600 bash scripts/gpu_prof_k.sh 4 "primal_coarse|tv_pass" cfg4_coarse 2 > gpurun_out/prof_cfg4.log 2>&1
timeout 600 bash scripts/gpu_prof_k.sh 3 "cbar_pool" cfg3_pool 2 > gpurun_out/prof_cfg3_pool.log 2>&1
CMD64="python bench.py --precision fp64 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD64 > gpurun_out/prof_fp64_plain.json 2> gpurun_out/prof_fp64_plain.err && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"cbar_exact2d|pruned_ct_kernel" -c 2 \
    -o gpurun_out/prof_fp64 $CMD64 > gpurun_out/ncu_fp64.log 2>&1
echo "fp64 exit $?" >> gpurun_out/ncu_fp64.log
bash scripts/ncu_export.sh
