#!/bin/bash
# ncu evidence for the bench: launch list of one step (cold, serialised) and a
# full-set capture of the dominant kernels.  Each ncu command runs only after
# the identical plain command exited 0 (B200_PROFILING.md).
set -x
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.json 2> gpurun_out/prof_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches exit $?"
$CMD > gpurun_out/prof_plain2.json 2> gpurun_out/prof_plain2.err && \
ncu --set full --clock-control none --import-source on \
    -k regex:"cbar_diag|pruned_ct|ipf_fast|price_kernel|cbar_moments|sep_tile|moments_tv" -c 12 \
    -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
echo "full exit $?"
