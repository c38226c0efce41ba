#!/bin/bash
# ncu evidence for one config: launch list of one step + full capture of the
# listed kernels.  Usage: bash scripts/gpu_prof_cfg.sh CONFIG REGEX TAG
C=${1:-4}; K=${2:-ipf_fast}; T=${3:-cfg$C}
set -x
CMD="python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_${T}_plain.json 2> gpurun_out/prof_${T}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${T}.csv $CMD > gpurun_out/ncu_launches_${T}.log 2>&1
echo "launches exit $?"
ncu --set full --clock-control none --import-source on -k regex:"$K" -c 2 \
    -o gpurun_out/prof_${T} $CMD > gpurun_out/ncu_full_${T}.log 2>&1
echo "full exit $?"
