#!/bin/bash
# full ncu capture of kernels matching $2 in bench config $1 (after a plain run)
C=${1:-3}; K=${2:-pruned}; T=${3:-k}
CMD="python bench.py --config $C --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_${T}_plain.json 2> gpurun_out/prof_${T}_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:"$K" -c ${4:-2} \
    -o gpurun_out/prof_${T} $CMD > gpurun_out/ncu_${T}.log 2>&1
echo "exit $?"
