#!/bin/bash
# C-bar diag: fast-path tests, tile-shape sweep (GDT_DG_VARIANT), optional ncu capture
timeout 600 python -m pytest tests/test_gpu_fast_paths.py -x -q > gpurun_out/pytest_fast.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_fast.log
grep -q "pytest exit 0" gpurun_out/pytest_fast.log || exit 1
for V in ${VARIANTS:-0 1 2 3}; do
  GDT_DG_VARIANT=$V timeout 240 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dg_v$V.json 2> gpurun_out/dg_v$V.err
done
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:cbar_diag -c 2 \
    -o gpurun_out/prof_dg python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_dg.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_dg.log
fi
