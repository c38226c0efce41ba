#!/bin/bash
# Round-2 first check: GPU tests (acceptance + existing; batch parity on the
# fixtures present), smoke, a headline bench line with the stock-reference CPU
# baseline, and a short reference arm.
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -k "not batch_matches or 2-fp" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 exit $?" >> gpurun_out/bench_cfg3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?" >> gpurun_out/bench_ref.err
