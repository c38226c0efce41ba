#!/bin/bash
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err
