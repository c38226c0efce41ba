#!/bin/bash
# iteration loop of round 2: the exact-IPF tests, then device-only bench lines
# of the fp64 configs (cfg5, cfg1, cfg3 in fp64 mode) and the headline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_gpu_batch_parity.py -q -m gpu -x > gpurun_out/pytest_iter.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_iter.log
tail -5 gpurun_out/pytest_iter.log
for C in 5 1; do
  timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/it_cfg$C.json 2> gpurun_out/it_cfg$C.err; echo "cfg$C exit $?"
done
timeout 600 python bench.py --config 3 --precision fp64 --no-cpu-baseline --no-e2e > gpurun_out/it_cfg3_fp64.json 2> gpurun_out/it_cfg3_fp64.err; echo "cfg3 fp64 exit $?"
python - <<'PY'
import json
for n in ("cfg5","cfg1","cfg3_fp64"):
    try:
        l=[x for x in open(f"gpurun_out/it_{n}.json") if x.startswith("{")]
        d=json.loads(l[-1]); print(n, round(d["value"],1), round(d["ms_per_step"],4), {k:v for k,v in d["config"]["stage_ms"].items() if "primal" in k})
    except Exception as e: print(n, "failed", e)
PY
python scripts/probe_dadd.py
for A in "5 64 2" "5 64 1" "3 45 3" "3 45 2"; do
  GRIDOT_B200_LIB=paper_2506_00976_b200/csrc/_trace/libgridot_b200.so timeout 300 python scripts/ipf_cl_trace.py $A 2>&1 | tail -2
done
