#!/bin/bash
# iteration loop for the fp32 headline path: fast-path + parity tests, then the device bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fast_paths.py tests/test_gpu_batch_parity.py tests/test_gpu_configs.py -q -m gpu -x > gpurun_out/pytest_iter3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_iter3.log
tail -3 gpurun_out/pytest_iter3.log
for C in 3 4; do
timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/it3_cfg$C.json 2> gpurun_out/it3_cfg$C.err; echo "cfg$C exit $?"
done
python - <<'PY'
import json
for n in ("cfg3","cfg4"):
    l=[x for x in open(f"gpurun_out/it3_{n}.json") if x.startswith("{")]
    d=json.loads(l[-1]); print(n, round(d["value"],1), round(d["ms_per_step"],4), d["config"].get("serial_ms_per_step")); print(d["config"]["stage_ms"])
PY
