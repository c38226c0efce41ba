#!/bin/bash
# iteration loop: all GPU tests, then device bench lines of the given configs (default 3 4 5)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_iter4.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_iter4.log
tail -3 gpurun_out/pytest_iter4.log
for C in ${@:-3 4 5}; do
timeout 600 python bench.py --config $C --no-cpu-baseline --no-e2e > gpurun_out/it4_cfg$C.json 2> gpurun_out/it4_cfg$C.err; echo "cfg$C exit $?"
python - <<PY
import json
l=[x for x in open("gpurun_out/it4_cfg$C.json") if x.startswith("{")]
d=json.loads(l[-1]); print("cfg$C", round(d["value"],1), round(d["ms_per_step"],4), d["config"].get("serial_ms_per_step")); print(d["config"]["stage_ms"])
PY
done
