#!/bin/bash
tail -2 gpurun_out/pytest_gpu.log
for f in "$@"; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/{f}.json"))
except Exception as e:
    print(f, "ERR", e); sys.exit()
print(f, round(d["value"], 1), "ms/step", round(d["ms_per_step"], 3), "e2e",
      round(d.get("e2e", {}).get("value", 0), 2), "ipf frac", round(d["roofline_ipf"]["frac"], 4))
print("   ", {k: v for k, v in d["config"]["stage_ms"].items()})
PY
done
