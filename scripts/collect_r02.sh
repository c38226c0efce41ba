#!/bin/bash
# gpurun_out/ of scripts/gpu_r02_measure.sh -> profiles/r02_* (bench lines, launch list, ncu summaries, traces)
cd "$(dirname "$0")/.."
G=gpurun_out; P=profiles
python - <<'PY'
import json
for n in ("cfg3","ref","cfg3_fp64","cfg4","cfg2","cfg5","cfg1"):
    l=[x for x in open(f"gpurun_out/r02_bench_{n}.json") if x.startswith("{")]
    json.dump(json.loads(l[-1]), open(f"profiles/r02_bench_{n}.json","w"), indent=1)
PY
cp $G/launches.csv $P/r02_cfg3_launches.csv
python -c "import json,sys; d=json.loads(open('$G/ct_trace.json').read().strip().splitlines()[-1]); json.dump(d, open('$P/r02_ct_tiles.json','w'))" || echo 'ct_trace.json invalid: profiles/r02_ct_tiles.json kept'
python scripts/summarize_profile.py $G/launches.csv $G/prof_full.raw.csv $P/r02_cfg3_ncu.md $P/r02_bench_cfg3.json >/dev/null
python scripts/ncu_traffic.py 3 $G/prof_full.raw.csv $G/prof_cfg3_pool.raw.csv > /dev/null
python scripts/ncu_traffic.py 1 $G/prof_cfg1_ipf.raw.csv > /dev/null
python scripts/ncu_traffic.py 4 $G/prof_cfg4_coarse.raw.csv >/dev/null
python scripts/ncu_traffic.py 5 $G/prof_cfg5_ipf.raw.csv > /dev/null
for n in cfg1_ipf cfg4_coarse fp64 cfg5_ipf; do python scripts/ncu_brief.py $G/prof_$n.raw.csv > $P/r02_${n}_ncu.txt; done
python - <<'PY'
s=open("profiles/r02_ipf_trace.txt").read()
fin=[l for l in open("gpurun_out/ipf_trace.txt").read().splitlines() if "cluster 1" not in l and "barrier -" not in l]
s=s.split("# -- final build")[0]
s+="# -- final build (scripts/gpu_r02_measure.sh) --\n"+"\n".join(fin)+"\n"
open("profiles/r02_ipf_trace.txt","w").write(s)
PY
