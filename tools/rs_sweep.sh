#!/bin/bash
# padded row stride for n = 4, 8, 12, 16: parity, then every variant at E=4096
cd ${GRAFT_REPO_ROOT:-.}
timeout 900 python -m pytest -q -x tests/test_gpu_parity.py -k "ax" 2>&1 | tail -1
timeout 1500 python tools/ax_sweep.py --n 4,8,12,16 --E 4096 --reps 30 > gpurun_out/sweep_rs.jsonl 2>&1
python - <<'PY'
import json
rows=[json.loads(l) for l in open("gpurun_out/sweep_rs.jsonl") if l.startswith("{") and '"us"' in l]
for n in (4,8,12,16):
    r=sorted([x for x in rows if x["n"]==n], key=lambda x:x["us"])
    print(n, [(x["variant"],x["us"],x["frac"]) for x in r[:5]], "default:", [(x["us"],x["frac"]) for x in r if x["variant"]==0])
PY
