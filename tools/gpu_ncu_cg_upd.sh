#!/bin/bash
# ncu --set full of the CG update kernel (row or element form) at E = 4096
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for m in ${MODES:-1 0}; do
  SEM_CG_UPD_ELEM=$m timeout 600 ncu --set full --clock-control none -k regex:cg_update -s 5 -c 1 \
    -o /tmp/upd$m -f python tools/cg_time.py 4096 > gpurun_out/ncu_upd$m.log 2>&1
  python tools/ncu_brief.py /tmp/upd$m.ncu-rep > gpurun_out/upd${m}_brief.txt 2>&1
  ncu -i /tmp/upd$m.ncu-rep --page raw --csv 2>/dev/null | python tools/ncu_stalls.py > gpurun_out/upd${m}_stalls.txt 2>&1
done
