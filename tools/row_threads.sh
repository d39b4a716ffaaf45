#!/bin/bash
# row-kernel block size x blocks/SM (one wave) for the CG update
cd ${GRAFT_REPO_ROOT:-.}
for cfg in "256 3" "128 6" "256 3" "128 6"; do
  set -- $cfg
  SEM_NVCC_DEFS="SEM_ROW_THREADS=$1 SEM_UPD_MINB=$2" python -m paper_2005_13425_b200.build --force > /dev/null 2>&1
  echo "threads=$1 minb=$2 $(timeout 120 python tools/cg_phases.py 4096 32768 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})') solve $(timeout 200 python tools/cg_time.py 4096 32768)"
done
