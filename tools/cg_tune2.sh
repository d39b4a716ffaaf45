#!/bin/bash
# CG tail/head tuning matrix: correctness of each option on the CG parity
# tests, then per-phase device times (tools/cg_phases.py) at E=4096, 32768.
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for opt in "SEM_CG_UPD=1" "SEM_CG_AX_CFG=6" "SEM_CG_AX_CFG=6 SEM_CG_UPD=1"; do
  echo "== tests with $opt"
  env $opt timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" tests/test_dist_gpu.py 2>&1 | tail -2
done
for ax in 0 6 7 8; do for upd in "0 0" "1 1184" "1 2368" "1 4736"; do
  set -- $upd
  echo "ax=$ax upd=$1 blocks=$2 $(SEM_CG_AX_CFG=$ax SEM_CG_UPD=$1 SEM_CG_UPD_BLOCKS=$2 timeout 120 python tools/cg_phases.py 4096 32768 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})')"
done; done
