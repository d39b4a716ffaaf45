#!/bin/bash
# CG Ax staging modes with the tuned update (888 blocks) and the deferred Ax reduction
cd ${GRAFT_REPO_ROOT:-.}
echo "== tests (defaults) and SEM_CG_AX_CFG=9"
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" tests/test_dist_gpu.py 2>&1 | tail -1
SEM_CG_AX_CFG=9 timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" 2>&1 | tail -1
for ax in 0 4 9 10 0 9; do
  echo "ax=$ax $(SEM_CG_AX_CFG=$ax timeout 120 python tools/cg_phases.py 4096 32768 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})')"
done
