#!/bin/bash
cd ${GRAFT_REPO_ROOT:-.}
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" 2>&1 | tail -1
SEM_CG_PDL=2 timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" 2>&1 | tail -1
for pdl in 0 2 1 0 2 1; do
  echo "pdl=$pdl us/it $(SEM_CG_PDL=$pdl timeout 200 python tools/cg_time.py 4096 32768)"
done
