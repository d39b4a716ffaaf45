#!/bin/bash
# programmatic dependent launch of the CG chain: tests, then solve time with / without
cd ${GRAFT_REPO_ROOT:-.}
timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" tests/test_dist_gpu.py 2>&1 | tail -1
for pdl in 0 1 0 1; do
  echo "pdl=$pdl us/it $(SEM_CG_PDL=$pdl timeout 200 python tools/cg_time.py 4096 32768)"
done
