#!/bin/bash
# deferred reductions (SEM_CG_FIN=1) x Ax staging x update grid
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
echo "== tests with SEM_CG_FIN=1"
SEM_CG_FIN=1 timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" 2>&1 | tail -2
for fin in 0 1; do for ax in 0 4 6; do for ub in 0 740 2368 4736; do
  echo "fin=$fin ax=$ax blocks=$ub $(SEM_CG_FIN=$fin SEM_CG_AX_CFG=$ax SEM_CG_UPD_BLOCKS=$ub timeout 120 python tools/cg_phases.py 4096 32768 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})')"
done; done; done
