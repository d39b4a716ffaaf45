#!/bin/bash
# software-pipelined update (SEM_CG_UPD=2) at 4 and 3 blocks/SM vs the default row kernel
cd ${GRAFT_REPO_ROOT:-.}
SEM_CG_UPD=2 timeout 600 python -m pytest -q -x tests/test_gpu_parity.py -k "cg" tests/test_dist_gpu.py 2>&1 | tail -1
for mb in 4 3; do
  SEM_NVCC_DEFS="SEM_UPD4_MINB=$mb" python -m paper_2005_13425_b200.build --force > /dev/null 2>&1
  cuobjdump -res-usage paper_2005_13425_b200/libsem.so 2>/dev/null | grep -A1 "cg_update4_kernelILi10ELb0" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | tr '\n' ' '; echo
  for upd in 0 2 0 2; do
    echo "minb4=$mb upd=$upd $(SEM_CG_UPD=$upd timeout 120 python tools/cg_phases.py 4096 32768 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})')"
  done
done
