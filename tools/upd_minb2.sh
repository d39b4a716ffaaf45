#!/bin/bash
# update2 occupancy x one-wave grid: rebuild with __launch_bounds__ min blocks
# MINB, grid = k * MINB * 148 (k = 1, 2), Ax reduction deferred.
cd ${GRAFT_REPO_ROOT:-.}
for mb in 5 6 8; do
  SEM_NVCC_DEFS="SEM_UPD_MINB=$mb" python -m paper_2005_13425_b200.build --force > /dev/null 2>&1
  cuobjdump -res-usage paper_2005_13425_b200/libsem.so 2>/dev/null | grep -A1 "cg_update2_kernelILi10ELb0" | grep -o "REG:[0-9]*\|STACK:[0-9]*" | tr '\n' ' '; echo
  for k in 1 2; do for fin in 2 1; do
    ub=$((k * mb * 148))
    echo "minb=$mb blocks=$ub fin=$fin $(SEM_CG_FIN=$fin SEM_CG_UPD_BLOCKS=$ub timeout 120 python tools/cg_phases.py 4096 32768 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})')"
  done; done
done
