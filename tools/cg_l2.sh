#!/bin/bash
# Fused CG per-iteration time with an L2 access-policy window over the
# iteration's hot vectors (cg.py _l2_window): modes x hit ratios.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
python -c "
import ctypes, torch; torch.cuda.init()
from paper_2005_13425_b200._lib import load
a,b,c=ctypes.c_int64(),ctypes.c_int64(),ctypes.c_int64()
load().sem_l2_props(ctypes.byref(a),ctypes.byref(b),ctypes.byref(c)); print('persist_max',a.value,'window_max',b.value,'l2',c.value)"
for mode in off rw prw xprw; do
  for hit in ${HITS:-1.0 0.7}; do
    [ $mode = off ] && [ $hit != 1.0 ] && continue
    echo "mode=$mode hit=$hit $(SEM_CG_L2=$mode SEM_CG_L2_HIT=$hit timeout 300 python tools/cg_time.py ${SIZES:-4096 32768} 2>&1 | tail -1)"
  done
done
