#!/bin/bash
# source-level stall attribution of the Ax kernel at given n/variant pairs
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for nv in ${NV:-15:0 16:0}; do
  n=${nv%%:*}; v=${nv##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ax_ -s 4 -c 1 \
    -o /tmp/src_n$n -f python tools/ax_sweep.py --n $n --E 4096 --variants $v --reps 5 > /dev/null 2>&1
  ncu -i /tmp/src_n$n.ncu-rep --page source --csv --print-source cuda,sass 2>&1 | head -c 3000000 > gpurun_out/src_n${n}_raw.csv
  ncu -i /tmp/src_n$n.ncu-rep --page source --csv --print-source sass 2>&1 | head -c 3000000 > gpurun_out/src_n${n}_sass.csv
done
