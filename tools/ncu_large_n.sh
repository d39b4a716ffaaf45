#!/bin/bash
# ncu --set full of the default Ax kernel at the large degrees (E = 4096);
# only the text summaries are kept (full reports exceed the pull-back limit)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for n in ${NS:-13 14 15 16}; do
  timeout 600 ncu --set full --clock-control none -k regex:ax_ -s 4 -c 1 \
    -o /tmp/ax_n${n}_full -f python tools/ax_sweep.py --n $n --E 4096 --variants ${VARIANT:-0} --reps 5 \
    > gpurun_out/ncu_n${n}.log 2>&1
  python tools/ncu_brief.py /tmp/ax_n${n}_full.ncu-rep > gpurun_out/ax_n${n}_brief.txt 2>&1
  ncu -i /tmp/ax_n${n}_full.ncu-rep --page raw --csv 2>/dev/null | python tools/ncu_stalls.py > gpurun_out/ax_n${n}_stalls.txt 2>&1
done
