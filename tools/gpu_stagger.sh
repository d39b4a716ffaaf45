#!/bin/bash
# SEM_AX_STAGGER probe: the second resident CTA of every SM waits X ns at
# entry so the two elements per SM run their phases out of step (large n).
# STAGGER_SPEC="n:variant:ns ns ...;..." (0 = no stagger)
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
OUT=gpurun_out/${STAGGER_OUT:-stagger2.jsonl}
: > $OUT
IFS=';' read -ra SPECS <<< "${STAGGER_SPEC}"
for rep in $(seq 1 ${STAGGER_REPS:-2}); do
for spec in "${SPECS[@]}"; do
  n=$(echo $spec | cut -d: -f1); v=$(echo $spec | cut -d: -f2); vals=$(echo $spec | cut -d: -f3)
  for st in $vals; do
    SEM_AX_STAGGER=$st timeout 300 python tools/ax_sweep.py --n $n --E 4096 --variants $v --reps 30 --repeat 3 --cool 0.3 | sed "s/^/{\"stagger\": \"$st\", \"r\": /; s/\$/}/" >> $OUT
  done
done
done
cat $OUT
