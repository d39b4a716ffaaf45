#!/bin/bash
# SEM_CG_STAGGER probe on the fused CG (E = 4096): the second resident Ax
# CTA per SM idles X ns at entry of every Ax launch.  Then the large-n
# defaults (stagger counted in SM cycles) re-timed.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/cg_stagger.jsonl
for rep in 1 2; do
  for st in 0 1500 3000 4500; do
    echo -n "{\"stagger\": $st, \"r\": " >> gpurun_out/cg_stagger.jsonl
    SEM_CG_STAGGER=$st CG_E=4096 CG_GRAPH_KS=10 CG_REPS=2 timeout 300 python tools/cg_ab.py | tr -d '\n' >> gpurun_out/cg_stagger.jsonl
    echo "}" >> gpurun_out/cg_stagger.jsonl
  done
done
timeout 600 python tools/ax_sweep.py --n 12,13,14,15,16 --E 4096 --variants 0 --reps 30 --repeat 3 --cool 0.3 > gpurun_out/large_n_cycles.jsonl 2>&1
cat gpurun_out/cg_stagger.jsonl gpurun_out/large_n_cycles.jsonl
