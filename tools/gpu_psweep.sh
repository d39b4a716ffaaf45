#!/bin/bash
# p-sweep (all variants, best of 3 graph timings, same-bytes copy beside each n)
# and the E-sweep at n = 10
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python tools/ax_sweep.py --n ${NS:-2,3,4,5,6,7,8,9,10,11,12,13,14,15,16} --E 4096 --reps 30 --repeat 3 --copy > gpurun_out/psweep.jsonl 2> gpurun_out/psweep.err
timeout 600 python tools/ax_sweep.py --n 10 --E 512,1024,2048,4096,8192 --variants 0,34,52 --reps 50 --repeat 3 --copy > gpurun_out/esweep.jsonl 2> gpurun_out/esweep.err
