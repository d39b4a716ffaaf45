#!/bin/bash
# Ax variant sweep at the paper's small sizes (n=10, E=1024/2048), a CG launch
# list and one ncu --set full capture of each CG kernel (E=4096).
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 python tools/ax_sweep.py --n 10 --E 1024,2048 --reps 200 > gpurun_out/sweep_smallE.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/cg_launches.csv \
    python tools/cg_time.py 4096 > gpurun_out/cg_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ax_pencil|cg_update2|cg_settle" -s 60 -c 3 \
    -o gpurun_out/cg_full -f python tools/cg_time.py 4096 > gpurun_out/cg_full.log 2>&1
tail -3 gpurun_out/cg_full.log
sort -t: -k5 -n gpurun_out/sweep_smallE.jsonl | head -3
