#!/bin/bash
# One GPU session: parity tests, smoke, bench, launch list, one ncu --set full
# capture of the Ax kernel, and the all-n sweep.  Outputs land in gpurun_out/.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
(nproc; lscpu | grep "Model name") >> gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 20 --warmup 3 --soak 0 --no-cpu --e2e-steps 0 --cg 0 --cg-weak 0 --cg-slab1 0 --ax-sizes 0 --psweep 0 > gpurun_out/bench_ncu.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:ax_pencil -s 8 -c 1 -o gpurun_out/ax_full -f \
      python bench.py --steps 10 --warmup 3 --soak 0 --no-cpu --cg 0 --cg-weak 0 --cg-slab1 0 --e2e-steps 0 --ax-sizes 0 --psweep 0 > gpurun_out/ncu_full.log 2>&1
fi
if [ "${SWEEP:-1}" = "1" ]; then
  timeout 900 python tools/ax_sweep.py --n 2,3,4,5,6,7,8,9,10,11,12,13,14,15,16 --E 4096 --reps 30 > gpurun_out/sweep_all.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/bench.log | cut -c1-400; tail -1 gpurun_out/bench_ref.log | cut -c1-300
