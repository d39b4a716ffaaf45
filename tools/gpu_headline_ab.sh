#!/bin/bash
# Headline bench (driver flags, headline key only) alternating the default
# build behaviour (B) with an environment override (A: $AB_ENV_A), 4 x each.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ax_tuning.py tests/test_gpu_parity.py -q -m gpu > gpurun_out/hl_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hl_tests.log
: > gpurun_out/headline_ab.txt
FL="--gpus 1 --steps 20 --warmup 5 --no-cpu --e2e-steps 0 --cg 0 --cg-weak 0 --cg-slab1 0 --ax-sizes 0 --psweep 0"
for rep in 1 2 3 4; do
  for arm in A B; do
    if [ $arm = A ]; then
      env $AB_ENV_A timeout 300 python bench.py $FL 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('A', d['ms_per_step']*1e3, d['roofline']['frac'], d['clocks']['sm_mhz'])" >> gpurun_out/headline_ab.txt
    else
      timeout 300 python bench.py $FL 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('B', d['ms_per_step']*1e3, d['roofline']['frac'], d['clocks']['sm_mhz'])" >> gpurun_out/headline_ab.txt
    fi
  done
done
tail -2 gpurun_out/hl_tests.log; cat gpurun_out/headline_ab.txt
