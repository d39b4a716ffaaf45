#!/bin/bash
# SEM_CG_FIN A/B (2: <r, r> finished by the update's last block; 3: folded
# into the next Ax CTAs + settle): CG mode tests, then idle-gapped whole
# solves alternating the two settings in separate processes.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_cg_modes.py -q -m gpu > gpurun_out/fin_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fin_tests.log
SEM_CG_FIN=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "cg or CG" > gpurun_out/fin3_parity.log 2>&1; echo "rc=$?" >> gpurun_out/fin3_parity.log
: > gpurun_out/fin_ab.jsonl
for rep in 1 2 3; do
  for fin in 2 3; do
    for e in 4096 32768; do
      SEM_CG_FIN=$fin CG_E=$e CG_GRAPH_KS=10 CG_REPS=2 timeout 300 python tools/cg_ab.py >> gpurun_out/fin_ab.jsonl 2>> gpurun_out/fin_ab.err
    done
  done
done
tail -3 gpurun_out/fin_tests.log; tail -2 gpurun_out/fin3_parity.log; cat gpurun_out/fin_ab.jsonl
