#!/bin/bash
# Fused-CG A/B of two environment settings (AB_ENV_A vs AB_ENV_B; one
# process per setting, alternated 3 x, tools/cg_ab.py idle-gapped solves).
# TESTS=paths runs those pytest files first.
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest $TESTS -q -m gpu > gpurun_out/env_ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/env_ab_tests.log
fi
: > gpurun_out/env_ab.jsonl
for rep in 1 2 3; do
  for arm in A B; do
    for e in ${CG_ES:-4096 32768}; do
      if [ $arm = A ]; then EV="$AB_ENV_A"; else EV="$AB_ENV_B"; fi
      echo -n "{\"arm\": \"$arm\", \"r\": " >> gpurun_out/env_ab.jsonl
      env $EV CG_E=$e CG_GRAPH_KS=10 CG_REPS=2 timeout 300 python tools/cg_ab.py | tr -d '\n' >> gpurun_out/env_ab.jsonl
      echo "}" >> gpurun_out/env_ab.jsonl
    done
  done
done
[ -n "${TESTS:-}" ] && tail -3 gpurun_out/env_ab_tests.log
cat gpurun_out/env_ab.jsonl
