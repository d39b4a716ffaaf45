#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py,
# default kernels and the opt-in CG forms (cube update, folded settle)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/sanitize.txt
: > $out
for envs in ${ENVS:-"" "SEM_CG_UPD_ELEM=1" "SEM_CG_SETTLE=0"}; do
  for tool in memcheck racecheck synccheck; do
    echo "== ${envs:-default} compute-sanitizer --tool $tool python tools/sanitize.py" >> $out
    env $envs timeout 1200 compute-sanitizer --tool $tool python tools/sanitize.py 2>&1 | grep -E "COMPUTE-SANITIZER|SUMMARY|ok|rror" | head -20 >> $out
  done
done
