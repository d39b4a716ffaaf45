#!/bin/bash
# A/B of two builds of libsem.so (ab/libsem_base.so = A, the in-tree build = B)
# on the fused CG: idle-gapped whole solves (tools/cg_ab.py), alternating the
# builds in separate processes.  TESTS=path runs that pytest file first (B).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
if [ -n "${TESTS:-}" ]; then
  timeout 900 python -m pytest $TESTS -q -m gpu > gpurun_out/ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tests.log
fi
: > gpurun_out/lib_ab.jsonl
for rep in 1 2 3; do
  for lib in A B; do
    for e in ${CG_ES:-4096 32768}; do
      if [ $lib = A ]; then L=ab/libsem_base.so; else L=paper_2005_13425_b200/libsem.so; fi
      echo -n "{\"lib\": \"$lib\", \"r\": " >> gpurun_out/lib_ab.jsonl
      SEM_LIBRARY=$L CG_E=$e CG_GRAPH_KS=10 CG_REPS=2 timeout 300 python tools/cg_ab.py | tr -d '\n' >> gpurun_out/lib_ab.jsonl 2>> gpurun_out/lib_ab.err
      echo "}" >> gpurun_out/lib_ab.jsonl
    done
  done
done
[ -n "${TESTS:-}" ] && tail -3 gpurun_out/ab_tests.log
cat gpurun_out/lib_ab.jsonl
