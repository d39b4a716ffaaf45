cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -q -m gpu -k "cg or CG or dist or interop or harness or c_client or random" > gpurun_out/cg_tests.log 2>&1
for rep in 1 2 3; do
  SEM_CG_PDL=2 SEM_CG_UPD_REV=0 SEM_CG_ALT=0 CG_REPS=2 CG_GRAPH_KS=1 python tools/cg_ab.py
  CG_REPS=2 CG_GRAPH_KS=10 python tools/cg_ab.py
done > gpurun_out/cg_total.txt 2>&1
for rep in 1 2; do
  SEM_CG_PDL=2 SEM_CG_UPD_REV=0 SEM_CG_ALT=0 CG_E=32768 CG_REPS=2 CG_GRAPH_KS=1 python tools/cg_ab.py
  CG_E=32768 CG_REPS=2 CG_GRAPH_KS=10 python tools/cg_ab.py
done >> gpurun_out/cg_total.txt 2>&1
