cd $GRAFT_REPO_ROOT
for rep in 1 2 3 4; do for env in "SEM_CG_ALT=1" "SEM_CG_ALT=2"; do env $env CG_REPS=2 CG_GRAPH_KS=10 python tools/cg_ab.py; done; done > gpurun_out/cg_alt3.txt 2>&1
for env in "SEM_CG_ALT=1" "SEM_CG_ALT=2"; do env $env CG_E=32768 CG_REPS=2 CG_GRAPH_KS=10 python tools/cg_ab.py; done >> gpurun_out/cg_alt3.txt 2>&1
