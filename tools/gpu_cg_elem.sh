cd $GRAFT_REPO_ROOT
for rep in 1 2 3 4; do for env in "SEM_CG_ALT=0" "SEM_CG_ALT=1"; do env $env CG_REPS=2 CG_GRAPH_KS=10 python tools/cg_ab.py; done; done > gpurun_out/cg_alt2.txt 2>&1
