cd $GRAFT_REPO_ROOT
for env in "SEM_CG_AX_CFG=0" "SEM_CG_AX_CFG=11" "SEM_CG_AX_CFG=12" "SEM_CG_AX_CFG=9" "SEM_CG_AX_CFG=0"; do echo "$env $(env $env timeout 300 python tools/cg_time.py 4096 32768 2>&1 | tail -1)"; done > gpurun_out/cg_elem.txt
