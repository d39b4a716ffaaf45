cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cg_modes.py -q -x > gpurun_out/cg_modes.log 2>&1
for env in "SEM_CG_UPD_PF=0" "SEM_CG_UPD_PF=1" "SEM_CG_UPD_PF=1 SEM_CG_PDL=1" "SEM_CG_UPD_PF=0 SEM_CG_PDL=1" "SEM_CG_UPD_PF=1 SEM_CG_ROW_THREADS=128"; do echo "$env $(env $env timeout 300 python tools/cg_time.py 4096 32768 2>&1 | tail -1)"; done > gpurun_out/cg_elem.txt
