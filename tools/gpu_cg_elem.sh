cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cg_modes.py tests/test_gpu_parity.py -q -x -k "cg or mode" > gpurun_out/cg_modes.log 2>&1
for rep in 1 2 3 4; do for env in "SEM_CG_PX_EARLY=0" "SEM_CG_PX_EARLY=1"; do env $env CG_REPS=2 CG_GRAPH_KS=10 python tools/cg_ab.py; done; done > gpurun_out/cg_px.txt 2>&1
for env in "SEM_CG_PX_EARLY=0" "SEM_CG_PX_EARLY=1"; do env $env CG_E=32768 CG_REPS=2 CG_GRAPH_KS=10 python tools/cg_ab.py; done >> gpurun_out/cg_px.txt 2>&1
