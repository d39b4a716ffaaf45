# update2 occupancy experiment: rebuild with different __launch_bounds__ minimum
# blocks for cg_update2_kernel and time the CG phases.
cd ${GRAFT_REPO_ROOT:-.}
for mb in 1 6 8; do
  SEM_NVCC_DEFS="SEM_UPD_MINB=$mb" python -m paper_2005_13425_b200.build --force > /dev/null 2>&1
  echo "minb=$mb $(timeout 300 python tools/cg_phases.py | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})')"
done
