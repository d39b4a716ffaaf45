cd $GRAFT_REPO_ROOT
for c in 0 1 2 3 4 5; do for ub in 1184 4736; do
  echo "cfg=$c upd_blocks=$ub $(SEM_CG_AX_CFG=$c SEM_CG_UPD_BLOCKS=$ub timeout 120 python tools/cg_phases.py 4096 32768 | python -c 'import json,sys; d=json.load(sys.stdin); print({k:(round(v["ax_us"],1), round(v["update_us"],1)) for k,v in d.items()})')"
done; done
