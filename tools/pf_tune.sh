# L2 prefetch distance sweep for the large-n Ax variants (SEM_AX_PFDIST =
# elements ahead of the CTA's own element; 0 = its own element).
cd ${GRAFT_REPO_ROOT:-.}
for d in default 0 1 4 16 148; do
  if [ "$d" = default ]; then unset SEM_AX_PFDIST; else export SEM_AX_PFDIST=$d; fi
  echo "pfdist=$d"
  timeout 300 python tools/ax_sweep.py --n 12,13,14,15,16 --E 4096 --reps 20 --variants 0,44 | grep '"us"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['n'], d['variant'], d['us'], d['frac'])"
done
