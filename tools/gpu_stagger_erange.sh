cd "${GRAFT_REPO_ROOT}"
mkdir -p gpurun_out
: > gpurun_out/stagger_erange.jsonl
for rep in 1 2; do
for arm in off on; do
  if [ $arm = off ]; then EV="SEM_AX_STAGGER=0"; else EV="SEM_AX_NOP=1"; fi
  env $EV timeout 600 python tools/ax_sweep.py --n 10,15,16 --E 2048,32768 --variants 0 --reps 10 --repeat 2 --cool 0.3 | sed "s/^/{\"arm\": \"$arm\", \"r\": /; s/\$/}/" >> gpurun_out/stagger_erange.jsonl
done
done
cat gpurun_out/stagger_erange.jsonl
