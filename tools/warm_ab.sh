#!/bin/bash
# headline protocol A/B: warm burst length and sync before the timed window
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
F="--steps 20 --warmup 5 --soak 0 --no-cpu --cg 0 --cg-weak 0 --cg-slab1 0 --ax-sizes 0 --psweep 0 --e2e-steps 0"
for rep in 1 2 3; do
for ws in 1 0; do for wm in 10 40 100; do
  echo "sync=$ws warm_ms=$wm $(python bench.py $F --warm-sync $ws --warm-ms $wm 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,2), round(d["roofline"]["frac"],4))')"
done; done; done
