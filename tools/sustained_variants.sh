# Sustained (power-capped) Ax time per kernel variant at E=4096, p=9: the
# bench protocol (1.5 s soak + 2000 timed steps), one process per variant.
cd ${GRAFT_REPO_ROOT:-.}
for v in ${VARIANTS:-0 26 25 35 37 38 40 41 53 5 8 19}; do
  sleep 3
  timeout 120 python bench.py --variant $v --no-cpu --e2e-steps 0 --cg 0 --cg-weak 0 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read())['sustained']; print($v, round(d['ms_per_step']*1e3,2), round(d['hbm_frac'],4), d['clocks']['sm_mhz'], d['clocks']['power_w_max'], round(d['same_bytes_copy']['ax_frac_of_copy'],4))"
done
