"""Per-solve times of back-to-back fused CG solves (E = 4096, 100 iterations)
to locate occasional slow solves: as-is, with the cyclic GC disabled, and
with the stop-flag polling off."""
import gc
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import cg as C  # noqa: E402

dev = torch.device("cuda", 0)
n, E, iters = 10, 4096, 100
b = sb.build_basis(n)
mesh = sb.build_mesh(*sb.factor_elements(E), n, 1.0)
topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
op = sb.GlobalOperator(geom, b, topo)
ws = sb.CgWorkspace(topo, iters, dev)
junk = [{"a": [i] * 3} for i in range(300000)]  # a bench-sized heap


def run(label, count=10):
    sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
    torch.cuda.synchronize()
    out = []
    for _ in range(count):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        out.append(round(e0.elapsed_time(e1) * 1e3 / iters, 2))
    print(json.dumps({label: out}), flush=True)


run("default")
gc.disable()
run("gc_off")
gc.enable()
C.POLL_EVERY = 10 ** 9
run("no_poll")
C.POLL_EVERY = 8

# fixed per-solve cost: solves of 12 and 112 iterations (both graph-replayed)
def solve_ms(it):
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sb.cg_solve(f, op, topo, sb.CgConfig(it, 0.0), workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


ws = sb.CgWorkspace(topo, 112, dev)
sb.cg_solve(f, op, topo, sb.CgConfig(112, 0.0), workspace=ws)
a, b2 = solve_ms(12), solve_ms(112)
per_it = (b2 - a) / 100
print(json.dumps({"per_iteration_us": round(per_it * 1e3, 2), "fixed_per_solve_us": round((a - 12 * per_it) * 1e3, 1)}))
