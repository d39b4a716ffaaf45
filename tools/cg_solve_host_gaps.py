"""Host time before the first launch and after the last one in cg_solve:
CUDA events recorded on the solve's stream by wrappers around the libsem
entry points (the GPU is idle around a solve, so an event's GPU timestamp is
the moment the host enqueued it)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200._lib import load  # noqa: E402

dev = torch.device("cuda", 0)
n, E, iters = 10, 4096, 100
b = sb.build_basis(n)
mesh = sb.build_mesh(*sb.factor_elements(E), n, 1.0)
topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
op = sb.GlobalOperator(geom, b, topo)
ws = sb.CgWorkspace(topo, iters, dev)
lib = load()
marks = []


def wrap(name):
    orig = getattr(lib, name)

    def w(*a):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((name, e))
        return orig(*a)
    setattr(lib, name, w)


for nm in ("sem_consistent_box", "sem_cg_init", "sem_cg_run_at", "sem_cg_finalize"):
    wrap(nm)
for _ in range(2):
    sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
torch.cuda.synchronize()
rows = []
for _ in range(5):
    marks.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    rows.append({"total_us": round(e0.elapsed_time(e1) * 1e3, 1),
                 **{f"{i}:{nm}": round(e0.elapsed_time(e) * 1e3, 1) for i, (nm, e) in enumerate(marks)}})
for r in rows:
    print(json.dumps(r))
