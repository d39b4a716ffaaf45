"""A/B of fused-CG launch structures at E = 4096 with idle gaps (the whole
solve is power-sensitive: back-to-back solves drift 5-10% slower).  Each
configuration: 1 s idle, then the best of 3 100-iteration solves (CUDA
events around cg_solve).  GRAPH_ITERATIONS from CG_GRAPH_KS; other knobs
from the environment (read once per process)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import cg as C  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n, E, iters = 10, int(os.environ.get("CG_E", "4096")), 100
b = sb.build_basis(n)
mesh = sb.build_mesh(*sb.factor_elements(E), n, 1.0)
topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
op = sb.GlobalOperator(geom, b, topo)
ks = [int(x) for x in os.environ.get("CG_GRAPH_KS", "1,5").split(",")]
out = {k: [] for k in ks}
for rep in range(int(os.environ.get("CG_REPS", "3"))):
    for k in ks:
        C.GRAPH_ITERATIONS = k
        ws = sb.CgWorkspace(topo, iters, dev)
        sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)  # capture + warm
        torch.cuda.synchronize()
        time.sleep(float(os.environ.get("CG_IDLE", "1.0")))
        best = None
        for _ in range(3):
            if os.environ.get("CG_WARM"):  # a short burst of iterations first
                sb.cg_solve(f, op, topo, sb.CgConfig(int(os.environ["CG_WARM"]), 0.0), workspace=ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / iters
            best = us if best is None else min(best, us)
        out[k].append(round(best, 2))
print(json.dumps({"E": E, "env": {k: v for k, v in os.environ.items() if k.startswith("SEM_CG")},
                  "us_per_iteration_by_graph_k": out}))
