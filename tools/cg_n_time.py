"""CG solve time per iteration for several n at a fixed element count
(graph-replayed solver, CUDA events), e.g. to catch a slow fallback tiling."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
E = 4096
out = {}
for n in [int(a) for a in (sys.argv[1:] or ["4", "6", "8", "10", "12"])]:
    b = sb.build_basis(n)
    mesh = sb.build_mesh(*sb.factor_elements(E), n, 1.0)
    topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
    f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
    op = sb.GlobalOperator(geom, b, topo)
    ws = sb.CgWorkspace(topo, 50, dev)
    sb.cg_solve(f, op, topo, sb.CgConfig(50, 0.0), workspace=ws)  # warm-up (captures)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sb.cg_solve(f, op, topo, sb.CgConfig(50, 0.0), workspace=ws)
    e1.record()
    torch.cuda.synchronize(dev)
    us = e0.elapsed_time(e1) * 1e3 / 50
    out[n] = {"us_per_it": round(us, 1), "GBps_120B": round(120 * E * n ** 3 / us / 1e3, 1)}
print(json.dumps(out))
