"""Timeline of the fused CG iteration chain (needs a -DSEM_TRACE build:
SEM_NVCC_DEFS=SEM_TRACE python -m paper_2005_13425_b200.build --force).
Per kernel of an iteration (K1 = Ax + iteration head, settle, update): the
earliest CTA entry, the earliest return from griddep_wait and the latest CTA
exit, in us relative to K1's first entry, averaged over the steady
iterations of a graph-replayed 100-iteration solve at E = 4096, p = 9."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import cg as C  # noqa: E402
from paper_2005_13425_b200.cg import ctypes_sizeof_state  # noqa: E402

C.GRAPH_ITERATIONS = int(os.environ.get("CG_GRAPH_K", "1"))

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n = 10
E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = 100
b = sb.build_basis(n)
mesh = sb.build_mesh(*sb.factor_elements(E), n, 1.0)
topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
op = sb.GlobalOperator(geom, b, topo)
ws = sb.CgWorkspace(topo, iters, dev)
S = ctypes_sizeof_state()
NK, SLOTS = 4, 128
big = torch.zeros(S + NK * SLOTS * 3 * 8, dtype=torch.uint8, device=dev)
ws.state = big
sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)   # warm-up (configures, captures)
tr = big[S:].view(torch.int64).view(NK, SLOTS, 3)
tr[:, :, 0:2] = torch.iinfo(torch.int64).max
tr[:, :, 2] = 0
torch.cuda.synchronize()
res = sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.float64)
print("nonzero exits per kernel:", [(int((t[k, :, 2] > 0).sum())) for k in range(3)], "iterations", res.iterations_run,
      file=sys.stderr)
rows = []
for it in range(10, 90):
    k0 = t[0, it, 0]
    if t[0, it, 2] == 0 or t[2, it, 2] == 0:
        continue
    rel = lambda x: (x - k0) / 1e3  # noqa: E731
    nxt = t[0, it + 1, 0]
    rows.append([rel(t[0, it, 1]), rel(t[0, it, 2]), rel(t[1, it, 0]), rel(t[1, it, 1]), rel(t[1, it, 2]),
                 rel(t[2, it, 0]), rel(t[2, it, 1]), rel(t[2, it, 2]), rel(nxt)])
a = np.median(np.array(rows), axis=0)
names = ["K1 waited", "K1 end", "settle entry", "settle waited", "settle end", "update entry",
         "update waited", "update end", "next K1 entry"]
ms = None
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"E": E, "graph_k": C.GRAPH_ITERATIONS, "us_per_iteration": round(e0.elapsed_time(e1) * 1e3 / iters, 2),
                  "iterations_used": len(rows),
                  "median_us_from_K1_entry": {k: round(v, 2) for k, v in zip(names, a)}}, indent=1))
