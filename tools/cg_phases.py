"""Per-phase device time of the fused single-GPU CG iteration (sem_cg_run_phases)
at the BASELINE CG sizes; prints JSON."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200.cg import CgWorkspace, fused_phase_seconds  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
for E in [int(a) for a in (sys.argv[1:] or ["4096", "32768"])]:
    n, iters = 10, 100
    mesh = sb.build_mesh(*sb.factor_elements(E), n, 1.0)
    b = sb.build_basis(n)
    topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
    f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
    op = sb.GlobalOperator(geom, b, topo)
    ws = CgWorkspace(topo, iters, dev)
    fused_phase_seconds(f, op, topo, 5, ws)
    t = fused_phase_seconds(f, op, topo, iters, ws)
    dofs = E * n ** 3
    out[f"E{E}"] = {"ax_us": t[0] / iters * 1e6, "update_us": t[1] / iters * 1e6,
                    "ax_GBps_96B": 96 * dofs / (t[0] / iters) / 1e9,
                    "update_GBps_24B": 24 * dofs / (t[1] / iters) / 1e9}
print(json.dumps(out, indent=1))
