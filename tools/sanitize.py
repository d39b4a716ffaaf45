"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every kernel family once on tiny inputs."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200.kernels import apply_ax_into  # noqa: E402

dev = torch.device("cuda", 0)
for n in (3, 4, 6, 7, 8, 10, 11, 12, 14, 16):
    E = 5
    b = sb.build_basis(n)
    u = sb.random_field(E, n, 1, device=dev)
    g = sb.GeomFactors(values=sb.random_field(6 * E, n, 2, device=dev).reshape(E, 6, n, n, n))
    for v in ("layered", "reference") + (("scratch",) if n <= 10 else ()):
        sb.apply_ax(u, g, b, v)
    w = torch.empty_like(u)
    for var in (0, 34, 40, 47, 48, 50):
        apply_ax_into(u, g.values, b, w, var)
    sb.apply_ax(u.cpu().pin_memory(), g, b)          # zero-copy host path
    sb.apply_ax(u.cpu().numpy(), g, b)               # staged numpy path
    mesh = sb.build_mesh(2, 2, 2, n, 1.0)
    topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
    f = sb.make_rhs(8, n, topo, sb.mix64(1, 8), device=dev)
    sb.cg_solve(f, sb.GlobalOperator(geom, b, topo), topo, sb.CgConfig(4, 0.0))
    if n in (7, 10):  # graph-replayed iterations with programmatic launches
        sb.cg_solve(f, sb.GlobalOperator(geom, b, topo), topo, sb.CgConfig(25, 0.0))
    sb.cg_solve(f, lambda x: sb.apply_global(x, geom, b, topo), topo, sb.CgConfig(3, 0.0))
    sb.weighted_dot(f, f, topo)
# large-n tilings with the wave-ahead u prefetch need more elements than one
# resident wave (E > 2 x 148) to engage it
for n in (12, 13):
    E = 320
    b = sb.build_basis(n)
    u = sb.random_field(E, n, 3, device=dev)
    gv = sb.random_field(6 * E, n, 4, device=dev).reshape(E, 6, n, n, n)
    w = torch.empty_like(u)
    for var in (0, 71, 72, 73, 74, 75):
        apply_ax_into(u, gv, b, w, var)
import warnings  # noqa: E402
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    sb.measure_bandwidth(64 * 1000, repetitions=10)   # streaming-copy probe kernel
torch.cuda.synchronize()
print("sanitize workload ok")
