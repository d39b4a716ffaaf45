import cProfile, pstats, sys, time, os
sys.path.insert(0, '/root/repo')
import torch
import paper_2005_13425_b200 as sb
dev = torch.device('cuda', 0)
n, E, iters = 10, 64, 30
b = sb.build_basis(n)
mesh = sb.build_mesh(4, 4, 4, n, 1.0)
topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
op = sb.GlobalOperator(geom, b, topo)
ws = sb.CgWorkspace(topo, iters, dev)
for _ in range(3): sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
torch.cuda.synchronize()
print("wall per solve us", (time.perf_counter() - t0) / 20 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(50): sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
pr.disable()
st = pstats.Stats(pr); st.sort_stats('tottime')
rows = sorted(st.stats.items(), key=lambda kv: -kv[1][2])[:25]
for k, v in rows: print(f"{v[2]/50*1e6:8.1f} us  {k[2]} {k[0].split('/')[-1]}:{k[1]}")
