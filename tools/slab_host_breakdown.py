"""Host time per call category of the z-slab CG driver loop (NCCL world 1):
where the Python side of an iteration goes."""
import collections
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import dist as D  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29583")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
E, n, iters = 4096, 10, 200
ex, ey, ez = sb.factor_elements(E)
b = sb.build_basis(n)
part = D.SlabPartition(ex, ey, ez, n, 1, 0)
geom = sb.build_geom(sb.build_mesh(ex, ey, ez, n, 1.0), b, device=dev)
topo = sb.build_topology(sb.build_mesh(ex, ey, ez, n, 1.0))
f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
comm = D.SlabComm(part)
ops = D.CudaSlabOps(part, geom.values, b, iters, dev)
acc = collections.Counter()
cnt = collections.Counter()


def wrap(obj, name, label):
    fn = getattr(obj, name)

    def w(*a, **k):
        t0 = time.perf_counter()
        r = fn(*a, **k)
        acc[label] += time.perf_counter() - t0
        cnt[label] += 1
        return r
    setattr(obj, name, w)


for nm in ("ax_layers", "plane_top", "plane_bottom", "update", "finish", "local_sum"):
    wrap(ops, nm, "ops." + nm)
for nm in ("allgather", "exchange_up_start", "exchange_up_wait", "exchange_down"):
    wrap(comm, nm, "comm." + nm)
D.dist_cg_solve(ops, comm, f, 3)
torch.cuda.synchronize(dev)
acc.clear(); cnt.clear()
t0 = time.perf_counter()
D.dist_cg_solve(ops, comm, f, iters)
total = time.perf_counter() - t0
torch.cuda.synchronize(dev)
out = {k: round(v / iters * 1e6, 1) for k, v in sorted(acc.items(), key=lambda kv: -kv[1])}
out["total_us_per_it"] = round(total / iters * 1e6, 1)
print(json.dumps(out))
dist.destroy_process_group()
