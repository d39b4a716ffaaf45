"""Host enqueue time vs device time per iteration of the z-slab CG solver
(dist.py) on one GPU (NCCL world 1): is the Python driver loop the bound?"""
import json
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200.dist import CudaSlabOps, SlabComm, SlabPartition, dist_cg_solve  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29581")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
out = {}
for E in (4096, 32768):
    n, iters = 10, 100
    ex, ey, ez = sb.factor_elements(E)
    b = sb.build_basis(n)
    part = SlabPartition(ex, ey, ez, n, 1, 0)
    geom = sb.build_geom(sb.build_mesh(ex, ey, ez, n, 1.0), b, device=dev)
    topo = sb.build_topology(sb.build_mesh(ex, ey, ez, n, 1.0))
    f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
    comm = SlabComm(part)
    ops = CudaSlabOps(part, geom.values, b, iters, dev)
    dist_cg_solve(ops, comm, f, 3)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    # dist_cg_solve ends with a device->host read of the state (result()):
    # time the enqueue of the loop by the wall clock up to that point
    res = dist_cg_solve(ops, comm, f, iters)
    e1.record()
    t_host = time.perf_counter() - t0
    torch.cuda.synchronize(dev)
    out[f"E{E}"] = {"device_us_per_it": e0.elapsed_time(e1) * 1e3 / iters,
                    "host_wall_us_per_it": t_host * 1e6 / iters}
print(json.dumps(out))
dist.destroy_process_group()
