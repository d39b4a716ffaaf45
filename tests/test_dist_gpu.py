"""The distributed (z-slab) CG path with the CUDA per-rank kernels.

Only one GPU is available to the test tiers, so:
  * world size 1 over NCCL exercises the NCCL code path end to end and must
    reproduce the fused single-GPU solve bit-for-bit;
  * world sizes 2 and 4 run as processes SHARING cuda:0 over gloo (NCCL
    refuses two ranks on one device); the CUDA slab kernels and the halo
    protocol must give a dssum bit-identical to the global one and the
    single-GPU residual history.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

BOX = (4, 3, 8)
N = 6
ITERS = 40


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _global_problem(sb, dev):
    ex, ey, ez = BOX
    b = sb.build_basis(N)
    mesh = sb.build_mesh(ex, ey, ez, N, 1.0)
    topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
    E = mesh.num_elements
    f = sb.make_rhs(E, N, topo, sb.mix64(1, E), device=dev)
    return b, topo, geom, f


def _run_rank(rank, world, port, backend, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import paper_2005_13425_b200 as sb
    from paper_2005_13425_b200.dist import (CudaSlabOps, SlabComm, SlabPartition, dist_cg_solve,
                                            dist_dssum)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, topo, geom, f = _global_problem(sb, dev)
        ex, ey, ez = BOX
        part = SlabPartition(ex, ey, ez, N, world, rank)
        e0, e1 = part.element_range
        comm = SlabComm(part)
        g_local = geom.values[e0:e1].contiguous()
        ops = CudaSlabOps(part, g_local, b, ITERS, dev)
        field = sb.random_field(topo.num_elements, N, 5, device=dev)
        d_local = dist_dssum(ops, comm, field[e0:e1].contiguous(), apply_mask=True)
        res = dist_cg_solve(ops, comm, f[e0:e1].contiguous(), ITERS)
        q.put((rank, d_local.cpu().numpy(), res.residual_history.tolist(), res.iterations_run,
               res.solution.cpu().numpy(), (e0, e1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo"), (4, "gloo")])
def test_dist_cg_on_gpu(cuda, world, backend):
    import paper_2005_13425_b200 as sb
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_rank, args=(r, world, port, backend, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dev = torch.device("cuda", 0)
    b, topo, geom, f = _global_problem(sb, dev)
    field = sb.random_field(topo.num_elements, N, 5, device=dev)
    want = sb.mask(sb.dssum(field, topo), topo).cpu().numpy()
    ref = sb.cg_solve(f, sb.GlobalOperator(geom, b, topo), topo, sb.CgConfig(ITERS, 0.0))
    x_ref = ref.solution.cpu().numpy()
    for rank, d_local, hist, iters, x, (e0, e1) in out:
        assert np.array_equal(d_local, want[e0:e1]), f"rank {rank} dssum"
        assert iters == ref.iterations_run
        h = np.asarray(hist)
        rel = np.max(np.abs(h - ref.residual_history) / np.abs(ref.residual_history))
        # the slab solver reduces <p, w2>_c over the assembled field, the
        # single-GPU solver sums p . A_local p per element (ax_pencil.cuh,
        # CGM = 2): equal in exact arithmetic, rounding-level apart
        assert rel <= 1e-12
        assert np.max(np.abs(x - x_ref[e0:e1])) <= 1e-12 * np.max(np.abs(x_ref))
