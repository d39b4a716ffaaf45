"""Multi-rank (z-slab) host logic on CPU with the gloo backend.

The distributed driver (paper_2005_13425_b200/dist.py: partition, ordered
two-step halo, rank-ordered scalar combine, CG choreography) runs here over
world sizes 2, 3 and 4 with a numpy implementation of the per-rank compute
(test infrastructure; the product's per-rank compute is CudaSlabOps).  The
distributed dssum must equal the GLOBAL oracle dssum bit-for-bit, and the
distributed CG must reproduce the global oracle's residual history.
"""

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2005_13425_b200.dist import (SlabComm, SlabPartition, dist_cg_solve, dist_dssum)


class NumpySlabOps:
    """Per-rank compute in numpy, mirroring CudaSlabOps' interface and the
    device kernels' scalar semantics (csrc/cg.cu fin_* functions, the fused
    Ax prologue/epilogue of ax_pencil.cuh)."""

    def __init__(self, part: SlabPartition, g_global, dx, dxt, topo_global, max_iterations):
        self.part = part
        e0, e1 = part.element_range
        self.g = g_global[e0:e1]
        self.dx, self.dxt = dx, dxt
        n = part.n
        self.gid = topo_global.global_id[e0:e1]
        self.maskv = topo_global.mask[e0:e1]
        self.invm = (1.0 / topo_global.multiplicity[e0:e1].astype(np.float64))
        nx = part.ex * (n - 1) + 1
        k = np.arange(n).reshape(1, n, 1, 1)
        j = np.arange(n).reshape(1, 1, n, 1)
        i = np.arange(n).reshape(1, 1, 1, n)
        el = np.arange(part.num_elements)
        ix = (el % part.ex).reshape(-1, 1, 1, 1)
        iy = ((el // part.ex) % part.ey).reshape(-1, 1, 1, 1)
        izl = (el // (part.ex * part.ey)).reshape(-1, 1, 1, 1)
        shape = (part.num_elements, n, n, n)
        self.plane_idx = np.broadcast_to((iy * (n - 1) + j) * nx + (ix * (n - 1) + i), shape)
        self.on_bot = np.broadcast_to((izl == 0) & (k == 0), shape)
        self.on_top = np.broadcast_to((izl == part.ez - 1) & (k == n - 1), shape)
        ps = part.plane_size
        self.bottom_prefix = torch.zeros(ps, dtype=torch.float64)
        self.top_totals = torch.zeros(ps, dtype=torch.float64)
        self.history = np.zeros(max_iterations)
        self.st = dict(rtz=0.0, rtz_old=1.0, pap=0.0, alpha=0.0, it=0, iters=0, stop=0,
                       bit=0, tol=0.0, xpend=False)
        self.local = torch.zeros(1, dtype=torch.float64)

    def scalar_buffer(self, world):
        return torch.zeros(world, dtype=torch.float64)

    def local_sum(self):
        return self.local

    def _wdot(self, a, b):
        return float(np.sum((a * b) * self.invm))

    def init(self, f, max_iterations, tolerance):
        self.r = f * self.maskv
        self.x = np.zeros_like(self.r)
        self.p = np.zeros_like(self.r)
        self.st.update(tol=tolerance)
        self.local[0] = self._wdot(self.r, self.r)

    def finish(self, phase, gathered):
        st = self.st
        if phase != 0 and st["stop"]:
            return
        total = 0.0
        for v in gathered.tolist():
            total += v
        if phase == 0:
            st.update(rtz=total, rtz_old=1.0, it=0, iters=0, stop=0)
        elif phase == 1:
            st["pap"] = total
            st["xpend"] = False
            if total <= 0.0:
                st["stop"], st["bit"] = 2, st["it"] + 1
            else:
                st["alpha"] = st["rtz"] / total
        else:
            it = st["it"] + 1
            rn = math.sqrt(total)
            self.history[it - 1] = rn
            st.update(iters=it, rtz_old=st["rtz"], rtz=total, it=it, xpend=True)
            if st["tol"] > 0.0 and rn < st["tol"]:
                st["stop"] = 3

    def settle(self):
        """Mirror of sem_cg_settle_slab: ax_layers already accumulated."""

    def ax_layers(self, l0, l1, first):
        """Mirror of sem_cg_ax_slab: owed x update, p = beta p + r, w = A_local p
        and the local sum of p.(A_local p) on element layers [l0, l1)."""
        st = self.st
        if l1 <= l0 or st["stop"]:
            return
        it = st["it"] + 1
        if st["rtz"] == 0.0:
            self.history[it - 1] = 0.0
            st.update(iters=it, stop=1)
            return
        beta = 0.0 if it == 1 else st["rtz"] / st["rtz_old"]
        if not hasattr(self, "w") or self.w is None or self.w.shape != self.p.shape:
            self.w = np.zeros_like(self.p)
        per = self.part.ex * self.part.ey
        a, b = l0 * per, l1 * per
        if st["xpend"]:
            xs = np.ascontiguousarray(self.x[a:b])
            O.axpy_into(xs, np.ascontiguousarray(self.p[a:b]), st["alpha"])
            self.x[a:b] = xs
        ps = np.ascontiguousarray(self.p[a:b])
        O.scale_add(ps, np.ascontiguousarray(self.r[a:b]), beta)
        self.p[a:b] = ps
        self.w[a:b] = O.ax_layered(ps, self.g[a:b], self.dx, self.dxt)
        part = float(np.sum(ps * self.w[a:b]))
        self.local[0] = part if first else float(self.local[0]) + part

    def finalize(self):
        st = self.st
        if st["xpend"] and st["stop"] != 2:
            O.axpy_into(self.x, self.p, st["alpha"])
            st["xpend"] = False

    def _plane(self, field, sel, prefix):
        acc = np.zeros(self.part.plane_size) if prefix is None else prefix.numpy().copy()
        np.add.at(acc, self.plane_idx[sel], field[sel])  # ascending local index order
        return torch.from_numpy(acc)

    def plane_top(self, field):
        return self._plane(field, self.on_top, None)

    def plane_bottom(self, field, prefix):
        return self._plane(field, self.on_bot, prefix)

    def dssum(self, field, bot, top, apply_mask=False):
        gid = self.gid.ravel()
        uniq, inv = np.unique(gid, return_inverse=True)
        acc = np.bincount(inv, weights=field.ravel(), minlength=uniq.size)
        out = acc[inv].reshape(field.shape)
        if bot is not None:
            out[self.on_bot] = bot.numpy()[self.plane_idx[self.on_bot]]
        if top is not None:
            out[self.on_top] = top.numpy()[self.plane_idx[self.on_top]]
        return out * self.maskv if apply_mask else out

    def update(self, bot, top):
        if self.st["stop"]:
            return
        a = self.st["alpha"]
        w2 = self.dssum(self.w, bot, top, apply_mask=True)
        O.axpy_into(self.r, np.ascontiguousarray(w2), -a)
        self.local[0] = self._wdot(self.r, self.r)

    def update_alpha(self, bot, top, gathered):
        """Mirror of sem_cg_update_slab_alpha: finish(1) folded into update."""
        self.finish(1, gathered)
        self.update(bot, top)

    def result(self):
        st = self.st
        return (self.x, self.history[:st["iters"]].copy(), st["iters"], st["stop"], st["pap"],
                st["bit"])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


BOX = (3, 2, 5)
N = 4
ITERS = 25


def _problem(box=BOX):
    ex, ey, ez = box
    E = ex * ey * ez
    b_nodes = None  # basis from the golden fixture (pinned to the reference)
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))
    dx, dxt, wts = G[f"basis/{N}/diff"], G[f"basis/{N}/diff_t"], G[f"basis/{N}/weights"]
    T = O.BoxTopology(ex, ey, ez, N)
    g = O.box_geom(ex, ey, ez, wts, 1.0)
    f = O.mask(O.dssum(O.random_field(E, N, O.mix64(1, E)), T), T)
    return dx, dxt, T, g, f, b_nodes


def _worker(rank, world, port, q, box=BOX):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dx, dxt, T, g, f, _ = _problem(box)
        ex, ey, ez = box
        part = SlabPartition(ex, ey, ez, N, world, rank)
        e0, e1 = part.element_range
        comm = SlabComm(part)
        # 1. distributed dssum of a random field, bit-exact vs the global one
        ops = NumpySlabOps(part, g, dx, dxt, T, ITERS)
        field = O.random_field(T.num_elements, N, 99)
        field.ravel()[::37] = -0.0
        got = dist_dssum(ops, comm, np.ascontiguousarray(field[e0:e1]), apply_mask=True)
        want = O.mask(O.dssum(field, T), T)[e0:e1]
        ok_dssum = bool(np.array_equal(got, want))
        # 2. distributed CG vs the global oracle CG
        ops = NumpySlabOps(part, g, dx, dxt, T, ITERS)
        res = dist_cg_solve(ops, comm, np.ascontiguousarray(f[e0:e1]), ITERS)
        q.put((rank, ok_dssum, res.residual_history.tolist(), res.iterations_run,
               res.solution.copy(), (e0, e1)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,box", [(2, BOX), (3, BOX), (4, BOX),
                                       (8, (2, 2, 8))])  # world 8: one element layer per rank
def test_dist_dssum_and_cg_gloo(world, box):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, box)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dx, dxt, T, g, f, _ = _problem(box)
    x_ref, hist_ref, its = O.cg(f, lambda p: O.apply_global(p, g, dx, dxt, T), T, ITERS)
    hists = {r: h for r, _, h, _, _, _ in out}
    for rank, ok_dssum, hist, iters, x, (e0, e1) in out:
        assert ok_dssum, f"rank {rank}: distributed dssum differs from the global one"
        assert iters == its
        assert hist == hists[0], "ranks disagree on the residual history"
        h = np.asarray(hist)
        assert np.max(np.abs(h - hist_ref) / np.abs(hist_ref)) <= 1e-10
        assert O.rel_diff(x, x_ref[e0:e1]) <= 1e-10


def test_partition_layers():
    sizes = [SlabPartition(4, 4, 10, 5, 4, r).ez for r in range(4)]
    assert sizes == [3, 3, 2, 2]
    p0, p3 = SlabPartition(4, 4, 10, 5, 4, 0), SlabPartition(4, 4, 10, 5, 4, 3)
    assert p0.lower is None and p0.upper == 1 and p3.upper is None and p3.lower == 2
    assert p3.element_range == (8 * 16, 10 * 16)
    assert p0.plane_size == 17 * 17
    with pytest.raises(ValueError):
        SlabPartition(2, 2, 3, 4, 4, 0)
