"""Multi-GPU CG on an element-partitioned box (BASELINE config 5).

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The
reference's element order e = ix + ex*(iy + ey*iz) (sembench/assembly.py:
76-79) makes contiguous element ranges z-slabs, so rank r owns global element
layers [z0, z1) and its local fields are exactly the slice [z0*ex*ey,
z1*ex*ey) of the global arrays.

Per CG iteration (the recurrence of sembench/cg.py:148-186), the single-GPU
solver's two kernels per rank (csrc/cg.cu):

    Ax launch(es): x += alpha_prev p_old (owed from the previous
        iteration), p = beta p + r, w = A_local p, local sum of p.(A_local p)
        -- bottom/top element layers first, the interior overlapping the
        first halo step                                       (sem_cg_ax_slab)
    halo, step 1: top-face partial sums  -> rank r+1               (plane_top)
    halo, step 2: continue the prefix with own bottom-face copies
                  -> interface totals    -> rank r-1               (plane_bottom)
    all_gather of the <p, A p> partials; every update CTA combines them
         in rank order -> alpha (finish 1 folded into the update launch)
    r -= alpha mask(dssum(w)) with the faces taken from the totals,
         local <r, r>_c partial -> all_gather                (update, finish 2)

and after the loop the owed x += alpha p (sem_cg_finalize).  <p, A p> is the
sum over elements of p.(A_local p), each element owned by exactly one rank,
so the rank partials need no halo (p is continuous and masked; see
ax_pencil.cuh).  The second exchange overlaps the settle of <p, A p> and
its gather.

With one rank there is no halo and no gather (the slab is the box, a rank's
partial is the total), so the iteration is one Ax launch, one settle, the
update and finish 2.  Over NCCL the iteration is captured once in a CUDA
graph and replayed (the launches are parameter-stable: scalars live in the
device state), so the driver loop is not host-bound at small slabs; early
exits are device-side (stop flag) and polled without blocking.

The two-step halo reproduces the reference's bincount order bit-for-bit:
every copy on rank r-1's side of an interface has a lower element id than
any copy on rank r's side, so rank r-1's ordered partial IS the prefix of the
reference's sum.  Dot products combine per-rank partials in rank order on
every rank (deterministic, identical scalars everywhere; the early-exit
flags therefore agree across ranks).

The driver is written against two small interfaces -- ``SlabOps`` (the
per-rank compute) and ``SlabComm`` (the exchanges) -- so the choreography is
exercised on CPU with the gloo backend in tests/test_dist_gloo.py; the
product implementation of ``SlabOps`` is ``CudaSlabOps`` (libsem kernels).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _device as dv
from ._lib import check, load, sem_cg_state

_STOP_OFFSET = sem_cg_state.stop.offset

__all__ = ["SlabPartition", "SlabComm", "CudaSlabOps", "dist_cg_solve", "dist_dssum",
           "dist_cg_phases", "halo_exchange", "DistCgResult"]


@dataclass(frozen=True)
class SlabPartition:
    """Rank `rank` of `world` owns global element layers [z0, z1)."""

    ex: int
    ey: int
    ez_global: int
    n: int
    world: int
    rank: int

    def __post_init__(self):
        if not (0 <= self.rank < self.world):
            raise ValueError(f"rank {self.rank} outside world of size {self.world}")
        if self.ez_global < self.world:
            raise ValueError(f"{self.ez_global} element layers cannot be split over "
                             f"{self.world} ranks (each needs >= 1 layer)")

    @staticmethod
    def layer_range(ez_global: int, world: int, rank: int) -> tuple[int, int]:
        base, extra = divmod(ez_global, world)
        z0 = rank * base + min(rank, extra)
        return z0, z0 + base + (1 if rank < extra else 0)

    @property
    def z0(self) -> int:
        return self.layer_range(self.ez_global, self.world, self.rank)[0]

    @property
    def z1(self) -> int:
        return self.layer_range(self.ez_global, self.world, self.rank)[1]

    @property
    def ez(self) -> int:
        return self.z1 - self.z0

    @property
    def num_elements(self) -> int:
        return self.ex * self.ey * self.ez

    @property
    def element_range(self) -> tuple[int, int]:
        per = self.ex * self.ey
        return self.z0 * per, self.z1 * per

    @property
    def lower(self):
        return self.rank - 1 if self.z0 > 0 else None

    @property
    def upper(self):
        return self.rank + 1 if self.z1 < self.ez_global else None

    @property
    def plane_size(self) -> int:
        return (self.ex * (self.n - 1) + 1) * (self.ey * (self.n - 1) + 1)


class SlabComm:
    """The two halo exchanges and the scalar all-gather over torch.distributed.

    NCCL moves device tensors directly; with gloo (CPU tests, or several
    processes sharing one GPU) device tensors are staged through host memory.
    """

    def __init__(self, part: SlabPartition, group=None):
        self.part = part
        self.group = group
        self.backend = dist.get_backend(group)
        self.stage = self.backend != "nccl"

    def _xfer(self, sends: list, recvs: list) -> None:
        ops = []
        staged = []
        for t, peer in sends:
            src = t.cpu() if (self.stage and t.is_cuda) else t
            ops.append(dist.P2POp(dist.isend, src, peer, self.group))
        for t, peer in recvs:
            dst = torch.empty(t.shape, dtype=t.dtype) if (self.stage and t.is_cuda) else t
            staged.append((t, dst))
            ops.append(dist.P2POp(dist.irecv, dst, peer, self.group))
        if not ops:
            return
        for req in dist.batch_isend_irecv(ops):
            req.wait()
        for t, dst in staged:
            if dst is not t:
                t.copy_(dst)

    def exchange_up(self, top_partial, bottom_prefix) -> None:
        """Send this slab's top-face partial to rank+1; receive rank-1's."""
        self.exchange_up_wait(self.exchange_up_start(top_partial, bottom_prefix))

    def exchange_up_start(self, top_partial, bottom_prefix):
        """Non-blocking form: returns a handle for exchange_up_wait().  Over NCCL
        the transfer runs on the communicator's stream, so kernels enqueued on
        the current stream before the wait overlap it."""
        p = self.part
        sends = [(top_partial, p.upper)] if p.upper is not None else []
        recvs = [(bottom_prefix, p.lower)] if p.lower is not None else []
        if self.stage:
            self._xfer(sends, recvs)
            return None
        ops = [dist.P2POp(dist.isend, t, peer, self.group) for t, peer in sends]
        ops += [dist.P2POp(dist.irecv, t, peer, self.group) for t, peer in recvs]
        return dist.batch_isend_irecv(ops) if ops else None

    @staticmethod
    def exchange_up_wait(handle) -> None:
        for req in handle or []:
            req.wait()

    def exchange_down(self, bottom_totals, top_totals) -> None:
        """Send the bottom interface totals to rank-1; receive rank+1's."""
        self.exchange_up_wait(self.exchange_down_start(bottom_totals, top_totals))

    def exchange_down_start(self, bottom_totals, top_totals):
        """Non-blocking form of exchange_down (see exchange_up_start)."""
        p = self.part
        sends = [(bottom_totals, p.lower)] if p.lower is not None else []
        recvs = [(top_totals, p.upper)] if p.upper is not None else []
        if self.stage:
            self._xfer(sends, recvs)
            return None
        ops = [dist.P2POp(dist.isend, t, peer, self.group) for t, peer in sends]
        ops += [dist.P2POp(dist.irecv, t, peer, self.group) for t, peer in recvs]
        return dist.batch_isend_irecv(ops) if ops else None

    @property
    def capturable(self) -> bool:
        """Collectives of this communicator can be captured in a CUDA graph:
        NCCL, and (untested beyond one rank on this project's hardware) for
        world > 1 only when SEM_DIST_GRAPH=1."""
        if self.stage:
            return False
        return self.part.world == 1 or os.environ.get("SEM_DIST_GRAPH", "0") == "1"

    def allgather(self, local: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        """All ranks' partials in rank order.  One rank: the partial itself."""
        if self.part.world == 1:
            return local
        if self.stage and local.is_cuda:
            tmp = torch.empty(out.shape, dtype=out.dtype)
            dist.all_gather_into_tensor(tmp, local.cpu(), group=self.group)
            out.copy_(tmp)
        else:
            dist.all_gather_into_tensor(out, local, group=self.group)
        return out


class CudaSlabOps:
    """Per-rank compute of the distributed CG on the GPU (csrc/cg.cu, slab.cu)."""

    def __init__(self, part: SlabPartition, g_local: torch.Tensor, basis, max_iterations: int,
                 device: torch.device):
        self.part, self.basis, self.dev = part, basis, device
        n = part.n
        shape = (part.num_elements, n, n, n)
        mk = lambda: torch.empty(shape, dtype=torch.float64, device=device)  # noqa: E731
        self.x, self.r, self.p, self.w, self.w2 = mk(), mk(), mk(), mk(), mk()
        self.g = g_local
        self.history = torch.zeros(max(1, max_iterations), dtype=torch.float64, device=device)
        self.state = torch.zeros(ctypes.sizeof(sem_cg_state), dtype=torch.uint8, device=device)
        self.scratch = torch.zeros(int(load().sem_reduce_scratch_bytes()), dtype=torch.uint8,
                                   device=device)
        ps = part.plane_size
        self.top_partial = torch.zeros(ps, dtype=torch.float64, device=device)
        self.bottom_prefix = torch.zeros(ps, dtype=torch.float64, device=device)
        self.bottom_totals = torch.zeros(ps, dtype=torch.float64, device=device)
        self.top_totals = torch.zeros(ps, dtype=torch.float64, device=device)
        self.dx = np.ascontiguousarray(basis.diff, dtype=np.float64)
        self.dxt = np.ascontiguousarray(basis.diff_t, dtype=np.float64)
        self.lib = load()
        self._local = self.state.view(torch.float64)[9:10]  # sem_cg_state.local_sum
        # per-iteration calls with their ctypes arguments converted once (the
        # driver loop is host-bound at small slabs: ~12 calls per iteration)
        self._bound: dict = {}

    def _invoke(self, key, build, what: str) -> None:
        """Call a libsem entry with memoised arguments: `build()` returns
        (fn, args) once per (key, stream)."""
        s = torch.cuda.current_stream(self.dev).cuda_stream
        ent = self._bound.get((key, s))
        if ent is None:
            ent = build()
            self._bound[(key, s)] = ent
        check(ent[0](*ent[1]), what)

    # geometry of this slab as the C-ABI expects it
    def _slab(self):
        p = self.part
        return (p.ex, p.ey, p.ez, p.n, p.z0, p.ez_global)

    def _s(self):
        return dv.stream_handle(self.dev)

    def init(self, f: torch.Tensor, max_iterations: int, tolerance: float) -> None:
        check(self.lib.sem_cg_init_slab(dv.ptr(f), dv.ptr(self.x), dv.ptr(self.r), dv.ptr(self.p),
                                        dv.ptr(self.state), dv.ptr(self.history), max_iterations,
                                        float(tolerance), *self._slab(), dv.ptr(self.scratch),
                                        self._s()), "dist cg init")

    def local_sum(self) -> torch.Tensor:
        return self._local

    def finish(self, phase: int, gathered: torch.Tensor) -> None:
        self._invoke(("finish", phase, gathered.data_ptr(), gathered.numel()), lambda: (
            self.lib.sem_cg_finish, (dv.ptr(self.state), dv.ptr(gathered), gathered.numel(),
                                     phase, dv.ptr(self.history), self._s())), "dist cg finish")

    def ax_layers(self, l0: int, l1: int, first: bool) -> None:
        """Iteration head + w = A_local p on element layers [l0, l1), leaving
        the per-element <p, A p> partials in their slots of w2 (`first` is
        the iteration's first range; settle() then sums every slot)."""
        p = self.part
        if l1 <= l0:
            return

        def build():
            per = p.ex * p.ey
            e0, ne = l0 * per, (l1 - l0) * per
            off = lambda t, width: ctypes.c_void_p(t.data_ptr() + e0 * width * 8)  # noqa: E731
            nnn = p.n ** 3
            return self.lib.sem_cg_ax_slab, (
                off(self.p, nnn), off(self.r, nnn), off(self.x, nnn), off(self.g, 6 * nnn),
                dv.host_f64_ptr(self.dx), dv.host_f64_ptr(self.dxt), off(self.w, nnn), ne, p.n,
                dv.ptr(self.state), dv.ptr(self.history), off(self.w2, 1),
                dv.ptr(self.scratch), -1, self._s())
        self._invoke(("ax", l0, l1, bool(first)), build, "dist cg ax")

    def settle(self) -> None:
        """local_sum = the fixed-order sum of every element slot's <p, A p>
        partial (all of this iteration's ax_layers ranges)."""
        self._invoke(("settle",), lambda: (
            self.lib.sem_cg_settle_slab, (dv.ptr(self.w2), self.part.num_elements,
                                          dv.ptr(self.state), 0, self._s())), "dist cg settle")

    def plane_top(self, field: torch.Tensor) -> torch.Tensor:
        p = self.part
        self._invoke(("top", field.data_ptr()), lambda: (
            self.lib.sem_slab_plane_top, (dv.ptr(field), dv.ptr(self.top_partial), p.ex, p.ey,
                                          p.ez, p.n, self._s())), "plane top")
        return self.top_partial

    def plane_bottom(self, field: torch.Tensor, prefix) -> torch.Tensor:
        p = self.part
        self._invoke(("bottom", field.data_ptr(), prefix.data_ptr()), lambda: (
            self.lib.sem_slab_plane_bottom, (dv.ptr(field), dv.ptr(prefix),
                                             dv.ptr(self.bottom_totals), p.ex, p.ey, p.ez, p.n,
                                             self._s())), "plane bottom")
        return self.bottom_totals

    def dssum(self, field: torch.Tensor, bottom_totals, top_totals, apply_mask: bool = False):
        """Standalone distributed dssum of `field` (faces from the halo totals)."""
        p = self.part
        out = torch.empty_like(field)
        ptr = lambda t: dv.ptr(t) if t is not None else ctypes.c_void_p(0)  # noqa: E731
        check(self.lib.sem_dssum_slab(dv.ptr(field), dv.ptr(out), ptr(bottom_totals),
                                      ptr(top_totals), p.ex, p.ey, p.ez, p.n, p.z0, p.ez_global,
                                      1 if apply_mask else 0, self._s()), "dist dssum")
        return out

    def update(self, bottom_totals, top_totals) -> None:
        """r -= alpha mask(dssum(w)) (faces from the halo totals); <r,r>_c partial."""
        ptr = lambda t: dv.ptr(t) if t is not None else ctypes.c_void_p(0)  # noqa: E731
        key = ("update", None if bottom_totals is None else bottom_totals.data_ptr(),
               None if top_totals is None else top_totals.data_ptr())
        self._invoke(key, lambda: (
            self.lib.sem_cg_update_slab, (dv.ptr(self.w), dv.ptr(self.r), ptr(bottom_totals),
                                          ptr(top_totals), dv.ptr(self.state), *self._slab(),
                                          dv.ptr(self.scratch), self._s())), "dist update")

    def update_alpha(self, bottom_totals, top_totals, gathered: torch.Tensor) -> None:
        """finish(1) folded into the update launch: alpha from the gathered
        <p, A p> partials (rank order) in every CTA, then update()."""
        ptr = lambda t: dv.ptr(t) if t is not None else ctypes.c_void_p(0)  # noqa: E731
        key = ("update_alpha", None if bottom_totals is None else bottom_totals.data_ptr(),
               None if top_totals is None else top_totals.data_ptr(), gathered.data_ptr(),
               gathered.numel())
        self._invoke(key, lambda: (
            self.lib.sem_cg_update_slab_alpha, (dv.ptr(self.w), dv.ptr(self.r), ptr(bottom_totals),
                                                ptr(top_totals), dv.ptr(self.state),
                                                dv.ptr(gathered), gathered.numel(), *self._slab(),
                                                dv.ptr(self.scratch), self._s())),
            "dist update (alpha)")

    def iteration_graph(self, enqueue):
        """CUDA graph of one iteration (`enqueue()` launches it), captured on
        a side stream once per ops object."""
        if getattr(self, "_graph", None) is None:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.dev)
            side.wait_stream(torch.cuda.current_stream(self.dev))
            with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
                enqueue()
            torch.cuda.current_stream(self.dev).wait_stream(side)
            self._graph = g
        return self._graph

    def stop_flag(self) -> torch.Tensor:
        """Device int32 view of sem_cg_state.stop (early-exit polling)."""
        return self.state[_STOP_OFFSET:_STOP_OFFSET + 4].view(torch.int32)

    def finalize(self) -> None:
        """The owed x += alpha p of the last iteration run."""
        check(self.lib.sem_cg_finalize(dv.ptr(self.x), dv.ptr(self.p), dv.ptr(self.state),
                                       self.x.numel(), self._s()), "dist finalize")

    def scalar_buffer(self, world: int) -> torch.Tensor:
        return torch.zeros(world, dtype=torch.float64, device=self.dev)

    def result(self):
        raw = self.state.cpu().numpy().tobytes()
        st = sem_cg_state.from_buffer_copy(raw)
        iters = int(st.iterations_run)
        hist = self.history[:iters].cpu().numpy().copy()
        return self.x, hist, iters, int(st.stop), float(st.pap), int(st.breakdown_it)


def halo_exchange(ops, comm: SlabComm, field, overlap=None):
    """The two-step ordered halo of one assembled field.  Returns the
    (bottom_totals, top_totals) planes this rank needs (None = no neighbour).
    `overlap()` (optional) is enqueued while the first exchange is in flight."""
    part = comm.part
    top = ops.plane_top(field) if part.upper is not None else None
    handle = comm.exchange_up_start(top, ops.bottom_prefix if part.lower is not None else None)
    if overlap is not None:
        overlap()
    comm.exchange_up_wait(handle)
    bot = ops.plane_bottom(field, ops.bottom_prefix) if part.lower is not None else None
    comm.exchange_down(bot, ops.top_totals if part.upper is not None else None)
    return bot, (ops.top_totals if part.upper is not None else None)


def dist_dssum(ops, comm: SlabComm, field, apply_mask: bool = False):
    """dssum of a slab-partitioned field, bit-identical to the global one."""
    bot, top = halo_exchange(ops, comm, field)
    return ops.dssum(field, bot, top, apply_mask)


@dataclass
class DistCgResult:
    solution: object          # this rank's slice of the solution
    residual_history: np.ndarray
    iterations_run: int
    stop: int


def _ax_ranges(part: SlabPartition):
    """(edge ranges, interior range or None): with a neighbour the interface
    planes need only the bottom / top element layers, so they go first and
    the interior overlaps the first exchange; without one, one launch."""
    ez = part.ez
    if part.lower is None and part.upper is None:
        return [(0, ez)], None
    edge = [(0, 1)] if ez == 1 else [(0, 1), (ez - 1, ez)]
    return edge, ((1, ez - 1) if ez > 2 else None)


def _iteration(ops, comm: SlabComm, gathered, phase=None) -> None:
    """Enqueue one distributed CG iteration (every rank).  `phase(name)`, if
    given, is called at each phase boundary (instrumentation)."""
    mark = phase or (lambda name: None)
    part = comm.part
    edge, interior = _ax_ranges(part)
    mark("ax")
    for q, (l0, l1) in enumerate(edge):
        ops.ax_layers(l0, l1, first=(q == 0))
    if part.lower is None and part.upper is None:
        bot = top = None
    else:
        mark("halo")
        top_p = ops.plane_top(ops.w) if part.upper is not None else None
        handle = comm.exchange_up_start(top_p, ops.bottom_prefix if part.lower is not None
                                        else None)
        if interior is not None:  # overlaps the first exchange
            ops.ax_layers(*interior, first=False)
        comm.exchange_up_wait(handle)
        bot = ops.plane_bottom(ops.w, ops.bottom_prefix) if part.lower is not None else None
        top = ops.top_totals if part.upper is not None else None
        handle = comm.exchange_down_start(bot, top)
    mark("pap")
    ops.settle()  # overlaps the second exchange
    g1 = comm.allgather(ops.local_sum(), gathered)
    if part.lower is not None or part.upper is not None:
        comm.exchange_up_wait(handle)
    mark("update")
    if hasattr(ops, "update_alpha"):
        ops.update_alpha(bot, top, g1)
    else:
        ops.finish(1, g1)
        ops.update(bot, top)
    mark("rr")
    ops.finish(2, comm.allgather(ops.local_sum(), gathered))
    mark("end")


POLL_EVERY = 8


def dist_cg_solve(ops, comm: SlabComm, f_local, max_iterations: int, tolerance: float = 0.0,
                  graph: bool | None = None) -> DistCgResult:
    """Distributed CG; every rank calls this with its slab (same arguments).
    `graph` (default: comm.capturable and a CUDA ops object) captures one
    iteration in a CUDA graph and replays it."""
    part = comm.part
    gathered = ops.scalar_buffer(part.world)
    ops.init(f_local, max_iterations, tolerance)
    ops.finish(0, comm.allgather(ops.local_sum(), gathered))
    if graph is None:
        graph = comm.capturable and isinstance(ops, CudaSlabOps) and max_iterations > 2
    if not graph:
        for _ in range(max_iterations):
            _iteration(ops, comm, gathered)
    else:
        dev = ops.dev
        _iteration(ops, comm, gathered)  # iteration 1 eagerly: configures the kernels
        g = ops.iteration_graph(lambda: _iteration(ops, comm, gathered))
        stream = torch.cuda.current_stream(dev)
        stop_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        stop_event = None
        for q in range(max_iterations - 1):
            g.replay()
            if (q + 1) % POLL_EVERY == 0:  # every rank sees the same flag
                if stop_event is not None and stop_event.query() and int(stop_host[0]) != 0:
                    break
                stop_host.copy_(ops.stop_flag(), non_blocking=True)
                stop_event = torch.cuda.Event()
                stop_event.record(stream)
    ops.finalize()
    x, hist, iters, stop, pap, bit = ops.result()
    if stop == 2:
        from .cg import CgBreakdownError
        raise CgBreakdownError(f"<p, A p>_c = {pap:.3e} at iteration {bit}; "
                               "operator is not SPD here")
    return DistCgResult(solution=x, residual_history=hist, iterations_run=iters, stop=stop)


def dist_cg_phases(ops, comm: SlabComm, f_local, iterations: int) -> dict:
    """Per-rank device time (ms, summed over `iterations` eager iterations)
    of the iteration's phases -- ax (Ax launches up to the first exchange),
    halo (planes, exchanges, overlapped interior Ax), pap (settle + gather),
    update (alpha + r update), rr (gather + finish) -- from CUDA events on
    the compute stream.  Measurement only (bench.py --gpus N)."""
    part = comm.part
    gathered = ops.scalar_buffer(part.world)
    ops.init(f_local, iterations, 0.0)
    ops.finish(0, comm.allgather(ops.local_sum(), gathered))
    stream = torch.cuda.current_stream(ops.dev)
    marks: list = []

    def phase(name):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        marks.append((name, ev))

    for _ in range(iterations):
        _iteration(ops, comm, gathered, phase)
    torch.cuda.synchronize(ops.dev)
    out: dict = {}
    for (name, e0), (_, e1) in zip(marks, marks[1:]):
        if name != "end":
            out[name] = out.get(name, 0.0) + e0.elapsed_time(e1)
    return out
