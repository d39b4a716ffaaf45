"""Unpreconditioned CG with multiplicity-weighted inner products on the B200
(contract of sembench/cg.py:53-193).

Two execution paths share the reference recurrence:

* **fused** -- when ``operator`` is a :class:`GlobalOperator` (the box
  apply_global), the whole solve runs as device-resident launches
  (``sem_cg_init`` + ``sem_cg_run``, csrc/cg.cu): alpha/beta never leave the
  GPU, reductions are deterministic, early exits are device flags.  The host
  synchronises once at the end (or once per iteration if a callback is set).
* **generic** -- any other callable: each iteration calls ``operator(p)`` on
  a CUDA tensor and uses the same sm_100a vector kernels (add2s1, add2s2,
  glsc3).

Errors follow the reference: ``CgBreakdownError`` when <p,Ap>_c <= 0, and
``ValueError`` for a bad configuration.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from ._lib import check, load, sem_cg_state
from .assembly import GlobalOperator, Topology, _mask_dev, _wdot_dev, as_topology
from .fields import validate_field
from .kernels import TrafficCounters

__all__ = ["CgConfig", "CgResult", "CgBreakdownError", "weighted_dot", "cg_solve",
           "CG_VECTOR_FLOPS_PER_POINT", "CgWorkspace", "fused_phase_seconds"]

CG_VECTOR_FLOPS_PER_POINT = 12
USE_GRAPHS = True  # replay captured iterations (fused path)
# iterations per captured graph: 10.  Inside one graph the next iteration's
# Ax is a programmatic dependent of the previous update (csrc/cg.cu cg_pdl),
# so its CTAs start loading the metric while the update drains; between graph
# launches that overlap is lost.  tools/cg_ab.py with idle gaps between
# configurations (profiles/r02_cg_graph_pdl.txt): E = 4096 98.0-99.2 us per
# iteration at 1 -> 93.8-94.9 us at 10; round 1's "1 is best" came from
# back-to-back solves whose power-cap drift hid the difference.
GRAPH_ITERATIONS = 10
# graph replays between non-blocking polls of the device stop flag
POLL_EVERY = 8
_STOP_OFFSET = sem_cg_state.stop.offset


class CgBreakdownError(RuntimeError):
    """<p, A p>_c was non-positive: the operator is not SPD on this subspace."""


@dataclass
class CgConfig:
    max_iterations: int = 100
    tolerance: float = 0.0

    def __post_init__(self):
        if self.max_iterations < 1:
            raise ValueError("max_iterations must be at least 1")
        if self.tolerance < 0.0:
            raise ValueError("tolerance must be non-negative")


@dataclass
class CgResult:
    solution: object
    residual_history: np.ndarray
    iterations_run: int
    counters: TrafficCounters = field(default_factory=TrafficCounters)


def _glsc3_box_dev(a: torch.Tensor, b: torch.Tensor, topo,
                   out: torch.Tensor | None = None) -> torch.Tensor:
    return _wdot_dev(a, b, topo, out)


def weighted_dot(u, v, topo) -> float:
    """sum(u * v / multiplicity) -- deterministic device reduction."""
    topo = as_topology(topo)
    validate_field(u, topo.num_elements, topo.n, "u")
    validate_field(v, topo.num_elements, topo.n, "v")
    dev = u.device if dv.is_tensor(u) else (v.device if dv.is_tensor(v) else None)
    ud = dv.as_device_f64(u, dev, "u")
    vd = dv.as_device_f64(v, ud.device, "v")
    with torch.cuda.device(ud.device):
        out = _glsc3_box_dev(ud, vd, topo)
        return float(out.item())


def _consistency_flag(f_dev: torch.Tensor, topo: Topology) -> torch.Tensor:
    """Device int32: 0 iff mask(f) is interface-consistent (equal copies of
    every shared node).  Enqueued only -- nothing waits on it here."""
    flag = torch.empty(1, dtype=torch.int32, device=f_dev.device)
    check(load().sem_consistent_box(dv.ptr(f_dev), topo.ex, topo.ey, topo.ez, topo.n,
                                    dv.ptr(flag), dv.stream_handle(f_dev.device)),
          "cg_solve consistency check")
    return flag


def _consistent(f_dev: torch.Tensor, topo: Topology) -> bool:
    """Is mask(f) interface-consistent (equal copies of every shared node)?"""
    return int(_consistency_flag(f_dev, topo).item()) == 0


class CgWorkspace:
    """Device vectors and state of one fused solve (reusable across solves)."""

    def __init__(self, topo: Topology, max_iterations: int, device: torch.device):
        topo = as_topology(topo)
        shape = (topo.num_elements, topo.n, topo.n, topo.n)
        self.box = (topo.ex, topo.ey, topo.ez, topo.n)
        # one allocation, [x | p | r | w | w2]: the vectors an iteration
        # re-reads soonest (r, w; then p) are adjacent, so one L2 access-policy
        # window can cover them (_l2_window)
        # (each vector starts on a 16-byte boundary: the kernels move even-n
        # rows as 128-bit accesses and the settle reads the partials so)
        m = topo.num_elements * topo.n ** 3
        mp = m + (m & 1)
        self._buf = torch.empty(3 * mp + 2 * m, dtype=torch.float64, device=device)
        v = [self._buf[q * mp:q * mp + m].view(shape) for q in range(3)]
        self.x, self.p, self.r = v
        self.w = self._buf[3 * mp:].view((2,) + shape)
        self._m = m
        self._mp = mp
        self.history = torch.zeros(max(1, max_iterations), dtype=torch.float64, device=device)
        self.state = torch.zeros(ctypes_sizeof_state(), dtype=torch.uint8, device=device)
        self.scratch = torch.zeros(int(load().sem_reduce_scratch_bytes()), dtype=torch.uint8,
                                   device=device)
        self.device = device
        self.max_iterations = max_iterations
        self._graph = None
        self._graph_key = None
        # pinned mirror of state.stop for the replay loop's non-blocking poll
        self._stop_host = torch.zeros(1, dtype=torch.int32, pin_memory=True)
        self._stop_event = None
        self._poll_stream = None

    def fits(self, topo: Topology, max_iterations: int, device: torch.device) -> bool:
        """Usable for a solve on `topo` (same box and n: the launches index the
        vectors by the box) with this iteration budget on this device."""
        return (self.box == (topo.ex, topo.ey, topo.ez, topo.n)
                and self.max_iterations >= max_iterations and self.device == device)

    def poll_stream(self) -> torch.cuda.Stream:
        """Side stream for the non-blocking stop-flag copies."""
        if self._poll_stream is None:
            self._poll_stream = torch.cuda.Stream(self.device)
        return self._poll_stream

    def iteration_graph(self, launch_one, key):
        """CUDA graph of one fused iteration (captured once per workspace and
        operator: `key` identifies the captured geometry / basis / box)."""
        if self._graph is None or self._graph_key != key:
            self._graph_key = key
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    launch_one()
            torch.cuda.current_stream(self.device).wait_stream(side)
            self._graph = g
        return self._graph

    def read_state(self) -> sem_cg_state:
        raw = self.state.cpu().numpy().tobytes()
        return sem_cg_state.from_buffer_copy(raw)


def _l2_window(ws: CgWorkspace, stream) -> bool:
    """Keep the vectors an iteration re-reads soonest L2-resident across its
    launches: an access-policy window over [p | r | w] (SEM_CG_L2 = "rw",
    "prw" or "off"; SEM_CG_L2_HIT = hit ratio)."""
    import os
    mode = os.environ.get("SEM_CG_L2", "off")
    if mode == "off":
        return False
    m8 = ws._mp * 8
    first = {"rw": 2, "prw": 1, "xprw": 0}[mode]
    base = ws._buf.data_ptr() + first * m8
    nbytes = (4 - first) * m8
    hit = float(os.environ.get("SEM_CG_L2_HIT", "1.0"))
    import ctypes
    pm, wm, l2 = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    lib = load()
    check(lib.sem_l2_props(ctypes.byref(pm), ctypes.byref(wm), ctypes.byref(l2)), "L2 props")
    setaside = int(os.environ.get("SEM_CG_L2_SETASIDE", str(pm.value)))
    check(lib.sem_l2_window(base, nbytes, hit, setaside, stream), "cg_solve L2 window")
    return True


def ctypes_sizeof_state() -> int:
    import ctypes
    return ctypes.sizeof(sem_cg_state)


def _fused_solve(f_dev: torch.Tensor, op: GlobalOperator, topo: Topology, cfg: CgConfig,
                 callback, host: bool, ws: CgWorkspace | None = None):
    lib = load()
    dev = f_dev.device
    if ws is None or not ws.fits(topo, cfg.max_iterations, dev):
        ws = CgWorkspace(topo, cfg.max_iterations, dev)
    s = dv.stream_handle(dev)
    g = op.geom.device_values(dev)
    dx = np.ascontiguousarray(op.basis.diff, dtype=np.float64)
    dxt = np.ascontiguousarray(op.basis.diff_t, dtype=np.float64)
    box = (topo.ex, topo.ey, topo.ez, topo.n)
    check(lib.sem_cg_init(dv.ptr(f_dev), dv.ptr(ws.x), dv.ptr(ws.r), dv.ptr(ws.p),
                          dv.ptr(ws.state), dv.ptr(ws.history), cfg.max_iterations,
                          float(cfg.tolerance), *box, dv.ptr(ws.scratch), s), "cg_solve init")

    win = _l2_window(ws, s)

    def run(k: int, first: int):
        # iterations first .. first+k-1 (1-based, global: the kernels alternate
        # their element walk by its parity).  The stream is looked up at call
        # time: inside graph capture it is the capture stream.
        check(lib.sem_cg_run_at(dv.ptr(g), dv.host_f64_ptr(dx), dv.host_f64_ptr(dxt),
                                dv.ptr(ws.x), dv.ptr(ws.r), dv.ptr(ws.p), dv.ptr(ws.w),
                                dv.ptr(ws.state), dv.ptr(ws.history), k, first, *box,
                                dv.ptr(ws.scratch), dv.stream_handle(dev)), "cg_solve run")

    m = ws.x.numel()

    def finalize():  # the deferred x += alpha p of the last iteration run
        check(lib.sem_cg_finalize(dv.ptr(ws.x), dv.ptr(ws.p), dv.ptr(ws.state), m,
                                  dv.stream_handle(dev)), "cg_solve finalize")

    timers = op.timers
    if callback is None and timers is not None:
        # the same launches with CUDA events between them (sem_cg_run_phases):
        # the operator's timers receive the device time of the Ax phase (Ax
        # with the fused p update and <p, A p>) and of the assembly phase
        # (dssum + mask fused with the r update and <r, r>)
        import ctypes
        ms = (ctypes.c_double * 3)(0.0, 0.0, 0.0)
        check(lib.sem_cg_run_phases(dv.ptr(g), dv.host_f64_ptr(dx), dv.host_f64_ptr(dxt),
                                    dv.ptr(ws.x), dv.ptr(ws.r), dv.ptr(ws.p), dv.ptr(ws.w),
                                    dv.ptr(ws.state), dv.ptr(ws.history), cfg.max_iterations,
                                    *box, dv.ptr(ws.scratch), ms, s), "cg_solve run")
        timers.ax_seconds += ms[0] * 1e-3
        timers.dssum_seconds += (ms[1] + ms[2]) * 1e-3
        finalize()
        st = ws.read_state()
    elif callback is None:
        if cfg.max_iterations > max(2, GRAPH_ITERATIONS + 1) and USE_GRAPHS:
            # iteration 1 launched directly (configures the kernels), then
            # GRAPH_ITERATIONS iterations are captured into one CUDA graph and
            # replayed: the launches are parameter-stable (scalars live in the
            # device state), so replay == relaunch without the host overhead.
            # Early exits are device-side (queued launches become no-ops); the
            # host also polls the stop flag without blocking (an async copy
            # into pinned memory every POLL_EVERY replays, read once its event
            # has completed) and stops replaying once the solve has ended.
            run(1, 1)
            rest = cfg.max_iterations - 1
            # always the same graph size (a short solve runs its iterations
            # directly instead of capturing -- and evicting -- another graph);
            # even, so every replay starts on an even global iteration, the
            # parity the graph was captured with
            k = max(2, GRAPH_ITERATIONS + (GRAPH_ITERATIONS & 1))
            key = (g.data_ptr(), box, dx.tobytes(), k)
            graph = ws.iteration_graph(lambda: run(k, 2), key)
            stream = torch.cuda.current_stream(dev)
            ws._stop_host.zero_()
            ws._stop_event = None
            for q in range(rest // k):
                graph.replay()
                if (q + 1) % max(1, POLL_EVERY // k) == 0:
                    if ws._stop_event is not None and ws._stop_event.query() \
                            and int(ws._stop_host[0]) != 0:
                        break
                    # the flag is copied on a side stream that waits for this
                    # replay: a copy on the solve's own stream would sit
                    # between two replays (~1% of an E = 4096 iteration)
                    done = torch.cuda.Event()
                    done.record(stream)
                    ps = ws.poll_stream()
                    ps.wait_event(done)
                    with torch.cuda.stream(ps):
                        ws._stop_host.copy_(ws.state[_STOP_OFFSET:_STOP_OFFSET + 4]
                                            .view(torch.int32), non_blocking=True)
                    ws._stop_event = torch.cuda.Event()
                    ws._stop_event.record(ps)
            else:
                if rest % k:
                    run(rest % k, 2 + (rest // k) * k)
        else:
            run(cfg.max_iterations, 1)
        finalize()
        st = ws.read_state()
    else:
        st = None
        for it in range(1, cfg.max_iterations + 1):
            run(1, it)
            finalize()
            st = ws.read_state()
            if st.iterations_run >= it and st.stop != 2:
                x = dv.to_numpy(ws.x) if host else ws.x
                r = dv.to_numpy(ws.r) if host else ws.r
                callback(it, x, r)
            if st.stop:
                break
    if win:
        check(lib.sem_l2_window(None, 0, 0.0, 0, s), "cg_solve L2 window reset")
    if st.stop == 2:
        ppc = float(_glsc3_box_dev(ws.p, ws.p, topo).item())
        raise CgBreakdownError(
            f"<p, A p>_c = {st.pap:.3e} at iteration {st.breakdown_it} "
            f"(scale <p, p>_c = {ppc:.3e}); operator is not SPD here")
    iters = int(st.iterations_run)
    history = dv.to_numpy(ws.history[:iters]).copy()
    zero_exit = st.stop == 1
    solution = ws.x.clone()
    return solution, history, iters, zero_exit


def fused_phase_seconds(f, op: GlobalOperator, topo: Topology, iterations: int,
                        workspace: CgWorkspace | None = None) -> tuple[float, float, float]:
    """Device seconds of the fused solve's three phases over `iterations`
    eagerly launched iterations (sem_cg_run_phases: CUDA events between the
    launches): (Ax with the fused p update, assemble = dssum + mask + <p,w>,
    x/r updates + <r,r>).  Measurement helper for harness.py; the solve's
    result is discarded."""
    import ctypes
    lib = load()
    fd = dv.as_device_f64(f, None, "f")
    dev = fd.device
    ws = workspace
    topo = as_topology(topo)
    if ws is None or not ws.fits(topo, iterations, dev):
        ws = CgWorkspace(topo, iterations, dev)
    box = (topo.ex, topo.ey, topo.ez, topo.n)
    g = op.geom.device_values(dev)
    dx = np.ascontiguousarray(op.basis.diff, dtype=np.float64)
    dxt = np.ascontiguousarray(op.basis.diff_t, dtype=np.float64)
    ms = (ctypes.c_double * 3)(0.0, 0.0, 0.0)
    with torch.cuda.device(dev):
        s = dv.stream_handle(dev)
        check(lib.sem_cg_init(dv.ptr(fd), dv.ptr(ws.x), dv.ptr(ws.r), dv.ptr(ws.p),
                              dv.ptr(ws.state), dv.ptr(ws.history), iterations, 0.0, *box,
                              dv.ptr(ws.scratch), s), "cg_solve init")
        check(lib.sem_cg_run_phases(dv.ptr(g), dv.host_f64_ptr(dx), dv.host_f64_ptr(dxt),
                                    dv.ptr(ws.x), dv.ptr(ws.r), dv.ptr(ws.p), dv.ptr(ws.w),
                                    dv.ptr(ws.state), dv.ptr(ws.history), iterations, *box,
                                    dv.ptr(ws.scratch), ms, s), "cg phase timing")
    return ms[0] * 1e-3, ms[1] * 1e-3, ms[2] * 1e-3


def _generic_solve(f_dev: torch.Tensor, operator, topo: Topology, cfg: CgConfig, counters,
                   callback, host: bool):
    lib = load()
    dev = f_dev.device
    s = dv.stream_handle(dev)
    m = f_dev.numel()
    r = _mask_dev(f_dev, topo)
    x = torch.zeros_like(r)
    p = torch.zeros_like(r)
    dofs = topo.dofs
    history: list[float] = []
    rtz, iters, zero_exit = 1.0, 0, False

    def dot(a, b) -> float:
        return float(_glsc3_box_dev(a, b, topo).item())

    for it in range(1, cfg.max_iterations + 1):
        rtz_old = rtz
        rtz = dot(r, r)
        if rtz == 0.0:
            iters = it
            history.append(0.0)
            zero_exit = True
            if callback is not None:
                callback(it, dv.to_numpy(x) if host else x, dv.to_numpy(r) if host else r)
            break
        beta = 0.0 if it == 1 else rtz / rtz_old
        check(lib.sem_add2s1(dv.ptr(p), dv.ptr(r), beta, m, s), "add2s1")
        w = operator(dv.to_numpy(p) if host else p)
        w = dv.as_device_f64(w, dev, "operator output")
        pap = dot(p, w)
        if pap <= 0.0:
            ppc = dot(p, p)
            raise CgBreakdownError(
                f"<p, A p>_c = {pap:.3e} at iteration {it} "
                f"(scale <p, p>_c = {ppc:.3e}); operator is not SPD here")
        alpha = rtz / pap
        check(lib.sem_add2s2(dv.ptr(x), dv.ptr(p), alpha, m, s), "add2s2")
        check(lib.sem_add2s2(dv.ptr(r), dv.ptr(w), -alpha, m, s), "add2s2")
        rnorm = math.sqrt(dot(r, r))
        history.append(rnorm)
        iters = it
        counters.add(reads=(9 + 6) * dofs, writes=3 * dofs,
                     flops=CG_VECTOR_FLOPS_PER_POINT * dofs)
        if callback is not None:
            callback(it, dv.to_numpy(x) if host else x, dv.to_numpy(r) if host else r)
        if cfg.tolerance > 0.0 and rnorm < cfg.tolerance:
            break
    if zero_exit:
        counters.add(reads=3 * dofs, flops=2 * dofs)
    return x, np.asarray(history, dtype=np.float64), iters


def cg_solve(f, operator, topo, cfg: CgConfig,
             counters: TrafficCounters | None = None, callback=None,
             workspace: CgWorkspace | None = None) -> CgResult:
    """Run CG on A x = f (reference recurrence, cg.py:139-186).

    The fused device-resident solve runs when ``operator`` is a
    :class:`GlobalOperator` on this (box) topology and mask(f) is
    interface-consistent (the fused <p, A p> is the element-local sum, equal
    to the reference's assembled one only for continuous iterates);
    otherwise the generic path calls ``operator`` every iteration."""
    if counters is None:
        counters = TrafficCounters()
    topo = as_topology(topo)
    validate_field(f, topo.num_elements, topo.n, "f")
    fd, kind = dv.to_device_io(f, "f")
    host = kind != "device"
    dofs = topo.dofs
    # r = mask(f) on entry (cg.py:139)
    counters.add(reads=2 * dofs, writes=dofs)
    with torch.cuda.device(fd.device):
        fused = (isinstance(operator, GlobalOperator) and isinstance(topo, Topology)
                 and operator.topo == topo)
        out = None
        if fused and callback is None:
            # optimistic: the consistency check is enqueued ahead of the fused
            # solve and read once the solve's own final synchronisation has
            # happened (no host round trip before the first launch); an
            # inconsistent rhs -- rare, the fused <p, A p> assumes a
            # continuous p -- discards the result and takes the generic path
            flag = _consistency_flag(fd, topo)
            try:
                out = _fused_solve(fd, operator, topo, cfg, callback, host, workspace)
            except CgBreakdownError:
                if int(flag.item()) == 0:
                    raise
                out = None
            if out is not None and int(flag.item()) != 0:
                out = None
        elif fused and _consistent(fd, topo):  # callbacks see every iterate: check first
            out = _fused_solve(fd, operator, topo, cfg, callback, host, workspace)
        if out is not None:
            x, history, iters, zero_exit = out
            full = iters - (1 if zero_exit else 0)
            counters.add(reads=15 * dofs * full, writes=3 * dofs * full,
                         flops=CG_VECTOR_FLOPS_PER_POINT * dofs * full)
            if zero_exit:
                counters.add(reads=3 * dofs, flops=2 * dofs)
            operator.account(full)
        else:
            x, history, iters = _generic_solve(fd, operator, topo, cfg, counters, callback, host)
    return CgResult(solution=dv.from_device_io(x, kind), residual_history=history,
                    iterations_run=iters, counters=counters.copy())
