"""Direct-stiffness summation, Dirichlet mask and the global operator on the
B200 (contract of sembench/assembly.py:37-155).

The topology of a box mesh is pure lattice arithmetic, so the device
kernels (csrc/assembly.cu) recompute global ids, multiplicities and the mask
from element coordinates instead of reading them.  The host-side arrays of
the reference ``Topology`` (``global_id``, ``multiplicity``, ``mask``,
``inv_multiplicity``) are still available, built lazily with the
reference's integer recipe, for callers that inspect them.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from ._lib import check, load
from .basis import PolynomialBasis
from .fields import validate_field
from .kernels import KernelVariant, TrafficCounters, apply_ax
from .mesh import BoxMesh, GeomFactors, as_geom

__all__ = ["Topology", "CsrTopology", "OperatorTimers", "build_topology", "as_topology",
           "dssum", "mask", "apply_global", "GlobalOperator"]


@dataclass(frozen=True)
class Topology:
    """Global node identification of an ex*ey*ez box with n points per edge."""

    num_elements: int
    n: int
    ex: int
    ey: int
    ez: int
    num_global: int
    _host: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def dofs(self) -> int:
        return self.num_elements * self.n ** 3

    @property
    def box(self) -> tuple[int, int, int]:
        return (self.ex, self.ey, self.ez)

    # -- host arrays of the reference Topology (lazy; assembly.py:69-110) --
    def _build_host(self) -> dict:
        if self._host:
            return self._host
        n, ex, ey, ez = self.n, self.ex, self.ey, self.ez
        nx, ny, nz = ex * (n - 1) + 1, ey * (n - 1) + 1, ez * (n - 1) + 1
        elem = np.arange(self.num_elements, dtype=np.int64)
        cx = (elem % ex).reshape(-1, 1, 1, 1) * (n - 1)
        cy = ((elem // ex) % ey).reshape(-1, 1, 1, 1) * (n - 1)
        cz = (elem // (ex * ey)).reshape(-1, 1, 1, 1) * (n - 1)
        loc = np.arange(n, dtype=np.int64)
        gx = cx + loc.reshape(1, 1, 1, n)
        gy = cy + loc.reshape(1, 1, n, 1)
        gz = cz + loc.reshape(1, n, 1, 1)
        gid = (gz * ny + gy) * nx + gx
        mult = np.bincount(gid.ravel(), minlength=self.num_global)[gid]
        inner = ((gx > 0) & (gx < nx - 1) & (gy > 0) & (gy < ny - 1) & (gz > 0) & (gz < nz - 1))
        host = {
            "global_id": gid,
            "multiplicity": mult,
            "mask": inner.astype(np.float64),
            "inv_multiplicity": (1.0 / mult.astype(np.float64)).ravel(),
        }
        for arr in host.values():
            arr.flags.writeable = False
        self._host.update(host)
        return self._host

    @property
    def global_id(self) -> np.ndarray:
        return self._build_host()["global_id"]

    @property
    def multiplicity(self) -> np.ndarray:
        return self._build_host()["multiplicity"]

    @property
    def mask(self) -> np.ndarray:
        return self._build_host()["mask"]

    @property
    def inv_multiplicity(self) -> np.ndarray:
        return self._build_host()["inv_multiplicity"]


@dataclass
class OperatorTimers:
    """Scoped accumulators (seconds) for the global operator pieces; on the GPU
    they are measured with CUDA events around each launch."""

    ax_seconds: float = 0.0
    dssum_seconds: float = 0.0
    applies: int = 0


def build_topology(mesh: BoxMesh) -> Topology:
    n = mesh.n
    num_global = ((mesh.ex * (n - 1) + 1) * (mesh.ey * (n - 1) + 1) * (mesh.ez * (n - 1) + 1))
    return Topology(num_elements=mesh.num_elements, n=n, ex=mesh.ex, ey=mesh.ey, ez=mesh.ez,
                    num_global=num_global)


class CsrTopology:
    """A reference-style topology whose numbering is NOT the box lattice.

    Built from any object carrying the reference ``Topology`` fields
    (``num_elements``, ``n``, ``num_global``, ``global_id``, ``mask``,
    ``multiplicity``, ``inv_multiplicity``; sembench/assembly.py:37-53).
    dssum runs the ordered CSR gather (``sem_dssum_csr``: each id class
    summed in ascending local index from +0.0, bit-identical to the
    reference's ``np.bincount``), mask multiplies by the caller's mask array
    (``sem_mask_array``), weighted dots read ``inv_multiplicity``
    (``sem_glsc3``).  The device copies are made once per device.
    """

    def __init__(self, src):
        self.num_elements = int(src.num_elements)
        self.n = int(src.n)
        self.num_global = int(src.num_global)
        shape = (self.num_elements, self.n, self.n, self.n)
        self.global_id = np.asarray(src.global_id).reshape(shape)
        self.multiplicity = np.asarray(src.multiplicity).reshape(shape)
        self.mask = np.asarray(src.mask, dtype=np.float64).reshape(shape)
        self.inv_multiplicity = np.asarray(src.inv_multiplicity, dtype=np.float64).ravel()
        gid = self.global_id.ravel().astype(np.int64, copy=False)
        if gid.size >= 2 ** 31:
            raise ValueError("general topologies are limited to 2^31 - 1 local points")
        if gid.size and (gid.min() < 0 or gid.max() >= self.num_global):
            raise ValueError("global_id outside [0, num_global)")
        counts = np.bincount(gid, minlength=self.num_global)
        self._off = np.zeros(self.num_global + 1, dtype=np.int32)
        np.cumsum(counts, out=self._off[1:])
        self._idx = np.argsort(gid, kind="stable").astype(np.int32)
        self._dev: dict = {}

    @property
    def dofs(self) -> int:
        return self.num_elements * self.n ** 3

    def device_arrays(self, device: torch.device):
        """(seg_off, seg_idx, mask, inv_multiplicity) on `device`."""
        ent = self._dev.get(device.index)
        if ent is None:
            ent = tuple(torch.from_numpy(np.array(a)).to(device) for a in
                        (self._off, self._idx, self.mask, self.inv_multiplicity))
            self._dev[device.index] = ent
        return ent


_converted: dict = {}


def _box_of(t):
    """The (ex, ey, ez) box whose lattice numbering t.global_id might be, or None."""
    n, E = int(t.n), int(t.num_elements)
    gid = np.asarray(t.global_id)
    if E < 1 or n < 2 or gid.shape != (E, n, n, n) or int(gid[0, 0, 0, 0]) != 0:
        return None
    nx = int(gid[0, 0, 1, 0])
    if nx < n or (nx - 1) % (n - 1):
        return None
    ny = int(gid[0, 1, 0, 0]) // nx
    if ny < n or (ny - 1) % (n - 1):
        return None
    ex, ey = (nx - 1) // (n - 1), (ny - 1) // (n - 1)
    if E % (ex * ey):
        return None
    return ex, ey, E // (ex * ey)


def as_topology(topo):
    """This package's topology for `topo`.

    Our own :class:`Topology` / :class:`CsrTopology` pass through.  Any other
    object with the reference ``Topology`` fields (e.g. one built by
    ``sembench.build_topology``) is checked against the box lattice: when
    its ``global_id``, ``multiplicity``, ``mask`` and ``inv_multiplicity``
    are exactly the lattice's (assembly.py:69-110), the analytic box
    topology is returned (every fused kernel applies); otherwise a
    :class:`CsrTopology` (general ordered gather).  Conversions of objects
    whose arrays are read-only are cached."""
    if isinstance(topo, (Topology, CsrTopology)):
        return topo
    needed = ("num_elements", "n", "num_global", "global_id", "multiplicity", "mask",
              "inv_multiplicity")
    if not all(hasattr(topo, a) for a in needed):
        raise TypeError(f"not a topology: {type(topo).__name__} lacks the reference "
                        "Topology fields")
    ent = _converted.get(id(topo))
    if ent is not None and ent[0]() is topo:
        return ent[1]
    frozen = all(not getattr(getattr(topo, a), "flags", None) or
                 not getattr(topo, a).flags.writeable
                 for a in ("global_id", "multiplicity", "mask", "inv_multiplicity"))
    box = _box_of(topo)
    out = None
    if box is not None:
        cand = build_topology(BoxMesh(*box, int(topo.n), 1.0))
        if cand.num_global == int(topo.num_global) and \
                np.array_equal(cand.global_id, np.asarray(topo.global_id)) and \
                np.array_equal(cand.multiplicity, np.asarray(topo.multiplicity)) and \
                np.array_equal(cand.mask, np.asarray(topo.mask)) and \
                np.array_equal(cand.inv_multiplicity, np.asarray(topo.inv_multiplicity).ravel()):
            out = cand
    if out is None:
        out = CsrTopology(topo)
    if frozen:
        try:
            ref = weakref.ref(topo)
        except TypeError:
            return out
        if len(_converted) > 64:
            _converted.clear()
        _converted[id(topo)] = (ref, out)
    return out


def _dssum_dev(f: torch.Tensor, topo, apply_mask: bool) -> torch.Tensor:
    out = torch.empty_like(f)
    if isinstance(topo, CsrTopology):
        off, idx, msk, _ = topo.device_arrays(f.device)
        s = dv.stream_handle(f.device)
        check(load().sem_dssum_csr(dv.ptr(f), dv.ptr(out), dv.ptr(off), dv.ptr(idx),
                                   topo.num_global, s), "dssum")
        if apply_mask:
            check(load().sem_mask_array(dv.ptr(out), dv.ptr(msk), dv.ptr(out), out.numel(), s),
                  "mask")
        return out
    check(load().sem_dssum_box(dv.ptr(f), dv.ptr(out), topo.ex, topo.ey, topo.ez, topo.n,
                               1 if apply_mask else 0, dv.stream_handle(f.device)), "dssum")
    return out


def _mask_dev(f: torch.Tensor, topo) -> torch.Tensor:
    out = torch.empty_like(f)
    if isinstance(topo, CsrTopology):
        msk = topo.device_arrays(f.device)[2]
        check(load().sem_mask_array(dv.ptr(f), dv.ptr(msk), dv.ptr(out), out.numel(),
                                    dv.stream_handle(f.device)), "mask")
        return out
    check(load().sem_mask_box(dv.ptr(f), dv.ptr(out), topo.ex, topo.ey, topo.ez, topo.n,
                              dv.stream_handle(f.device)), "mask")
    return out


def _wdot_dev(a: torch.Tensor, b: torch.Tensor, topo, out: torch.Tensor | None = None
              ) -> torch.Tensor:
    """<a, b>_c = sum(a * b * inv_multiplicity) into a device scalar."""
    dev = a.device
    if out is None:
        out = torch.empty(1, dtype=torch.float64, device=dev)
    s, scratch = dv.stream_handle(dev), dv.reduce_scratch(dev)
    if isinstance(topo, CsrTopology):
        invm = topo.device_arrays(dev)[3]
        check(load().sem_glsc3(dv.ptr(a), dv.ptr(b), dv.ptr(invm), a.numel(), dv.ptr(out),
                               dv.ptr(scratch), s), "weighted_dot")
    else:
        check(load().sem_glsc3_box(dv.ptr(a), dv.ptr(b), topo.ex, topo.ey, topo.ez, topo.n,
                                   dv.ptr(out), dv.ptr(scratch), s), "weighted_dot")
    return out


def dssum(f, topo: Topology, counters: TrafficCounters | None = None):
    """Sum every class of coincident nodes; all copies receive the total.

    Bit-identical to the reference's ``np.bincount`` order."""
    topo = as_topology(topo)
    validate_field(f, topo.num_elements, topo.n)
    fd, kind = dv.to_device_io(f, "f")
    with torch.cuda.device(fd.device):
        out = _dssum_dev(fd, topo, False)
    if counters is not None:
        counters.add(reads=topo.dofs, writes=topo.dofs)
    return dv.from_device_io(out, kind)


def mask(f, topo: Topology, counters: TrafficCounters | None = None):
    """Zero the boundary nodes (pointwise product with the 0/1 mask)."""
    topo = as_topology(topo)
    validate_field(f, topo.num_elements, topo.n)
    fd, kind = dv.to_device_io(f, "f")
    with torch.cuda.device(fd.device):
        out = _mask_dev(fd, topo)
    if counters is not None:
        counters.add(reads=2 * topo.dofs, writes=topo.dofs)
    return dv.from_device_io(out, kind)


def apply_global(u, geom: GeomFactors, basis: PolynomialBasis, topo: Topology,
                 variant: KernelVariant = KernelVariant.LAYERED,
                 counters: TrafficCounters | None = None,
                 timers: OperatorTimers | None = None, workspace=None):
    """Global masked Poisson operator mask(dssum(A_local(mask(u))))."""
    topo = as_topology(topo)
    geom = as_geom(geom)
    validate_field(u, topo.num_elements, topo.n)
    ud, kind = dv.to_device_io(u, "u")
    with torch.cuda.device(ud.device):
        um = _mask_dev(ud, topo)
        if counters is not None:
            counters.add(reads=2 * topo.dofs, writes=topo.dofs)
        if timers is None:
            w = apply_ax(um, geom, basis, variant, counters, workspace)
            w = _dssum_dev(w, topo, True)
        else:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record()
            w = apply_ax(um, geom, basis, variant, counters, workspace)
            ev[1].record()
            w = _dssum_dev(w, topo, True)
            ev[2].record()
            ev[2].synchronize()
            timers.ax_seconds += ev[0].elapsed_time(ev[1]) / 1e3
            timers.dssum_seconds += ev[1].elapsed_time(ev[2]) / 1e3
            timers.applies += 1
    if counters is not None:
        # dssum and the output mask, fused into one launch above
        counters.add(reads=topo.dofs, writes=topo.dofs)
        counters.add(reads=2 * topo.dofs, writes=topo.dofs)
    return dv.from_device_io(w, kind)


class GlobalOperator:
    """Callable ``op(u) = apply_global(u, geom, basis, topo)``.

    ``cg_solve`` recognises this type and runs its fused, device-resident
    iteration (csrc/cg.cu) instead of calling back into Python per step.
    """

    def __init__(self, geom: GeomFactors, basis: PolynomialBasis, topo: Topology,
                 counters: TrafficCounters | None = None, timers: OperatorTimers | None = None):
        geom, topo = as_geom(geom), as_topology(topo)
        if basis.n != topo.n or geom.n != topo.n or geom.num_elements != topo.num_elements:
            raise ValueError("geometry, basis and topology disagree on n or element count")
        self.geom, self.basis, self.topo = geom, basis, topo
        self.counters, self.timers = counters, timers

    def __call__(self, u):
        return apply_global(u, self.geom, self.basis, self.topo, KernelVariant.LAYERED,
                            self.counters, self.timers)

    def account(self, applies: int) -> None:
        """Counter/timer bookkeeping for `applies` fused applications."""
        if self.counters is not None and applies > 0:
            d, n = self.topo.dofs, self.topo.n
            per_r = 2 * d + 7 * d + d + 2 * d  # mask, Ax, dssum, mask
            per_w = d + d + d + d
            self.counters.add(reads=per_r * applies, writes=per_w * applies,
                              flops=d * (12 * n + 15) * applies)
        if self.timers is not None:
            self.timers.applies += applies
