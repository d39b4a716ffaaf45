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

import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from ._lib import check, load
from .basis import PolynomialBasis
from .fields import validate_field
from .kernels import KernelVariant, TrafficCounters, apply_ax
from .mesh import BoxMesh, GeomFactors

__all__ = ["Topology", "OperatorTimers", "build_topology", "dssum", "mask", "apply_global",
           "GlobalOperator"]


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


def _dssum_dev(f: torch.Tensor, topo: Topology, apply_mask: bool) -> torch.Tensor:
    out = torch.empty_like(f)
    check(load().sem_dssum_box(dv.ptr(f), dv.ptr(out), topo.ex, topo.ey, topo.ez, topo.n,
                               1 if apply_mask else 0, dv.stream_handle(f.device)), "dssum")
    return out


def _mask_dev(f: torch.Tensor, topo: Topology) -> torch.Tensor:
    out = torch.empty_like(f)
    check(load().sem_mask_box(dv.ptr(f), dv.ptr(out), topo.ex, topo.ey, topo.ez, topo.n,
                              dv.stream_handle(f.device)), "mask")
    return out


def dssum(f, topo: Topology, counters: TrafficCounters | None = None):
    """Sum every class of coincident nodes; all copies receive the total.

    Bit-identical to the reference's ``np.bincount`` order."""
    validate_field(f, topo.num_elements, topo.n)
    fd, kind = dv.to_device_io(f, "f")
    with torch.cuda.device(fd.device):
        out = _dssum_dev(fd, topo, False)
    if counters is not None:
        counters.add(reads=topo.dofs, writes=topo.dofs)
    return dv.from_device_io(out, kind)


def mask(f, topo: Topology, counters: TrafficCounters | None = None):
    """Zero the boundary nodes (pointwise product with the 0/1 mask)."""
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
    validate_field(u, topo.num_elements, topo.n)
    ud, kind = dv.to_device_io(u, "u")
    with torch.cuda.device(ud.device):
        um = mask(ud, topo, counters)
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
