"""Box mesh and geometric factors (contract of sembench/mesh.py:20-91).

``GeomFactors.values`` keeps the reference layout ``[E, 6, n, n, n]``
(index ``[e, m, k, j, i]``, m = g1..g6).  It may be a CUDA tensor (used in
place), a read-only numpy array (the reference's frozen geometry: copied to
the GPU once and cached), a writable numpy array (copied on EVERY use -- the
caller may mutate it in place, and a cached copy would go stale) or a CPU
tensor (cached, re-copied whenever its version counter moves).
``build_geom`` generates the affine box metric on the GPU with the
reference's exact rounding (``((w_k*w_j)*w_i)*(h/2)``); with ``device=`` the
result stays there (a 32768-element geometry, 1.6 GB, never crosses PCIe),
without it a frozen numpy array is returned like the reference's.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from ._lib import check, load
from .basis import PolynomialBasis

__all__ = ["BoxMesh", "GeomFactors", "build_mesh", "build_geom", "as_geom"]


@dataclass(frozen=True)
class BoxMesh:
    ex: int
    ey: int
    ez: int
    n: int
    element_extent: float

    @property
    def num_elements(self) -> int:
        return self.ex * self.ey * self.ez

    @property
    def dofs(self) -> int:
        return self.num_elements * self.n ** 3


@dataclass(frozen=True)
class GeomFactors:
    """Symmetric metric (g1 g2 g3; g2 g4 g5; g3 g5 g6) per nodal point."""

    values: object  # np.ndarray or torch.Tensor, shape (E, 6, n, n, n)
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def num_elements(self) -> int:
        return int(self.values.shape[0])

    @property
    def n(self) -> int:
        return int(self.values.shape[2])

    @property
    def shape(self):
        return tuple(self.values.shape)

    def device_values(self, device: torch.device | None = None) -> torch.Tensor:
        """The metric as a contiguous float64 CUDA tensor on `device`."""
        dev = device or dv.current_device()
        v = self.values
        if isinstance(v, torch.Tensor):
            if v.device == dev and v.dtype == torch.float64 and v.is_contiguous():
                return v
            key = (dev.index, v._version)  # an in-place write bumps the version
        elif isinstance(v, np.ndarray) and not v.flags.writeable:
            key = (dev.index, None)
        else:  # writable numpy: the caller may change it between calls
            self._cache.pop(dev.index, None)
            return dv.as_device_f64(v, dev, "geometry")
        ent = self._cache.get(dev.index)
        if ent is None or ent[0] != key:
            ent = (key, dv.as_device_f64(v, dev, "geometry"))
            self._cache[dev.index] = ent
        return ent[1]


_wrapped: dict = {}


def as_geom(geom) -> GeomFactors:
    """This package's GeomFactors for `geom`: ours pass through; any object
    with a ``values`` array of the reference layout (e.g. a
    ``sembench.GeomFactors``) is wrapped, the wrapper cached per object so
    its device copy is reused (sembench/mesh.py:40-58)."""
    if isinstance(geom, GeomFactors):
        return geom
    v = getattr(geom, "values", None)
    if v is None or len(getattr(v, "shape", ())) != 5 or v.shape[1] != 6:
        raise TypeError(f"not a geometry: {type(geom).__name__} has no [E, 6, n, n, n] values")
    ent = _wrapped.get(id(geom))
    if ent is not None and ent[0]() is geom and ent[1].values is v:
        return ent[1]
    out = GeomFactors(values=v)
    try:
        ref = weakref.ref(geom)
    except TypeError:
        return out
    if len(_wrapped) > 64:
        _wrapped.clear()
    _wrapped[id(geom)] = (ref, out)
    return out


def build_mesh(ex: int, ey: int, ez: int, n: int, element_extent: float) -> BoxMesh:
    for name, v in (("ex", ex), ("ey", ey), ("ez", ez), ("n", n)):
        if not isinstance(v, (int, np.integer)) or v < 1:
            raise ValueError(f"{name} must be a positive integer, got {v!r}")
    if n < 2:
        raise ValueError(f"n must be at least 2, got {n}")
    if not element_extent > 0.0:
        raise ValueError(f"element_extent must be positive, got {element_extent!r}")
    return BoxMesh(int(ex), int(ey), int(ez), int(n), float(element_extent))


def build_geom(mesh: BoxMesh, basis: PolynomialBasis, device: torch.device | None = None
               ) -> GeomFactors:
    """Affine box metric, generated on the GPU (sem_box_geom).  With
    ``device`` the values stay there; without it they are returned as a
    frozen numpy array, the reference's type (mesh.py:72-91)."""
    if basis.n != mesh.n:
        raise ValueError(f"basis has n={basis.n} but mesh has n={mesh.n}")
    dev = device or dv.current_device()
    n = mesh.n
    g = torch.empty((mesh.num_elements, 6, n, n, n), dtype=torch.float64, device=dev)
    w = np.ascontiguousarray(basis.weights, dtype=np.float64)
    with torch.cuda.device(dev):
        check(load().sem_box_geom(dv.ptr(g), mesh.num_elements, n, dv.host_f64_ptr(w),
                                  float(mesh.element_extent), dv.stream_handle(dev)),
              "build_geom")
    if device is not None:
        return GeomFactors(values=g)
    host = dv.to_numpy(g)
    host.flags.writeable = False
    out = GeomFactors(values=host)
    out._cache[dev.index] = ((dev.index, None), g)  # the device copy is already made
    return out
