"""Box mesh and geometric factors (contract of sembench/mesh.py:20-91).

``GeomFactors.values`` keeps the reference layout ``[E, 6, n, n, n]``
(index ``[e, m, k, j, i]``, m = g1..g6).  It may be a numpy array (copied to
the GPU once, on first use, and cached) or a CUDA tensor.  ``build_geom``
generates the affine box metric directly on the GPU with the reference's
exact rounding (``((w_k*w_j)*w_i)*(h/2)``), so a 32768-element geometry
(1.6 GB) never crosses PCIe.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _device as dv
from ._lib import check, load
from .basis import PolynomialBasis

__all__ = ["BoxMesh", "GeomFactors", "build_mesh", "build_geom"]


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
        """The metric as a contiguous float64 CUDA tensor (cached per device)."""
        dev = device or dv.current_device()
        v = self.values
        if isinstance(v, torch.Tensor) and v.device == dev and v.dtype == torch.float64 \
                and v.is_contiguous():
            return v
        t = self._cache.get(dev.index)
        if t is None:
            t = dv.as_device_f64(v, dev, "geometry")
            self._cache[dev.index] = t
        return t


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
    """Affine box metric, generated on the GPU (sem_box_geom)."""
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
    return GeomFactors(values=g)
