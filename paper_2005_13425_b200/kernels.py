"""Element-local Poisson operator ``apply_ax`` on the B200 (contract of
sembench/kernels.py:413-468).

Every variant name the reference accepts runs its own sm_100a kernel, with
the reference's validation and error behaviour (``ValueError`` for shape /
name problems, ``ScratchCapacityError`` for SCRATCH beyond n=10, the
analytic ``TrafficCounters`` inventory): LAYERED is the tuned pencil kernel
of csrc/ax.cu (the paper's §IV-C design and the north-star path, 1e-12 of
the reference); REFERENCE and SCRATCH are the paper's baselines
(csrc/ax_variants.cu, bit-identical to the reference, REFERENCE leaving the
metric-scaled gradients in its workspace just as sembench does).
"""

from __future__ import annotations

import ctypes
import enum
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from ._lib import check, load
from .basis import PolynomialBasis
from .mesh import GeomFactors, as_geom

__all__ = ["KernelVariant", "TrafficCounters", "ScratchCapacityError", "apply_ax",
           "apply_ax_into", "flops_per_apply", "apply_read_words", "apply_write_words",
           "reference_workspace", "SCRATCH_MAX_POINTS", "SCRATCH_WORD_BUDGET",
           "ax_bytes_per_apply"]

SCRATCH_MAX_POINTS = 10
SCRATCH_WORD_BUDGET = 6144


class KernelVariant(enum.Enum):
    REFERENCE = "reference"
    SCRATCH = "scratch"
    LAYERED = "layered"

    @classmethod
    def parse(cls, name: str) -> "KernelVariant":
        try:
            return cls(name.lower())
        except (ValueError, AttributeError):
            valid = ", ".join(v.value for v in cls)
            raise ValueError(f"unknown kernel variant {name!r} (expected one of {valid})") from None


class ScratchCapacityError(ValueError):
    """The scratch variant cannot stage an element of this size."""


@dataclass
class TrafficCounters:
    """Analytic word/flop inventory (sembench/kernels.py:95-118)."""

    reads: int = 0
    writes: int = 0
    flops: int = 0

    def add(self, reads: int = 0, writes: int = 0, flops: int = 0) -> None:
        if reads < 0 or writes < 0 or flops < 0:
            raise ValueError("counter increments must be non-negative")
        self.reads += reads
        self.writes += writes
        self.flops += flops

    def copy(self) -> "TrafficCounters":
        return TrafficCounters(self.reads, self.writes, self.flops)


def flops_per_apply(dofs: int, n: int) -> int:
    """D (12 n + 15): the equal-weight flop count of one apply."""
    if dofs < 1 or n < 1:
        raise ValueError("dofs and n must be positive")
    return dofs * (12 * n + 15)


def apply_read_words(variant: KernelVariant, dofs: int) -> int:
    return dofs * (13 if variant is KernelVariant.REFERENCE else 7)


def apply_write_words(variant: KernelVariant, dofs: int) -> int:
    return dofs * (7 if variant is KernelVariant.REFERENCE else 1)


def ax_bytes_per_apply(dofs: int) -> int:
    """Algorithmic HBM bytes of the layered GPU kernel: u + 6 g + w = 64 B/point."""
    return 64 * dofs


def reference_workspace(num_elements: int, n: int, device=None):
    """The REFERENCE variant's three full-size intermediates (kernels.py:
    :138-146).  numpy arrays by default (the reference's type: the GPU pass
    results are copied back into them); ``device=`` gives CUDA tensors that
    the kernels write in place."""
    shape = (num_elements, n, n, n)
    if device is not None:
        return tuple(torch.empty(shape, dtype=torch.float64, device=device) for _ in range(3))
    return np.empty(shape), np.empty(shape), np.empty(shape)


def _validate(u, g_shape, n: int) -> None:
    shp = tuple(u.shape)
    if len(shp) != 4 or shp[1:] != (n, n, n):
        raise ValueError(f"field shape {shp} does not match basis n={n}")
    if tuple(g_shape) != (shp[0], 6, n, n, n):
        raise ValueError(f"geometry shape {tuple(g_shape)} does not match field {shp}")


_basis_ptrs: dict = {}


def _basis_host_ptrs(basis: PolynomialBasis):
    """(dx, dxt) as contiguous float64 arrays with their ctypes pointers,
    converted once per basis (the basis arrays are frozen)."""
    ent = _basis_ptrs.get(id(basis))
    if ent is None or ent[0] is not basis:
        if len(_basis_ptrs) > 64:
            _basis_ptrs.clear()
        dx = np.ascontiguousarray(basis.diff, dtype=np.float64)
        dxt = np.ascontiguousarray(basis.diff_t, dtype=np.float64)
        ent = (basis, dx, dxt, dv.host_f64_ptr(dx), dv.host_f64_ptr(dxt))
        _basis_ptrs[id(basis)] = ent
    return ent[3], ent[4]


def apply_ax_into(u: torch.Tensor, g: torch.Tensor, basis: PolynomialBasis, w: torch.Tensor,
                  variant: int = 0) -> torch.Tensor:
    """Device-only fast path: w <- A_local u (no validation, no allocation;
    the per-call host work is a handful of attribute reads, so back-to-back
    launches keep the GPU fed)."""
    pdx, pdxt = _basis_host_ptrs(basis)
    check(load().sem_ax_variant(u.data_ptr(), g.data_ptr(), pdx, pdxt, w.data_ptr(),
                                u.shape[0], basis.n, variant,
                                torch.cuda.current_stream(u.device).cuda_stream), "apply_ax")
    return w


def apply_ax(u, geom: GeomFactors, basis: PolynomialBasis,
             variant: KernelVariant = KernelVariant.LAYERED,
             counters: TrafficCounters | None = None, workspace=None):
    """w = A_local u.  numpy in -> numpy out (H2D/D2H); CUDA tensor in -> CUDA
    tensor out (zero-copy).  Returns a fresh array; inputs are not modified."""
    if not isinstance(variant, KernelVariant):
        variant = KernelVariant.parse(variant)
    geom = as_geom(geom)
    n = basis.n
    _validate(u, geom.shape, n)
    if variant is KernelVariant.REFERENCE and workspace is not None:
        if any(tuple(a.shape) != tuple(u.shape) for a in workspace):
            raise ValueError("workspace arrays must match the field shape")
    if variant is KernelVariant.SCRATCH and n > SCRATCH_MAX_POINTS:
        raise ScratchCapacityError(
            f"scratch variant supports at most {SCRATCH_MAX_POINTS} points per "
            f"dimension, got n={n}")
    kind = dv.io_kind(u)
    if variant is not KernelVariant.LAYERED:
        result = _apply_ax_variant(u, kind, geom, basis, variant, workspace)
    elif kind == "device":
        with torch.cuda.device(u.device):
            ud = dv.as_device_f64(u, u.device, "u")
            gd = geom.device_values(ud.device)
            wd = torch.empty_like(ud)
            if ud.shape[0] > 0:
                apply_ax_into(ud, gd, basis, wd)
        result = wd
    else:
        result = _apply_ax_host(u, kind, geom, basis)
    if counters is not None:
        dofs = math.prod(tuple(u.shape))
        counters.add(reads=apply_read_words(variant, dofs),
                     writes=apply_write_words(variant, dofs),
                     flops=flops_per_apply(dofs, n))
    return result


_ref_scratch: dict = {}


def _apply_ax_variant(u, kind: str, geom: GeomFactors, basis: PolynomialBasis,
                      variant: KernelVariant, workspace):
    """REFERENCE / SCRATCH on the GPU (csrc/ax_variants.cu), bit-exact with the
    reference.  Host inputs are copied to the device and the result back; a
    host workspace receives the intermediates like the reference's does."""
    ud, kind = dv.to_device_io(u, "u")
    dev = ud.device
    n, E = basis.n, int(ud.shape[0])
    dx = np.ascontiguousarray(basis.diff, dtype=np.float64)
    with torch.cuda.device(dev):
        gd = geom.device_values(dev)
        wd = torch.empty_like(ud)
        stream = dv.stream_handle(dev)
        if variant is KernelVariant.SCRATCH:
            check(load().sem_ax_scratch(dv.ptr(ud), dv.ptr(gd), dv.host_f64_ptr(dx), dv.ptr(wd),
                                        E, n, stream), "apply_ax")
        else:
            dxt = np.ascontiguousarray(basis.diff_t, dtype=np.float64)
            on_dev = workspace is not None and all(
                isinstance(a, torch.Tensor) and a.device == dev and a.dtype == torch.float64
                and a.is_contiguous() for a in workspace)
            if on_dev:
                ws = tuple(workspace)
            else:
                key = (dev.index, E * n ** 3)
                buf = _ref_scratch.get(key)
                if buf is None:
                    _ref_scratch.clear()
                    buf = torch.empty((3,) + tuple(ud.shape), dtype=torch.float64, device=dev)
                    _ref_scratch[key] = buf
                ws = (buf[0], buf[1], buf[2])
            check(load().sem_ax_reference(dv.ptr(ud), dv.ptr(gd), dv.host_f64_ptr(dx),
                                          dv.host_f64_ptr(dxt), *(dv.ptr(a) for a in ws),
                                          dv.ptr(wd), E, n, stream), "apply_ax")
            if workspace is not None and not on_dev:
                for dst, src in zip(workspace, ws):
                    if isinstance(dst, torch.Tensor):
                        dst.copy_(src)
                    else:
                        dst[...] = src.cpu().numpy()
    return dv.from_device_io(wd, kind)


# elements per streamed chunk for host-buffer calls: 8 MB of u was the
# best point of the chunk sweep on B200 + PCIe Gen5 (tools/e2e_probe.py)
HOST_CHUNK_BYTES = 8 << 20
# pieces a pageable input is staged in (host copy overlapping the GPU;
# tools/numpy_e2e_probe.py: numpy in 1.50 ms unpiped, 1.15 / 1.19 / 1.32 ms with
# 2 / 4 / 8 pieces, pinned input 0.92 ms)
STAGE_CHUNKS = 2
_host_scratch: dict = {}


def _host_device_scratch(dev: torch.device, numel: int):
    """Device staging halves (u, w) of at least numel doubles each, kept per
    device; the sliced views are cached with the buffer."""
    ent = _host_scratch.get(dev.index)
    if ent is None or ent[0].shape[1] < numel:
        buf = torch.empty((2, numel), dtype=torch.float64, device=dev)
        ent = (buf, {})
        _host_scratch[dev.index] = ent
    views = ent[1].get(numel)
    if views is None:
        views = (ent[0][0, :numel], ent[0][1, :numel])
        ent[1][numel] = views
    return views


def _apply_ax_host(u, kind: str, geom: GeomFactors, basis: PolynomialBasis):
    """Host arrays in/out through sem_ax_host: chunked H2D / Ax / D2H on
    library-owned copy streams (csrc/host.cu).  Pageable inputs are first
    staged into pinned memory; the result is a pinned CPU tensor (numpy view
    for numpy callers).  The per-call Python work is kept to the minimum
    (tools/host_overhead_probe.py): this is the reference's call shape."""
    dv.require_cuda()
    dev = torch.device("cuda", torch.cuda.current_device())
    shape = tuple(u.shape)
    E, n = shape[0], basis.n
    if E == 0:
        out = torch.empty(shape, dtype=torch.float64)
        return out.numpy() if kind == "numpy" else out
    if kind == "numpy":
        src = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64))
    else:
        src = u if (u.dtype == torch.float64 and u.is_contiguous()) else \
            u.to(torch.float64).contiguous()
    out_np = dv.pinned_pool.array(shape)
    pdx, pdxt = _basis_host_ptrs(basis)
    gd = geom.device_values(dev)
    ud, wd = _host_device_scratch(dev, E * n ** 3)
    stream = torch.cuda.current_stream()
    chunk = max(1, HOST_CHUNK_BYTES // (8 * n ** 3))
    lib = load()
    per = n ** 3 * 8  # bytes per element of u / w
    staged = None
    if src.is_pinned():
        check(lib.sem_ax_host(src.data_ptr(), gd.data_ptr(), pdx, pdxt,
                              out_np.ctypes.data, E, n, ud.data_ptr(), wd.data_ptr(),
                              chunk, stream.cuda_stream), "apply_ax")
    else:
        # pageable input (a reference-style numpy array): staged into a
        # recycled pinned block in STAGE_CHUNKS pieces, each piece's apply
        # enqueued as soon as it is staged, so the host copy of piece k+1
        # overlaps the GPU's PCIe traffic for piece k
        staged = dv.pinned_pool.scratch(src.numel() * 8)
        st = staged.view(torch.float64)[:src.numel()].view(shape)
        pieces = min(STAGE_CHUNKS, E)
        for q in range(pieces):
            e0, e1 = E * q // pieces, E * (q + 1) // pieces
            st[e0:e1].copy_(src[e0:e1])
            check(lib.sem_ax_host(st.data_ptr() + e0 * per, gd.data_ptr() + 6 * e0 * per,
                                  pdx, pdxt, out_np.ctypes.data + e0 * per, e1 - e0, n,
                                  ud.data_ptr() + e0 * per, wd.data_ptr() + e0 * per, chunk,
                                  stream.cuda_stream), "apply_ax")
    stream.synchronize()
    if staged is not None:
        dv.pinned_pool.release(staged)
    return out_np if kind == "numpy" else torch.from_numpy(out_np)
