"""Element-local fields and the seeded generator (contract of sembench/fields.py).

A field is ``[E, n, n, n]`` float64 indexed ``[e, k, j, i]`` (i fastest).
``random_field`` is the reference's counter-based SplitMix64 stream; it is
generated on the GPU (``sem_random_field``) bit-for-bit.  Like the
reference, the builders return numpy arrays; ``device=`` returns a CUDA
tensor on that device instead (no host round trip).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dv
from ._lib import check, load

__all__ = ["zeros_field", "constant_field", "random_field", "validate_field", "mix64"]

_MASK64 = (1 << 64) - 1
_FNV_PRIME = 0x100000001B3


def _splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def mix64(a: int, b: int = 0) -> int:
    """Seed mixer of sembench/fields.py:28-31 (exact 64-bit integer arithmetic)."""
    return _splitmix64((a * _FNV_PRIME + b) & _MASK64)


def zeros_field(num_elements: int, n: int, device=None):
    """Zero field: numpy (the reference's type), or a CUDA tensor on `device`."""
    if device is None:
        return np.zeros((num_elements, n, n, n))
    return torch.zeros((num_elements, n, n, n), dtype=torch.float64, device=device)


def constant_field(num_elements: int, n: int, value: float = 1.0, device=None):
    """Constant field: numpy (the reference's type), or a CUDA tensor on `device`."""
    if device is None:
        return np.full((num_elements, n, n, n), float(value))
    return torch.full((num_elements, n, n, n), float(value), dtype=torch.float64,
                      device=device)


def random_field(num_elements: int, n: int, seed: int, device=None, host: bool | None = None):
    """Uniform [-1, 1) field, value q = 2*(splitmix64(seed+q) >> 11)*2^-53 - 1,
    generated on the GPU.  Returns numpy unless `device` is given (``host=True``
    forces numpy, ``host=False`` a tensor on the current device)."""
    if host is None:
        host = device is None
    dev = device or dv.current_device()
    out = torch.empty((num_elements, n, n, n), dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        check(load().sem_random_field(dv.ptr(out), out.numel(), int(seed) & _MASK64,
                                      dv.stream_handle(dev)), "random_field")
    return dv.to_numpy(out) if host else out


def validate_field(f, num_elements: int, n: int, name: str = "field") -> None:
    expected = (num_elements, n, n, n)
    if not isinstance(f, (np.ndarray, torch.Tensor)) or tuple(f.shape) != expected:
        got = getattr(f, "shape", None)
        got = tuple(got) if got is not None else None
        raise ValueError(f"{name} must have shape {expected}, got {got}")
