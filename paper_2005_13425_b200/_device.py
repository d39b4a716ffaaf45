"""Device-buffer plumbing: torch supplies CUDA memory and streams, libsem
supplies the compute.  Fields are float64 CUDA tensors; numpy inputs are
copied host->device (and results back) so reference-style callers work
unchanged."""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import SemLibraryError, load

_scratch: dict = {}


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise SemLibraryError("no CUDA device visible: the sm_100a path has no CPU fallback")
    load()


def current_device() -> torch.device:
    require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(device: torch.device | None = None) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def is_tensor(x) -> bool:
    return isinstance(x, torch.Tensor)


def as_device_f64(x, device: torch.device | None = None, name: str = "array") -> torch.Tensor:
    """C-contiguous float64 CUDA tensor view/copy of x (numpy or torch)."""
    if isinstance(x, torch.Tensor):
        if x.device.type != "cuda":
            dev = device or current_device()
            x = x.to(dev)
        if x.dtype != torch.float64:
            x = x.to(torch.float64)
        return x.contiguous()
    if isinstance(x, np.ndarray):
        dev = device or current_device()
        arr = np.ascontiguousarray(x, dtype=np.float64)
        return torch.from_numpy(arr).to(dev, non_blocking=False)
    raise ValueError(f"{name} must be a numpy array or a torch tensor, got {type(x).__name__}")


def ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


def host_f64_ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def reduce_scratch(device: torch.device) -> torch.Tensor:
    """Zero-initialised reduction scratch, one per (device, stream)."""
    key = (device.index, torch.cuda.current_stream(device).cuda_stream)
    buf = _scratch.get(key)
    if buf is None:
        nbytes = int(load().sem_reduce_scratch_bytes())
        buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _scratch[key] = buf
    return buf


def to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def io_kind(x) -> str:
    """'numpy' | 'host' (CPU tensor) | 'device' (CUDA tensor)."""
    if isinstance(x, torch.Tensor):
        return "device" if x.device.type == "cuda" else "host"
    return "numpy"


def to_device_io(x, name: str = "array"):
    """(CUDA float64 tensor, io kind) for an API input."""
    kind = io_kind(x)
    dev = x.device if kind == "device" else None
    return as_device_f64(x, dev, name), kind


def from_device_io(t: torch.Tensor, kind: str):
    """Return a result in the caller's memory space: numpy in -> numpy out,
    CPU tensor in -> CPU tensor out, CUDA tensor in -> CUDA tensor out."""
    if kind == "numpy":
        return to_numpy(t)
    if kind == "host":
        return t.cpu()
    return t
