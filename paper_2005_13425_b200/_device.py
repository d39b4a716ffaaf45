"""Device-buffer plumbing: torch supplies CUDA memory and streams, libsem
supplies the compute.  Fields are float64 CUDA tensors; numpy inputs are
copied host->device (and results back) so reference-style callers work
unchanged."""

from __future__ import annotations

import ctypes
import math
import threading
import warnings
import weakref

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
        with warnings.catch_warnings():  # read-only arrays (frozen geometry) are only read
            warnings.simplefilter("ignore", UserWarning)
            src = torch.from_numpy(arr)
        return src.to(dev, non_blocking=False)
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


class PinnedPool:
    """Recycled page-locked host blocks for host-buffer results.

    Pinning a fresh 32 MB buffer costs ~1.2 ms on the B200 boxes (more than
    the PCIe transfer it enables), so results are carved from recycled pinned
    blocks.  Each call still returns a FRESH array (reference semantics: the
    result never aliases an earlier one): the block returns to the pool only
    when the numpy array handed out -- and every numpy/torch view of it --
    has been garbage collected (weakref.finalize on the owning array).
    """

    def __init__(self, keep_per_size: int = 4):
        self._free: dict[int, list] = {}
        self._lock = threading.Lock()
        self._keep = keep_per_size

    def _take(self, nbytes: int) -> torch.Tensor:
        with self._lock:
            lst = self._free.get(nbytes)
            if lst:
                return lst.pop()
        return torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)

    def _give(self, nbytes: int, blk: torch.Tensor) -> None:
        with self._lock:
            lst = self._free.setdefault(nbytes, [])
            if len(lst) < self._keep:
                lst.append(blk)

    def array(self, shape, dtype=np.float64) -> np.ndarray:
        """A fresh pinned numpy array; its memory is recycled after it dies."""
        nbytes = math.prod(shape) * np.dtype(dtype).itemsize
        size = max(nbytes, 1)
        blk = self._take(size)
        # a per-call owner object exports the block's memory; every numpy
        # view (and torch.from_numpy of one) chains its .base to it, so the
        # block is recycled only when the LAST view dies -- a finalizer on the
        # returned array itself would fire while a reshape/ravel view lives
        owner = (ctypes.c_char * size).from_address(blk.data_ptr())
        owner._block = blk
        weakref.finalize(owner, self._give, size, blk)
        arr = np.frombuffer(owner, dtype=np.uint8, count=nbytes).view(dtype).reshape(shape)
        return arr

    def scratch(self, nbytes: int) -> torch.Tensor:
        """A pinned staging block the caller returns with release()."""
        return self._take(nbytes)

    def release(self, blk: torch.Tensor) -> None:
        self._give(blk.numel(), blk)


pinned_pool = PinnedPool()
