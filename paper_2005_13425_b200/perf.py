"""Cost model and roofline arithmetic (contract of sembench/perf.py:56-221),
plus the B200 measurement helpers used by bench.py.

The paper's per-CG-iteration model (Eq. 1/2): D(12n+34) flops and 240 D bytes
(24 D reads + 6 D writes), intensity (12n+34)/240.  The Ax-only headline
metric uses (12n+15) D flops (kernels.py:121-125) over 64 D algorithmic
bytes (u 8 + g 48 + w 8 per point).
"""

from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass

import numpy as np

__all__ = ["measure_bandwidth", "B200_L2_BYTES", "model_flops_per_iteration", "model_bytes_per_iteration",
           "model_read_bytes_per_iteration", "model_write_bytes_per_iteration", "intensity",
           "roofline_peak", "probe_byte_accounting", "evaluate_roofline", "RooflineResult",
           "CostModel", "CACHE_EFFECT_THRESHOLD", "LLC_WARN_BYTES", "ax_intensity",
           "measured_peaks"]

WORD_BYTES = 8
MODEL_READ_WORDS_PER_POINT = 24
MODEL_WRITE_WORDS_PER_POINT = 6
CACHE_EFFECT_THRESHOLD = 1.2
LLC_WARN_BYTES = 64 * 1024 * 1024


def model_flops_per_iteration(dofs: int, n: int) -> int:
    if dofs < 1 or n < 0:
        raise ValueError("dofs must be positive and n non-negative")
    return dofs * (12 * n + 34)


def model_bytes_per_iteration(dofs: int) -> int:
    if dofs < 1:
        raise ValueError("dofs must be positive")
    return WORD_BYTES * (MODEL_READ_WORDS_PER_POINT + MODEL_WRITE_WORDS_PER_POINT) * dofs


def model_read_bytes_per_iteration(dofs: int) -> int:
    return WORD_BYTES * MODEL_READ_WORDS_PER_POINT * dofs


def model_write_bytes_per_iteration(dofs: int) -> int:
    return WORD_BYTES * MODEL_WRITE_WORDS_PER_POINT * dofs


def intensity(n: int) -> float:
    if n < 2:
        raise ValueError(f"n must be at least 2, got {n}")
    return (12 * n + 34) / 240.0


def ax_intensity(n: int) -> float:
    """Ax-only intensity (12n+15)/64 flop/byte (2.109 at n=10)."""
    return (12 * n + 15) / 64.0


def roofline_peak(bandwidth: float, n: int) -> float:
    if not bandwidth > 0.0:
        raise ValueError(f"bandwidth must be positive, got {bandwidth!r}")
    if n < 2:
        raise ValueError(f"n must be at least 2, got {n}")
    return bandwidth * (12 * n + 34) / 240.0


@dataclass(frozen=True)
class CostModel:
    dofs: int
    n: int

    def __post_init__(self):
        if self.dofs < 1 or self.n < 2:
            raise ValueError("require dofs >= 1 and n >= 2")

    @property
    def flops_per_iteration(self) -> int:
        return model_flops_per_iteration(self.dofs, self.n)

    @property
    def bytes_per_iteration(self) -> int:
        return model_bytes_per_iteration(self.dofs)

    @property
    def intensity(self) -> float:
        return intensity(self.n)


@dataclass(frozen=True)
class RooflineResult:
    measured_bandwidth: float
    intensity: float
    peak_flops: float
    achieved_flops: float
    fraction: float
    flags: tuple = ()

    def __post_init__(self):
        for name in ("measured_bandwidth", "intensity", "peak_flops", "achieved_flops"):
            v = getattr(self, name)
            if not (np.isfinite(v) and v > 0.0):
                raise ValueError(f"{name} must be positive and finite, got {v!r}")


def probe_byte_accounting(dofs: int) -> tuple[int, int]:
    payload = model_bytes_per_iteration(dofs)
    return payload, 2 * payload


def evaluate_roofline(run_flops: int, run_seconds: float, bandwidth: float, n: int
                      ) -> RooflineResult:
    if run_flops <= 0 or not run_seconds > 0.0:
        raise ValueError("run_flops and run_seconds must be positive")
    achieved = run_flops / run_seconds
    peak = roofline_peak(bandwidth, n)
    frac = achieved / peak
    flags = ("cache-effect",) if frac > CACHE_EFFECT_THRESHOLD else ()
    return RooflineResult(measured_bandwidth=bandwidth, intensity=intensity(n),
                          peak_flops=peak, achieved_flops=achieved, fraction=frac, flags=flags)


_MIN_REPETITIONS = 10
# The reference's 1 ms floor guards a host perf_counter; CUDA events resolve
# ~0.5 us, so the device probe's floor is 20 us of timed copies (40x the
# event resolution) -- a 64-element probe (15 MB) takes ~0.1 ms for 10 reps.
_MIN_ELAPSED_SECONDS = 2e-5
# B200 L2 (126 MB): a probe payload below it streams partly from L2, so the
# GPU analog of the reference's last-level-cache warning uses the larger of
# the two thresholds.
B200_L2_BYTES = 126 * 1024 * 1024


def measure_bandwidth(dofs: int, repetitions: int = 10, warmup: int = 2, device=None) -> float:
    """Device streaming-copy bandwidth in bytes/second at the model's buffer
    size (the contract of sembench/perf.py:162-203 on the GPU).

    Allocates a source and a destination of 240 D bytes each in HBM, copies
    source to destination once per repetition with the library's streaming
    copy kernel (sem_stream_copy), times each repetition with CUDA events and
    reports the median rate counting read plus write streams.  Warm-up
    repetitions are excluded.  Same errors as the reference: ValueError for
    fewer than 10 repetitions, RuntimeWarning when the payload may fit in
    cache, MemoryError when the buffers cannot be allocated, RuntimeError when
    the timed region is below timer resolution.
    """
    import warnings

    import torch

    from . import _device as dv
    from ._lib import check, load

    if repetitions < _MIN_REPETITIONS:
        raise ValueError(f"repetitions must be at least {_MIN_REPETITIONS}, got {repetitions}")
    payload, counted = probe_byte_accounting(dofs)
    limit = max(LLC_WARN_BYTES, B200_L2_BYTES)
    if payload < limit:
        warnings.warn(f"probe payload {payload} bytes may fit in cache (below {limit}); "
                      "bandwidth may read high", RuntimeWarning, stacklevel=2)
    dev = torch.device(device) if device is not None else dv.current_device()
    nwords = payload // WORD_BYTES
    try:
        src = torch.ones(nwords, dtype=torch.float64, device=dev)
        dst = torch.empty(nwords, dtype=torch.float64, device=dev)
    except torch.OutOfMemoryError as exc:
        raise MemoryError(f"cannot allocate two {payload}-byte probe buffers") from exc
    lib = load()
    with torch.cuda.device(dev):
        stream = torch.cuda.current_stream(dev)
        handle = ctypes.c_void_p(stream.cuda_stream)

        def copy():
            check(lib.sem_stream_copy(dv.ptr(dst), dv.ptr(src), nwords, handle), "measure_bandwidth")

        for _ in range(max(warmup, 1)):
            copy()
        events = [torch.cuda.Event(enable_timing=True) for _ in range(repetitions + 1)]
        events[0].record(stream)
        for rep in range(repetitions):
            copy()
            events[rep + 1].record(stream)
        events[-1].synchronize()
    times = np.array([events[r].elapsed_time(events[r + 1]) * 1e-3 for r in range(repetitions)])
    if times.sum() < _MIN_ELAPSED_SECONDS:
        raise RuntimeError(f"probe finished in {times.sum():.2e} s, below timer resolution; "
                           "increase repetitions or the problem size")
    rates = np.where(times > 0.0, counted / np.maximum(times, 1e-300), np.inf)
    return float(np.median(rates))


_FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback when the driver file is absent


def measured_peaks(repo_root: str | None = None) -> dict:
    """MEASURED_PEAKS.json (driver-written) or the documented fallback."""
    root = repo_root or os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        d["source"] = "measured"
        return d
    return {"hbm_gbs": _FALLBACK_HBM_GBS, "source": "fallback"}
