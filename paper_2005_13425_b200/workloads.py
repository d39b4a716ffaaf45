"""Benchmark input definitions reused from the reference harness
(sembench/bench.py:100-125): the most-cubic element box and the seeded,
interface-consistent, masked right-hand side."""

from __future__ import annotations

import torch

from .assembly import _dssum_dev, _mask_dev, as_topology
from .fields import random_field

__all__ = ["factor_elements", "make_rhs"]


def factor_elements(count: int) -> tuple[int, int, int]:
    """Most cubic ex >= ey >= ez factorisation, minimising (ex/ez, ex-ez)."""
    if count < 1:
        raise ValueError("element count must be positive")
    best, best_key = (count, 1, 1), (count / 1, count + 2)
    cbrt = round(count ** (1 / 3))
    for ez in range(1, cbrt + 1):
        if count % ez:
            continue
        rest = count // ez
        ey = ez
        while ey * ey <= rest:
            if rest % ey == 0:
                ex = rest // ey
                key = (ex / ez, ex - ez)
                if key < best_key:
                    best_key, best = key, (ex, ey, ez)
            ey += 1
    return best


def make_rhs(num_elements: int, n: int, topo, seed: int, device=None, host: bool | None = None):
    """mask(dssum(random_field(E, n, seed))) generated on the GPU.  numpy like
    the reference (bench.py:122-125) unless `device` is given."""
    if host is None:
        host = device is None
    topo = as_topology(topo)
    f = random_field(num_elements, n, seed, device=device, host=False)
    with torch.cuda.device(f.device):
        out = _mask_dev(_dssum_dev(f, topo, False), topo)
    return out.cpu().numpy() if host else out
