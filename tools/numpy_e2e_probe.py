"""apply_ax with reference-style numpy arrays (pageable in, numpy out) vs a
pinned CPU tensor, E = 4096, p = 9: median ms per call."""
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
n, E = 10, 4096
b = sb.build_basis(n)
u = sb.random_field(E, n, 1, device=dev)
g = sb.GeomFactors(values=sb.random_field(6 * E, n, 2, device=dev).reshape(E, 6, n, n, n))
u_np = u.cpu().numpy().copy()
u_pin = u.cpu().pin_memory()


def med(x, reps=30):
    w = None
    for _ in range(3):
        w = sb.apply_ax(x, g, b)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        w = sb.apply_ax(x, g, b)
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(statistics.median(ts), 3)


t0 = time.perf_counter()
tmp = np.empty_like(u_np)
for _ in range(10):
    np.copyto(tmp, u_np)
memcpy_ms = (time.perf_counter() - t0) / 10 * 1e3
print({"numpy_in_ms": med(u_np), "pinned_in_ms": med(u_pin), "host_memcpy_32MB_ms": round(memcpy_ms, 3),
       "torch_threads": torch.get_num_threads()})

from paper_2005_13425_b200 import kernels as K  # noqa: E402
for c in (2, 4, 8, 16):
    K.STAGE_CHUNKS = c
    print({"stage_chunks": c, "numpy_in_ms": med(u_np)})
