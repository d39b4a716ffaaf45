"""Host-buffer Ax (pinned in/out) per transfer mode and chunk size."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import kernels as K  # noqa: E402

dev = torch.device("cuda", 0)
n, E = 10, 4096
b = sb.build_basis(n)
u = sb.random_field(E, n, 1, device=dev)
g = sb.GeomFactors(values=sb.random_field(6 * E, n, 2, device=dev).reshape(E, 6, n, n, n))
uh = u.cpu().pin_memory()


def med(reps=30):
    w = None
    for _ in range(4):
        w = sb.apply_ax(uh, g, b)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        w = sb.apply_ax(uh, g, b)
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(statistics.median(ts), 3)


for mode, chunks in (("1", [8]), ("2", [2, 4, 8, 16]), ("0", [4, 8]), ("1", [8])):
    os.environ["SEM_HOST_MODE"] = mode
    for c in chunks:
        K.HOST_CHUNK_BYTES = c << 20
        print({"mode": mode, "chunk_MB": c, "ms": med()})
