"""Host-buffer Ax path: per-step wall-time distribution and chunk sweep."""
import ctypes
import json
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import _device as dv  # noqa: E402
from paper_2005_13425_b200 import kernels as K  # noqa: E402
from paper_2005_13425_b200._lib import load  # noqa: E402

E, n = 4096, 10
b = sb.build_basis(n)
u = sb.random_field(E, n, 1)
geom = sb.GeomFactors(values=sb.random_field(6 * E, n, 2).reshape(E, 6, n, n, n))
u_pin = u.cpu().pin_memory()
res = {}
for chunk_mb in (2, 4, 8, 16, 32):
    K.HOST_CHUNK_BYTES = chunk_mb << 20
    for _ in range(5):
        w = sb.apply_ax(u_pin, geom, b)
    ts = []
    for _ in range(40):
        t0 = time.perf_counter()
        w = sb.apply_ax(u_pin, geom, b)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    res[f"chunk{chunk_mb}MB"] = {"median_ms": statistics.median(ts), "min_ms": ts[0],
                                 "p90_ms": ts[int(0.9 * len(ts))], "max_ms": ts[-1]}
print(json.dumps(res, indent=1))
