"""Host-buffer Ax path: per-step wall-time distribution and chunk/ramp sweep
(SEM_HOST_RAMP overrides the first/last-chunk ramp of csrc/host.cu)."""
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
u = sb.random_field(E, n, 1, device="cuda")
geom = sb.GeomFactors(values=sb.random_field(6 * E, n, 2, device="cuda").reshape(E, 6, n, n, n))
u_pin = u.cpu().pin_memory()
w_dev = sb.apply_ax(u.cuda(), geom, b).cpu()
import os  # noqa: E402
res = {}
for mode, chunk_mb, ramp in ((0, 8, 1), (0, 8, 4), (1, 8, 1), (2, 8, 1), (2, 4, 1), (2, 2, 1),
                             (2, 1, 1), (2, 4, 4), (3, 8, 1), (3, 4, 1), (3, 2, 1), (3, 1, 1),
                             (3, 4, 4)):
    K.HOST_CHUNK_BYTES = chunk_mb << 20
    os.environ["SEM_HOST_RAMP"] = str(ramp)
    os.environ["SEM_HOST_MODE"] = str(mode)
    for _ in range(5):
        w = sb.apply_ax(u_pin, geom, b)
    ts = []
    for _ in range(40):
        t0 = time.perf_counter()
        w = sb.apply_ax(u_pin, geom, b)
        ts.append((time.perf_counter() - t0) * 1e3)
    ts.sort()
    res[f"mode{mode}_chunk{chunk_mb}MB_ramp{ramp}"] = {"median_ms": statistics.median(ts), "min_ms": ts[0],
                                 "p90_ms": ts[int(0.9 * len(ts))], "max_ms": ts[-1],
                                 "max_abs_diff_vs_device": float((w - w_dev).abs().max())}
print(json.dumps(res, indent=1))
