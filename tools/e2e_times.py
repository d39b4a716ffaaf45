"""Per-call wall times of the host-buffer Ax (public API), to locate outliers."""
import gc
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402

E, n = 4096, 10
b = sb.build_basis(n)
dev = torch.device("cuda", 0)
u = sb.random_field(E, n, 1, device=dev)
geom = sb.GeomFactors(values=sb.random_field(6 * E, n, 2, device=dev).reshape(E, 6, n, n, n))
u_host = u.cpu().pin_memory()
out = {}
for label, gc_on in (("gc_on", True), ("gc_off", False)):
    if not gc_on:
        gc.disable()
    for _ in range(5):
        w = sb.apply_ax(u_host, geom, b)
    torch.cuda.synchronize()
    ts = []
    for _ in range(60):
        t0 = time.perf_counter()
        w = sb.apply_ax(u_host, geom, b)
        ts.append(round((time.perf_counter() - t0) * 1e3, 3))
    gc.enable()
    out[label] = ts
print(json.dumps(out))
