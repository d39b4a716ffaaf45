"""Host time per apply_ax_into call (the bench step) vs its GPU time."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200.kernels import apply_ax_into  # noqa: E402

dev = torch.device("cuda", 0)
n, E = 10, 4096
b = sb.build_basis(n)
u = sb.random_field(E, n, 1, device=dev)
g = sb.random_field(6 * E, n, 2, device=dev).reshape(E, 6, n, n, n)
w = torch.empty_like(u)
for _ in range(20):
    apply_ax_into(u, g, b, w)
torch.cuda.synchronize()
# host cost alone: tiny problem so the GPU never lags
us, gs = u[:1].contiguous(), g[:1].contiguous()
ws = torch.empty_like(us)
t0 = time.perf_counter()
for _ in range(2000):
    apply_ax_into(us, gs, b, ws)
host_us = (time.perf_counter() - t0) / 2000 * 1e6
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(2000):
    apply_ax_into(u, g, b, w)
e1.record()
torch.cuda.synchronize()
print({"host_us_per_launch": round(host_us, 2), "stream_us_per_apply": round(e0.elapsed_time(e1) / 2000 * 1e3, 2)})
