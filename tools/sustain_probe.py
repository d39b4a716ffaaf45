"""Burst vs sustained: is the power-capped Ax slowdown the kernel or the chip?

Times, with the bench protocol (soak, then K back-to-back launches, CUDA
events), (1) a 262 MB D2D copy (read 131 MB + write 131 MB = the Ax apply's
algorithmic bytes) and (2) the Ax apply at E=4096, p=9, each at several soak
lengths, sampling SM clocks / power with nvidia-smi.  Prints one JSON object.
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200.kernels import apply_ax_into  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n, E = 10, 4096
basis = sb.build_basis(n)
sets = []
for s in range(2):
    u = sb.random_field(E, n, 1 + 10 * s, device=dev)
    g = sb.random_field(6 * E, n, 2 + 10 * s, device=dev).reshape(E, 6, n, n, n)
    sets.append((u, g, torch.empty_like(u)))
half = 131072000 // 8
cp = [(torch.rand(half, dtype=torch.float64, device=dev), torch.empty(half, dtype=torch.float64, device=dev))
      for _ in range(2)]


def ax(i):
    u, g, w = sets[i % 2]
    apply_ax_into(u, g, basis, w, 0)


def copy(i):
    a, b = cp[i % 2]
    b.copy_(a)


def timed(fn, soak, steps):
    for i in range(5):
        fn(i)
    torch.cuda.synchronize()
    with bench.ClockSampler(0) as clk:
        t0 = time.perf_counter()
        i = 0
        while time.perf_counter() - t0 < soak:
            for _ in range(100):
                fn(i)
                i += 1
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(steps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / steps
    c = clk.summary()
    return {"us": us, "GBps": 262144000 / us / 1e3, "sm_mhz": c["sm_mhz"],
            "reasons": c["reasons"], "power_w_max": c.get("power_w_max")}


out = {}
for soak, steps in ((0.0, 50), (0.0, 500), (0.0, 2000), (1.5, 2000), (4.0, 2000)):
    for name, fn in (("copy", copy), ("ax", ax)):
        time.sleep(2.0)  # let the chip cool back to burst state
        out[f"{name}_soak{soak}_steps{steps}"] = timed(fn, soak, steps)
print(json.dumps(out, indent=1))
