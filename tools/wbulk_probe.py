"""Bulk-store (TMA) write-back of w (variants 63/64) vs the default Ax:
zero-copy host buffers (the e2e path) and device-resident, n = 10, E = 4096."""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import _device as dv  # noqa: E402
from paper_2005_13425_b200._lib import check, load  # noqa: E402
from paper_2005_13425_b200.kernels import apply_ax_into  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n, E = 10, 4096
b = sb.build_basis(n)
u = sb.random_field(E, n, 1, device=dev)
g = sb.random_field(6 * E, n, 2, device=dev).reshape(E, 6, n, n, n)
w_ref = torch.empty_like(u)
apply_ax_into(u, g, b, w_ref, 0)
u_pin = u.cpu().pin_memory()
w_pin = torch.empty(u.shape, dtype=torch.float64).pin_memory()
dxh, dxth = b.diff.copy(), b.diff_t.copy()


def ax_raw(uu, ww, v):
    check(load().sem_ax_variant(dv.ptr(uu), dv.ptr(g), dv.host_f64_ptr(dxh), dv.host_f64_ptr(dxth),
                                dv.ptr(ww), E, n, v, dv.stream_handle(dev)), "ax")


def wall(fn, reps=60):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(statistics.median(ts), 4)


out = {}
wd = torch.empty_like(u)
for v in (0, 34, 63, 64, 0, 63):
    w_pin.zero_()
    zc = wall(lambda: ax_raw(u_pin, w_pin, v))
    diff = float((w_pin.to(dev) - w_ref).abs().max())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(20):
        ax_raw(u, wd, v)
    ev0.record()
    for _ in range(200):
        ax_raw(u, wd, v)
    ev1.record()
    torch.cuda.synchronize()
    dd = float((wd - w_ref).abs().max())
    out[f"v{v}_{len(out)}"] = {"zerocopy_ms": zc, "zc_max_abs_diff": diff,
                               "device_us": round(ev0.elapsed_time(ev1) / 200 * 1e3, 2),
                               "dev_max_abs_diff": dd}
print(json.dumps(out, indent=1))
