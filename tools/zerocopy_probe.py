"""Host-buffer Ax without copy engines: the kernel reads u from and writes w
to page-locked host memory directly (mapped, UVA), so the PCIe reads and
writes of all elements run concurrently inside one launch.

Compares, per variant, the time and result against the device-resident
apply, and against the chunked copy-engine pipeline (sem_ax_host)."""
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
geom = sb.GeomFactors(values=g)
out = {}
dxh, dxth = b.diff.copy(), b.diff_t.copy()


def ax_raw(uu, ww, v):
    check(load().sem_ax_variant(dv.ptr(uu), dv.ptr(g), dv.host_f64_ptr(dxh), dv.host_f64_ptr(dxth),
                                dv.ptr(ww), E, n, v, dv.stream_handle(dev)), "ax")


def wall(fn, reps=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return {"median_ms": statistics.median(ts), "min_ms": min(ts)}


for v in (0, 1, 19, 25, 34, 35, 36, 38, 5):
    try:
        w_pin.zero_()
        r = wall(lambda: ax_raw(u_pin, w_pin, v))
        r["max_abs_diff"] = float((w_pin.to(dev) - w_ref).abs().max())
        out[f"zerocopy_v{v}"] = r
    except Exception as exc:  # noqa: BLE001
        out[f"zerocopy_v{v}"] = {"error": str(exc)[:200]}
# device-resident u, host w (writes only over PCIe) and the reverse
out["dev_u_host_w_v0"] = wall(lambda: ax_raw(u, w_pin, 0))
wd = torch.empty_like(u)
out["host_u_dev_w_v0"] = wall(lambda: ax_raw(u_pin, wd, 0))
out["chunked_public_api"] = wall(lambda: sb.apply_ax(u_pin, geom, b))
print(json.dumps(out, indent=1))
