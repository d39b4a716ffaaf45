"""Break down the host-buffer Ax path: chunk sizes, allocation, copies."""
import ctypes
import json
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
out = torch.empty_like(u_pin).pin_memory()
ud, wd = torch.empty_like(u), torch.empty_like(u)
dx = np.ascontiguousarray(b.diff)
lib = load()
st = torch.cuda.current_stream()


def run(chunk):
    rc = lib.sem_ax_host(ctypes.c_void_p(u_pin.data_ptr()), dv.ptr(geom.values), dv.host_f64_ptr(dx),
                         dv.host_f64_ptr(dx), ctypes.c_void_p(out.data_ptr()), E, n, dv.ptr(ud),
                         dv.ptr(wd), chunk, ctypes.c_void_p(st.cuda_stream))
    assert rc == 0, lib.sem_last_error()


res = {}
for chunk in [4096, 2048, 1024, 512, 256, 128, 64]:
    for _ in range(3):
        run(chunk)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        run(chunk)
        st.synchronize()
    res[f"chunk{chunk}_ms"] = (time.perf_counter() - t0) / 20 * 1e3
# side stream as the compute stream
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    st = torch.cuda.current_stream()
    for _ in range(3):
        run(256)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        run(256)
        st.synchronize()
    res["chunk256_sidestream_ms"] = (time.perf_counter() - t0) / 20 * 1e3
# full API path
for _ in range(3):
    sb.apply_ax(u_pin, geom, b)
t0 = time.perf_counter()
for _ in range(20):
    w = sb.apply_ax(u_pin, geom, b)
res["api_ms"] = (time.perf_counter() - t0) / 20 * 1e3
t0 = time.perf_counter()
for _ in range(20):
    o = torch.empty_like(u_pin, pin_memory=True)
res["pinned_alloc_ms"] = (time.perf_counter() - t0) / 20 * 1e3
print(json.dumps(res))
