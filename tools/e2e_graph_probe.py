"""Host-buffer Ax (E = 4096, p = 9, pinned u in, pinned w out): per-call wall
time of sem_ax_host launched directly vs captured once into a CUDA graph and
replayed, for the transfer modes x chunk sizes (csrc/host.cu):
  mode 0: chunked copy engines both ways, mode 2: copy-engine u + mapped w,
  mode 1: the kernel reads u / writes w in mapped host memory (one launch).
Prints one JSON line per configuration."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200._lib import load  # noqa: E402
from paper_2005_13425_b200.kernels import _basis_host_ptrs  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
E, n = 4096, 10
per = n ** 3
b = sb.build_basis(n)
u_d = sb.random_field(E, n, 1, device="cuda")
g_d = sb.random_field(6 * E, n, 2, device="cuda").reshape(E, 6, n, n, n)
ref = torch.empty_like(u_d)
load().sem_ax(u_d.data_ptr(), g_d.data_ptr(), *_basis_host_ptrs(b), ref.data_ptr(), E, n,
              torch.cuda.current_stream().cuda_stream)
ref = ref.cpu()
u_h = u_d.cpu().pin_memory()
w_h = torch.empty(u_h.shape, dtype=torch.float64).pin_memory()
ud = torch.empty_like(u_d)
wd = torch.empty_like(u_d)
lib = load()
pdx, pdxt = _basis_host_ptrs(b)


def call(chunk, stream):
    rc = lib.sem_ax_host(u_h.data_ptr(), g_d.data_ptr(), pdx, pdxt, w_h.data_ptr(), E, n,
                         ud.data_ptr(), wd.data_ptr(), chunk, stream)
    assert rc == 0, lib.sem_last_error()


def timed(fn, steps=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3, min(ts) * 1e3


for mode in (0, 2, 1):
    os.environ["SEM_HOST_MODE"] = str(mode)
    for mb in ((0.25, 0.5, 1, 2, 4, 8) if mode != 1 else (32,)):
        chunk = max(1, int(mb * 2 ** 20 // (8 * per)))
        s = torch.cuda.current_stream().cuda_stream
        med, mn = timed(lambda: call(chunk, torch.cuda.current_stream().cuda_stream))
        w_h.zero_()
        call(chunk, s)
        torch.cuda.synchronize()
        ok = bool(torch.equal(w_h, ref))
        row = {"mode": mode, "chunk_mb": mb, "direct_ms": round(med, 4), "direct_min_ms": round(mn, 4),
               "exact": ok}
        try:
            graph = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side), torch.cuda.graph(graph, stream=side):
                call(chunk, side.cuda_stream)
            torch.cuda.current_stream().wait_stream(side)
            gmed, gmn = timed(graph.replay)
            w_h.zero_()
            graph.replay()
            torch.cuda.synchronize()
            row.update({"graph_ms": round(gmed, 4), "graph_min_ms": round(gmn, 4),
                        "graph_exact": bool(torch.equal(w_h, ref))})
        except Exception as exc:  # noqa: BLE001
            row["graph_error"] = str(exc)[:200]
        print(json.dumps(row), flush=True)
