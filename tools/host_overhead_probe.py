"""Fixed per-call cost of the host-buffer apply_ax wrapper: the Python API vs
the raw sem_ax_host call, at E = 1 (kernel time negligible) and E = 4096."""
import cProfile
import json
import pstats
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2005_13425_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
n = 10
b = sb.build_basis(n)
out = {}
for E in (1, 4096):
    u = sb.random_field(E, n, 1, device=dev)
    g = sb.random_field(6 * E, n, 2, device=dev).reshape(E, 6, n, n, n)
    geom = sb.GeomFactors(values=g)
    uh = u.cpu().pin_memory()
    w = None
    for _ in range(10):
        w = sb.apply_ax(uh, geom, b)
    ts = []
    for _ in range(100):
        t0 = time.perf_counter()
        w = sb.apply_ax(uh, geom, b)
        ts.append((time.perf_counter() - t0) * 1e6)
    out[f"api_E{E}_us"] = round(statistics.median(ts), 1)
    if E == 1:
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(200):
            w = sb.apply_ax(uh, geom, b)
        pr.disable()
        st = pstats.Stats(pr)
        st.sort_stats("tottime")
        rows = sorted(st.stats.items(), key=lambda kv: -kv[1][2])[:15]
        out["top_tottime_us_per_call"] = [(f"{k[2]}:{k[0].split('/')[-1]}:{k[1]}", round(v[2] / 200 * 1e6, 1)) for k, v in rows]
print(json.dumps(out, indent=1))
