"""Where the fixed per-solve cost of cg_solve goes: a torch.profiler (CUPTI)
trace of one 100-iteration solve at E = 4096, printing the host-side
Python / launch spans and the GPU kernel spans of the first and last
microseconds of the solve."""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2005_13425_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
n, E, iters = 10, 4096, 100
b = sb.build_basis(n)
mesh = sb.build_mesh(*sb.factor_elements(E), n, 1.0)
topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b, device=dev)
f = sb.make_rhs(E, n, topo, sb.mix64(1, E), device=dev)
op = sb.GlobalOperator(geom, b, topo)
ws = sb.CgWorkspace(topo, iters, dev)
for _ in range(2):
    sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    with torch.profiler.record_function("cg_solve"):
        sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0), workspace=ws)
    torch.cuda.synchronize()
path = "/tmp/cg_trace.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
spans = [e for e in ev if e.get("ph") == "X"]
solve = [e for e in spans if e["name"] == "cg_solve" and e.get("cat") == "user_annotation"]
t0 = solve[0]["ts"] if solve else min(e["ts"] for e in spans)
t1 = t0 + (solve[0]["dur"] if solve else 0)
gpu = sorted([e for e in spans if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")], key=lambda e: e["ts"])
print(f"cg_solve host span: {t1 - t0:.1f} us")
print("first GPU activities (us from cg_solve entry):")
for e in gpu[:6]:
    print(f"  {e['ts'] - t0:9.1f} +{e['dur']:7.1f}  {e['name'][:70]}")
print("last GPU activities:")
for e in gpu[-6:]:
    print(f"  {e['ts'] - t0:9.1f} +{e['dur']:7.1f}  {e['name'][:70]}")
cpu = sorted([e for e in spans if e.get("cat") in ("cpu_op", "cuda_runtime", "python_function")
              and t0 <= e["ts"] <= t1], key=lambda e: e["ts"])
print("host calls in the first 300 us:")
for e in cpu:
    if e["ts"] - t0 > 300:
        break
    print(f"  {e['ts'] - t0:9.1f} +{e['dur']:7.1f}  {e.get('cat')}: {e['name'][:60]}")
last_gpu_end = max(e["ts"] + e["dur"] for e in gpu)
print(f"last GPU end {last_gpu_end - t0:.1f} us, host span end {t1 - t0:.1f} us")
