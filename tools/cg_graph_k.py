"""CG solve time per iteration vs iterations captured per CUDA graph."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import cg as C  # noqa: E402

dev = torch.device("cuda", 0)
out = {}
KS = [int(x) for x in os.environ.get("CG_GRAPH_KS", "1,5,10,20,1,10").split(",")]
for k in KS:
    C.GRAPH_ITERATIONS = k
    row = {}
    for E in (4096, 32768):
        bench.E_HEAD = E
        row[E] = round(min(bench.bench_cg(sb, dev, 100)["ms_per_iteration"] for _ in range(3)) * 1e3, 1)
    out[f"k{k}_{len(out)}"] = row
print(json.dumps(out))
