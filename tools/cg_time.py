"""Whole-solve CG timing (100 iterations, the bench protocol: CUDA events
around cg_solve, graph-replayed iterations) at E = 4096 and 32768; prints
ms per iteration.  Tuning knobs come from the environment (SEM_CG_*)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import bench  # noqa: E402
import paper_2005_13425_b200 as sb  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
out = {}
for E in [int(a) for a in (sys.argv[1:] or ["4096", "32768"])]:
    bench.E_HEAD = E
    best = min(bench.bench_cg(sb, dev, 100)["ms_per_iteration"] for _ in range(3))
    out[f"E{E}"] = round(best * 1e3, 1)
print(json.dumps(out))
