#!/usr/bin/env python
"""Small-E probe (BASELINE config 2, E = 1024 / 2048): per E, time sem_ax
variants and a same-bytes streaming copy under one protocol -- one apply per
rotating input set (sets x 64 B x E n^3 >= 2 x L2) captured in a CUDA graph,
graph replays timed with CUDA events -- so a variant's fraction of the HBM
roofline can be read next to what a pure data mover reaches at that size.
Each variant is checked against the oracle on a few elements."""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import _device as dv  # noqa: E402
from paper_2005_13425_b200._lib import load  # noqa: E402
from paper_2005_13425_b200.kernels import apply_ax_into  # noqa: E402
from paper_2005_13425_b200.perf import measured_peaks  # noqa: E402


def graph_time(calls, reps):
    """Mean microseconds per call: all `calls` captured once in a graph."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for c in calls:
            c()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(graph, stream=side):
        for c in calls:
            c()
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * len(calls))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=10)
    ap.add_argument("--E", default="512,1024,2048,4096")
    ap.add_argument("--variants", default="0")
    ap.add_argument("--reps", type=int, default=60)
    args = ap.parse_args()
    n = args.n
    hbm = float(measured_peaks(ROOT)["hbm_gbs"])
    lib = load()
    basis = sb.build_basis(n)
    for E in [int(x) for x in args.E.split(",")]:
        nbytes = 64 * E * n ** 3
        nsets = max(2, -(-2 * 126 * 2 ** 20 // nbytes))
        sets = []
        for s in range(nsets):
            u = sb.random_field(E, n, 1 + s, device="cuda")
            g = sb.random_field(6 * E, n, 100 + s, device="cuda").reshape(E, 6, n, n, n)
            sets.append((u, g, torch.empty_like(u)))
        idx = sorted({0, 1, E // 2, E - 1})
        ref = O.ax_layered(sets[0][0][idx].cpu().numpy(), sets[0][1][idx].cpu().numpy(),
                           basis.diff, basis.diff_t)
        # same-bytes copy: 64 E n^3 B moved = 32 E n^3 B read + written
        words = 4 * E * n ** 3
        bufs = [(torch.empty(words, dtype=torch.float64, device="cuda"),
                 torch.empty(words, dtype=torch.float64, device="cuda")) for _ in range(nsets)]
        def copy_call(b):
            def c():
                h = dv.stream_handle()
                rc = lib.sem_stream_copy(dv.ptr(b[1]), dv.ptr(b[0]), words, h)
                assert rc == 0
            return c
        us_copy = graph_time([copy_call(b) for b in bufs], args.reps)
        us_tcopy = graph_time([(lambda b=b: b[1].copy_(b[0])) for b in bufs], args.reps)
        print(json.dumps({"n": n, "E": E, "what": "sem_stream_copy", "us": round(us_copy, 2),
                          "frac": round(nbytes / (us_copy * 1e3) / hbm, 4)}), flush=True)
        print(json.dumps({"n": n, "E": E, "what": "torch copy_", "us": round(us_tcopy, 2),
                          "frac": round(nbytes / (us_tcopy * 1e3) / hbm, 4)}), flush=True)
        del bufs
        for v in [int(x) for x in args.variants.split(",")]:
            try:
                us = graph_time([(lambda s=s: apply_ax_into(s[0], s[1], basis, s[2], v))
                                 for s in sets], args.reps)
            except Exception as exc:  # noqa: BLE001
                print(json.dumps({"n": n, "E": E, "variant": v, "error": str(exc)}), flush=True)
                continue
            u, g, w = sets[0]
            apply_ax_into(u, g, basis, w, v)
            err = O.rel_diff(w[idx].cpu().numpy(), ref)
            print(json.dumps({"n": n, "E": E, "variant": v, "us": round(us, 2),
                              "frac": round(nbytes / (us * 1e3) / hbm, 4),
                              "fallbacks": int(lib.sem_fallback_count()),
                              "rel_err": err}), flush=True)
        del sets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
