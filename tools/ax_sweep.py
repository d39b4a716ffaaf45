#!/usr/bin/env python
"""Tuning sweep: time every sem_ax variant for a set of n / E (CUDA events,
two rotating input sets larger than L2), check each against the oracle on a
few elements, print one JSON line per (n, E, variant)."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200._lib import load  # noqa: E402
from paper_2005_13425_b200.kernels import apply_ax_into  # noqa: E402
from paper_2005_13425_b200.perf import measured_peaks  # noqa: E402


def time_variant(sets, basis, variant, reps):
    """Launches captured in a CUDA graph so small-n timings are not bound by
    the Python launch path."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            u, g, w = sets[i % len(sets)]
            apply_ax_into(u, g, basis, w, variant)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(reps):
            u, g, w = sets[i % len(sets)]
            apply_ax_into(u, g, basis, w, variant)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def time_copy(nbytes, nsets, reps):
    """Same-bytes reference: sem_stream_copy of nbytes/2 read + nbytes/2
    written per launch, rotating over nsets buffer pairs, graph-timed like
    the Ax launches (the size-matched copy roofline: L2-resident and
    launch-bound regimes included)."""
    lib = load()
    half = nbytes // 2 // 8
    bufs = [(torch.empty(half, dtype=torch.float64, device="cuda").fill_(1.0),
             torch.empty(half, dtype=torch.float64, device="cuda")) for _ in range(nsets)]

    def run(i):
        src, dst = bufs[i % nsets]
        rc = lib.sem_stream_copy(dst.data_ptr(), src.data_ptr(), half,
                                 torch.cuda.current_stream().cuda_stream)
        assert rc == 0
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3):
            run(i)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(reps):
            run(i)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", default="10")
    ap.add_argument("--E", default="4096")
    ap.add_argument("--variants", default="all")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--copy", action="store_true", help="also time a same-bytes copy")
    ap.add_argument("--repeat", type=int, default=1, help="timings per variant (best kept)")
    ap.add_argument("--cool", type=float, default=0.0,
                    help="seconds idle before each timing (back-to-back timings soak the "
                         "1000 W power cap and bias a sweep toward the variants timed first)")
    args = ap.parse_args()
    hbm = float(measured_peaks(ROOT)["hbm_gbs"])
    lib = load()
    for n in [int(x) for x in args.n.split(",")]:
        basis = sb.build_basis(n)
        nv = lib.sem_ax_num_variants(n)
        variants = range(nv) if args.variants == "all" else [int(v) for v in args.variants.split(",")]
        for E in [int(x) for x in args.E.split(",")]:
            per_set = E * n ** 3 * 64
            nsets = max(2, int(np.ceil(3 * 126e6 / per_set)))
            nsets = min(nsets, 8)
            sets = []
            for s in range(nsets):
                u = sb.random_field(E, n, 1 + s, device="cuda")
                g = sb.random_field(6 * E, n, 100 + s, device="cuda").reshape(E, 6, n, n, n)
                sets.append((u, g, torch.empty_like(u)))
            idx = sorted({0, 1, E // 2, E - 1})
            ref = O.ax_layered(sets[0][0][idx].cpu().numpy(), sets[0][1][idx].cpu().numpy(),
                               basis.diff, basis.diff_t)
            for v in variants:
                try:
                    ts = []
                    for _ in range(args.repeat):
                        if args.cool > 0:
                            time.sleep(args.cool)
                        ts.append(time_variant(sets, basis, v, args.reps))
                    ms = min(ts)
                except Exception as exc:  # noqa: BLE001
                    print(json.dumps({"n": n, "E": E, "variant": v, "error": str(exc)}))
                    continue
                u, g, w = sets[0]
                apply_ax_into(u, g, basis, w, v)
                err = O.rel_diff(w[idx].cpu().numpy(), ref)
                gbs = E * n ** 3 * 64 / (ms * 1e-3) / 1e9
                print(json.dumps({"n": n, "E": E, "variant": v, "us": round(ms * 1e3, 2),
                                  "gflops": round(E * n ** 3 * (12 * n + 15) / (ms * 1e-3) / 1e9, 1),
                                  "gbs": round(gbs, 1), "frac": round(gbs / hbm, 4),
                                  "rel_err": err}), flush=True)
            if args.copy:
                cms = min(time_copy(per_set, nsets, args.reps) for _ in range(args.repeat))
                cgbs = per_set / (cms * 1e-3) / 1e9
                print(json.dumps({"n": n, "E": E, "what": "same-bytes copy", "us": round(cms * 1e3, 2),
                                  "gbs": round(cgbs, 1), "frac": round(cgbs / hbm, 4),
                                  "sets": nsets}), flush=True)
            del sets
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
