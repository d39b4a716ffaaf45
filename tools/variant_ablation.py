"""Paper Figs. 2-3 on B200: the three storage strategies (REFERENCE,
SCRATCH, LAYERED) as GPU kernels.

1. Ax-only at E=4096 for p = 3..9 (n <= 10, SCRATCH's capacity): device time
   per apply (CUDA events, mean of 50 applies over two rotating input sets
   larger than L2), GFLOP/s, and HBM GB/s against each variant's OWN
   algorithmic traffic (REFERENCE 160 B/point, the others 64 B/point).
2. The reference protocol (harness.run_sweep, variant="all", 100 CG
   iterations) over the default sweep 64..4096, emitted as sembench-1 CSV and
   gnuplot next to each other under the output directory.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2005_13425_b200 as sb  # noqa: E402
from paper_2005_13425_b200 import perf  # noqa: E402


def ax_only(n, E=4096, reps=50):
    dev = torch.device("cuda", 0)
    b = sb.build_basis(n)
    sets = []
    for s in range(2):
        u = sb.random_field(E, n, 1 + s, device=dev)
        g = sb.random_field(6 * E, n, 3 + s, device=dev).reshape(E, 6, n, n, n)
        sets.append((u, sb.GeomFactors(values=g)))
    ws = sb.reference_workspace(E, n, device=dev)
    out = {}
    for v in ("reference", "scratch", "layered"):
        kw = {"workspace": ws} if v == "reference" else {}
        for i in range(3):
            sb.apply_ax(sets[i % 2][0], sets[i % 2][1], b, v, **kw)
        torch.cuda.synchronize()
        # one apply per input set captured in a CUDA graph, replayed: device
        # time without the Python call overhead (~25 us per apply_ax call)
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side), torch.cuda.graph(graph, stream=side):
            for i in range(2):
                sb.apply_ax(sets[i][0], sets[i][1], b, v, **kw)
        torch.cuda.current_stream().wait_stream(side)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps // 2):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / (2 * (reps // 2)) * 1e-3
        dofs = E * n ** 3
        words = sb.apply_read_words(sb.KernelVariant(v), dofs) + \
            sb.apply_write_words(sb.KernelVariant(v), dofs)
        out[v] = {"us": t * 1e6, "gflops": sb.flops_per_apply(dofs, n) / t / 1e9,
                  "hbm_gbs_own_traffic": 8 * words / t / 1e9}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out")
    ap.add_argument("--iterations", type=int, default=100)
    args = ap.parse_args()
    os.makedirs(args.out, exist_ok=True)
    res = {"ax_only_E4096": {f"n{n}": ax_only(n) for n in range(4, 11)},
           "peak_hbm_gbs": perf.measured_peaks()["hbm_gbs"]}
    rows = sb.run_sweep(sb.BenchConfig(iterations=args.iterations, variant="all"))
    with open(os.path.join(args.out, "variants_sweep.csv"), "w") as fh:
        fh.write(sb.emit_csv(rows))
    with open(os.path.join(args.out, "variants_sweep.gnuplot"), "w") as fh:
        fh.write(sb.emit_gnuplot(rows))
    res["cg_sweep"] = [{"variant": r.variant, "elements": r.elements,
                        "ms_per_iteration": r.seconds_per_iteration * 1e3,
                        "achieved_gflops": r.achieved_gflops,
                        "roofline_fraction": r.roofline_fraction,
                        "measured_bandwidth_gbs": r.measured_bandwidth / 1e9,
                        "ax_ms": r.ax_seconds * 1e3, "dssum_ms": r.dssum_seconds * 1e3,
                        "flags": r.flags} for r in rows]
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
