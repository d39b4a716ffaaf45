"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container, where the reference package is importable:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``sembench`` from /root/reference/pkg/src (read-only; numba needs
a writable cache dir) and records outputs of the reference's own public API
on seeded inputs.  The fixtures pin both the CPU oracle (oracle/) and the
host-side input builders of the product package; the GPU box never sees
/root/reference, only these committed .npz files.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("SEMBENCH_SRC", "/root/reference/pkg/src")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# (E-box, n, seed_u, seed_g) for Ax with a RANDOM metric (all six components
# independent, so the off-diagonal g2/g3/g5 wiring is pinned -- the reference's
# own suite only exercises the diagonal build_geom metric).
AX_CASES = [
    ((1, 1, 1), 2, 11, 12),
    ((2, 2, 2), 3, 13, 14),
    ((2, 2, 2), 4, 15, 16),
    ((2, 2, 1), 5, 17, 18),
    ((2, 1, 1), 7, 19, 20),
    ((2, 2, 2), 10, 21, 22),
    ((3, 1, 1), 9, 23, 24),
    ((1, 1, 1), 16, 25, 26),
]
DSSUM_CASES = [((1, 1, 1), 3), ((2, 1, 1), 2), ((2, 2, 2), 4), ((3, 2, 2), 5),
               ((3, 3, 3), 3), ((2, 3, 2), 6)]
CG_CASES = [((2, 2, 2), 6, 50), ((4, 4, 4), 10, 100), ((3, 2, 2), 4, 30)]
FACTOR_COUNTS = [1, 7, 12, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768,
                 65536, 131072, 262144]


def main() -> int:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF_SRC)
    import sembench as sb
    from sembench import verify

    d: dict[str, np.ndarray] = {}

    for n in range(2, 17):
        b = sb.build_basis(n)
        d[f"basis/{n}/nodes"] = np.array(b.nodes)
        d[f"basis/{n}/weights"] = np.array(b.weights)
        d[f"basis/{n}/diff"] = np.array(b.diff)
        d[f"basis/{n}/diff_t"] = np.array(b.diff_t)

    seeds = [0, 1, 2, 12345, sb.fields.mix64(1, 4096)]
    d["random/seeds"] = np.array(seeds, dtype=np.uint64)
    for s in seeds:
        d[f"random/{s}"] = sb.random_field(2, 5, s).ravel()[:250]
    mix_args = [(1, 64), (1, 4096), (3, 7), (0, 0), (1, 32768)]
    d["mix64/args"] = np.array(mix_args, dtype=np.int64)
    d["mix64/values"] = np.array([sb.fields.mix64(a, b) for a, b in mix_args], dtype=np.uint64)

    for dims, n, su, sg in AX_CASES:
        E = dims[0] * dims[1] * dims[2]
        basis = sb.build_basis(n)
        u = sb.random_field(E, n, su)
        g = sb.random_field(6 * E, n, sg).reshape(E, 6, n, n, n)
        geom = sb.GeomFactors(values=g)
        key = f"ax/{E}x{n}"
        d[key + "/meta"] = np.array([E, n, su, sg], dtype=np.int64)
        d[key + "/layered"] = sb.apply_ax(u, geom, basis, "layered")
        ws = sb.reference_workspace(E, n)
        d[key + "/reference"] = sb.apply_ax(u, geom, basis, "reference", workspace=ws)
        # the REFERENCE variant leaves the metric-scaled gradients in its workspace
        for name, a in zip(("ur", "us", "ut"), ws):
            d[key + "/reference_ws_" + name] = np.array(a)
        if n <= sb.kernels.SCRATCH_MAX_POINTS:
            d[key + "/scratch"] = sb.apply_ax(u, geom, basis, "scratch")
        if n <= 5:
            d[key + "/dense"] = verify.apply_dense(basis, geom, u)

    # box geometry (the benchmark's diagonal metric)
    basis = sb.build_basis(10)
    mesh = sb.build_mesh(2, 2, 1, 10, 0.5)
    geom = sb.build_geom(mesh, basis)
    d["geom/2x2x1n10h0.5"] = np.array(geom.values)
    u = sb.random_field(mesh.num_elements, 10, 5)
    d["ax_box/2x2x1n10"] = sb.apply_ax(u, geom, basis, "layered")

    for dims, n in DSSUM_CASES:
        basis, mesh, geom, topo = verify._setup(*dims, n)
        E = mesh.num_elements
        f = sb.random_field(E, n, 100 + n)
        key = f"dssum/{dims[0]}x{dims[1]}x{dims[2]}n{n}"
        d[key + "/out"] = sb.dssum(f, topo)
        d[key + "/mask"] = sb.mask(f, topo)
        d[key + "/gid"] = np.array(topo.global_id)
        d[key + "/mult"] = np.array(topo.multiplicity)
        d[key + "/bcmask"] = np.array(topo.mask)
        v = sb.random_field(E, n, 200 + n)
        d[key + "/wdot"] = np.array([sb.weighted_dot(f, v, topo), sb.weighted_dot(f, f, topo)])
        d[key + "/global"] = sb.apply_global(verify.consistent_random_field(E, n, topo, 7),
                                             geom, basis, topo)

    for dims, n, iters in CG_CASES:
        E = dims[0] * dims[1] * dims[2]
        basis = sb.build_basis(n)
        mesh = sb.build_mesh(*dims, n, 1.0)
        geom = sb.build_geom(mesh, basis)
        topo = sb.build_topology(mesh)
        f = sb.make_rhs(E, n, topo, sb.fields.mix64(1, E))

        def op(v, geom=geom, basis=basis, topo=topo):
            return sb.apply_global(v, geom, basis, topo)

        res = sb.cg_solve(f, op, topo, sb.CgConfig(iters, 0.0))
        key = f"cg/{dims[0]}x{dims[1]}x{dims[2]}n{n}"
        # the reference's OWN sensitivity to reassociation: LAYERED vs
        # REFERENCE-variant Ax inside the same CG (bounds any faithful port)
        alt = sb.cg_solve(f, lambda v, geom=geom, basis=basis, topo=topo:
                          sb.apply_global(v, geom, basis, topo, "reference"),
                          topo, sb.CgConfig(iters, 0.0))
        h0, h1 = res.residual_history, alt.residual_history
        d[key + "/variant_spread"] = np.array([np.max(np.abs(h1 - h0) / np.abs(h0))])
        d[key + "/meta"] = np.array([dims[0], dims[1], dims[2], n, iters], dtype=np.int64)
        d[key + "/history"] = res.residual_history
        if E * n ** 3 <= 20000:
            d[key + "/solution"] = res.solution
        d[key + "/solution_norm"] = np.array([np.linalg.norm(res.solution)])

    d["factor/counts"] = np.array(FACTOR_COUNTS, dtype=np.int64)
    d["factor/boxes"] = np.array([sb.factor_elements(c) for c in FACTOR_COUNTS], dtype=np.int64)

    # report serialisations emitted by the reference (sembench-1 schema)
    from sembench import report as R
    rows = []
    for q, (variant, elements) in enumerate([("reference", 64), ("scratch", 64), ("layered", 64),
                                             ("layered", 4096), ("reference", 4096)]):
        rows.append(R.PerfReport(
            schema_version=R.SCHEMA_VERSION, variant=variant, elements=elements,
            box="4x4x4" if elements == 64 else "16x16x16", n=10, dofs=elements * 1000,
            iterations=100, workers=148, seed=1, include_dssum=(q % 2 == 1),
            total_seconds=0.1 + q / 3.0, seconds_per_iteration=(0.1 + q / 3.0) / 100,
            ax_seconds=1e-3 * (q + 1) / 7.0, dssum_seconds=2.5e-4 / (q + 3),
            model_flops_per_iteration=elements * 1000 * 154,
            model_bytes_per_iteration=elements * 1000 * 240,
            model_read_bytes_per_iteration=elements * 1000 * 192,
            model_write_bytes_per_iteration=elements * 1000 * 48,
            instr_flops=elements * 1000 * 147 * 100, instr_read_words=elements * 1000 * 36 * 100,
            instr_write_words=elements * 1000 * 8 * 100, achieved_gflops=5303.914826095655 / (q + 1),
            measured_bandwidth=6.0931e12 + q, roofline_peak_gflops=3909.8 + q / 10.0,
            roofline_fraction=1.2616330551493 / (q + 1),
            flags="" if q < 2 else ("probe-under-llc" if q < 4 else "probe-under-llc;cache-effect")))
    # deterministic integer fields of the reference's own benchmark rows
    # (traffic / flop inventory of a 10-iteration solve, every variant)
    sb.set_workers(2)
    bench_rows = sb.run_bench(sb.BenchConfig(elements=64, iterations=10, variant="all",
                                             probe_repetitions=10))
    int_fields = ["elements", "n", "dofs", "iterations", "seed", "model_flops_per_iteration",
                  "model_bytes_per_iteration", "model_read_bytes_per_iteration",
                  "model_write_bytes_per_iteration", "instr_flops", "instr_read_words",
                  "instr_write_words"]
    d["bench64/int_fields"] = np.frombuffer(",".join(int_fields).encode(), dtype=np.uint8)
    d["bench64/variants"] = np.frombuffer(",".join(r.variant for r in bench_rows).encode(),
                                          dtype=np.uint8)
    d["bench64/values"] = np.array([[getattr(r, k) for k in int_fields] for r in bench_rows],
                                   dtype=np.int64)
    d["bench64/roofline_keys"] = np.frombuffer(
        ",".join(sb.run_roofline(sb.BenchConfig(elements=64)).keys()).encode(), dtype=np.uint8)
    for fmt, text in (("csv", R.emit_csv(rows)), ("json", R.emit_json(rows)),
                      ("gnuplot", R.emit_gnuplot(rows))):
        d[f"report/{fmt}"] = np.frombuffer(text.encode(), dtype=np.uint8)

    np.savez_compressed(OUT, **d)
    print(f"wrote {OUT}: {len(d)} arrays, {os.path.getsize(OUT)} bytes")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
