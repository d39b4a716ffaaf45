"""Seeded random sweep over box shapes and degrees (the edge cases a fixed
list misses: one-element-thick boxes, odd point counts, n = 2 and 16, E
not a multiple of any tile): Ax, dssum + mask, apply_global and a short
fused CG through the public API vs the CPU oracle, at the module's bars."""

import numpy as np
import pytest

import oracle as O
import paper_2005_13425_b200 as sb

pytestmark = pytest.mark.gpu

_rng = np.random.default_rng(20261017)
CASES = []
for _ in range(24):
    n = int(_rng.integers(2, 17))
    box = tuple(int(v) for v in _rng.integers(1, 6, size=3))
    if box[0] * box[1] * box[2] * n ** 3 > 600_000:  # keep the oracle CG fast
        box = (box[0], box[1], 1)
    CASES.append((box, n))


@pytest.mark.parametrize("box,n", CASES, ids=[f"{b[0]}x{b[1]}x{b[2]}n{n}" for b, n in CASES])
def test_random_box(cuda, box, n):
    ex, ey, ez = box
    E = ex * ey * ez
    b = sb.build_basis(n)
    mesh = sb.build_mesh(ex, ey, ez, n, 1.0)
    topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b)
    T = O.BoxTopology(ex, ey, ez, n)
    seed = 1000 * E + n
    u = O.random_field(E, n, seed)
    g = O.random_field(6 * E, n, seed + 1).reshape(E, 6, n, n, n)
    # Ax on a random metric (numpy in -> numpy out through the host path)
    w = sb.apply_ax(u, sb.GeomFactors(values=g), b)
    assert O.rel_diff(np.asarray(w), O.ax_layered(u, g, b.diff, b.diff_t)) <= 1e-12
    # assembly: bit-exact
    assert np.array_equal(np.asarray(sb.dssum(u, topo)), O.dssum(u, T))
    assert np.array_equal(np.asarray(sb.mask(u, topo)), O.mask(u, T))
    # the global operator on the box geometry
    gb = O.box_geom(ex, ey, ez, b.weights, 1.0)
    got = np.asarray(sb.apply_global(u, geom, b, topo))
    assert O.rel_diff(got, O.apply_global(u, gb, b.diff, b.diff_t, T)) <= 1e-12
    # a short fused CG
    f = sb.make_rhs(E, n, topo, sb.mix64(1, E))
    res = sb.cg_solve(f, sb.GlobalOperator(geom, b, topo), topo, sb.CgConfig(12, 0.0))
    _, hist, it_ref = O.cg(np.asarray(f), lambda p: O.apply_global(p, gb, b.diff, b.diff_t, T), T, 12)
    hr = np.asarray(hist)
    assert res.iterations_run == it_ref
    if hr.size and hr[0] > 0:
        sig = hr > 1e-12 * hr[0]
        h = np.asarray(res.residual_history)
        assert float(np.max(np.abs(h[sig] - hr[sig]) / hr[sig])) <= 1e-10
