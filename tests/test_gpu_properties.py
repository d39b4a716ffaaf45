"""The reference's own property suite (sembench/verify.py:229-511), restated
against the GPU path: every Ax variant, the fused and the generic CG, the
assembly kernels.  These complement the oracle / golden parity tests with
the mathematical invariants the reference checks on itself."""

import numpy as np
import pytest
import torch

import oracle as O
import paper_2005_13425_b200 as sb

pytestmark = pytest.mark.gpu

VARIANTS = ("reference", "scratch", "layered")


def _box(ex, ey, ez, n):
    b = sb.build_basis(n)
    mesh = sb.build_mesh(ex, ey, ez, n, 1.0)
    return b, mesh, sb.build_geom(mesh, b), sb.build_topology(mesh)


def _consistent(E, n, topo, seed):
    """Masked, interface-consistent random field (verify.py:91-98)."""
    return sb.mask(sb.dssum(sb.random_field(E, n, seed), topo), topo)


def _host(t):
    return t.cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)


@pytest.mark.parametrize("variant", VARIANTS)
def test_ax_null_space_linearity_symmetry(cuda, variant):
    """Constants are in the null space; A_local is linear, symmetric and PSD
    (verify.py:229-235, 270-293)."""
    b, mesh, geom, _ = _box(2, 2, 2, 5)
    E = mesh.num_elements
    c = sb.apply_ax(sb.constant_field(E, 5, 2.5), geom, b, variant)
    op_scale = (5 * np.max(np.abs(b.diff))) ** 2 * float(geom.values.max())
    assert float(np.abs(_host(c)).max()) <= 1e-12 * 2.5 * op_scale
    u, v = _host(sb.random_field(E, 5, 11)), _host(sb.random_field(E, 5, 12))
    au, av = _host(sb.apply_ax(u, geom, b, variant)), _host(sb.apply_ax(v, geom, b, variant))
    lin = _host(sb.apply_ax(1.5 * u - 0.25 * v, geom, b, variant))
    assert O.rel_diff(lin, 1.5 * au - 0.25 * av) <= 1e-12
    nu, nv = np.linalg.norm(u), np.linalg.norm(v)
    scale = max(np.linalg.norm(au) / nu, np.linalg.norm(av) / nv)
    assert abs(np.vdot(v, au) - np.vdot(u, av)) <= 1e-12 * nu * nv * scale
    assert np.vdot(u, au) >= -1e-12 * nu * nu * scale


def test_variants_agree_seeds(cuda):
    """Cross-variant equivalence at n = 10, E = 64 over 20 seeds (
    verify.py:250-258 uses 3)."""
    b = sb.build_basis(10)
    g = sb.GeomFactors(values=sb.random_field(6 * 64, 10, 999).reshape(64, 6, 10, 10, 10))
    for seed in range(20):
        u = sb.random_field(64, 10, seed)
        outs = [_host(sb.apply_ax(u, g, b, v)) for v in VARIANTS]
        assert O.rel_diff(outs[0], outs[2]) <= 1e-12 and O.rel_diff(outs[1], outs[2]) <= 1e-12


def test_dssum_identity_linearity_conservation(cuda):
    """verify.py:362-380: identity on one element; exact linearity on
    integer-valued fields; sum(dssum(f)/mult) == sum(f)."""
    _, _, _, t1 = _box(1, 1, 1, 3)
    f = _host(sb.random_field(1, 3, 5))
    assert np.array_equal(_host(sb.dssum(f, t1)), f)
    _, _, _, t2 = _box(2, 1, 1, 2)
    a = np.floor(5 * _host(sb.random_field(2, 2, 1)))
    c = np.floor(5 * _host(sb.random_field(2, 2, 2)))
    assert np.array_equal(_host(sb.dssum(2.0 * a + 3.0 * c, t2)),
                          2.0 * _host(sb.dssum(a, t2)) + 3.0 * _host(sb.dssum(c, t2)))
    _, mesh, _, t3 = _box(3, 2, 2, 4)
    f = _host(sb.random_field(mesh.num_elements, 4, 9))
    after = float(np.sum(_host(sb.dssum(f, t3)) / t3.multiplicity))
    assert abs(after - float(np.sum(f))) <= 1e-12 * max(1.0, abs(float(np.sum(f))))


def test_mask_and_boundary_null(cuda):
    """verify.py:383-416: one interior node on a 1x1x1 n=3 box; mask is
    idempotent; the global operator annihilates boundary-only fields."""
    _, _, _, t1 = _box(1, 1, 1, 3)
    m = _host(sb.mask(sb.constant_field(1, 3, 1.0), t1))
    assert np.count_nonzero(m) == 1 and m[0, 1, 1, 1] == 1.0
    assert np.array_equal(_host(sb.mask(m, t1)), m)
    b, mesh, geom, topo = _box(2, 2, 2, 3)
    bnd = _host(sb.random_field(mesh.num_elements, 3, 31)) * (1.0 - topo.mask)
    for variant in VARIANTS:
        out = _host(sb.apply_global(bnd, geom, b, topo, variant))
        assert np.array_equal(out, np.zeros_like(out))


@pytest.mark.parametrize("variant", VARIANTS)
def test_global_symmetry_psd(cuda, variant):
    """<v, A u>_c == <u, A v>_c and <u, A u>_c > 0 on consistent fields (verify.py:393-404)."""
    b, mesh, geom, topo = _box(2, 2, 2, 4)
    u, v = _consistent(mesh.num_elements, 4, topo, 21), _consistent(mesh.num_elements, 4, topo, 22)
    au, av = sb.apply_global(u, geom, b, topo, variant), sb.apply_global(v, geom, b, topo, variant)
    vau, uav = sb.weighted_dot(v, au, topo), sb.weighted_dot(u, av, topo)
    assert abs(vau - uav) <= 1e-12 * max(abs(vau), abs(uav), 1e-30)
    assert sb.weighted_dot(u, au, topo) > 0.0


def test_weighted_dot_anchors(cuda):
    """verify.py:424-437: all-ones on a 2x1x1 n=2 box is exactly 12."""
    _, _, _, t = _box(2, 1, 1, 2)
    assert sb.weighted_dot(sb.constant_field(2, 2, 1.0), sb.constant_field(2, 2, 1.0), t) == 12.0
    assert sb.weighted_dot(sb.constant_field(2, 2, 0.0), sb.constant_field(2, 2, 0.0), t) == 0.0
    w = sb.random_field(2, 2, 3)
    assert sb.weighted_dot(w, w, t) > 0.0


@pytest.mark.parametrize("fused", [True, False])
def test_cg_fixed_protocol_and_scaling(cuda, fused):
    """verify.py:493-511: exactly 100 operator applications and iterations
    with tolerance 0; the solution scales with the right-hand side."""
    b, mesh, geom, topo = _box(2, 2, 2, 3)
    timers = sb.OperatorTimers()
    op = sb.GlobalOperator(geom, b, topo, timers=timers) if fused else \
        (lambda x: sb.apply_global(x, geom, b, topo, timers=timers))
    f = _consistent(mesh.num_elements, 3, topo, 6)
    res = sb.cg_solve(f, op, topo, sb.CgConfig(100, 0.0))
    assert timers.applies == 100 and res.iterations_run == 100
    assert res.residual_history.shape == (100,)
    f2 = _consistent(mesh.num_elements, 3, topo, 15)
    base = sb.cg_solve(f2, op, topo, sb.CgConfig(20, 0.0))
    scaled = sb.cg_solve(3.5 * f2, op, topo, sb.CgConfig(20, 0.0))
    assert scaled.iterations_run == base.iterations_run
    assert O.rel_diff(_host(scaled.solution), 3.5 * _host(base.solution)) <= 1e-12
