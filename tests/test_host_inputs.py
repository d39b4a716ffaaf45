"""CPU tests of the product package's host-side logic: input builders are
bit-identical to the reference (golden fixtures), cost-model anchors of
sembench/verify.py:519-547, and the reference's validation/error behaviour.
None of these launch a kernel."""

import numpy as np
import pytest

import paper_2005_13425_b200 as sb
from paper_2005_13425_b200 import perf
from paper_2005_13425_b200.kernels import KernelVariant


@pytest.mark.parametrize("n", range(2, 17))
def test_basis_bitexact_vs_reference(golden, n):
    b = sb.build_basis(n)
    for name in ("nodes", "weights", "diff", "diff_t"):
        assert np.array_equal(getattr(b, name), golden[f"basis/{n}/{name}"]), name
        assert not getattr(b, name).flags.writeable


def test_basis_rejects_bad_n():
    for bad in (1, 0, -3, 17, 2.0):
        with pytest.raises(ValueError):
            sb.build_basis(bad)


def test_basis_frozen_values():
    # sembench/verify.py:114-124
    b2 = sb.build_basis(2)
    assert np.array_equal(b2.nodes, [-1.0, 1.0]) and np.array_equal(b2.weights, [1.0, 1.0])
    b3 = sb.build_basis(3)
    assert np.max(np.abs(b3.weights - [1 / 3, 4 / 3, 1 / 3])) <= 1e-14
    b4 = sb.build_basis(4)
    assert np.max(np.abs(b4.nodes[1:3] - np.array([-1, 1]) / np.sqrt(5.0))) <= 1e-14


def test_mix64_and_factor(golden):
    for (a, b), v in zip(golden["mix64/args"], golden["mix64/values"]):
        assert sb.mix64(int(a), int(b)) == int(v)
    for c, box in zip(golden["factor/counts"], golden["factor/boxes"]):
        assert sb.factor_elements(int(c)) == tuple(int(v) for v in box)
    with pytest.raises(ValueError):
        sb.factor_elements(0)


@pytest.mark.parametrize("key", ["1x1x1n3", "2x2x2n4", "3x2x2n5", "2x3x2n6"])
def test_topology_host_arrays(golden, key):
    dims, n = key.split("n")
    ex, ey, ez = (int(v) for v in dims.split("x"))
    topo = sb.build_topology(sb.build_mesh(ex, ey, ez, int(n), 1.0))
    base = f"dssum/{key}"
    assert np.array_equal(topo.global_id, golden[base + "/gid"])
    assert np.array_equal(topo.multiplicity, golden[base + "/mult"])
    assert np.array_equal(topo.mask, golden[base + "/bcmask"])
    assert topo.num_global == int(golden[base + "/gid"].max()) + 1
    assert abs(np.sum(1.0 / topo.multiplicity) - topo.num_global) <= 1e-9


def test_mesh_arithmetic_and_errors():
    m = sb.build_mesh(16, 16, 16, 10, 0.25)
    assert m.num_elements == 4096 and m.dofs == 4_096_000
    for bad in ((0, 1, 1, 3, 1.0), (1, -1, 1, 3, 1.0), (1, 1, 1, 3, 0.0), (1, 1, 1, 1, 1.0)):
        with pytest.raises(ValueError):
            sb.build_mesh(*bad)


def test_cost_model_anchors():
    # sembench/verify.py:519-537 and kernels.py:121-125
    assert sb.flops_per_apply(1, 10) == 135
    assert sb.flops_per_apply(64000, 10) == 8_640_000
    assert perf.model_flops_per_iteration(1, 10) == 154
    assert perf.model_flops_per_iteration(4_096_000, 10) == 630_784_000
    assert perf.model_flops_per_iteration(1, 0) == 34
    assert perf.model_bytes_per_iteration(64000) == 15_360_000
    assert perf.model_read_bytes_per_iteration(1) == 192
    assert perf.model_write_bytes_per_iteration(1) == 48
    assert perf.intensity(10) == 154 / 240
    assert perf.roofline_peak(720e9, 10) == 462.0e9
    assert perf.roofline_peak(900e9, 10) == 577.5e9
    res = perf.evaluate_roofline(462, 1.0, 720.0, 10)
    assert res.fraction == 1.0 and res.flags == ()
    assert "cache-effect" in perf.evaluate_roofline(1000, 1.0, 720.0, 10).flags
    payload, counted = perf.probe_byte_accounting(64000)
    assert payload == 15_360_000 and counted == 30_720_000


def test_variant_parse_and_counters():
    assert KernelVariant.parse("LAYERED") is KernelVariant.LAYERED
    with pytest.raises(ValueError):
        KernelVariant.parse("fastest")
    assert sb.apply_read_words(KernelVariant.REFERENCE, 10) == 130
    assert sb.apply_write_words(KernelVariant.SCRATCH, 10) == 10
    c = sb.TrafficCounters()
    c.add(reads=1, writes=2, flops=3)
    assert (c.reads, c.writes, c.flops) == (1, 2, 3)
    with pytest.raises(ValueError):
        c.add(reads=-1)


def test_apply_ax_validates_before_launch():
    # shape errors surface as ValueError (kernels.py:433-436) without a GPU
    basis = sb.build_basis(4)
    geom = sb.GeomFactors(values=np.zeros((2, 6, 4, 4, 4)))
    with pytest.raises(ValueError):
        sb.apply_ax(np.zeros((2, 4, 4, 5)), geom, basis)
    with pytest.raises(ValueError):
        sb.apply_ax(np.zeros((3, 4, 4, 4)), geom, basis)
    with pytest.raises(ValueError):
        sb.apply_ax(np.zeros((2, 4, 4, 4)), geom, basis, "bogus")
    big = sb.build_basis(11)
    g11 = sb.GeomFactors(values=np.zeros((1, 6, 11, 11, 11)))
    with pytest.raises(sb.ScratchCapacityError):
        sb.apply_ax(np.zeros((1, 11, 11, 11)), g11, big, "scratch")


def test_cg_config_errors():
    with pytest.raises(ValueError):
        sb.CgConfig(0, 0.0)
    with pytest.raises(ValueError):
        sb.CgConfig(10, -1.0)
