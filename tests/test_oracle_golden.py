"""Pin the CPU oracle against fixtures produced by the reference itself.

tests/golden/golden.npz was written by tests/golden/make_golden.py, which
imports the reference package (sembench) and records its outputs on seeded
inputs.  Every oracle routine must reproduce them BIT-FOR-BIT (the oracle
keeps the reference's operation order), which is what licenses using the
oracle as the parity checker for the CUDA path.
"""

import numpy as np
import pytest

import oracle as O


def _box_from_key(key):
    dims, n = key.split("n")
    a, b, c = (int(v) for v in dims.split("x"))
    return a, b, c, int(n)


def test_random_field_and_mix64(golden):
    for s in golden["random/seeds"]:
        s = int(s)
        got = O.random_field(2, 5, s).ravel()[:250]
        assert np.array_equal(got, golden[f"random/{s}"])
    for (a, b), v in zip(golden["mix64/args"], golden["mix64/values"]):
        assert O.mix64(int(a), int(b)) == int(v)


@pytest.mark.parametrize("key", ["1x2", "8x3", "8x4", "4x5", "2x7", "8x10", "3x9", "1x16"])
def test_ax_layered_bitexact(golden, key):
    E, n, su, sg = (int(v) for v in golden[f"ax/{key}/meta"])
    u = O.random_field(E, n, su)
    g = O.random_field(6 * E, n, sg).reshape(E, 6, n, n, n)
    w = O.ax_layered(u, g, golden[f"basis/{n}/diff"], golden[f"basis/{n}/diff_t"])
    assert np.array_equal(w, golden[f"ax/{key}/layered"])
    # and the reference's own REFERENCE variant agrees to reassociation
    assert O.rel_diff(w, golden[f"ax/{key}/reference"]) <= 1e-14
    if n <= 5:
        # independent dense Kronecker oracle (verify.py:45-77)
        dense = O.dense_apply(u, g, golden[f"basis/{n}/diff"])
        assert O.rel_diff(dense, golden[f"ax/{key}/dense"]) <= 1e-14
        assert O.rel_diff(w, dense) <= 1e-12


@pytest.mark.parametrize("key", ["1x2", "8x3", "8x4", "4x5", "2x7", "8x10", "3x9", "1x16"])
def test_ax_reference_scratch_bitexact(golden, key):
    """REFERENCE (kernels.py:159-205, including the intermediates it leaves in
    its workspace) and SCRATCH (:213-259) restatements, bit-for-bit."""
    E, n, su, sg = (int(v) for v in golden[f"ax/{key}/meta"])
    u = O.random_field(E, n, su)
    g = O.random_field(6 * E, n, sg).reshape(E, 6, n, n, n)
    dx, dxt = golden[f"basis/{n}/diff"], golden[f"basis/{n}/diff_t"]
    w, ur, us, ut = O.ax_reference(u, g, dx, dxt)
    assert np.array_equal(w, golden[f"ax/{key}/reference"])
    for name, a in (("ur", ur), ("us", us), ("ut", ut)):
        assert np.array_equal(a, golden[f"ax/{key}/reference_ws_{name}"])
    if n <= 10:
        assert np.array_equal(O.ax_scratch(u, g, dx), golden[f"ax/{key}/scratch"])


def test_ax_box_geometry(golden):
    w = golden["basis/10/weights"]
    g = O.box_geom(2, 2, 1, w, 0.5)
    assert np.array_equal(g, golden["geom/2x2x1n10h0.5"])
    u = O.random_field(4, 10, 5)
    out = O.ax_layered(u, g, golden["basis/10/diff"], golden["basis/10/diff_t"])
    assert np.array_equal(out, golden["ax_box/2x2x1n10"])


@pytest.mark.parametrize("key", ["1x1x1n3", "2x1x1n2", "2x2x2n4", "3x2x2n5", "3x3x3n3",
                                 "2x3x2n6"])
def test_assembly_bitexact(golden, key):
    ex, ey, ez, n = _box_from_key(key)
    T = O.BoxTopology(ex, ey, ez, n)
    base = f"dssum/{key}"
    assert np.array_equal(T.global_id, golden[base + "/gid"])
    assert np.array_equal(T.multiplicity, golden[base + "/mult"])
    assert np.array_equal(T.mask, golden[base + "/bcmask"])
    E = T.num_elements
    f = O.random_field(E, n, 100 + n)
    assert np.array_equal(O.dssum(f, T), golden[base + "/out"])
    assert np.array_equal(O.mask(f, T), golden[base + "/mask"])
    v = O.random_field(E, n, 200 + n)
    wd = golden[base + "/wdot"]
    assert O.wdot3(f, v, T.inv_multiplicity) == wd[0]
    assert O.wdot3(f, f, T.inv_multiplicity) == wd[1]


def test_factor_elements(golden):
    for c, box in zip(golden["factor/counts"], golden["factor/boxes"]):
        assert tuple(O.factor_elements(int(c))) == tuple(int(v) for v in box)


@pytest.mark.parametrize("key", ["2x2x2n6", "3x2x2n4", "4x4x4n10"])
def test_cg_history_bitexact(golden, key):
    ex, ey, ez, n, iters = (int(v) for v in golden[f"cg/{key}/meta"])
    E = ex * ey * ez
    T = O.BoxTopology(ex, ey, ez, n)
    g = O.box_geom(ex, ey, ez, golden[f"basis/{n}/weights"], 1.0)
    dx, dxt = golden[f"basis/{n}/diff"], golden[f"basis/{n}/diff_t"]
    f = O.mask(O.dssum(O.random_field(E, n, O.mix64(1, E)), T), T)
    x, hist, its = O.cg(f, lambda p: O.apply_global(p, g, dx, dxt, T), T, iters)
    assert its == iters
    assert np.array_equal(hist, golden[f"cg/{key}/history"])
    if f"cg/{key}/solution" in golden.files:
        assert np.array_equal(x, golden[f"cg/{key}/solution"])
