"""The fused CG's launch-structure options agree with each other and with the
CPU oracle (csrc/cg.cu tuning hooks, read once per process, so each mode runs
in its own subprocess):

  * SEM_CG_FIN   0 fused reductions (last-CTA finish), 1 both deferred to a
                 settle block, 2 (default) the <p, A p> reduction deferred;
  * SEM_CG_PDL   0 plain launches, 1 every launch a programmatic dependent,
                 2 (default) the settle and update launches only;
  * SEM_CG_AX_CFG 0 (default, GMODE 4: p / r / x / g bulk-copied before the
                 scalars are read) vs 4 (metric only staged, p / r / x via
                 registers);
  * SEM_CG_UPD_ELEM 1 element-granular update (extended cube in shared
                 memory) vs 0 the row kernel.

Every mode is deterministic run to run; modes with the same reduction trees
(PDL, Ax staging) agree bit-for-bit with the default, and all agree with the
oracle's residual history to the north-star 1e-10.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import paper_2005_13425_b200 as sb
n, (ex, ey, ez) = 10, (6, 5, 4)
b = sb.build_basis(n)
mesh = sb.build_mesh(ex, ey, ez, n, 1.0)
topo, geom = sb.build_topology(mesh), sb.build_geom(mesh, b)
E = mesh.num_elements
f = sb.make_rhs(E, n, topo, sb.mix64(1, E))
op = sb.GlobalOperator(geom, b, topo)
tol = float(os.environ.get("CG_TEST_TOL", "0"))
out = []
for _ in range(2):
    res = sb.cg_solve(f, op, topo, sb.CgConfig(40, tol))
    out.append([float(v) for v in res.residual_history])
x = res.solution
print(json.dumps({{"hist": out, "xsum": float(abs(x).sum()), "iters": int(res.iterations_run)}}))
"""

MODES = {
    "default": {},
    "fin0": {"SEM_CG_FIN": "0"},
    "fin1": {"SEM_CG_FIN": "1"},
    "pdl0": {"SEM_CG_PDL": "0"},
    "pdl1": {"SEM_CG_PDL": "1"},
    "axcfg4": {"SEM_CG_AX_CFG": "4"},
    "updrow": {"SEM_CG_UPD_ELEM": "0"},
    "updelem": {"SEM_CG_UPD_ELEM": "1"},
    "settle0": {"SEM_CG_SETTLE": "0"},
    "settle1": {"SEM_CG_SETTLE": "1"},
    "updfwd": {"SEM_CG_UPD_REV": "0"},
    "noalt": {"SEM_CG_ALT": "0"},
}


def _run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def runs(cuda):
    return {k: _run(v) for k, v in MODES.items()}


@pytest.fixture(scope="module")
def oracle_hist():
    import oracle as O
    import paper_2005_13425_b200 as sb
    n, (ex, ey, ez) = 10, (6, 5, 4)
    b = sb.build_basis(n)
    T = O.BoxTopology(ex, ey, ez, n)
    g = O.box_geom(ex, ey, ez, b.weights, 1.0)
    E = ex * ey * ez
    f0 = O.random_field(E, n, O.mix64(1, E))
    f = O.mask(O.dssum(f0, T), T)
    _, hist, _ = O.cg(f, lambda p: O.apply_global(p, g, b.diff, b.diff_t, T), T, 40)
    return np.asarray(hist)


@pytest.mark.parametrize("mode", sorted(MODES))
def test_cg_mode_deterministic_and_matches_oracle(runs, oracle_hist, mode):
    r = runs[mode]
    h0, h1 = np.asarray(r["hist"][0]), np.asarray(r["hist"][1])
    assert np.array_equal(h0, h1), f"{mode}: not reproducible run to run"
    rel = float(np.max(np.abs(h0 - oracle_hist) / np.abs(oracle_hist)))
    assert rel <= 1e-10, f"{mode}: residual history vs oracle {rel:.3e}"


def test_cg_modes_same_trees_bitexact(runs):
    # PDL and the Ax staging mode change no arithmetic or reduction tree:
    # bit-identical to the default (FIN changes the final combine's tree)
    base = runs["default"]["hist"][0]
    for mode in ("pdl0", "pdl1", "axcfg4"):
        assert runs[mode]["hist"][0] == base, mode


def test_cg_tolerance_exit_mid_graph(cuda, oracle_hist):
    # a tolerance first met at iteration 23 (inside the third 10-iteration
    # graph): the stop flag turns the rest of the graph into no-ops -- same
    # iteration count and history as the oracle's early exit
    import oracle as O
    import paper_2005_13425_b200 as sb
    tol = float(oracle_hist[22]) * (1.0 + 1e-6)
    assert tol < float(np.min(oracle_hist[:22]))
    r = _run({"CG_TEST_TOL": repr(tol)})
    n, (ex, ey, ez) = 10, (6, 5, 4)
    b = sb.build_basis(n)
    T = O.BoxTopology(ex, ey, ez, n)
    g = O.box_geom(ex, ey, ez, b.weights, 1.0)
    E = ex * ey * ez
    f0 = O.random_field(E, n, O.mix64(1, E))
    f = O.mask(O.dssum(f0, T), T)
    _, hist, _ = O.cg(f, lambda p: O.apply_global(p, g, b.diff, b.diff_t, T), T, 40, tol)
    h = np.asarray(r["hist"][0])
    assert r["iters"] == len(hist) == 23
    assert float(np.max(np.abs(h - hist) / np.abs(hist))) <= 1e-10
