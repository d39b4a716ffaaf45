"""The C-ABI from a plain C program (tests/c_client/sem_client.c, built with
gcc against include/sem.h and libsem.so, no Python or torch in its process):
Ax, dssum + mask and a fused CG solve on seeded inputs, checked against the
CPU oracle with the same bars as the Python-level parity tests (Ax <= 1e-12
max-norm relative, dssum bit-exact, CG history <= 1e-10)."""

import os
import shutil
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_2005_13425_b200 as sb

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2005_13425_b200")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


@pytest.fixture(scope="module")
def client(tmp_path_factory):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path_factory.mktemp("cclient") / "sem_client")
    cmd = ["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"),
           "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "c_client", "sem_client.c"),
           "-L", LIBDIR, "-lsem", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


@pytest.mark.parametrize("box,n,iters", [((4, 3, 2), 10, 30), ((3, 3, 3), 7, 20)])
def test_c_client_matches_oracle(cuda, client, tmp_path, box, n, iters):
    ex, ey, ez = box
    E = ex * ey * ez
    b = sb.build_basis(n)
    seed = int(sb.mix64(1, E))
    np.ascontiguousarray(b.diff, dtype=np.float64).tofile(tmp_path / "dx.bin")
    np.ascontiguousarray(b.diff_t, dtype=np.float64).tofile(tmp_path / "dxt.bin")
    np.ascontiguousarray(b.weights, dtype=np.float64).tofile(tmp_path / "weights.bin")
    (tmp_path / "meta.txt").write_text(f"{n} {ex} {ey} {ez} {iters} {seed}\n")
    out = subprocess.run([client, str(tmp_path)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    shape = (E, n, n, n)
    load = lambda name, cnt=None: np.fromfile(tmp_path / name, dtype=np.float64)  # noqa: E731
    u = O.random_field(E, n, 1)
    g = O.random_field(6 * E, n, 2).reshape(E, 6, n, n, n)
    T = O.BoxTopology(ex, ey, ez, n)
    assert O.rel_diff(load("w.bin").reshape(shape), O.ax_layered(u, g, b.diff, b.diff_t)) <= 1e-12
    assert np.array_equal(load("dssum.bin").reshape(shape), O.mask(O.dssum(u, T), T))
    f = O.mask(O.dssum(O.random_field(E, n, seed), T), T)
    gh = O.box_geom(ex, ey, ez, b.weights, 1.0)
    x_ref, hist, _ = O.cg(f, lambda p: O.apply_global(p, gh, b.diff, b.diff_t, T), T, iters)
    got = load("hist.bin")
    assert got.shape == (iters,)
    assert float(np.max(np.abs(got - hist) / np.abs(hist))) <= 1e-10
    assert O.rel_diff(load("x.bin").reshape(shape), x_ref) <= 1e-10
    # host buffers: pageable (chunked copy engines) and mapped (zero-copy)
    w_dev = load("w.bin")
    assert np.array_equal(load("w_host.bin"), w_dev)
    assert O.rel_diff(load("w_mapped.bin"), w_dev) <= 1e-12
    # weighted dot (deterministic tree: rounding-level vs the oracle) and the
    # unfused vector updates (bit-exact: multiply rounded, then add)
    wv = w_dev.reshape(shape)
    dot_ref = O.wdot3(u, wv, T.inv_multiplicity)
    assert abs(float(load("dot.bin")[0]) - dot_ref) <= 1e-13 * max(1.0, abs(dot_ref))
    p1 = w_dev.copy()
    O.scale_add(p1, u.reshape(-1), 0.75)              # p = 0.75 p + z
    assert np.array_equal(load("add2s1.bin"), p1)
    x1 = u.reshape(-1).copy()
    O.axpy_into(x1, g.reshape(-1)[:u.size], -1.25)    # x += -1.25 y
    assert np.array_equal(load("add2s2.bin"), x1)
