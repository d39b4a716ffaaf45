"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 hot path.

This package restates the reference (``sembench``, arXiv 2005.13425 proxy)
hot path on the CPU so tests can check the CUDA path against it.  It is
imported only by ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py``; the product
package ``paper_2005_13425_b200`` never imports it (tests/test_boundary.py
enforces that).

Arithmetic kernels live in ``sem_oracle.c`` (built by ``oracle/Makefile``
into ``oracle/_build/libsem_oracle.so``); mesh/topology bookkeeping is
restated here in numpy.  Parity is PINNED: tests/test_oracle_golden.py
checks every routine bit-for-bit against fixtures produced by the reference
itself (tests/golden/make_golden.py, run in the build container where
/root/reference is importable).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libsem_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the C oracle with its Makefile (gcc, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB_PATH):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_ax_layered.argtypes = [_dp, _dp, _dp, _dp, _dp, ctypes.c_int64,
                                        ctypes.c_int, ctypes.c_int]
        L.oracle_ax_layered.restype = ctypes.c_int
        L.oracle_ax_reference.argtypes = [_dp] * 8 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.oracle_ax_reference.restype = ctypes.c_int
        L.oracle_ax_scratch.argtypes = [_dp] * 4 + [ctypes.c_int64, ctypes.c_int, ctypes.c_int]
        L.oracle_ax_scratch.restype = ctypes.c_int
        L.oracle_dssum.argtypes = [_dp, _i64p, ctypes.c_int64, ctypes.c_int64, _dp]
        L.oracle_dssum.restype = ctypes.c_int
        L.oracle_mask.argtypes = [_dp, _dp, _dp, ctypes.c_int64]
        L.oracle_mask.restype = None
        L.oracle_wdot3.argtypes = [_dp, _dp, _dp, ctypes.c_int64, ctypes.c_int]
        L.oracle_wdot3.restype = ctypes.c_double
        L.oracle_axpy_into.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_int64, ctypes.c_int]
        L.oracle_axpy_into.restype = None
        L.oracle_scale_add.argtypes = [_dp, _dp, ctypes.c_double, ctypes.c_int64, ctypes.c_int]
        L.oracle_scale_add.restype = None
        L.oracle_random_field.argtypes = [ctypes.c_uint64, ctypes.c_int64, _dp]
        L.oracle_random_field.restype = None
        L.oracle_max_threads.argtypes = []
        L.oracle_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(_dp if a.dtype == np.float64 else _i64p)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


# ---------------------------------------------------------------------------
# seeded inputs -- sembench/fields.py:16-54
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1


def _splitmix_int(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return z ^ (z >> 31)


def mix64(a: int, b: int = 0) -> int:
    """sembench/fields.py:28-31: splitmix of (a * FNV-prime + b) mod 2^64."""
    return _splitmix_int((a * 0x100000001B3 + b) & _M64)


def random_field(num_elements: int, n: int, seed: int) -> np.ndarray:
    out = np.empty((num_elements, n, n, n))
    lib().oracle_random_field(ctypes.c_uint64(int(seed) & _M64), out.size, _p(out))
    return out


# ---------------------------------------------------------------------------
# mesh, geometry, topology -- sembench/mesh.py:72-91, assembly.py:69-110,
# bench.py:100-125
# ---------------------------------------------------------------------------

def factor_elements(count: int):
    """Most cubic ex >= ey >= ez box, minimising (ex/ez, ex-ez) (bench.py:100-119)."""
    best, best_key = (count, 1, 1), (float(count), count + 2)
    ez = 1
    while ez <= round(count ** (1.0 / 3.0)):
        if count % ez == 0:
            rest = count // ez
            ey = ez
            while ey * ey <= rest:
                if rest % ey == 0:
                    ex = rest // ey
                    key = (ex / ez, ex - ez)
                    if key < best_key:
                        best_key, best = key, (ex, ey, ez)
                ey += 1
        ez += 1
    return best


def box_geom(ex: int, ey: int, ez: int, weights: np.ndarray, extent: float) -> np.ndarray:
    n = weights.size
    wk = weights.reshape(n, 1, 1)
    wj = weights.reshape(1, n, 1)
    wi = weights.reshape(1, 1, n)
    diag = (wk * wj * wi) * (extent / 2.0)
    g = np.zeros((ex * ey * ez, 6, n, n, n))
    for comp in (0, 3, 5):
        g[:, comp] = diag
    return g


class BoxTopology:
    """Global lattice numbering of an ex*ey*ez box (assembly.py:69-110)."""

    def __init__(self, ex: int, ey: int, ez: int, n: int):
        E = ex * ey * ez
        nx, ny, nz = ex * (n - 1) + 1, ey * (n - 1) + 1, ez * (n - 1) + 1
        e = np.arange(E, dtype=np.int64)
        ax = (e % ex)[:, None, None, None]
        ay = ((e // ex) % ey)[:, None, None, None]
        az = (e // (ex * ey))[:, None, None, None]
        q = np.arange(n, dtype=np.int64)
        gx = ax * (n - 1) + q[None, None, None, :]
        gy = ay * (n - 1) + q[None, None, :, None]
        gz = az * (n - 1) + q[None, :, None, None]
        self.num_elements, self.n = E, n
        self.global_id = np.ascontiguousarray((gz * ny + gy) * nx + gx)
        self.num_global = nx * ny * nz
        counts = np.bincount(self.global_id.ravel(), minlength=self.num_global)
        self.multiplicity = counts[self.global_id]
        inside = ((gx > 0) & (gx < nx - 1) & (gy > 0) & (gy < ny - 1)
                  & (gz > 0) & (gz < nz - 1))
        self.mask = inside.astype(np.float64)
        self.inv_multiplicity = (1.0 / self.multiplicity.astype(np.float64)).ravel()


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------

def ax_layered(u: np.ndarray, g: np.ndarray, dx: np.ndarray, dxt: np.ndarray,
               nthreads: int = 0) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    dxt = np.ascontiguousarray(dxt, dtype=np.float64)
    E, n = u.shape[0], u.shape[-1]
    assert g.shape == (E, 6, n, n, n)
    w = np.empty_like(u)
    rc = lib().oracle_ax_layered(_p(u), _p(g), _p(dx), _p(dxt), _p(w), E, n, nthreads)
    if rc != 0:
        raise RuntimeError(f"oracle_ax_layered failed ({rc})")
    return w


def ax_reference(u: np.ndarray, g: np.ndarray, dx: np.ndarray, dxt: np.ndarray,
                 nthreads: int = 0):
    """REFERENCE variant (sembench/kernels.py:159-205): returns (w, ur, us, ut),
    the intermediates as the reference leaves them in its workspace."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    dxt = np.ascontiguousarray(dxt, dtype=np.float64)
    E, n = u.shape[0], u.shape[-1]
    assert g.shape == (E, 6, n, n, n)
    w, ur, us, ut = (np.empty_like(u) for _ in range(4))
    rc = lib().oracle_ax_reference(_p(u), _p(g), _p(dx), _p(dxt), _p(ur), _p(us), _p(ut),
                                   _p(w), E, n, nthreads)
    if rc != 0:
        raise RuntimeError(f"oracle_ax_reference failed ({rc})")
    return w, ur, us, ut


def ax_scratch(u: np.ndarray, g: np.ndarray, dx: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """SCRATCH variant (sembench/kernels.py:213-259)."""
    u = np.ascontiguousarray(u, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    dx = np.ascontiguousarray(dx, dtype=np.float64)
    E, n = u.shape[0], u.shape[-1]
    assert g.shape == (E, 6, n, n, n)
    w = np.empty_like(u)
    rc = lib().oracle_ax_scratch(_p(u), _p(g), _p(dx), _p(w), E, n, nthreads)
    if rc != 0:
        raise RuntimeError(f"oracle_ax_scratch failed ({rc})")
    return w


def dssum(f: np.ndarray, topo: BoxTopology) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty_like(f)
    gid = np.ascontiguousarray(topo.global_id, dtype=np.int64)
    rc = lib().oracle_dssum(_p(f), _p(gid), f.size, topo.num_global, _p(out))
    if rc != 0:
        raise MemoryError("oracle_dssum accumulator allocation failed")
    return out


def mask(f: np.ndarray, topo: BoxTopology) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty_like(f)
    lib().oracle_mask(_p(f), _p(np.ascontiguousarray(topo.mask)), _p(out), f.size)
    return out


def apply_global(u, g, dx, dxt, topo, nthreads: int = 0):
    """mask(dssum(A_local(mask(u)))) -- assembly.py:132-155."""
    return mask(dssum(ax_layered(mask(u, topo), g, dx, dxt, nthreads), topo), topo)


def wdot3(a: np.ndarray, b: np.ndarray, wt: np.ndarray, nthreads: int = 0) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64).ravel()
    b = np.ascontiguousarray(b, dtype=np.float64).ravel()
    wt = np.ascontiguousarray(wt, dtype=np.float64).ravel()
    return float(lib().oracle_wdot3(_p(a), _p(b), _p(wt), a.size, nthreads))


def axpy_into(x: np.ndarray, y: np.ndarray, alpha: float, nthreads: int = 0) -> None:
    lib().oracle_axpy_into(_p(x), _p(np.ascontiguousarray(y)), float(alpha), x.size, nthreads)


def scale_add(p: np.ndarray, z: np.ndarray, beta: float, nthreads: int = 0) -> None:
    lib().oracle_scale_add(_p(p), _p(np.ascontiguousarray(z)), float(beta), p.size, nthreads)


def cg(f: np.ndarray, operator, topo: BoxTopology, max_iterations: int,
       tolerance: float = 0.0, nthreads: int = 0):
    """Unpreconditioned CG, the recurrence of sembench/cg.py:139-186.

    Returns (x, history, iterations).  Raises RuntimeError on <p,Ap> <= 0.
    """
    r = mask(f, topo)
    x = np.zeros_like(r)
    p = np.zeros_like(r)
    invm = topo.inv_multiplicity
    history = []
    rtz, iterations = 1.0, 0
    for it in range(1, max_iterations + 1):
        rtz_old = rtz
        rtz = wdot3(r, r, invm, nthreads)
        if rtz == 0.0:
            history.append(0.0)
            iterations = it
            break
        beta = 0.0 if it == 1 else rtz / rtz_old
        scale_add(p, r, beta, nthreads)
        w = operator(p)
        pap = wdot3(p, w, invm, nthreads)
        if pap <= 0.0:
            raise RuntimeError(f"breakdown at iteration {it}: pap={pap}")
        alpha = rtz / pap
        axpy_into(x, p, alpha, nthreads)
        axpy_into(r, np.ascontiguousarray(w), -alpha, nthreads)
        rnorm = math.sqrt(wdot3(r, r, invm, nthreads))
        history.append(rnorm)
        iterations = it
        if tolerance > 0.0 and rnorm < tolerance:
            break
    return x, np.asarray(history), iterations


# ---------------------------------------------------------------------------
# comparison metric and independent dense oracle -- sembench/verify.py:37-77
# ---------------------------------------------------------------------------

def rel_diff(a: np.ndarray, b: np.ndarray) -> float:
    """Max-norm difference relative to the larger operand (verify.py:37-42)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(a))), float(np.max(np.abs(b))))
    return 0.0 if scale == 0.0 else float(np.max(np.abs(a - b)) / scale)


_SYM = ((0, 1, 2), (1, 3, 4), (2, 4, 5))


def dense_apply(u: np.ndarray, g: np.ndarray, dx: np.ndarray) -> np.ndarray:
    """w_e = K_e u_e with K_e = sum_ab Da^T diag(g_ab) Db built from Kronecker
    products (no sum factorisation) -- the independent oracle of verify.py:45-77."""
    n = dx.shape[0]
    I = np.eye(n)
    ops = (np.kron(I, np.kron(I, dx)), np.kron(I, np.kron(dx, I)), np.kron(dx, np.kron(I, I)))
    out = np.empty_like(u)
    for e in range(u.shape[0]):
        K = np.zeros((n ** 3, n ** 3))
        for a in range(3):
            for b in range(3):
                K += ops[a].T @ (g[e, _SYM[a][b]].reshape(-1)[:, None] * ops[b])
        out[e] = (K @ u[e].reshape(-1)).reshape(n, n, n)
    return out
