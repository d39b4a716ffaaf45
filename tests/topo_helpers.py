"""Reference-shaped topology objects for the interop tests.

``RefTopology`` has exactly the fields of the reference's frozen
``Topology`` dataclass (sembench/assembly.py:37-53), so code that accepts a
reference topology can be driven without importing the reference (which is
absent on the GPU box).  ``box_topology`` builds it with the reference's
lattice recipe (via the oracle's restatement, assembly.py:69-110);
``periodic_x_topology`` wraps the x lattice (a NON-box numbering the
analytic box kernels cannot express).
"""

from dataclasses import dataclass, field

import numpy as np

import oracle as O


@dataclass(frozen=True)
class RefTopology:
    num_elements: int
    n: int
    global_id: np.ndarray
    multiplicity: np.ndarray
    mask: np.ndarray
    num_global: int
    inv_multiplicity: np.ndarray = field(repr=False)

    @property
    def dofs(self) -> int:
        return self.num_elements * self.n ** 3


def _freeze(*arrays):
    for a in arrays:
        a.flags.writeable = False


def box_topology(ex, ey, ez, n, frozen=True) -> RefTopology:
    T = O.BoxTopology(ex, ey, ez, n)
    arrs = (T.global_id.copy(), T.multiplicity.copy(), T.mask.copy(), T.inv_multiplicity.copy())
    if frozen:
        _freeze(*arrs)
    return RefTopology(T.num_elements, n, arrs[0], arrs[1], arrs[2], T.num_global, arrs[3])


def periodic_x_topology(ex, ey, ez, n) -> RefTopology:
    """Periodic in x (the x = max face is the x = 0 face), Dirichlet in y, z."""
    E = ex * ey * ez
    nxp, ny, nz = ex * (n - 1), ey * (n - 1) + 1, ez * (n - 1) + 1
    e = np.arange(E, dtype=np.int64)
    q = np.arange(n, dtype=np.int64)
    gx = ((e % ex)[:, None, None, None] * (n - 1) + q[None, None, None, :]) % nxp
    gy = ((e // ex) % ey)[:, None, None, None] * (n - 1) + q[None, None, :, None]
    gz = (e // (ex * ey))[:, None, None, None] * (n - 1) + q[None, :, None, None]
    gid = np.ascontiguousarray((gz * ny + gy) * nxp + gx)
    num_global = nxp * ny * nz
    mult = np.bincount(gid.ravel(), minlength=num_global)[gid]
    inner = (gy > 0) & (gy < ny - 1) & (gz > 0) & (gz < nz - 1)
    msk = np.ascontiguousarray(np.broadcast_to(inner, gid.shape).astype(np.float64))
    invm = (1.0 / mult.astype(np.float64)).ravel()
    _freeze(gid, mult, msk, invm)
    return RefTopology(E, n, gid, mult, msk, num_global, invm)


def relabelled(topo: RefTopology, seed: int = 0) -> RefTopology:
    """The same id classes under a random permutation of the id labels."""
    perm = np.random.default_rng(seed).permutation(topo.num_global)
    gid = perm[topo.global_id]
    _freeze(gid)
    return RefTopology(topo.num_elements, topo.n, gid, topo.multiplicity, topo.mask,
                       topo.num_global, topo.inv_multiplicity)


def sembench_or_none():
    """The installed reference package (baseline/_ref), if present."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    ref = os.path.join(root, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "sembench")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/sem_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import sembench
    except Exception:  # noqa: BLE001 -- numba missing etc.
        return None
    return sembench
