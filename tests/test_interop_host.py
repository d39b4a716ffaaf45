"""Host-side interop (no GPU): reference-shaped topology / geometry objects
are recognised (box lattice -> analytic box topology, anything else -> the
ordered CSR), the CSR follows np.bincount's summation order, and pooled
pinned results stay alive as long as any view of them does."""

import gc

import numpy as np
import pytest
import torch

import oracle as O
import paper_2005_13425_b200 as sb
from paper_2005_13425_b200.assembly import CsrTopology, Topology, as_topology
from topo_helpers import box_topology, periodic_x_topology, relabelled, sembench_or_none


@pytest.mark.parametrize("box,n", [((1, 1, 1), 2), ((3, 2, 2), 5), ((4, 1, 3), 3),
                                   ((2, 3, 4), 10)])
def test_box_topology_recognised(box, n):
    ref = box_topology(*box, n)
    t = as_topology(ref)
    assert isinstance(t, Topology) and t.box == box and t.n == n
    assert t.num_global == ref.num_global
    assert np.array_equal(t.global_id, ref.global_id)
    assert as_topology(ref) is t  # frozen arrays: cached


def test_writable_topology_not_cached():
    ref = box_topology(2, 2, 2, 4, frozen=False)
    assert isinstance(as_topology(ref), Topology)
    assert as_topology(ref) is not as_topology(ref)


def test_non_box_numberings_take_the_csr():
    for ref in (periodic_x_topology(3, 2, 2, 4), relabelled(box_topology(3, 2, 2, 4))):
        t = as_topology(ref)
        assert isinstance(t, CsrTopology)
        gid = ref.global_id.ravel()
        # every class in ascending local index (np.bincount's order)
        for s in range(0, ref.num_global, 7):
            members = t._idx[t._off[s]:t._off[s + 1]]
            assert np.array_equal(members, np.flatnonzero(gid == s))


def test_modified_mask_is_not_the_box():
    ref = box_topology(2, 2, 2, 4)
    m = ref.mask.copy()
    m[0, 1, 1, 1] = 0.0
    m.flags.writeable = False
    other = type(ref)(ref.num_elements, ref.n, ref.global_id, ref.multiplicity, m,
                      ref.num_global, ref.inv_multiplicity)
    assert isinstance(as_topology(other), CsrTopology)


def test_sembench_topology_recognised():
    S = sembench_or_none()
    if S is None:
        pytest.skip("reference package not installed under baseline/_ref")
    ref = S.build_topology(S.build_mesh(3, 2, 4, 5, 1.0))
    t = as_topology(ref)
    assert isinstance(t, Topology) and t.box == (3, 2, 4)
    geom = S.build_geom(S.build_mesh(3, 2, 4, 5, 1.0), S.build_basis(5))
    g = sb.as_geom(geom)
    assert g.values is geom.values and sb.as_geom(geom) is g


def test_not_a_topology():
    with pytest.raises(TypeError):
        as_topology(object())


def test_pinned_pool_views_keep_the_block():
    """A caller holding only a view (reshape / ravel / torch.from_numpy) of a
    pooled result must keep its block out of the pool."""
    from paper_2005_13425_b200._device import PinnedPool

    class Pool(PinnedPool):
        def _take(self, nbytes):  # pageable stand-in: no CUDA needed
            with self._lock:
                lst = self._free.get(nbytes)
                if lst:
                    return lst.pop()
            return torch.empty(nbytes, dtype=torch.uint8)

    pool = Pool()
    a = pool.array((4, 3))
    a[...] = 1.0
    view = a.reshape(-1)[2:]
    del a
    gc.collect()
    b = pool.array((4, 3))
    b[...] = 2.0
    assert np.all(view == 1.0)  # b did not reuse view's block
    t = torch.from_numpy(view)
    del view
    gc.collect()
    c = pool.array((4, 3))
    c[...] = 3.0
    assert torch.all(t == 1.0)
    del t
    gc.collect()
    assert len(pool._free.get(96, [])) == 1  # the block came back once unreferenced


def test_oracle_dssum_is_bincount_for_any_numbering():
    """The oracle's ordered dssum (the checker of sem_dssum_csr) equals
    np.bincount for a non-box numbering, bit for bit."""
    ref = periodic_x_topology(3, 2, 2, 4)
    f = O.random_field(ref.num_elements, 4, 3)
    want = np.bincount(ref.global_id.ravel(), weights=f.ravel(),
                       minlength=ref.num_global)[ref.global_id]
    assert np.array_equal(O.dssum(f, ref), want)
