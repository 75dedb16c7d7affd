"""Device agglomeration against the host agglomerate, which
is itself tested against polydg's (tests/test_host.py): bit-identical
polytopic meshes, same MeshError conditions."""

import numpy as np
import pytest

import fixtures as F
from paper_2007_04881_b200.mesh import MeshError, SimplicialMesh, agglomerate

FIELDS = ("elem_ptr", "elem_simplices", "boxes", "elem_volumes", "face_owner", "face_neighbor", "face_normal",
          "face_measure", "face_ptr", "facet_vertices", "facet_owner_simplex", "facet_neighbor_simplex",
          "facet_measures", "iface_owner", "iface_neighbor", "iface_ptr", "iface_faces", "elem_bface_ptr",
          "elem_bfaces")


def _cases():
    from paper_2007_04881_b200.meshgen import voronoi_simplicial

    vb, va = voronoi_simplicial(300, seed=2)
    g10, c3, g6 = F.square_grid(10), F.cube_grid(3), F.square_grid(6)
    return [("voronoi300", vb, va), ("grid10_clusters", g10, F.grown_clusters(g10, 23, seed=2)),
            ("grid6_identity", g6, np.arange(g6.n_simplices)), ("grid8_blocks", F.square_grid(8),
                                                                 F.square_blocks(8, 2)),
            ("cube3_clusters", c3, F.grown_clusters(c3, 11, seed=3)), ("cube4_blocks", F.cube_grid(4),
                                                                       F.cube_blocks(4, 2))]


@pytest.mark.gpu
@pytest.mark.parametrize("case", _cases(), ids=lambda c: c[0])
def test_device_agglomerate_bit_identical(case):
    from paper_2007_04881_b200.meshprep import agglomerate_device

    _, base, agg = case
    ref = agglomerate(base, agg).flat
    got = agglomerate_device(base, agg).flat
    for k in FIELDS:
        a, b = getattr(ref, k), getattr(got, k)
        assert a.shape == b.shape, (k, a.shape, b.shape)
        assert np.array_equal(a, b), k


@pytest.mark.gpu
def test_device_agglomerate_zigzag_multiface():
    """One interface made of several planar faces (greedy co-hyperplanar split)."""
    from paper_2007_04881_b200.meshprep import agglomerate_device

    pm = F.zigzag(3)
    got = agglomerate_device(pm.base, pm.agg_map).flat
    for k in FIELDS:
        assert np.array_equal(getattr(pm.flat, k), getattr(got, k)), k


@pytest.mark.gpu
def test_device_agglomerate_errors():
    from paper_2007_04881_b200.meshprep import agglomerate_device

    g = F.square_grid(4)
    agg = np.zeros(g.n_simplices, np.int64)
    agg[0] = 1
    agg[-1] = 1  # two far-apart simplices: element 1 not facet-connected
    with pytest.raises(MeshError, match="not facet-connected"):
        agglomerate_device(g, agg)
    agglomerate_device(g, agg, check_connected=False)
    bad = np.arange(g.n_simplices) * 2  # not surjective
    with pytest.raises(MeshError):
        agglomerate_device(g, bad)
