"""Space-time slab path: the oracle (oracle/spacetime.py) against golden
fixtures from the real reference (tests/golden/make_golden_slab.py) and the
reference suite's space-time known answers (pkg/tests/test_spacetime.py);
the device engine against both (``-m gpu``)."""

import glob
import os

import numpy as np
import pytest

import fixtures as F
from compare import assert_parity
from oracle import sipg as O
from oracle import spacetime as OS
from paper_2007_04881_b200 import Family
from paper_2007_04881_b200.mesh import SimplicialMesh, agglomerate
from paper_2007_04881_b200.spacetime import TimePartition, build_slab

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "slab_*.npz")))


def load_slab_case(path):
    z = np.load(path, allow_pickle=False)
    base = SimplicialMesh(int(z["vertices"].shape[1]), z["vertices"], z["simplices"])
    pm = agglomerate(base, z["agg"])
    cname = str(z["coeffs"])
    coeffs, initial = getattr(F, cname)()
    fam = Family(str(z["family"]))
    p = int(z["degree"])
    slab, specs = build_slab(pm, (float(z["t0"]), float(z["t1"])), p, fam)
    if "prev_vec" in z.files:
        _, pspecs = build_slab(pm, (float(z["prev_t0"]), float(z["prev_t1"])), p, fam)
        prev = (pspecs, np.array(z["prev_vec"]))
    else:
        prev = initial
    ref = (z["row_ptr"], z["col_idx"], z["values"], z["rhs"])
    return slab, coeffs, specs, prev, F.slab_predicate(cname), ref


class _CSR:
    def __init__(self, rp, ci, v):
        self.row_ptr, self.col_idx, self.values = rp, ci, v


def _offsets(specs):
    return np.concatenate([[0], np.cumsum([s.n_funcs for s in specs])])


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_slab_oracle_reproduces_reference_golden(path):
    slab, coeffs, specs, prev, pred, ref = load_slab_case(path)
    rp, ci, v, r = OS.assemble_slab(slab.spatial, slab.t0, slab.t1, coeffs, specs, prev,
                                    dirichlet_predicate=pred)
    assert_parity(_CSR(rp, ci, v), r, ref, _offsets(specs), tol=1e-13)


def test_slab_golden_set_present():
    assert len(GOLDEN) >= 8  # 6 over 2D meshes, 2 over 3D meshes (3+1D prisms)


def test_time_partition_validation():
    """test_spacetime.py:49-55."""
    with pytest.raises(ValueError):
        TimePartition(np.array([0.0]))
    with pytest.raises(ValueError):
        TimePartition(np.array([0.0, 0.5, 0.5]))
    tp = TimePartition.uniform(1.0, 4)
    assert tp.n_steps == 4 and tp.interval(1) == (0.25, 0.5)


def test_build_slab_counts():
    """test_spacetime.py:57-65: prism boxes and PQ / P basis sizes."""
    pm = agglomerate(F.square_grid(4), F.square_blocks(4, 2))
    slab, specs = build_slab(pm, (0.0, 0.1), 1, Family.P)
    assert slab.dim == 3 and specs[0].n_funcs == 4
    assert np.allclose(specs[0].box[:, -1], [0.0, 0.1])
    _, pq = build_slab(pm, (0.0, 0.1), 1, Family.PQ)
    assert pq[0].n_funcs == 6
    assert np.isclose(sum(slab.prism_volume(e) for e in range(pm.n_elements)), 0.1)


def test_bottom_facet_block_is_scaled_spatial_mass():
    """test_spacetime.py:212-227 restated on the oracle: with no diffusion,
    reaction or lateral flux, the slab matrix is the bottom-facet mass block
    plus the (b.grad) volume term; on the bottom facet the time factor of the
    PQ basis is L~_k(-1) = (-1)^k sqrt(2k+1)/sqrt(tau)."""
    pm = agglomerate(F.square_grid(2), np.zeros(8, np.int64))
    import paper_2007_04881_b200.model as M

    C = M.PdeCoefficients(advection=M.constant_vector([0.0, 0.0, 1.0]))
    slab, specs = build_slab(pm, (0.0, 1.0), 1, Family.PQ)
    prob = OS.SlabProblem(pm, 0.0, 1.0, C, specs, lambda xy: np.zeros(len(xy)))
    blocks, _ = OS.slab_element_rows(prob, 0)
    # bottom block alone
    rule = O.simplex_rule(2, 4)
    Kb = np.zeros((6, 6))
    for s in pm.elements[0]:
        sp, sw = O.map_to_simplex(rule, pm.base.vertices[pm.base.simplices[s]])
        pts = np.concatenate([sp, np.zeros((sp.shape[0], 1))], axis=1)
        V, _ = O.tabulate(1, specs[0].box, pts, "PQ")
        Kb += np.einsum("q,iq,jq->ij", sw, V, V)
    sgn = np.array([1, 1, 1, -1, -1, -1]) * np.sqrt([1, 1, 1, 3, 3, 3])
    spatial = Kb / np.outer(sgn, sgn)
    # the spatial factor is the orthonormal spatial mass on the unit square = I
    assert np.allclose(spatial[:3, :3], np.eye(3), atol=1e-12)
    vol = blocks[0] - Kb
    # the volume term sum_q w (d_t phi_j) phi_i is strictly "upper" in time
    assert np.allclose(vol[:3, :3], 0.0, atol=1e-12)


# ---------------------------------------------------------------- device engine

@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_slab_engine_reproduces_reference_golden(path):
    from paper_2007_04881_b200.spacetime import assemble_slab

    slab, coeffs, specs, prev, pred, ref = load_slab_case(path)
    m, rhs, stats = assemble_slab(slab, coeffs, specs, prev, dirichlet_predicate=pred)
    assert_parity(m, rhs, ref, _offsets(specs))
    assert stats.nnz == m.nnz


@pytest.mark.gpu
@pytest.mark.parametrize("p,fam", [(0, "PQ"), (1, "PQ"), (2, "PQ"), (3, "PQ"), (4, "PQ"),
                                   (1, "P"), (3, "P"), (4, "P")])
def test_slab_engine_degrees_against_oracle(p, fam):
    from paper_2007_04881_b200.meshgen import voronoi_mesh
    from paper_2007_04881_b200.spacetime import assemble_slab

    pm = voronoi_mesh(40, seed=3)
    coeffs, initial = F.slab_heat()
    slab, specs = build_slab(pm, (0.2, 0.45), p, Family(fam))
    m, rhs, _ = assemble_slab(slab, coeffs, specs, initial)
    ref = OS.assemble_slab(pm, 0.2, 0.45, coeffs, specs, initial)
    assert_parity(m, rhs, ref, _offsets(specs))


@pytest.mark.gpu
def test_slab_engine_rows_partition_and_determinism():
    """Row-partitioned slab assembly reproduces the monolithic rows bit for bit
    (distribute.py:200-232 semantics) and repeated runs are bitwise equal."""
    from paper_2007_04881_b200.meshgen import voronoi_mesh
    from paper_2007_04881_b200.spacetime import SlabPlan

    pm = voronoi_mesh(60, seed=4)
    coeffs, initial = F.slab_adv_heat()
    slab, specs = build_slab(pm, (0.0, 0.1), 2, Family.PQ)
    full = SlabPlan(slab, coeffs, specs, initial, dirichlet_predicate=F.slab_predicate("slab_adv_heat"))
    full.run()
    full.check_flags()
    v0 = full.values.clone()
    full.run()
    full.check_flags()
    assert bool((full.values == v0).all())
    rows = np.arange(13, 41)
    part = SlabPlan(slab, coeffs, specs, initial, row_elements=rows,
                    dirichlet_predicate=F.slab_predicate("slab_adv_heat"))
    part.run()
    part.check_flags()
    off = full.t["val_off"].cpu().numpy()
    a, b = int(off[13]), int(off[41])
    assert np.array_equal(part.values.cpu().numpy(), v0.cpu().numpy()[a:b])
    ro = full.t["row_off"].cpu().numpy()
    rp = full.row_ptr.cpu().numpy()
    ci = full.col_idx.cpu().numpy()
    assert np.array_equal(part.col_idx.cpu().numpy(), ci[a:b])
    d0, d1 = int(full.dof.offsets[13]), int(full.dof.offsets[41])
    assert np.array_equal(part.rhs.cpu().numpy()[d0:d1], full.rhs.cpu().numpy()[d0:d1])
    assert int(ro[41] - ro[13]) == part.n_local_rows and rp[-1] == full.nnz


@pytest.mark.gpu
def test_march_two_slabs_against_oracle():
    """march (spacetime.py:434-481): the second slab's time jump uses the
    first slab's solution; both systems match the oracle."""
    from paper_2007_04881_b200.spacetime import ParabolicProblem, TimePartition, assemble_slab, march

    pm = agglomerate(F.square_grid(6), F.grown_clusters(F.square_grid(6), 9, seed=3))
    coeffs, initial = F.slab_heat()
    prob = ParabolicProblem(2, coeffs, initial, 0.5)
    sols, slabs = march(pm, TimePartition.uniform(0.5, 2), prob, 1, Family.PQ)
    assert len(sols) == 2
    slab2, specs2 = slabs[1]
    m, rhs, _ = assemble_slab(slab2, coeffs, specs2, (slabs[0][1], sols[0]))
    ref = OS.assemble_slab(pm, slab2.t0, slab2.t1, coeffs, specs2, (slabs[0][1], sols[0]))
    assert_parity(m, rhs, ref, _offsets(specs2))
    # the discrete solution approximates u = sin sin (1 - t) at the slab end
    assert np.all(np.isfinite(sols[1]))


@pytest.mark.gpu
@pytest.mark.parametrize("p,fam", [(0, "PQ"), (1, "PQ"), (2, "PQ"), (1, "P"), (2, "P"), (3, "P")])
def test_slab_engine_3d_spatial_against_oracle(p, fam):
    """3+1D prisms (spacetime over a 3D agglomerated mesh; polydg
    test_spacetime.py:278-290 exercises this dimension at p = 0)."""
    from paper_2007_04881_b200.spacetime import assemble_slab

    g = F.cube_grid(3)
    pm = agglomerate(g, F.grown_clusters(g, 9, seed=4))
    coeffs, initial = F.slab_heat3d()
    slab, specs = build_slab(pm, (0.1, 0.3), p, Family(fam))
    m, rhs, _ = assemble_slab(slab, coeffs, specs, initial)
    ref = OS.assemble_slab(pm, 0.1, 0.3, coeffs, specs, initial)
    assert_parity(m, rhs, ref, _offsets(specs))
