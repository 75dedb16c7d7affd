"""Host-side logic (no GPU): the C ABI library, mesh flattening routes,
coefficient lowering, partitioning and gather semantics."""

import os
import re

import numpy as np
import pytest

import fixtures as F
from paper_2007_04881_b200 import _lib, build_basis, classify_boundary_faces
from paper_2007_04881_b200 import model as M
from paper_2007_04881_b200.assembly import AssemblyError, CSRMatrix, DofMap
from paper_2007_04881_b200.distribute import (
    PartialMatrix,
    PartitionError,
    contiguous_partition,
    gather_and_verify,
    gather_load,
    partition_from_map,
    quadrature_cost_weights,
)
from paper_2007_04881_b200.mesh import FlatMesh, MeshError, SimplicialMesh, agglomerate
from paper_2007_04881_b200.meshgen import kuhn_agglomerated_mesh, voronoi_mesh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---- C ABI ---------------------------------------------------------------------

def test_library_loads_and_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "pdg.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(pdg_\w+)\(", header, flags=re.M))
    assert declared == set(_lib.EXPORTS), declared ^ set(_lib.EXPORTS)
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.pdg_abi_version() == _lib.ABI_VERSION == 3


def test_library_rejects_bad_arguments_without_a_gpu():
    import ctypes as C

    lib = _lib.load()
    rc = lib.pdg_adjacency(None, None, None, None, None, 0, None)
    assert rc == _lib.PDG_ERR_INVALID
    assert b"null" in lib.pdg_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)
    m = _lib.Mesh()
    m.dim = 5
    b = _lib.Basis()
    c = _lib.Coeffs()
    assert lib.pdg_assemble(C.byref(m), C.byref(b), C.byref(c), None, None, None, None, None, None,
                            None, 0, None, None, None) == _lib.PDG_ERR_UNSUPPORTED


def test_expand_block_cols_rebuilds_every_row_on_the_host():
    """pdg_expand_block_cols (host threads, no GPU): one packed column list per
    element -> the same list in each of the element's rows, for ragged row
    counts / lengths, empty lists and any thread count (HostIO's e2e path)."""
    rng = np.random.default_rng(3)
    n = 257
    ne = rng.integers(1, 7, n)
    L = rng.integers(0, 40, n)
    L[5] = 0
    row0 = np.concatenate([[0], np.cumsum(ne)]).astype(np.int64)
    row_len = np.repeat(L, ne)
    row_ptr = np.concatenate([[0], np.cumsum(row_len)]).astype(np.int64)
    lists = [np.sort(rng.choice(10_000, int(l), replace=False)).astype(np.int64) for l in L]
    packed = np.concatenate(lists).astype(np.int64)
    want = np.concatenate([np.tile(c, int(k)) for c, k in zip(lists, ne)]).astype(np.int64)
    lib = _lib.load()
    for nt in (1, 3, 16):
        out = np.full(row_ptr[-1], -1, np.int64)
        _lib.check(lib.pdg_expand_block_cols(n, row0.ctypes.data, row_ptr.ctypes.data, packed.ctypes.data,
                                             out.ctypes.data, nt))
        assert np.array_equal(out, want)
    assert lib.pdg_expand_block_cols(n, None, None, None, None, 1) == _lib.PDG_ERR_INVALID


# ---- meshes ------------------------------------------------------------------------

def _flat_equal(a: FlatMesh, b: FlatMesh):
    for k, va in a.arrays().items():
        vb = getattr(b, k)
        if k == "face_tag":
            continue
        assert va.shape == vb.shape, k
        if va.dtype.kind == "f":
            np.testing.assert_allclose(va, vb, rtol=1e-14, atol=1e-15, err_msg=k)
        else:
            assert np.array_equal(va, vb), k


@pytest.mark.reference
def test_vectorised_agglomerate_matches_reference(polydg):
    from polydg import mesh as RM

    cases = []
    g = F.square_grid(8)
    cases.append((g, F.square_blocks(8, 2)))
    g = F.square_grid(6)
    cases.append((g, F.grown_clusters(g, 7, seed=1)))
    g = F.cube_grid(3)
    cases.append((g, F.grown_clusters(g, 11, seed=3)))
    pm = voronoi_mesh(150, seed=5)
    cases.append((pm.base, pm.agg_map))
    pm3 = kuhn_agglomerated_mesh(6, 120)
    cases.append((pm3.base, pm3.agg_map))
    for base, agg in cases:
        ref = RM.agglomerate(RM.SimplicialMesh(base.dim, base.vertices, base.simplices), agg)
        _flat_equal(FlatMesh.from_polytopic(ref), agglomerate(base, agg).flat)


def test_object_and_flat_routes_agree():
    pm = F.zigzag(3)
    assert len(pm.interfaces[0].face_ids) == 3
    _flat_equal(FlatMesh.from_polytopic(pm), pm.flat)


def test_agglomerate_rejects_disconnected_and_bad_maps():
    g = F.square_grid(2)
    with pytest.raises(MeshError):
        agglomerate(g, np.array([0, 1, 1, 1, 1, 1, 1, 0]))  # element 0 split in two
    with pytest.raises(MeshError):
        agglomerate(g, np.array([0, 0, 0, 0, 2, 2, 2, 2]))  # not surjective
    with pytest.raises(MeshError):
        SimplicialMesh(2, np.zeros((3, 2)), np.array([[0, 1, 2]]))  # degenerate


def test_reorientation_swaps_last_two_vertices():
    V = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    m = SimplicialMesh(2, V, np.array([[0, 2, 1]]))
    assert m.simplices.tolist() == [[0, 1, 2]]
    assert abs(m.simplex_volumes[0] - 0.5) < 1e-15


def test_voronoi_generator_properties():
    pm = voronoi_mesh(300, seed=0)
    f = pm.flat
    assert pm.n_elements == 300
    assert abs(f.elem_volumes.sum() - 1.0) < 1e-12
    assert np.all(f.vertices >= 0.0) and np.all(f.vertices <= 1.0)
    assert np.all(np.diff(f.elem_ptr) >= 3)
    # 2D Voronoi: every interface is one face made of one sub-facet
    assert np.array_equal(np.diff(f.iface_ptr), np.ones(f.n_interfaces, np.int64))
    assert np.array_equal(np.diff(f.face_ptr)[: f.n_interfaces], np.ones(f.n_interfaces, np.int64))


# ---- coefficients ----------------------------------------------------------------------

def test_expr_numpy_evaluation_matches_numpy():
    rng = np.random.default_rng(0)
    p = rng.uniform(0, 1, (50, 2))
    e = 2 * np.pi ** 2 * M.sin(np.pi * M.X) * M.sin(np.pi * M.Y) + M.X ** 2 - M.exp(M.Y) / 3.0
    ref = 2 * np.pi ** 2 * np.sin(np.pi * p[:, 0]) * np.sin(np.pi * p[:, 1]) + p[:, 0] ** 2 - np.exp(p[:, 1]) / 3.0
    assert np.array_equal(e(p), ref)


def test_compile_coeffs_kinds_and_rejections():
    d = M.compile_coeffs(F.generic(2), 2)
    assert d["diffusion_kind"] == 1 and d["has_advection"] and d["has_reaction"]
    assert d["diffusion"][0][2] == 1  # constant 0.7 I folded to an isotropic constant
    d = M.compile_coeffs(F.anisotropic(2), 2)
    assert d["diffusion_kind"] == 2 and d["diffusion_symmetric"] == 1
    with pytest.raises(NotImplementedError):
        M.compile_coeffs(M.PdeCoefficients(source=lambda p: p[:, 0]), 2)
    src = M.policy_source(F.poisson_sine(2), 2)
    assert "sinpi(x[0])" in src and "diff_kind() { return 1; }" in src


def test_reference_builders_recognised(polydg):
    from polydg import model as Rm

    C = Rm.PdeCoefficients(diffusion=Rm.isotropic_diffusion(2.0, 2), advection=Rm.constant_vector([1.0, 0.5]),
                           reaction=Rm.constant_scalar(3.0))
    d = M.compile_coeffs(C, 2)
    assert d["diffusion_kind"] == 1 and d["diffusion"][0][3] == 2.0
    assert [p[3] for p in d["advection"]] == [1.0, 0.5]


def test_classification_matches_reference(polydg):
    from polydg import mesh as RM, model as Rm

    g = F.square_grid(6)
    agg = F.grown_clusters(g, 9, seed=2)
    for coeffs, pred in ((F.generic(2), None), (F.hyperbolic(2), None),
                         (F.anisotropic(2), lambda x: x[0] < 0.5)):
        mine = agglomerate(g, agg)
        classify_boundary_faces(mine, coeffs, pred)
        ref = RM.agglomerate(RM.SimplicialMesh(2, g.vertices, g.simplices), agg)
        Rm.classify_boundary_faces(ref, coeffs, pred)
        assert [f.tag.value for f in ref.faces] == [f.tag.value for f in mine.faces]


def test_straddling_boundary_face_raises():
    g = F.square_grid(2)
    pm = agglomerate(g, np.zeros(8, np.int64))
    rot = M.PdeCoefficients(advection=M.VectorField([M.Y - 0.5, 0.5 - M.X]))
    with pytest.raises(M.ClassificationError):
        classify_boundary_faces(pm, rot)


# ---- partitions and gather ----------------------------------------------------------

def test_contiguous_partition_balance_and_cut():
    pm = voronoi_mesh(400, seed=1)
    specs = build_basis(pm, 2)
    w = quadrature_cost_weights(pm, specs)
    for n in (1, 2, 4, 8):
        part = contiguous_partition(pm, n, w)
        assert part.n_parts == n
        assert sorted(np.concatenate(part.owned).tolist()) == list(range(pm.n_elements))
        assert np.max(part.weights) <= part.weights.mean() + w.max() + 1e-9
        part.validate(pm)
    with pytest.raises(PartitionError):
        contiguous_partition(pm, 0)
    with pytest.raises(PartitionError):
        partition_from_map(pm, np.r_[np.zeros(399, np.int64), [2]])  # part 1 empty


def test_contiguous_partition_skewed_weights_keep_every_part_nonempty():
    """One dominant weight used to collapse consecutive cuts onto the same index."""
    pm = voronoi_mesh(400, seed=1)
    w = np.ones(pm.n_elements)
    w[1] = 1e6
    for n in (2, 3, 4, 8):
        part = contiguous_partition(pm, n, w)
        assert all(o.size >= 1 for o in part.owned)
        assert np.all(np.diff(part.part_of) >= 0)


def test_quadrature_cost_weights_match_reference(polydg):
    from polydg import basis as RB, distribute as RD, mesh as RM

    g = F.square_grid(6)
    agg = F.grown_clusters(g, 9, seed=2)
    mine = agglomerate(g, agg)
    ref = RM.agglomerate(RM.SimplicialMesh(2, g.vertices, g.simplices), agg)
    degs = 1 + np.arange(9) % 3
    np.testing.assert_array_equal(quadrature_cost_weights(mine, build_basis(mine, degs)),
                                  RD.quadrature_cost_weights(ref, RB.build_basis(ref, degs)))


def _toy_partials():
    # 3 elements of 2 dofs; parts own {0, 2} and {1}
    def csr(rows, ncols=6):
        lens = [len(r) for r in rows]
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        ci = np.concatenate([np.arange(len(r)) for r in rows]).astype(np.int64)
        v = np.concatenate([np.asarray(r, float) for r in rows])
        return CSRMatrix(len(rows), ncols, rp, ci, v)

    p0 = PartialMatrix(0, [(0, 2), (4, 6)], csr([[1, 2], [3], [4, 5, 6], [7]]))
    p1 = PartialMatrix(1, [(2, 4)], csr([[8], [9, 10]]))
    return p0, p1


def test_gather_and_verify_stacks_and_detects_gaps():
    p0, p1 = _toy_partials()
    full = gather_and_verify([p1, p0], 6)
    assert full.row_ptr.tolist() == [0, 2, 3, 4, 6, 9, 10]
    assert full.values.tolist() == [1, 2, 3, 8, 9, 10, 4, 5, 6, 7]
    with pytest.raises(AssemblyError):
        gather_and_verify([p0], 6)
    with pytest.raises(AssemblyError):
        gather_and_verify([p0, p1, p1], 6)
    load = gather_load([np.array([1.0, 2, 5, 6]), np.array([3.0, 4])], [p0, p1], 6)
    assert load.tolist() == [1, 2, 3, 4, 5, 6]


def test_dofmap_and_csr_helpers():
    pm = F.one_square()
    dm = DofMap.from_specs(build_basis(pm, 3))
    assert dm.n_dofs == 10 and dm.count(0) == 10
    m = CSRMatrix(2, 3, np.array([0, 2, 3]), np.array([0, 2, 1]), np.array([1.0, 2.0, 3.0]))
    m.validate()
    bad = CSRMatrix(2, 3, np.array([0, 2, 3]), np.array([2, 0, 1]), np.array([1.0, 2.0, 3.0]))
    with pytest.raises(AssemblyError):
        bad.validate()
    assert m.max_relative_difference(m) == 0.0


# ---- per-rank sub-meshes (owned + one-ring halo) -----------------------------------

def _local_rows_equal_global(pm, coeffs, specs, n_parts, cfg=None):
    from oracle import sipg as oracle
    from paper_2007_04881_b200.assembly import AssemblyConfig, DofMap
    from paper_2007_04881_b200.distribute import local_problem
    from paper_2007_04881_b200.mesh import PolytopicMesh

    cfg = cfg or AssemblyConfig()
    part = contiguous_partition(pm, n_parts, quadrature_cost_weights(pm, specs))
    gdm = DofMap.from_specs(specs)
    cov = cfg.penalty.coverable
    for r in range(n_parts):
        own = part.owned[r]
        grp, gci, gv, grhs = oracle.assemble(pm, coeffs, specs, cfg.quad_increment, cfg.penalty.constant, cov,
                                             row_elements=own)
        lp = local_problem(pm, part, r, specs, cfg)
        assert lp.flat.n_elements < pm.n_elements or n_parts == 1
        lpm = PolytopicMesh.from_flat(lp.flat)
        lrp, lci, lv, lrhs = oracle.assemble(lpm, coeffs, lp.specs, cfg.quad_increment, cfg.penalty.constant,
                                             lp.config.penalty.coverable, row_elements=lp.owned_local)
        assert np.array_equal(lrp, grp)
        assert np.array_equal(lv, gv)  # bit for bit
        ldm = DofMap.from_specs(lp.specs)
        j = np.searchsorted(ldm.offsets, lci, "right") - 1
        assert np.array_equal(lp.col_dof[j] + (lci - ldm.offsets[j]), gci)
        lo = np.concatenate([np.arange(ldm.offsets[e], ldm.offsets[e + 1]) for e in lp.owned_local])
        go = np.concatenate([np.arange(gdm.offsets[e], gdm.offsets[e + 1]) for e in own])
        assert np.array_equal(lrhs[lo], grhs[go])


def test_submesh_rows_bit_identical_2d():
    """A rank's sub-mesh (owned + halo, monotone relabelling) reproduces the
    whole mesh's rows bit for bit, columns mapped through col_dof (oracle)."""
    import fixtures as F

    pm = voronoi_mesh(300, seed=3)
    coeffs = F.adr(2)
    classify_boundary_faces(pm, coeffs)
    _local_rows_equal_global(pm, coeffs, build_basis(pm, 2), 3)


def test_submesh_rows_bit_identical_3d_variable_degree_coverable():
    import fixtures as F
    from paper_2007_04881_b200.assembly import AssemblyConfig
    from paper_2007_04881_b200.mesh import agglomerate
    from paper_2007_04881_b200.model import PenaltyConfig

    g = F.cube_grid(3)
    pm = agglomerate(g, F.grown_clusters(g, 11, seed=3))
    coeffs = F.anisotropic(3)
    classify_boundary_faces(pm, coeffs, lambda x: x[0] < 0.5)
    deg = np.arange(pm.n_elements) % 2 + 1
    cov = np.arange(pm.n_elements) % 3 == 0
    _local_rows_equal_global(pm, coeffs, build_basis(pm, deg), 2,
                             AssemblyConfig(penalty=PenaltyConfig(constant=9.0, coverable=cov)))


def test_block_pattern_from_adjacency_matches_per_element_build():
    """Vectorised BlockPattern (ragged views of the device adjacency) equals the
    per-element construction of polydg (assembly.py:207-272); block_slots
    addresses the CSR exactly and misses raise PatternMissError."""
    from paper_2007_04881_b200.assembly import BlockPattern, DofMap, PatternMissError

    rng = np.random.default_rng(0)
    nel = 40
    deg = rng.integers(0, 4, nel)
    counts = np.array([(p + 1) * (p + 2) // 2 for p in deg], np.int64)
    dm = DofMap(np.concatenate([[0], np.cumsum(counts)]).astype(np.int64))
    adj = [sorted({e} | set(rng.choice(nel, rng.integers(1, 6), replace=False).tolist())) for e in range(nel)]
    nbr_ptr = np.concatenate([[0], np.cumsum([len(a) for a in adj])]).astype(np.int64)
    nbr_elem = np.concatenate(adj).astype(np.int32)
    rows = np.array([1, 4, 5, 17, 39])
    lens = np.concatenate([np.full(counts[e], counts[adj[e]].sum()) for e in rows])
    row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    col_idx = np.concatenate([np.tile(np.concatenate([np.arange(dm.offsets[j], dm.offsets[j + 1])
                                                      for j in adj[e]]), counts[e]) for e in rows])
    bp = BlockPattern.from_adjacency(dm, rows, nbr_ptr, nbr_elem, row_ptr, col_idx)
    assert len(bp.neighbors) == rows.size and bp.nnz == col_idx.size
    for k, e in enumerate(rows):
        assert np.array_equal(bp.neighbors[k], adj[e])
        st = np.concatenate([[0], np.cumsum(counts[adj[e]])[:-1]])
        assert np.array_equal(bp.col_starts[k], st)
        assert bp.local_block_start(int(e)) == k
        for j in adj[e]:
            slots = bp.block_slots(int(e), int(j))
            assert np.array_equal(col_idx[slots], np.broadcast_to(np.arange(dm.offsets[j], dm.offsets[j + 1]),
                                                                  slots.shape))
    assert np.array_equal(bp.global_rows, np.concatenate([np.arange(dm.offsets[e], dm.offsets[e + 1])
                                                          for e in rows]))
    with pytest.raises(PatternMissError):
        bp.block_slots(2, 2)
    missing = next(j for j in range(nel) if j not in adj[4])
    with pytest.raises(PatternMissError):
        bp.block_slots(4, missing)
