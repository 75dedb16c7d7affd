"""The single-item public kernels of polydg on the device:
interior_face_kernel / dirichlet_kernel / inflow_kernel /
neumann_outflow_kernel (assembly.py:1160-1234), penalty_side_data /
penalty_sigma (model.py:196-257), triplets_to_csr (assembly.py:1002-1031),
and the unit ABIs pdg_map_simplices / pdg_tabulate / pdg_eval_coeffs.

Two kinds of checks: the reference suite's hand cases
(pkg/tests/test_assembly.py:97-227, test_model.py:118-147) and face-by-face
parity with the CPU oracle on agglomerated meshes."""

import numpy as np
import pytest

import fixtures as F
from oracle import sipg as O
from paper_2007_04881_b200 import (
    AssemblyConfig,
    AssemblyError,
    BasisSpec,
    Family,
    PenaltyConfig,
    assemble_approach1,
    build_basis,
    classify_boundary_faces,
    dirichlet_kernel,
    element_kernel,
    inflow_kernel,
    interior_face_kernel,
    neumann_outflow_kernel,
    penalty_side_data,
    penalty_sigma,
    triplets_to_csr,
)
from paper_2007_04881_b200 import model as M
from paper_2007_04881_b200.mesh import BoundaryTag, agglomerate

# ---- CPU: host-side contract of triplets_to_csr ------------------------------------


def test_triplets_to_csr_empty_and_bounds_without_a_gpu():
    m = triplets_to_csr([], [], [], 3, 4)
    assert m.nnz == 0 and np.array_equal(m.row_ptr, np.zeros(4, np.int64))
    m = triplets_to_csr([-1, -1], [0, 1], [1.0, 2.0], 3, 4, sentinel=-1)
    assert m.nnz == 0
    with pytest.raises(AssemblyError):
        triplets_to_csr([0, 3], [0, 0], [1.0, 1.0], 3, 4)
    with pytest.raises(AssemblyError):
        triplets_to_csr([0, 1], [0, 4], [1.0, 1.0], 3, 4)


# ---- GPU --------------------------------------------------------------------------

gpu = pytest.mark.gpu


@gpu
def test_triplets_to_csr_matches_oracle_with_duplicates_and_sentinels():
    rng = np.random.default_rng(0)
    n_rows, n_cols, n = 50, 40, 5000
    rows = rng.integers(0, n_rows, n)
    cols = rng.integers(0, n_cols, n)
    vals = rng.standard_normal(n)
    rows[::17] = -7  # sentinel stripes (assembly.py:158-174)
    m = triplets_to_csr(rows, cols, vals, n_rows, n_cols, n_workers=4, sentinel=-7)
    rp, ci, v = O.triplets_to_csr(rows, cols, vals, n_rows, n_cols, sentinel=-7)
    assert np.array_equal(m.row_ptr, rp) and np.array_equal(m.col_idx, ci)
    # duplicates summed in stable input order: bit-identical to np.add.reduceat
    assert np.array_equal(m.values, v)
    m.validate()


@gpu
def test_interior_face_upwind_hand_case():
    """test_assembly.py:97-107: b = (1,0) across two unit squares."""
    pm = F.two_squares()
    coeffs = M.PdeCoefficients(advection=M.constant_vector([1.0, 0.0]))
    specs = build_basis(pm, 0)
    face = pm.faces[pm.interfaces[0].face_ids[0]]
    oo, on, no, nn = interior_face_kernel(pm, face, coeffs, specs[0], specs[1], 0.0)
    np.testing.assert_allclose(oo, [[0.0]], atol=1e-14)
    np.testing.assert_allclose(on, [[0.0]], atol=1e-14)
    np.testing.assert_allclose(nn, [[1.0]], atol=1e-14)
    np.testing.assert_allclose(no, [[-1.0]], atol=1e-14)


@gpu
def test_interior_face_sigma_only_pattern():
    """test_assembly.py:110-124: gradient terms off -> sigma |F| [+1 -1; -1 +1]."""
    pm = F.two_squares()
    coeffs = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2))
    specs = build_basis(pm, 0)
    face = pm.faces[pm.interfaces[0].face_ids[0]]
    oo, on, no, nn = interior_face_kernel(pm, face, coeffs, specs[0], specs[1], 7.5,
                                          include_gradient_terms=False)
    s = 7.5 * face.measure
    for blk, ref in ((oo, s), (nn, s), (on, -s), (no, -s)):
        np.testing.assert_allclose(blk, [[ref]], atol=1e-12)


@gpu
def test_boundary_kernels_hand_cases():
    """test_assembly.py:178-212: inflow +1/+1, zero data, Neumann 1, outflow 0."""
    pm = F.one_square()
    spec = BasisSpec(0, Family.P, pm.bounding_boxes[0])
    face = next(pm.faces[f] for f in pm.boundary_face_ids() if np.allclose(pm.faces[f].normal, [-1.0, 0.0]))
    C = M.PdeCoefficients(advection=M.constant_vector([1.0, 0.0]), dirichlet_data=M.constant_scalar(1.0))
    block, load = inflow_kernel(pm, face, C, spec)
    np.testing.assert_allclose(block, [[1.0]], atol=1e-14)
    np.testing.assert_allclose(load, [1.0], atol=1e-14)
    C0 = M.PdeCoefficients(advection=M.constant_vector([1.0, 0.0]), dirichlet_data=M.constant_scalar(0.0))
    block0, load0 = inflow_kernel(pm, face, C0, spec)
    np.testing.assert_allclose(block0, block)
    np.testing.assert_allclose(load0, [0.0], atol=1e-15)
    neu = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2), neumann_data=M.constant_scalar(1.0))
    face.tag = BoundaryTag.NEUMANN
    np.testing.assert_allclose(neumann_outflow_kernel(pm, face, neu, spec), [1.0], atol=1e-14)
    face.tag = BoundaryTag.OUTFLOW
    np.testing.assert_allclose(neumann_outflow_kernel(pm, face, neu, spec), [0.0])
    face.tag = BoundaryTag.INTERIOR


@gpu
def test_dirichlet_kernel_sign_bookkeeping():
    """test_assembly.py:215-227: p=0, A=0, b.n=-1, g=1: diagonal += 1, load += 1."""
    pm = F.one_square()
    spec = BasisSpec(0, Family.P, pm.bounding_boxes[0])
    face = next(pm.faces[f] for f in pm.boundary_face_ids() if np.allclose(pm.faces[f].normal, [-1.0, 0.0]))
    C = M.PdeCoefficients(advection=M.constant_vector([1.0, 0.0]), dirichlet_data=M.constant_scalar(1.0))
    block, load = dirichlet_kernel(pm, face, C, spec, sigma=0.0)
    np.testing.assert_allclose(block, [[1.0]], atol=1e-14)
    np.testing.assert_allclose(load, [1.0], atol=1e-14)


@gpu
def test_patch_contraction_continuous_functions():
    """test_assembly.py:127-175: interior-face terms cancel on continuous
    linear traces: v.(A u) with the full matrix == with volume + boundary only."""
    from paper_2007_04881_b200.kernels import face_sigma, map_simplices, tabulate
    from paper_2007_04881_b200.mesh import SimplicialMesh

    mesh = SimplicialMesh(2, np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]]),
                          np.array([[0, 1, 2], [0, 2, 3]]))
    coeffs = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2))
    pm = agglomerate(mesh, np.array([0, 1]))
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 1)
    config = AssemblyConfig(penalty=PenaltyConfig(constant=10.0))
    full, _, _ = assemble_approach1(pm, coeffs, specs, config)
    sig, _ = face_sigma(pm, coeffs, specs, config)
    no_int = np.zeros((6, 6))
    for el in (0, 1):
        block, _ = element_kernel(pm, el, coeffs, specs[el])
        no_int[3 * el:3 * el + 3, 3 * el:3 * el + 3] = block
    for fid in pm.boundary_face_ids():
        f = pm.faces[fid]
        block, _ = dirichlet_kernel(pm, f, coeffs, specs[f.owner], sig[fid])
        no_int[3 * f.owner:3 * f.owner + 3, 3 * f.owner:3 * f.owner + 3] += block

    def interpolant(fn):
        coefs = np.zeros(6)
        for el in (0, 1):
            gram, rhs = np.zeros((3, 3)), np.zeros(3)
            pts, w = map_simplices(pm, list(pm.elements[el]), 4)
            for s in range(pts.shape[0]):
                vals, _ = tabulate(specs[el], pts[s])
                gram += np.einsum("q,iq,jq->ij", w[s], vals, vals)
                rhs += vals @ (w[s] * fn(pts[s]))
            coefs[3 * el:3 * el + 3] = np.linalg.solve(gram, rhs)
        return coefs

    u = interpolant(lambda p: 2.0 * p[:, 0] - 3.0 * p[:, 1] + 0.25)
    v = interpolant(lambda p: -1.0 * p[:, 0] + 0.5 * p[:, 1] + 1.0)
    lhs = v @ (full.to_dense() @ u)
    rhs = v @ (no_int @ u)
    assert abs(lhs - rhs) < 1e-12 * max(1.0, abs(rhs))


@gpu
def test_penalty_hand_values():
    """test_model.py:118-147: sigma = 20 (inf cap), 10 (coverable), 0 (no diffusion)."""
    pm = F.one_square()
    spec = build_basis(pm, 1)[0]
    fid = next(i for i in pm.boundary_face_ids() if abs(pm.faces[i].measure - 1.0) < 1e-14)
    face = pm.faces[fid]
    from paper_2007_04881_b200.kernels import map_simplices

    pts, _ = map_simplices(pm, list(pm.elements[0]), 2 * 1 + 2)
    pts = pts.reshape(-1, 2)
    diff = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2))
    cfg = PenaltyConfig(constant=10.0)
    sd = penalty_side_data(pm, 0, face, 1, pts, diff, cfg)
    assert abs(penalty_sigma(face, sd, None, cfg) - 20.0) < 1e-12
    cov = PenaltyConfig(constant=10.0, coverable=np.array([True]))
    sd = penalty_side_data(pm, 0, face, 1, pts, diff, cov)
    assert abs(penalty_sigma(face, sd, None, cov) - 10.0) < 1e-12
    sd = penalty_side_data(pm, 0, face, 1, pts, M.PdeCoefficients(), cfg)
    assert penalty_sigma(face, sd, None, cfg) == 0.0


def _mesh(name):
    if name == "clusters10":
        g = F.square_grid(10)
        return agglomerate(g, F.grown_clusters(g, 23, seed=2))
    g = F.cube_grid(3)
    return agglomerate(g, F.grown_clusters(g, 11, seed=3))


def _close(a, b, tol=1e-12):
    scale = max(np.abs(b).max(), 1e-300)
    assert np.abs(a - b).max() <= tol * scale, (np.abs(a - b).max(), scale)


@gpu
@pytest.mark.parametrize("name,p,coeff", [("clusters10", 2, "generic"), ("clusters10", 3, "adr"),
                                          ("cube3", 2, "generic"), ("cube3", 1, "anisotropic")])
def test_face_kernels_match_oracle_face_by_face(name, p, coeff):
    """Every interior / Dirichlet / Neumann face of an agglomerated mesh:
    device unit kernels == oracle blocks summed over sub-facets (1e-12 per block)."""
    from paper_2007_04881_b200.kernels import face_sigma

    pm = _mesh(name)
    C = getattr(F, coeff)(pm.dim)
    pred = (lambda x: x[0] < 0.5) if coeff == "anisotropic" else None
    classify_boundary_faces(pm, C, pred)
    specs = build_basis(pm, p)
    prob = O.Problem(pm, C, specs)
    sig, flow = face_sigma(pm, C, specs)
    faces = pm.faces
    for fid in range(len(faces))[:: max(1, len(faces) // 40)]:
        f = faces[fid]
        sref = prob.sigma(f)
        if f.neighbor >= 0 or f.tag == BoundaryTag.DIRICHLET:  # the faces whose sigma the assembly reads
            assert abs(sig[fid] - sref) <= 1e-12 * max(abs(sref), 1e-300), (fid, sig[fid], sref)
        if f.neighbor >= 0:
            up = prob.upwind(f)
            got = interior_face_kernel(pm, f, C, specs[f.owner], specs[f.neighbor], sref)
            acc = None
            for pts, w in prob.face_quads(f):
                B = O.interior_blocks(prob.sp(f.owner), prob.sp(f.neighbor), pts, w, f.normal, C, sref, up)
                blk = [B[0][0], B[0][1], B[1][0], B[1][1]]
                acc = blk if acc is None else [a + b for a, b in zip(acc, blk)]
            for g_, r_ in zip(got, acc):
                _close(g_, r_)
            # explicit upwind side and gradient terms off
            got = interior_face_kernel(pm, f, C, specs[f.owner], specs[f.neighbor], 3.0,
                                       include_gradient_terms=False, upwind_side=1)
            acc = None
            for pts, w in prob.face_quads(f):
                B = O.interior_blocks(prob.sp(f.owner), prob.sp(f.neighbor), pts, w, f.normal, C, 3.0, 1,
                                      grad_terms=False)
                blk = [B[0][0], B[0][1], B[1][0], B[1][1]]
                acc = blk if acc is None else [a + b for a, b in zip(acc, blk)]
            for g_, r_ in zip(got, acc):
                _close(g_, r_)
        elif f.tag == BoundaryTag.DIRICHLET:
            wi = C.advection is not None and O.flow_is_inflow(pm, f.owner, f, C)
            K, L = dirichlet_kernel(pm, f, C, specs[f.owner], sref)
            Kr, Lr = 0.0, 0.0
            for pts, w in prob.face_quads(f):
                k, l = O.dirichlet_block(prob.sp(f.owner), pts, w, f.normal, C, sref, wi)
                Kr, Lr = Kr + k, Lr + l
            _close(K, Kr)
            _close(L, Lr)
        elif f.tag == BoundaryTag.NEUMANN:
            L = neumann_outflow_kernel(pm, f, C, specs[f.owner])
            Lr = sum(O.neumann_load(prob.sp(f.owner), pts, w, C) for pts, w in prob.face_quads(f))
            _close(L, Lr)


@gpu
@pytest.mark.parametrize("name", ["clusters10", "cube3"])
def test_face_sigma_matches_oracle_on_every_face(name):
    from paper_2007_04881_b200.kernels import face_sigma

    pm = _mesh(name)
    C = F.variable_diffusion(2) if pm.dim == 2 else F.anisotropic(3)
    classify_boundary_faces(pm, C)
    specs = build_basis(pm, 2)
    cov = np.arange(pm.n_elements) % 3 == 0
    cfg = AssemblyConfig(penalty=PenaltyConfig(constant=7.0, coverable=cov))
    sig, _ = face_sigma(pm, C, specs, cfg)
    prob = O.Problem(pm, C, specs, 2, 7.0, cov)
    ref = np.array([prob.sigma(f) for f in pm.faces])
    assert np.all(np.abs(sig - ref) <= 1e-13 * np.abs(ref))


@gpu
@pytest.mark.parametrize("name,order", [("clusters10", 2), ("clusters10", 9), ("cube3", 4), ("cube3", 6)])
def test_map_simplices_matches_oracle(name, order):
    """pdg_map_simplices vs map_to_simplex (quadrature.py:118-136) for every simplex."""
    from paper_2007_04881_b200.kernels import map_simplices

    pm = _mesh(name)
    d = pm.dim
    ids = np.arange(pm.base.simplices.shape[0])
    pts, w = map_simplices(pm, ids, order)
    rule = O.simplex_rule(d, order)
    for s in ids:
        rp, rw = O.map_to_simplex(rule, pm.base.vertices[pm.base.simplices[s]])
        np.testing.assert_allclose(pts[s], rp, rtol=0, atol=4e-16)
        np.testing.assert_allclose(w[s], rw, rtol=2e-15, atol=0)


@gpu
@pytest.mark.parametrize("d,p", [(2, 0), (2, 1), (2, 3), (2, 6), (3, 0), (3, 2), (3, 4)])
def test_tabulate_matches_oracle(d, p):
    """pdg_tabulate vs basis.tabulate (basis.py:129-164) at random points of
    the box and outside it (polytopes exceed their sub-boxes only at 0 here)."""
    from paper_2007_04881_b200.kernels import tabulate

    rng = np.random.default_rng(10 * d + p)
    lo = rng.uniform(-1, 0, d)
    box = np.stack([lo, lo + rng.uniform(0.01, 2.0, d)])
    pts = box[0] + rng.uniform(-0.1, 1.1, (57, d)) * (box[1] - box[0])
    spec = BasisSpec(p, Family.P, box)
    v, g = tabulate(spec, pts)
    rv, rg = O.tabulate(p, box, pts)
    assert v.shape == rv.shape and g.shape == rg.shape
    sv = max(np.abs(rv).max(), 1e-300)
    sg = max(np.abs(rg).max(), 1e-300)
    assert np.abs(v - rv).max() <= 1e-14 * sv
    assert np.abs(g - rg).max() <= 1e-14 * sg


@gpu
def test_eval_coefficients_matches_numpy():
    """pdg_eval_coeffs (interpreted fields) vs the numpy evaluation of the same Expr."""
    from paper_2007_04881_b200.kernels import eval_coefficients

    rng = np.random.default_rng(5)
    for C, d in ((F.advdiff3d(3), 3), (F.anisotropic(2), 2), (F.sine_dirichlet(2), 2)):
        pts = rng.uniform(0, 1, (200, d))
        pts[:5, 0] = 1.0  # on the boundary: sin(fl(pi)) = 1.2e-16, not 0
        got = eval_coefficients(C, pts)
        if C.dirichlet_data is not None:
            ref = C.dirichlet_data(pts)
            np.testing.assert_allclose(got["dirichlet"], ref, rtol=1e-15, atol=1e-300)  # libm vs CUDA sin: ulps
            assert np.all(got["dirichlet"][:5] != 0.0)
        np.testing.assert_allclose(got["source"], C.source(pts), rtol=1e-15, atol=1e-15)
        np.testing.assert_allclose(got["diffusion"], C.diffusion(pts), rtol=1e-15, atol=0)
