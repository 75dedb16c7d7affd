"""Known-answer tests of the reference suite, applied to the CPU oracle
(pins the oracle before it is trusted as the GPU checker).
Sources: pkg/tests/test_quadrature.py, test_basis.py, test_assembly.py,
test_model.py of the reference."""

import math

import numpy as np
import pytest

import fixtures as F
from oracle import sipg as O
from paper_2007_04881_b200 import build_basis, classify_boundary_faces
from paper_2007_04881_b200 import model as M


def exact_simplex_monomial(alpha):
    num = 1.0
    for a in alpha:
        num *= math.factorial(a)
    return num / math.factorial(sum(alpha) + len(alpha))


def monomials(d, order):
    if d == 1:
        return [(a,) for a in range(order + 1)]
    return [(a, *r) for a in range(order + 1) for r in monomials(d - 1, order - a)]


@pytest.mark.parametrize("d", [1, 2, 3])
@pytest.mark.parametrize("order", [0, 1, 2, 5, 8, 13, 20])
def test_rule_weight_sum_and_exactness(d, order):
    """test_quadrature.py:42-50."""
    x, w = O.simplex_rule(d, order)
    assert abs(w.sum() - 1.0 / math.factorial(d)) < 1e-14
    assert (w > 0).all()
    for al in monomials(d, order):
        approx = float(w @ np.prod(x ** np.array(al), axis=1))
        assert abs(approx - exact_simplex_monomial(al)) < 1e-13


def test_barycenter_and_x2y2():
    """test_quadrature.py:53-67."""
    x, w = O.simplex_rule(2, 1)
    np.testing.assert_allclose(x[0], [1 / 3, 1 / 3], atol=1e-15)
    assert abs(w[0] - 0.5) < 1e-15
    x, w = O.simplex_rule(2, 4)
    assert abs(float(w @ (x[:, 0] ** 2 * x[:, 1] ** 2)) - 1.0 / 180.0) < 1e-15


def test_interval_rule_points():
    """test_quadrature.py:78-87."""
    t, w = O.interval_rule(3)
    shift = 1.0 / (2.0 * math.sqrt(3.0))
    np.testing.assert_allclose(np.sort(t[:, 0]), [0.5 - shift, 0.5 + shift], atol=1e-15)
    np.testing.assert_allclose(w, [0.5, 0.5], atol=1e-15)


def test_map_hand_case_and_degeneracy():
    """test_quadrature.py:90-94, 114-117, 132-140."""
    pts, w = O.map_to_simplex(O.simplex_rule(2, 1), np.array([[0.0, 0.0], [2.0, 0.0], [0.0, 2.0]]))
    np.testing.assert_allclose(pts[0], [2 / 3, 2 / 3], atol=1e-14)
    assert abs(w[0] - 2.0) < 1e-14
    with pytest.raises(O.OracleQuadratureError):
        O.map_to_simplex(O.simplex_rule(2, 1), np.array([[0.0, 0.0], [1.0, 1.0], [2.0, 2.0]]))
    _, w = O.map_to_subsimplex(O.interval_rule(3), np.array([[0.0, 0.0], [3.0, 4.0]]))
    assert abs(w.sum() - 5.0) < 1e-13
    _, w3 = O.map_to_subsimplex(O.simplex_rule(2, 2), np.eye(3))
    assert abs(w3.sum() - math.sqrt(3.0) / 2.0) < 1e-14


def test_graded_lex_contract():
    """basis.py:9-16 ordering (test_basis.py:28-38)."""
    assert [tuple(r) for r in O.graded_lex(2, 2)] == [(0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0)]


def test_basis_constant_and_linear_modes():
    """test_basis.py:41-55: 1/sqrt|box| and sqrt(3)(2y-1) on the unit square."""
    box = np.array([[0.0, 0.0], [1.0, 1.0]])
    v, g = O.tabulate(1, box, np.array([[0.25, 0.75]]))
    assert abs(v[0, 0] - 1.0) < 1e-15
    assert abs(v[1, 0] - math.sqrt(3) * 0.5) < 1e-15      # (0,1): y mode
    assert abs(v[2, 0] - math.sqrt(3) * (-0.5)) < 1e-15   # (1,0): x mode
    np.testing.assert_allclose(g[1, :, 0], [0.0, 2 * math.sqrt(3)], atol=1e-14)
    v2, _ = O.tabulate(0, np.array([[0.0, 0.0], [2.0, 2.0]]), np.array([[0.3, 0.1]]))
    assert abs(v2[0, 0] - 0.5) < 1e-15


def test_basis_gradient_central_differences():
    """test_basis.py:75-98."""
    box = np.array([[0.1, -0.3, 0.0], [0.9, 0.4, 2.0]])
    x = np.array([[0.37, 0.11, 1.3]])
    v, g = O.tabulate(3, box, x)
    h = 1e-6
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        fd = (O.tabulate(3, box, x + e)[0] - O.tabulate(3, box, x - e)[0]) / (2 * h)
        np.testing.assert_allclose(g[:, k, 0], fd[:, 0], atol=1e-7)


def _square_mesh():
    return F.one_square()


def test_p0_stiffness_zero_and_mass_identity():
    """test_assembly.py:55-69."""
    pm = _square_mesh()
    diff = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2))
    mass = M.PdeCoefficients(reaction=M.constant_scalar(1.0))
    s0 = build_basis(pm, 0)[0]
    K, f = O.element_kernel(pm, 0, diff, s0)
    np.testing.assert_allclose(K, [[0.0]], atol=1e-15)
    for p in range(4):
        s = build_basis(pm, p)[0]
        K, _ = O.element_kernel(pm, 0, mass, s)
        np.testing.assert_allclose(K, np.eye(s.n_funcs), atol=1e-12)


def test_p1_stiffness_trace_24():
    """test_assembly.py:72-94 (sympy oracle: diag(0, 12, 12))."""
    pm = _square_mesh()
    K, _ = O.element_kernel(pm, 0, M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2)),
                            build_basis(pm, 1)[0])
    np.testing.assert_allclose(K, np.diag([0.0, 12.0, 12.0]), atol=1e-13)
    assert abs(np.trace(K) - 24.0) < 1e-12


def test_upwind_and_sigma_only_hand_cases():
    """test_assembly.py:97-124."""
    pm = F.two_squares()
    specs = build_basis(pm, 0)
    face = pm.faces[pm.interfaces[0].face_ids[0]]
    sp = [(0, specs[0].box), (0, specs[1].box)]
    adv = M.PdeCoefficients(advection=M.constant_vector([1.0, 0.0]))
    quads = O.Problem(pm, adv, specs).face_quads(face)
    up = O.Problem(pm, adv, specs).upwind(face)
    acc = np.zeros((2, 2))
    for pts, w in quads:
        B = O.interior_blocks(sp[0], sp[1], pts, w, face.normal, adv, 0.0, up)
        acc += np.array([[B[0][0][0, 0], B[0][1][0, 0]], [B[1][0][0, 0], B[1][1][0, 0]]])
    np.testing.assert_allclose(acc, [[0.0, 0.0], [-1.0, 1.0]], atol=1e-14)
    diff = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2))
    acc[:] = 0.0
    for pts, w in O.Problem(pm, diff, specs).face_quads(face):
        B = O.interior_blocks(sp[0], sp[1], pts, w, face.normal, diff, 7.5, -1, grad_terms=False)
        acc += np.array([[B[0][0][0, 0], B[0][1][0, 0]], [B[1][0][0, 0], B[1][1][0, 0]]])
    s = 7.5 * face.measure
    np.testing.assert_allclose(acc, [[s, -s], [-s, s]], atol=1e-12)


def test_boundary_kernel_hand_cases():
    """test_assembly.py:178-227: inflow +1/+1, Neumann 1, Dirichlet sign bookkeeping."""
    pm = _square_mesh()
    spec = build_basis(pm, 0)[0]
    fid = next(i for i in pm.boundary_face_ids() if np.allclose(pm.faces[i].normal, [-1.0, 0.0]))
    face = pm.faces[fid]
    C = M.PdeCoefficients(advection=M.constant_vector([1.0, 0.0]), dirichlet_data=M.constant_scalar(1.0))
    K, f = np.zeros((1, 1)), np.zeros(1)
    for pts, w in O.Problem(pm, C, [spec]).face_quads(face):
        k, l = O.inflow_block((0, spec.box), pts, w, face.normal, C)
        K += k
        f += l
    np.testing.assert_allclose([K[0, 0], f[0]], [1.0, 1.0], atol=1e-14)
    K[:] = 0.0
    f[:] = 0.0
    for pts, w in O.Problem(pm, C, [spec]).face_quads(face):
        k, l = O.dirichlet_block((0, spec.box), pts, w, face.normal, C, 0.0, True)
        K += k
        f += l
    np.testing.assert_allclose([K[0, 0], f[0]], [1.0, 1.0], atol=1e-14)
    N = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2), neumann_data=M.constant_scalar(1.0))
    f = sum(O.neumann_load((0, spec.box), pts, w, N) for pts, w in O.Problem(pm, N, [spec]).face_quads(face))
    np.testing.assert_allclose(f, [1.0], atol=1e-14)


def test_penalty_hand_values():
    """test_model.py:118-147: sigma = 20 (inf cap), 10 (coverable), 0 (no diffusion)."""
    pm = _square_mesh()
    spec = build_basis(pm, 1)[0]
    fid = next(i for i in pm.boundary_face_ids() if abs(pm.faces[i].measure - 1.0) < 1e-14)
    face = pm.faces[fid]
    diff = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2))
    prob = O.Problem(pm, diff, [spec], 2, 10.0)
    assert abs(prob.sigma(face) - 20.0) < 1e-12
    prob = O.Problem(pm, diff, [spec], 2, 10.0, np.array([True]))
    assert abs(prob.sigma(face) - 10.0) < 1e-12
    prob = O.Problem(pm, M.PdeCoefficients(), [spec], 2, 10.0)
    assert prob.sigma(face) == 0.0


def test_assembled_symmetry_and_spd():
    """test_assembly.py:411-437: symmetric form -> symmetric, SPD matrix."""
    from paper_2007_04881_b200.mesh import agglomerate

    g = F.square_grid(5)
    pm = agglomerate(g, F.grown_clusters(g, 9, seed=0))
    C = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2), reaction=M.constant_scalar(1.0))
    classify_boundary_faces(pm, C)
    specs = build_basis(pm, 2)
    rp, ci, v, _ = O.assemble(pm, C, specs)
    from scipy.sparse import csr_matrix

    Aa = csr_matrix((v, ci, rp)).toarray()
    assert np.max(np.abs(Aa - Aa.T)) < 1e-12 * np.max(np.abs(Aa))
    np.linalg.cholesky(0.5 * (Aa + Aa.T))


def test_partition_rows_equal_monolithic_oracle():
    """test_distribute.py:102-120 semantics at the oracle level."""
    from paper_2007_04881_b200.mesh import agglomerate

    g = F.square_grid(6)
    pm = agglomerate(g, F.grown_clusters(g, 12, seed=4))
    C = F.adr(2)
    classify_boundary_faces(pm, C)
    specs = build_basis(pm, 2)
    rp, ci, v, r = O.assemble(pm, C, specs)
    own = np.array([1, 4, 5, 9])
    prp, pci, pv, pr = O.assemble(pm, C, specs, row_elements=own)
    off = np.concatenate([[0], np.cumsum([s.n_funcs for s in specs])])
    loc = 0
    for e in own:
        for a in range(off[e], off[e + 1]):
            assert np.array_equal(pv[prp[loc]:prp[loc + 1]], v[rp[a]:rp[a + 1]])
            assert np.array_equal(pci[prp[loc]:prp[loc + 1]], ci[rp[a]:rp[a + 1]])
            loc += 1
        assert np.array_equal(pr[off[e]:off[e + 1]], r[off[e]:off[e + 1]])
