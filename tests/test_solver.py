"""Consumers of the device CSR: element-block SpMV and
block-Jacobi GMRES (polydg solver.py), Matrix Market IO (assembly.py:177-204)."""

import numpy as np
import pytest

import fixtures as F
from paper_2007_04881_b200 import assemble_approach2, build_basis, classify_boundary_faces
from paper_2007_04881_b200.assembly import CSRMatrix
from paper_2007_04881_b200.solver import read_matrix_market, write_matrix_market


def test_matrix_market_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    dense = np.where(rng.random((6, 5)) < 0.4, rng.standard_normal((6, 5)), 0.0)
    rows, cols = np.nonzero(dense)
    rp = np.zeros(7, np.int64)
    np.cumsum(np.bincount(rows, minlength=6), out=rp[1:])
    m = CSRMatrix(6, 5, rp, cols.astype(np.int64), dense[rows, cols])
    write_matrix_market(tmp_path / "a.mtx", m)
    b = read_matrix_market(tmp_path / "a.mtx")
    assert np.array_equal(b.row_ptr, m.row_ptr) and np.array_equal(b.col_idx, m.col_idx)
    assert np.array_equal(b.values, m.values)  # 17 significant digits: exact


def _system(coeff="poisson_sine", p=2):
    from paper_2007_04881_b200.mesh import agglomerate
    from paper_2007_04881_b200.meshgen import voronoi_mesh

    if coeff == "generic":  # b = (1 + x, 1) straddles some Voronoi faces: the grid clusters of the golden set
        g = F.square_grid(10)
        pm = agglomerate(g, F.grown_clusters(g, 23, seed=2))
    else:
        pm = voronoi_mesh(150, seed=1)
    C = getattr(F, coeff)(2)
    classify_boundary_faces(pm, C)
    specs = build_basis(pm, p)
    return assemble_approach2(pm, C, specs)


@pytest.mark.gpu
def test_blocked_spmv_matches_scipy():
    import torch

    from paper_2007_04881_b200.solver import DeviceSystem

    m, rhs, _, pattern = _system("adr", 3)
    sys_ = DeviceSystem(m, pattern.dof_map.offsets)
    x = np.random.default_rng(2).standard_normal(m.n_rows)
    y = sys_.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    ref = m.to_scipy() @ x
    assert np.allclose(y, ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())


@pytest.mark.gpu
@pytest.mark.parametrize("coeff", ["poisson_sine", "adr", "generic"])
def test_block_jacobi_gmres_solves(coeff):
    from paper_2007_04881_b200.solver import solve

    m, rhs, _, pattern = _system(coeff, 2)
    res = solve(m, rhs, tol=1e-10, dof_map=pattern.dof_map)
    assert res.converged and res.residual <= 1e-9
    x_ref = __import__("scipy.sparse.linalg", fromlist=["spsolve"]).spsolve(m.to_scipy().tocsc(), rhs)
    assert np.allclose(res.x, x_ref, rtol=1e-7, atol=1e-8 * np.abs(x_ref).max())


@pytest.mark.gpu
def test_block_inverses_against_numpy():
    import torch

    from paper_2007_04881_b200.solver import BlockJacobiPreconditioner, DeviceSystem

    m, _, _, pattern = _system("generic", 3)
    off = pattern.dof_map.offsets
    sys_ = DeviceSystem(m, off)
    pre = BlockJacobiPreconditioner(sys_)
    r = np.random.default_rng(3).standard_normal(m.n_rows)
    z = pre.apply(torch.from_numpy(r).cuda()).cpu().numpy()
    A = m.to_dense()
    for e in range(len(off) - 1):
        a, b = off[e], off[e + 1]
        ze = np.linalg.solve(A[a:b, a:b], r[a:b])
        assert np.allclose(z[a:b], ze, rtol=1e-10, atol=1e-12 * np.abs(ze).max())


@pytest.mark.gpu
def test_point_jacobi_zero_diagonal_substitutes_one():
    """polydg solver.py:102-104: a zero or missing diagonal entry acts as 1.0."""
    from paper_2007_04881_b200.solver import solve

    # [[0, 1, 0], [1, 2, 0], [0, 0, 3]] with row 0's diagonal missing from the pattern
    rp = np.array([0, 1, 3, 4], np.int64)
    ci = np.array([1, 0, 1, 2], np.int64)
    va = np.array([1.0, 1.0, 2.0, 3.0])
    m = CSRMatrix(3, 3, rp, ci, va)
    b = np.array([1.0, 2.0, 3.0])
    res = solve(m, b, tol=1e-12)
    assert res.converged
    assert np.allclose(res.x, np.linalg.solve(m.to_dense(), b), rtol=1e-10)


@pytest.mark.gpu
def test_block_jacobi_on_unstructured_csr_keeps_element_blocks():
    """A CSR without the assembled block structure (a dropped entry) still gets
    element-block Jacobi (polydg extracts the blocks from any CSR)."""
    from paper_2007_04881_b200.solver import BlockJacobiPreconditioner, _host_diagonal_blocks, solve

    m, rhs, _, pattern = _system("adr", 2)
    sp = m.to_scipy().tolil()
    r0 = int(pattern.dof_map.offsets[3])
    far = [c for c in sp.rows[r0] if c >= int(pattern.dof_map.offsets[4]) or c < int(pattern.dof_map.offsets[3])]
    sp[r0, far[-1]] = 0.0
    sp = sp.tocsr()
    sp.eliminate_zeros()
    m2 = CSRMatrix(m.n_rows, m.n_cols, sp.indptr.astype(np.int64), sp.indices.astype(np.int64), sp.data)
    blocks = _host_diagonal_blocks(m2, pattern.dof_map.offsets)
    A = m2.to_dense()
    off = pattern.dof_map.offsets
    for e in (0, 3, len(off) - 2):
        assert np.array_equal(blocks[e], A[off[e]:off[e + 1], off[e]:off[e + 1]])
    res = solve(m2, rhs, tol=1e-10, dof_map=pattern.dof_map)
    assert res.converged and res.residual <= 1e-9
