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
