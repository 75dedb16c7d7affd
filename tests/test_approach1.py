"""Approach 1 (stage-and-sort) on the device: per-item triplet stripes +
stable radix sort + reduce-by-key (polydg assembly.py:158-174, 977-1087).
Parity: the reference's own contract A1 == A2 within 1e-12
(test_assembly.py:379-389, test_acceptance.py:170-182), the golden fixtures,
and the merge against the oracle's restatement of triplets_to_csr."""

import glob
import os

import numpy as np
import pytest

import fixtures as F
from compare import assert_parity
from oracle import sipg as O
from paper_2007_04881_b200 import build_basis, classify_boundary_faces

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith("slab_"))


def test_oracle_triplet_merge_matches_dense_sum():
    rng = np.random.default_rng(0)
    n = 7
    rows = rng.integers(0, n, 200)
    cols = rng.integers(0, n, 200)
    vals = rng.standard_normal(200)
    rows[::17] = n  # sentinel
    rp, ci, v = O.triplets_to_csr(rows, cols, vals, n, n, sentinel=n)
    dense = np.zeros((n, n))
    keep = rows != n
    np.add.at(dense, (rows[keep], cols[keep]), vals[keep])
    got = np.zeros((n, n))
    for r in range(n):
        got[r, ci[rp[r]:rp[r + 1]]] = v[rp[r]:rp[r + 1]]
    assert np.allclose(got, dense, rtol=0, atol=1e-14)


@pytest.mark.gpu
def test_device_triplet_merge_against_oracle():
    import ctypes as C

    import torch

    from paper_2007_04881_b200 import _lib

    lib = _lib.load()
    rng = np.random.default_rng(1)
    n_rows, n_cols, m = 50, 40, 5000
    rows = rng.integers(0, n_rows, m)
    cols = rng.integers(0, n_cols, m)
    vals = rng.standard_normal(m)
    sent = rng.random(m) < 0.1
    keys = (rows * n_cols + cols).astype(np.uint64)
    keys[sent] = np.uint64(2 ** 64 - 1)
    rows_s = np.where(sent, n_rows, rows)
    rp, ci, v = O.triplets_to_csr(rows_s, cols, vals, n_rows, n_cols, sentinel=n_rows)
    dev = torch.device("cuda")
    tk = torch.from_numpy(keys.view(np.int64)).to(dev)
    tv = torch.from_numpy(vals).to(dev)
    ws_b = int(lib.pdg_triplets_workspace_bytes(m))
    ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
    orp = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    oci = torch.empty(m, dtype=torch.int64, device=dev)
    ov = torch.empty(m, dtype=torch.float64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    s = torch.cuda.current_stream()
    _lib.check(lib.pdg_triplets_to_csr(tk.data_ptr(), tv.data_ptr(), m, n_rows, n_cols, orp.data_ptr(),
                                       oci.data_ptr(), ov.data_ptr(), nnz.data_ptr(), ws.data_ptr(), ws_b,
                                       _lib.stream_ptr(s)))
    torch.cuda.synchronize()
    k = int(nnz.item())
    assert k == ci.size
    assert np.array_equal(orp.cpu().numpy(), rp)
    assert np.array_equal(oci[:k].cpu().numpy(), ci)
    assert np.array_equal(ov[:k].cpu().numpy(), v)  # numpy-order run sums: bit-identical


CASES = [("clusters10", lambda: F.square_grid(10), lambda g: F.grown_clusters(g, 23, seed=2)),
         ("cube3", lambda: F.cube_grid(3), lambda g: F.grown_clusters(g, 11, seed=3))]


@pytest.mark.gpu
@pytest.mark.parametrize("mesh_case", CASES, ids=lambda c: c[0])
@pytest.mark.parametrize("coeff", ["generic", "poisson_sine", "adr", "hyperbolic", "anisotropic"])
@pytest.mark.parametrize("p", [1, 2])
def test_approach1_equals_approach2(mesh_case, coeff, p):
    from paper_2007_04881_b200 import assemble_approach1, assemble_approach2
    from paper_2007_04881_b200.mesh import agglomerate

    _, mk, agg = mesh_case
    base = mk()
    pm = agglomerate(base, agg(base))
    C = getattr(F, coeff)(base.dim)
    classify_boundary_faces(pm, C)
    specs = build_basis(pm, p)
    m1, r1, s1 = assemble_approach1(pm, C, specs)
    m2, r2, s2, pattern = assemble_approach2(pm, C, specs)
    assert np.array_equal(m1.row_ptr, m2.row_ptr) and np.array_equal(m1.col_idx, m2.col_idx)
    assert m1.max_relative_difference(m2) <= 1e-12
    assert_parity(m1, r1, (m2.row_ptr, m2.col_idx, m2.values, r2), pattern.dof_map.offsets)
    assert s1.triplet_count > s1.nnz == m1.nnz  # duplicates merged


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_approach1_reproduces_reference_golden(path):
    from paper_2007_04881_b200 import assemble_approach1
    from test_oracle_golden import load_case

    pm, coeffs, specs, ref = load_case(path)
    m, rhs, _ = assemble_approach1(pm, coeffs, specs)
    off = np.concatenate([[0], np.cumsum([s.n_funcs for s in specs])])
    assert_parity(m, rhs, ref, off)
