"""Golden fixtures produced by the real reference (tests/golden/make_golden.py):
the oracle must reproduce them (CPU), and so must the CUDA engine (GPU)."""

import glob
import os

import numpy as np
import pytest

import fixtures as F
from compare import assert_parity
from oracle import sipg as oracle
from paper_2007_04881_b200 import build_basis, classify_boundary_faces
from paper_2007_04881_b200.mesh import SimplicialMesh, agglomerate

GOLDEN = sorted(p for p in glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))
                if not os.path.basename(p).startswith("slab_"))


def load_case(path):
    z = np.load(path, allow_pickle=False)
    base = SimplicialMesh(int(z["vertices"].shape[1]), z["vertices"], z["simplices"])
    pm = agglomerate(base, z["agg"])
    coeffs = getattr(F, str(z["coeffs"]))(base.dim)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, int(z["degree"]))
    ref = (z["row_ptr"], z["col_idx"], z["values"], z["rhs"])
    return pm, coeffs, specs, ref


class _CSR:
    def __init__(self, rp, ci, v):
        self.row_ptr, self.col_idx, self.values = rp, ci, v


@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_oracle_reproduces_reference_golden(path):
    pm, coeffs, specs, ref = load_case(path)
    rp, ci, v, r = oracle.assemble(pm, coeffs, specs)
    off = np.concatenate([[0], np.cumsum([s.n_funcs for s in specs])])
    # pinned tightly: the oracle restates the reference term by term
    assert_parity(_CSR(rp, ci, v), r, ref, off, tol=1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=lambda p: os.path.basename(p)[:-4])
def test_engine_reproduces_reference_golden(path):
    from paper_2007_04881_b200 import assemble_approach2

    pm, coeffs, specs, ref = load_case(path)
    m, rhs, _, pattern = assemble_approach2(pm, coeffs, specs)
    assert_parity(m, rhs, ref, pattern.dof_map.offsets)


def test_golden_set_present():
    assert len(GOLDEN) >= 8
