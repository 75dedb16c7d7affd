"""Parity at the BASELINE.json workload sizes (cfg1..cfg5, full meshes) by
the patch-oracle property of SURVEY §8c: any element's rows depend only on
the element and its face neighbours, so a seeded sample of elements of the
full-size device assembly is compared block by block with the oracle's
rows for those elements (values <= 1e-12 relative per block, columns and
RHS segments), plus the size-independent invariants of the whole CSR
(row_ptr = element row-length prefix, strictly increasing columns).

Sizes: cfg1 1k, cfg2 100k, cfg3 250k (p = 2..6), cfg4 207k (3D), cfg5 4M cells."""

import numpy as np
import pytest

from oracle import sipg as O

REL = 1e-12


def _sample(flat, k, seed):
    rng = np.random.default_rng(seed)
    nel = flat.n_elements
    bnd = np.unique(flat.face_owner[flat.face_neighbor < 0])
    pick = rng.choice(nel, size=min(k, nel), replace=False)
    extra = rng.choice(bnd, size=min(8, bnd.size), replace=False) if bnd.size else np.zeros(0, np.int64)
    return np.unique(np.concatenate([pick, extra, [0, nel - 1]]).astype(np.int64))


def _faces_index(flat, els):
    """oracle face lookup restricted to the sampled elements (the oracle's
    own index enumerates every face object of the mesh)."""
    out = {}
    own, nb = flat.face_owner, flat.face_neighbor
    for e in els:
        f = np.flatnonzero((own == e) | (nb == e))
        out[int(e)] = [int(x) for x in f]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3p2", "cfg3p3", "cfg3", "cfg3p5", "cfg3p6", "cfg4", "cfg5"])
def test_fullsize_sampled_rows_against_oracle(cfg):
    import torch

    from paper_2007_04881_b200 import build_basis, classify_boundary_faces
    from paper_2007_04881_b200.assembly import SipgPlan
    from paper_2007_04881_b200.problems import WORKLOADS, cached_mesh, coefficients

    w = WORKLOADS[cfg]
    pm = cached_mesh(w)
    coeffs = coefficients(w.coeffs, w.dim)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, w.degree)
    plan = SipgPlan(pm, coeffs, specs)
    plan.run()
    plan.check_flags()
    flat = plan.flat
    off = plan.dof.offsets
    counts = np.diff(off)

    # whole-CSR invariants
    rp = plan.row_ptr.cpu().numpy()
    assert rp[0] == 0 and rp[-1] == plan.nnz
    lens = np.diff(rp)
    assert np.all(lens > 0)
    row_len = plan.t["row_len"].cpu().numpy()
    assert np.array_equal(lens, np.repeat(row_len, counts))

    els = _sample(flat, 48 if cfg != "cfg5" else 32, seed=int(cfg[3]) * 10 + w.degree)
    O._FACE_INDEX[id(pm)] = (pm, _faces_index(flat, els))
    # oracle problem from the spec arrays (no per-element Python objects for 4M cells)
    prob = O.Problem.__new__(O.Problem)
    prob.mesh, prob.C, prob.deg, prob.box = pm, coeffs, specs.degrees, specs.boxes
    prob.n, prob.off = counts, off
    prob.inc, prob.pen, prob.cov, prob.d, prob._vpts = 2, 10.0, None, flat.dim, {}
    val_off = plan.t["val_off"].cpu().numpy()
    nbr_ptr = plan.t["nbr_ptr"].cpu().numpy()
    nbr_elem = plan.t["nbr_elem"].cpu().numpy()
    values, col_idx, rhs = plan.values, plan.col_idx, plan.rhs
    worst = 0.0
    for e in els:
        e = int(e)
        ne = int(counts[e])
        L = int(row_len[e])
        a, b = int(val_off[e]), int(val_off[e + 1])
        v = values[a:b].cpu().numpy().reshape(ne, L)
        c = col_idx[a:b].cpu().numpy().reshape(ne, L)
        blocks, r = O.element_rows(prob, e)
        nbrs = nbr_elem[nbr_ptr[e]:nbr_ptr[e + 1]]
        assert sorted(blocks) == sorted(int(j) for j in nbrs), (cfg, e)
        col = 0
        for j in nbrs:
            j = int(j)
            nj = int(counts[j])
            assert np.array_equal(c[:, col:col + nj], np.broadcast_to(np.arange(off[j], off[j + 1]), (ne, nj)))
            ref = blocks[j]
            got = v[:, col:col + nj]
            scale = max(np.abs(ref).max(), 1e-300)
            err = np.abs(got - ref).max() / scale
            worst = max(worst, err)
            assert err <= REL, (cfg, e, j, err)
            col += nj
        rr = rhs[int(off[e]):int(off[e + 1])].cpu().numpy()
        if np.abs(r).max() > 0:
            assert np.abs(rr - r).max() / np.abs(r).max() <= REL, (cfg, e)
    del O._FACE_INDEX[id(pm)]
    torch.cuda.empty_cache()
    print(f"{cfg}: {len(els)} sampled elements, worst block rel err {worst:.2e}")
