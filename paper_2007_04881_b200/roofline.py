"""Algorithmic work of one assembly -- the numerators of the
roofline fractions bench.py reports.

FLOPs are the canonical dense ``B^T diag(w) B`` contraction counts (FMA = 2),
independent of how the kernel organises them (symmetry savings, the upwind
terms folded into the penalty item, DMMA padding are NOT credited):

* volume sub-simplex:     2 n^2 nq_v (d + [b != 0] + [c != 0])
* interior sub-facet:     (16 + 4 [b != 0]) n^2 nq_f   (n = max of the two sides)
* Dirichlet sub-facet:    (4 + 2 [inflow]) n^2 nq_f
* inflow sub-facet:       2 n^2 nq_f

For a row-partitioned assembly an interior sub-facet counts (owned sides)/2
of its work, so the per-rank counts sum to the monolithic count.

Bytes are the compulsory HBM traffic: CSR values and col_idx written once
(8 B each per stored entry), the RHS, row_ptr, and the geometry reads
(simplex vertex coordinates, facet coordinates).
"""

from __future__ import annotations

import numpy as np

from .basis import num_basis
from .mesh import BOUNDARY, TAG_CODE
from .quadrature import points_per_axis


def _nq(order: np.ndarray, dim: int) -> np.ndarray:
    return ((order + 2) // 2).astype(np.float64) ** dim


def assembly_work(plan) -> dict:
    """-> {"flops": ..., "bytes": ..., "flops_element_kernel": ...} for a SipgPlan."""
    f = plan.flat
    d = f.dim
    deg = plan.degrees
    inc = plan.config.quad_increment
    desc = plan.cdesc
    nb = np.array([num_basis(int(p), d) for p in range(int(deg.max()) + 1)], np.float64)
    n = nb[deg]
    owned = np.zeros(f.n_elements, bool)
    owned[plan.row_elements] = True
    has_b = bool(desc["has_advection"])
    has_c = bool(desc["has_reaction"])
    has_a = desc["diffusion_kind"] != 0
    items = (d if has_a else 0) + int(has_b) + int(has_c)
    nsim = np.diff(f.elem_ptr).astype(np.float64)
    nqv = _nq(2 * deg + inc, d)
    vol = float(np.sum((nsim * 2.0 * n * n * nqv * items)[owned]))

    nfac = np.diff(f.face_ptr).astype(np.float64)
    o, nbh = f.face_owner, f.face_neighbor
    inter = nbh != BOUNDARY
    nbs = np.where(inter, nbh, 0)
    pmax = np.where(inter, np.maximum(deg[o], deg[nbs]), deg[o])
    nqf = _nq(2 * pmax + inc, d - 1)
    nmax = np.where(inter, np.maximum(n[o], n[nbs]), n[o])
    sides = owned[o].astype(np.float64) + np.where(inter, owned[nbs], False).astype(np.float64)
    face_int = float(np.sum(((16.0 + 4.0 * has_b) * nmax ** 2 * nqf * nfac * sides / 2.0)[inter]))
    tag = f.face_tag
    dirich = (~inter) & (tag == TAG_CODE["dirichlet"]) & owned[o]
    inflow = (~inter) & (tag == TAG_CODE["inflow"]) & owned[o]
    face_d = float(np.sum((4.0 * n[o] ** 2 * nqf * nfac)[dirich]))  # inflow part not known host-side
    face_i = float(np.sum((2.0 * n[o] ** 2 * nqf * nfac)[inflow]))
    neu = (~inter) & (tag == TAG_CODE["neumann"]) & owned[o]
    face_n = float(np.sum((2.0 * n[o] * nqf * nfac)[neu]))  # load only
    flops = vol + face_int + face_d + face_i

    nnz = float(plan.nnz)
    nrows = float(plan.n_local_rows)
    geo = float(np.sum(nsim[owned])) * 8.0 * d * (d + 1) + float(np.sum(nfac[inter | owned[o]])) * (8.0 * d * d + 32)
    bytes_ = 16.0 * nnz + 8.0 * nrows * 2 + geo
    return {"flops": flops, "bytes": bytes_, "flops_volume": vol, "flops_faces": face_int + face_d + face_i,
            "flops_interior": face_int, "flops_dirichlet": face_d, "flops_inflow": face_i,
            "flops_neumann": face_n, "nnz": nnz, "elements": float(owned.sum())}


def slab_work(plan) -> dict:
    """Canonical work of one slab assembly (SpacetimePlan), the counts above
    with the prism rules: volume sub-prism (p+2)^3 points, lateral sub-facet
    (p+2)^2, bottom facet (p+2)^2 per sub-triangle (2 n^2 nq, the inflow
    term); terms: the non-zero diagonal entries of A + [b] + [c]."""
    from .basis import family_name

    f = plan.flat
    deg = plan.degrees
    inc = plan.config.quad_increment
    n = np.diff(plan.dof.offsets).astype(np.float64)
    owned = np.zeros(f.n_elements, bool)
    owned[plan.row_elements] = True
    info = plan.policy_info
    S = f.dim
    items = (info["n_active"] if info["diag"] else S + 1) * (info["kind"] != 0) + int(info["adv"]) + int(info["reac"])
    nsim = np.diff(f.elem_ptr).astype(np.float64)
    m = ((2 * deg + inc + 2) // 2).astype(np.float64)
    vol = float(np.sum((nsim * 2.0 * n * n * m ** (S + 1) * items)[owned]))
    bottom = float(np.sum((nsim * 2.0 * n * n * m ** S)[owned])) if info["adv"] else 0.0
    nfac = np.diff(f.face_ptr).astype(np.float64)
    o, nbh = f.face_owner, f.face_neighbor
    inter = nbh != BOUNDARY
    nbs = np.where(inter, nbh, 0)
    pm = np.where(inter, np.maximum(deg[o], deg[nbs]), deg[o])
    mf = ((2 * pm + inc + 2) // 2).astype(np.float64)
    nmax = np.where(inter, np.maximum(n[o], n[nbs]), n[o])
    sides = owned[o].astype(np.float64) + np.where(inter, owned[nbs], False).astype(np.float64)
    up = 4.0 * float(info["adv_spatial"])
    face_int = float(np.sum(((16.0 + up) * nmax ** 2 * mf ** S * nfac * sides / 2.0)[inter]))
    tag = plan.lateral_tags
    dirich = (~inter) & (tag == TAG_CODE["dirichlet"]) & owned[o]
    face_d = float(np.sum((4.0 * n[o] ** 2 * mf ** S * nfac)[dirich]))
    flops = vol + bottom + face_int + face_d
    nnz = float(plan.nnz)
    geo = float(np.sum(nsim[owned])) * 8.0 * 6 + float(np.sum(nfac[inter | owned[o]])) * 40.0
    bytes_ = 16.0 * nnz + 16.0 * float(plan.n_local_rows) + geo
    return {"flops": flops, "bytes": bytes_, "flops_volume": vol, "flops_faces": face_int + face_d + bottom,
            "flops_interior": face_int, "flops_dirichlet": face_d, "flops_bottom": bottom,
            "nnz": nnz, "elements": float(owned.sum()), "family": family_name(plan.family)}
