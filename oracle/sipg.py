"""CPU ORACLE -- test infrastructure only, never the product path.

A plain numpy restatement of polydg's fp64 SIPG assembly path (reference
``/root/reference/pkg/src/polydg``), used ONLY by ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg, as the checker the CUDA engine is compared with.
Nothing in ``paper_2007_04881_b200`` imports this module.

Parity pinning: this restatement is checked against (1) the known-answer
tests of the reference's own suite (``tests/test_oracle_kats.py``) and (2)
golden CSR/RHS fixtures produced by running the real reference in the build
container (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``,
``tests/test_oracle_golden.py``).

Every function cites the reference code it restates.  The structure is
deliberately simple (dense per-item blocks summed into a dict keyed by
element pair) rather than a copy of the reference's work-plan executor; only
the summation order differs (<= 1e-14 relative).
"""

from __future__ import annotations

import math
import os
from functools import lru_cache

import numpy as np

BOUNDARY = -1
SIDE_OWNER, SIDE_NEIGHBOR = 0, 1
CLASSIFY_ORDER = 2  # model.py:26


def _tag(t) -> str:
    return getattr(t, "value", t)


# -- quadrature (quadrature.py:59-156) -----------------------------------------

def _gj01(n, alpha):
    """quadrature.py:59-66: n-point Gauss rule for (1-t)^alpha on (0,1)."""
    from scipy.special import roots_jacobi, roots_legendre

    x, w = roots_legendre(n) if alpha == 0 else roots_jacobi(n, alpha, 0.0)
    return 0.5 * (x + 1.0), w * 0.5 ** (alpha + 1)


@lru_cache(maxsize=None)
def simplex_rule(d: int, order: int):
    """quadrature.py:69-94: conical product, collapsed axes unfolded."""
    m = (order + 2) // 2
    ax = [_gj01(m, j) for j in range(d)]
    t = np.array(np.meshgrid(*[a[0] for a in ax], indexing="ij")).reshape(d, -1).T
    wg = np.array(np.meshgrid(*[a[1] for a in ax], indexing="ij")).reshape(d, -1).T
    w = np.prod(wg, axis=1) if d > 1 else wg[:, 0].copy()
    x = t.copy()
    for i in range(d):
        for j in range(i + 1, d):
            x[:, i] = x[:, i] * (1.0 - t[:, j])
    return x, w


@lru_cache(maxsize=None)
def interval_rule(order: int):
    """quadrature.py:97-103."""
    t, w = _gj01((order + 2) // 2, 0)
    return t[:, None], w


def face_rule(d, order):
    return interval_rule(order) if d == 2 else simplex_rule(d - 1, order)


class OracleQuadratureError(ValueError):
    pass


def map_to_simplex(rule, verts):
    """quadrature.py:118-136: x = v0 + xi E, w = w_hat |det E|."""
    xi, wh = rule
    verts = np.asarray(verts, float)
    E = verts[1:] - verts[0]
    det = np.linalg.det(E)
    scale = float(np.max(np.abs(E))) or 1.0
    if abs(det) < 1e-14 * scale ** verts.shape[1]:
        raise OracleQuadratureError("degenerate simplex in quadrature map")
    return verts[0] + xi @ E, wh * abs(det)


def map_to_subsimplex(rule, verts):
    """quadrature.py:139-156: w = w_hat sqrt(det(E E^T))."""
    xi, wh = rule
    verts = np.asarray(verts, float)
    E = verts[1:] - verts[0]
    g = np.linalg.det(E @ E.T)
    if g <= 0.0:
        raise OracleQuadratureError("degenerate sub-simplex in face quadrature map")
    return verts[0] + xi @ E, wh * math.sqrt(g)


# -- basis (basis.py:74-164) -----------------------------------------------------

@lru_cache(maxsize=None)
def graded_lex(p: int, d: int) -> np.ndarray:
    """basis.py:86-104 (family P): ascending total degree, lex within a level."""
    import itertools

    rows = [a for s in range(p + 1)
            for a in itertools.product(range(s + 1), repeat=d) if sum(a) == s]
    return np.array(rows, dtype=np.int64).reshape(-1, d)


@lru_cache(maxsize=None)
def multi_indices(p: int, d: int, family: str = "P") -> np.ndarray:
    """basis.py:93-104: family P = graded lex; family PQ (space-time) = spatial
    graded-lex multi-index of degree <= p times time degree k <= p, time outer."""
    if family == "P":
        return graded_lex(p, d)
    sp = graded_lex(p, d - 1)
    return np.array([(*a, k) for k in range(p + 1) for a in sp], dtype=np.int64).reshape(-1, d)


def tabulate(degree: int, box, pts, family: str = "P"):
    """basis.py:107-164: orthonormal box Legendre values (n,q) + grads (n,d,q)."""
    pts = np.atleast_2d(np.asarray(pts, float))
    box = np.asarray(box, float)
    lo, hi = box[0], box[1]
    d, q, p = pts.shape[1], pts.shape[0], degree
    half = 0.5 * (hi - lo)
    t = (pts - 0.5 * (lo + hi)) / half
    v1 = np.empty((d, p + 1, q))
    g1 = np.empty((d, p + 1, q))
    nrm = np.sqrt(2.0 * np.arange(p + 1) + 1.0)
    for i in range(d):
        L = np.empty((p + 1, q))
        dL = np.empty((p + 1, q))
        L[0], dL[0] = 1.0, 0.0
        if p >= 1:
            L[1], dL[1] = t[:, i], 1.0
        for k in range(1, p):
            L[k + 1] = (2 * k + 1) / (k + 1) * t[:, i] * L[k] - k / (k + 1) * L[k - 1]
            dL[k + 1] = (2 * k + 1) * L[k] + dL[k - 1]
        s = nrm / np.sqrt(hi[i] - lo[i])
        v1[i] = L * s[:, None]
        g1[i] = dL * (s / half[i])[:, None]
    al = multi_indices(p, d, family)
    dims = np.arange(d)[None, :]
    fv = v1[dims, al, :]                       # (n, d, q)
    vals = fv.prod(axis=1)
    fd = g1[dims, al, :]
    grads = np.empty((al.shape[0], d, q))
    for k in range(d):
        f = fv.copy()
        f[:, k, :] = fd[:, k, :]
        grads[:, k, :] = f.prod(axis=1)
    return vals, grads


# -- kernel mathematics (assembly.py:396-512) ----------------------------------------

def _tab(sp, pts):
    """sp = (degree, box[, family])."""
    return tabulate(sp[0], sp[1], pts, sp[2] if len(sp) > 2 else "P")


def volume_block(deg, box, pts, w, C, family="P"):
    """assembly.py:396-415: K_ij = sum_q w (A grad phi_j).grad phi_i + (b.grad phi_j) phi_i
    + c phi_j phi_i;  load_i = sum_q w f phi_i."""
    V, G = tabulate(deg, box, pts, family)
    K = np.zeros((V.shape[0], V.shape[0]))
    if C.diffusion is not None:
        AG = np.einsum("qab,nbq->naq", C.diffusion(pts), G)
        K += np.einsum("q,jaq,iaq->ij", w, AG, G)
    if C.advection is not None:
        K += np.einsum("q,jq,iq->ij", w, np.einsum("qa,naq->nq", C.advection(pts), G), V)
    if C.reaction is not None:
        K += np.einsum("q,jq,iq->ij", w * C.reaction(pts), V, V)
    f = V @ (w * C.source(pts)) if C.source is not None else np.zeros(V.shape[0])
    return K, f


def interior_blocks(sp_o, sp_n, pts, w, nrm, C, sigma, upwind, grad_terms=True):
    """assembly.py:418-463: blocks [[oo, on], [no, nn]] of one interior sub-facet."""
    Vo, Go = _tab(sp_o, pts)
    Vn, Gn = _tab(sp_n, pts)
    V = (Vo, Vn)
    s = (1.0, -1.0)
    B = [[np.zeros((V[a].shape[0], V[b].shape[0])) for b in range(2)] for a in range(2)]
    F = None
    if C.diffusion is not None and grad_terms:
        A = C.diffusion(pts)
        F = [np.einsum("qab,nbq,a->nq", A, g, nrm) for g in (Go, Gn)]
    for a in range(2):
        for b in range(2):
            if F is not None:
                B[a][b] -= 0.5 * s[a] * np.einsum("q,jq,iq->ij", w, F[b], V[a])
                B[a][b] -= 0.5 * s[b] * np.einsum("q,jq,iq->ij", w, V[b], F[a])
            if sigma:
                B[a][b] += sigma * s[a] * s[b] * np.einsum("q,jq,iq->ij", w, V[b], V[a])
    if upwind in (SIDE_OWNER, SIDE_NEIGHBOR) and C.advection is not None:
        wbn = w * (C.advection(pts) @ nrm)
        if upwind == SIDE_OWNER:
            B[0][0] -= np.einsum("q,jq,iq->ij", wbn, Vo, Vo)
            B[0][1] += np.einsum("q,jq,iq->ij", wbn, Vn, Vo)
        else:
            B[1][1] += np.einsum("q,jq,iq->ij", wbn, Vn, Vn)
            B[1][0] -= np.einsum("q,jq,iq->ij", wbn, Vo, Vn)
    return B


def dirichlet_block(sp, pts, w, nrm, C, sigma, with_inflow, grad_terms=True):
    """assembly.py:466-493."""
    V, G = _tab(sp, pts)
    n = V.shape[0]
    K, f = np.zeros((n, n)), np.zeros(n)
    g = C.dirichlet_data(pts) if C.dirichlet_data is not None else None
    F = None
    if C.diffusion is not None and grad_terms:
        F = np.einsum("qab,nbq,a->nq", C.diffusion(pts), G, nrm)
        K -= np.einsum("q,jq,iq->ij", w, F, V) + np.einsum("q,jq,iq->ij", w, V, F)
    if sigma:
        K += sigma * np.einsum("q,jq,iq->ij", w, V, V)
    if g is not None:
        if F is not None:
            f -= F @ (w * g)
        if sigma:
            f += sigma * (V @ (w * g))
    if with_inflow and C.advection is not None:
        wbn = w * (C.advection(pts) @ nrm)
        K -= np.einsum("q,jq,iq->ij", wbn, V, V)
        if g is not None:
            f -= V @ (wbn * g)
    return K, f


def inflow_block(sp, pts, w, nrm, C, g="dirichlet"):
    """assembly.py:496-505 (boundary values = geom.inflow_values: dirichlet_data,
    assembly.py:628-631, or the previous slab's trace, spacetime.py:355-362)."""
    V, _ = _tab(sp, pts)
    wbn = w * (C.advection(pts) @ nrm)
    K = -np.einsum("q,jq,iq->ij", wbn, V, V)
    if isinstance(g, str):
        g = C.dirichlet_data(pts) if C.dirichlet_data is not None else None
    f = np.zeros(V.shape[0]) if g is None else -(V @ (wbn * g))
    return K, f


def neumann_load(sp, pts, w, C):
    """assembly.py:508-512."""
    V, _ = _tab(sp, pts)
    if C.neumann_data is None:
        return np.zeros(V.shape[0])
    return V @ (w * C.neumann_data(pts))


# -- penalty and flow side (model.py:118-257) ---------------------------------------

def face_sample_points(mesh, face):
    """model.py:118-125: order-2 rule on every sub-facet."""
    d = mesh.dim
    rule = face_rule(d, CLASSIFY_ORDER)
    V = mesh.base.vertices
    return np.concatenate([map_to_subsimplex(rule, V[face.vertex_ids[r]])[0]
                           for r in range(face.vertex_ids.shape[0])])


def flow_is_inflow(mesh, elem, face, C) -> bool:
    """model.py:128-135 + 176-191: mean b.n_out < 0 (straddle raises)."""
    if C.advection is None:
        return False
    n = face.normal if elem == face.owner else -face.normal
    bn = C.advection(face_sample_points(mesh, face)) @ n
    tol = 1e-10 * max(1.0, float(np.abs(bn).max()))
    if bn.min() < -tol and bn.max() > tol:
        raise ValueError("advection flux changes sign across a face")
    return float(bn.mean()) < 0.0


def side_penalty(mesh, elem, face, degree, vol_pts, C, pen_const, coverable):
    """model.py:196-235 -> (volume, degree, a_bar, max_adjacent_volume, cov_cap)."""
    n = face.normal
    abar = 0.0 if C.diffusion is None else float(
        np.einsum("i,qij,j->q", n, C.diffusion(vol_pts), n).max())
    adj = face.owner_simplices if elem == face.owner else face.neighbor_simplices
    adj = np.asarray(adj)
    adj = adj[adj != BOUNDARY]
    mx = float(mesh.base.simplex_volumes[adj].max())
    d = mesh.dim
    cap = float(degree ** (2 * (d - 1))) if (coverable is not None and coverable[elem]) else np.inf
    return float(mesh.element_volumes[elem]), degree, abar, mx, cap


def sigma_of(face, sides, pen_const):
    """model.py:238-257."""
    best = 0.0
    for vol, p, abar, mx, cap in sides:
        best = max(best, min(vol / mx, cap) * abar * p ** 2 * face.measure / vol)
    return pen_const * best


# -- sparsity pattern (assembly.py:290-340) -----------------------------------------------

def block_pattern(offsets, pairs, row_elements):
    """Sorted neighbour lists and CSR skeleton (every row of an element has
    the concatenation of its neighbours' DoF ranges)."""
    nbrs = {int(e): {int(e)} for e in row_elements}
    for a, b in pairs:
        if a in nbrs:
            nbrs[a].add(b)
        if b in nbrs:
            nbrs[b].add(a)
    counts = np.diff(offsets)
    row_ptr = [0]
    cols = []
    nb_sorted = {}
    for e in row_elements:
        ns = sorted(nbrs[int(e)])
        nb_sorted[int(e)] = ns
        c = np.concatenate([np.arange(offsets[j], offsets[j + 1]) for j in ns])
        for _ in range(int(counts[e])):
            cols.append(c)
            row_ptr.append(row_ptr[-1] + c.size)
    col_idx = np.concatenate(cols).astype(np.int64) if cols else np.zeros(0, np.int64)
    return np.asarray(row_ptr, np.int64), col_idx, nb_sorted


# -- full assembly --------------------------------------------------------------------------

class Problem:
    """Everything one assembly reads, restated from ``MeshGeometry``
    (assembly.py:527-634) in oracle form."""

    def __init__(self, mesh, coeffs, specs, quad_increment=2, penalty_constant=10.0,
                 coverable=None):
        self.mesh = mesh
        self.C = coeffs
        self.deg = np.array([s.degree for s in specs], np.int64)
        self.box = [np.asarray(s.box, float) for s in specs]
        self.n = np.array([s.n_funcs for s in specs], np.int64)
        self.off = np.zeros(len(specs) + 1, np.int64)
        np.cumsum(self.n, out=self.off[1:])
        self.inc = quad_increment
        self.pen = penalty_constant
        self.cov = coverable
        self.d = mesh.dim
        self._vpts = {}

    def sp(self, e):
        return (int(self.deg[e]), self.box[e])

    def vol_quad(self, e, s):
        rule = simplex_rule(self.d, 2 * int(self.deg[e]) + self.inc)
        V = self.mesh.base.vertices[self.mesh.base.simplices[s]]
        return map_to_simplex(rule, V)

    def vol_points(self, e):
        if e not in self._vpts:
            self._vpts[e] = np.concatenate(
                [self.vol_quad(e, s)[0] for s in self.mesh.elements[e]])
        return self._vpts[e]

    def face_quads(self, face):
        p = int(self.deg[face.owner])
        if face.neighbor != BOUNDARY:
            p = max(p, int(self.deg[face.neighbor]))
        rule = face_rule(self.d, 2 * p + self.inc)
        V = self.mesh.base.vertices
        return [map_to_subsimplex(rule, V[face.vertex_ids[r]])
                for r in range(face.vertex_ids.shape[0])]

    def sigma(self, face):
        sides = [side_penalty(self.mesh, face.owner, face, int(self.deg[face.owner]),
                              self.vol_points(face.owner), self.C, self.pen, self.cov)]
        if face.neighbor != BOUNDARY:
            sides.append(side_penalty(self.mesh, face.neighbor, face,
                                      int(self.deg[face.neighbor]),
                                      self.vol_points(face.neighbor), self.C, self.pen,
                                      self.cov))
        return sigma_of(face, sides, self.pen)

    def upwind(self, face):
        """assembly.py:596-604."""
        if self.C.advection is None:
            return -1
        if flow_is_inflow(self.mesh, face.owner, face, self.C):
            return SIDE_OWNER
        if flow_is_inflow(self.mesh, face.neighbor, face, self.C):
            return SIDE_NEIGHBOR
        return -1


def element_rows(prob: Problem, e: int):
    """All blocks of element e's rows and its RHS segment.

    Returns ({col_element: (n_e, n_col) block}, rhs_e).  One-sided per
    element: interior faces contribute their e-rows only (the semantics of
    ``_SIDE_OWNER/_SIDE_NEIGHBOR``, assembly.py:685-696,778-788), so the
    result is independent of which other elements are assembled.
    """
    m, C = prob.mesh, prob.C
    ne = int(prob.n[e])
    blocks = {e: np.zeros((ne, ne))}
    rhs = np.zeros(ne)
    for s in m.elements[e]:
        pts, w = prob.vol_quad(e, s)
        K, f = volume_block(prob.deg[e], prob.box[e], pts, w, C)
        blocks[e] += K
        rhs += f
    for fid in _faces_of(m, e):
        face = m.faces[fid]
        tg = _tag(face.tag)
        if face.neighbor != BOUNDARY:
            side = 0 if face.owner == e else 1
            other = face.neighbor if side == 0 else face.owner
            sg, up = prob.sigma(face), prob.upwind(face)
            for pts, w in prob.face_quads(face):
                B = interior_blocks(prob.sp(face.owner), prob.sp(face.neighbor), pts, w,
                                    face.normal, C, sg, up)
                blocks[e] += B[side][side]
                blocks.setdefault(other, np.zeros((ne, int(prob.n[other]))))
                blocks[other] += B[side][1 - side]
        elif tg == "interior":
            raise ValueError(f"boundary face {fid} is unclassified; run classify_boundary_faces")
        elif tg == "dirichlet":
            sg = prob.sigma(face)
            wi = flow_is_inflow(m, e, face, C)
            for pts, w in prob.face_quads(face):
                K, f = dirichlet_block(prob.sp(e), pts, w, face.normal, C, sg, wi)
                blocks[e] += K
                rhs += f
        elif tg == "inflow":
            for pts, w in prob.face_quads(face):
                K, f = inflow_block(prob.sp(e), pts, w, face.normal, C)
                blocks[e] += K
                rhs += f
        elif tg == "neumann":
            for pts, w in prob.face_quads(face):
                rhs += neumann_load(prob.sp(e), pts, w, C)
    return blocks, rhs


_FACE_INDEX = {}


def _faces_of(mesh, e):
    key = id(mesh)
    idx = _FACE_INDEX.get(key)
    if idx is None or idx[0] is not mesh:
        by_el = {}
        for fid, f in enumerate(mesh.faces):
            by_el.setdefault(f.owner, []).append(fid)
            if f.neighbor != BOUNDARY:
                by_el.setdefault(f.neighbor, []).append(fid)
        idx = (mesh, by_el)
        _FACE_INDEX[key] = idx
    return idx[1].get(e, [])


def assemble(mesh, coeffs, specs, quad_increment=2, penalty_constant=10.0, coverable=None,
             row_elements=None, workers=1):
    """Oracle of ``_assemble_approach2`` (assembly.py:1102-1134):
    -> (row_ptr, col_idx, values, rhs[n_dofs]) for the rows of ``row_elements``."""
    prob = Problem(mesh, coeffs, specs, quad_increment, penalty_constant, coverable)
    nel = len(specs)
    rows = np.arange(nel) if row_elements is None else np.sort(np.asarray(row_elements))
    pairs = [(int(i.owner), int(i.neighbor)) for i in mesh.interfaces]
    row_ptr, col_idx, nbs = block_pattern(prob.off, pairs, rows)
    results = _run_elements(prob, rows, workers)
    values = np.zeros(col_idx.size)
    rhs = np.zeros(int(prob.off[-1]))
    pos = 0
    for e, (blocks, r) in zip(rows, results):
        e = int(e)
        ne = int(prob.n[e])
        rowblock = np.concatenate([blocks.get(j, np.zeros((ne, int(prob.n[j]))))
                                   for j in nbs[e]], axis=1)
        values[pos:pos + rowblock.size] = rowblock.ravel()
        pos += rowblock.size
        rhs[prob.off[e]:prob.off[e + 1]] = r
    return row_ptr, col_idx, values, rhs


_POOL_PROB = None


def _work(chunk):
    return [element_rows(_POOL_PROB, int(e)) for e in chunk]


def _run_elements(prob, rows, workers):
    global _POOL_PROB
    if workers <= 1 or len(rows) < 2 * workers:
        return [element_rows(prob, int(e)) for e in rows]
    import multiprocessing as mp

    _POOL_PROB = prob
    chunks = np.array_split(np.asarray(rows), workers * 8)
    try:
        with mp.get_context("fork").Pool(workers) as pool:
            parts = pool.map(_work, chunks)
    finally:
        _POOL_PROB = None
    return [r for part in parts for r in part]


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# -- single-item kernels (assembly.py:1139-1234) -----------------------------------------

def element_kernel(mesh, e, coeffs, spec, quad_increment=2):
    rule = simplex_rule(mesh.dim, 2 * spec.degree + quad_increment)
    n = spec.n_funcs
    K, f = np.zeros((n, n)), np.zeros(n)
    for s in mesh.elements[e]:
        pts, w = map_to_simplex(rule, mesh.base.vertices[mesh.base.simplices[s]])
        k, l = volume_block(spec.degree, spec.box, pts, w, coeffs)
        K += k
        f += l
    return K, f


# -- Approach 1 merge (assembly.py:1002-1031) ----------------------------------------------

def triplets_to_csr(rows, cols, vals, n_rows, n_cols, sentinel=None):
    """Stable sort by (row, col), duplicates summed in input order ->
    (row_ptr, col_idx, values)."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    vals = np.asarray(vals, float)
    if sentinel is not None:
        keep = rows != sentinel
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
    key = rows * np.int64(n_cols) + cols
    order = np.argsort(key, kind="stable")
    ks, vs = key[order], vals[order]
    if ks.size == 0:
        return np.zeros(n_rows + 1, np.int64), np.zeros(0, np.int64), np.zeros(0)
    starts = np.flatnonzero(np.concatenate([[True], ks[1:] != ks[:-1]]))
    sums = np.add.reduceat(vs, starts)
    uk = ks[starts]
    row_ptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(uk // n_cols, minlength=n_rows), out=row_ptr[1:])
    return row_ptr, (uk % n_cols).astype(np.int64), sums
