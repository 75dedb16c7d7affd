"""CPU ORACLE -- test infrastructure only, never the product path.

Plain numpy restatement of polydg's space-time slab provider
(``/root/reference/pkg/src/polydg/spacetime.py``: ``SlabGeometry``
:133-364, ``assemble_slab`` :391-413, previous-slab traces :367-388) feeding
the same kernel formulas as the spatial oracle (``oracle/sipg.py``).  Used
only by ``tests/`` and ``bench.py``'s CPU leg as the checker of the device
slab engine (``paper_2007_04881_b200/spacetime.py``).

Pinned by golden fixtures produced by the real reference
(``tests/golden/make_golden_slab.py`` -> ``tests/golden/slab_*.npz``) and by
the reference suite's space-time known answers restated in
``tests/test_slab_oracle.py``.
"""

from __future__ import annotations

import numpy as np

from . import sipg as O

BOUNDARY = O.BOUNDARY


def _tag(t):
    return getattr(t, "value", t)


def tensor_with_interval(bpts, bw, t0, t1, trule):
    """quadrature.py:159-178: base points x interval, time coordinate last
    (base index outer, time index inner)."""
    tp, tw = trule
    tau = t1 - t0
    tpts = t0 + tau * tp[:, 0]
    tws = tau * tw
    nb, nt = bw.shape[0], tws.shape[0]
    pts = np.empty((nb * nt, bpts.shape[1] + 1))
    pts[:, :-1] = np.repeat(bpts, nt, axis=0)
    pts[:, -1] = np.tile(tpts, nb)
    return pts, (bw[:, None] * tws[None, :]).ravel()


def checked_flow_sign(bn):
    """model.py:128-135."""
    tol = 1e-10 * max(1.0, float(np.abs(bn).max()))
    if bn.min() < -tol and bn.max() > tol:
        raise ValueError("advection flux changes sign across a lateral slab face")
    return float(bn.mean())


class SlabProblem:
    """Restatement of ``SlabGeometry`` (spacetime.py:133-364) for one slab
    (spatial mesh x (t0, t1)); ``previous`` is a callable of spatial points
    (initial data) or ``(prev_specs, prev_vec)`` (spacetime.py:367-388)."""

    def __init__(self, mesh, t0, t1, coeffs, specs, previous, quad_increment=2,
                 penalty_constant=10.0, coverable=None, dirichlet_predicate=None):
        self.mesh, self.t0, self.t1, self.tau = mesh, float(t0), float(t1), float(t1) - float(t0)
        self.C = coeffs
        self.s = mesh.dim
        self.d = self.s + 1
        self.deg = np.array([sp.degree for sp in specs], np.int64)
        self.fam = [getattr(sp.family, "value", sp.family) for sp in specs]
        self.box = [np.asarray(sp.box, float) for sp in specs]
        self.n = np.array([sp.n_funcs for sp in specs], np.int64)
        self.off = np.zeros(len(specs) + 1, np.int64)
        np.cumsum(self.n, out=self.off[1:])
        self.inc = quad_increment
        self.pen = penalty_constant
        self.cov = coverable
        self.previous = previous
        if previous is not None and not callable(previous):
            pspecs, pvec = previous
            self.prev_specs = pspecs
            self.prev_vec = np.asarray(pvec, float)
            self.prev_off = np.concatenate([[0], np.cumsum([sp.n_funcs for sp in pspecs])])
            if self.prev_off[-1] != self.prev_vec.shape[0]:
                raise ValueError("previous solution has the wrong number of dofs")
        self._vpts = {}
        self.lat_tag = {}
        for fid, f in enumerate(mesh.faces):
            if f.neighbor == BOUNDARY:
                self.lat_tag[fid] = self._classify_lateral(fid, dirichlet_predicate)

    # -- rules (spacetime.py:178-193, 265-285) ------------------------------
    def sp(self, e):
        return (int(self.deg[e]), self.box[e], self.fam[e])

    def order(self, *els):
        return 2 * max(int(self.deg[e]) for e in els) + self.inc

    def vol_quad(self, e, s):
        o = self.order(e)
        V = self.mesh.base.vertices[self.mesh.base.simplices[s]]
        bp, bw = O.map_to_simplex(O.simplex_rule(self.s, o), V)
        return tensor_with_interval(bp, bw, self.t0, self.t1, O.interval_rule(o))

    def vol_points(self, e):
        if e not in self._vpts:
            self._vpts[e] = np.concatenate([self.vol_quad(e, s)[0] for s in self.mesh.elements[e]])
        return self._vpts[e]

    def lateral_quads(self, f):
        els = (f.owner,) if f.neighbor == BOUNDARY else (f.owner, f.neighbor)
        o = self.order(*els)
        rule = O.face_rule(self.s, o)
        V = self.mesh.base.vertices
        out = []
        for r in range(f.vertex_ids.shape[0]):
            bp, bw = O.map_to_subsimplex(rule, V[f.vertex_ids[r]])
            out.append(tensor_with_interval(bp, bw, self.t0, self.t1, O.interval_rule(o)))
        return out

    def lateral_normal(self, f):
        n = np.zeros(self.d)
        n[:-1] = f.normal
        return n

    def lateral_samples(self, f):
        """spacetime.py:248-263: order-2 facet rule x order-2 interval rule."""
        rule = O.face_rule(self.s, 2)
        V = self.mesh.base.vertices
        chunks = []
        for r in range(f.vertex_ids.shape[0]):
            bp, bw = O.map_to_subsimplex(rule, V[f.vertex_ids[r]])
            chunks.append(tensor_with_interval(bp, bw, self.t0, self.t1, O.interval_rule(2))[0])
        return np.concatenate(chunks)

    # -- classification / flow / penalty (spacetime.py:229-246, 287-338) -------
    def _classify_lateral(self, fid, predicate):
        f = self.mesh.faces[fid]
        pts = self.lateral_samples(f)
        n = self.lateral_normal(f)
        mean = pts.mean(axis=0)[None, :]
        if self.C.diffusion is not None:
            a = self.C.diffusion(mean)[0]
            tol = 1e-12 * max(1.0, float(np.abs(a).max()))
            if float(n @ a @ n) > tol:
                if predicate is None or predicate(mean[0]):
                    return "dirichlet"
                return "neumann"
        if self.C.advection is None:
            return "outflow"
        sign = checked_flow_sign(self.C.advection(pts) @ n)
        return "inflow" if sign < 0.0 else "outflow"

    def lateral_sign(self, f):
        if self.C.advection is None:
            return 0.0
        return checked_flow_sign(self.C.advection(self.lateral_samples(f)) @ self.lateral_normal(f))

    def upwind(self, f):
        """spacetime.py:287-299."""
        sg = self.lateral_sign(f)
        return O.SIDE_OWNER if sg < 0.0 else (O.SIDE_NEIGHBOR if sg > 0.0 else -1)

    def side_penalty(self, f, e):
        """spacetime.py:319-351 (extruded-split adjacent volumes)."""
        n = self.lateral_normal(f)
        abar = 0.0 if self.C.diffusion is None else float(
            np.einsum("i,qij,j->q", n, self.C.diffusion(self.vol_points(e)), n).max())
        adj = np.asarray(f.owner_simplices if e == f.owner else f.neighbor_simplices)
        adj = adj[adj != BOUNDARY]
        mx = float(self.mesh.base.simplex_volumes[adj].max()) * self.tau / (self.s + 1)
        p = int(self.deg[e])
        cap = float(p ** (2 * (self.d - 1))) if (self.cov is not None and self.cov[e]) else np.inf
        return float(self.mesh.element_volumes[e] * self.tau), p, abar, mx, cap

    def sigma(self, f):
        sides = [self.side_penalty(f, f.owner)]
        if f.neighbor != BOUNDARY:
            sides.append(self.side_penalty(f, f.neighbor))
        best = 0.0
        for vol, p, abar, mx, cap in sides:
            best = max(best, min(vol / mx, cap) * abar * p ** 2 * (f.measure * self.tau) / vol)
        return self.pen * best

    # -- time-jump data (spacetime.py:367-388) ----------------------------------
    def previous_values(self, e, pts):
        if self.previous is None:
            raise ValueError("slab assembly needs initial data or a previous solution")
        if callable(self.previous):
            return self.previous(pts[:, :-1])
        ps = self.prev_specs[e]
        vals, _ = O.tabulate(ps.degree, np.asarray(ps.box, float), pts,
                             getattr(ps.family, "value", ps.family))
        return self.prev_vec[self.prev_off[e]:self.prev_off[e + 1]] @ vals


def slab_element_rows(prob: SlabProblem, e: int):
    """All blocks of prism e's rows and its RHS segment (one-sided per
    element like ``oracle.sipg.element_rows``)."""
    m, C = prob.mesh, prob.C
    ne = int(prob.n[e])
    blocks = {e: np.zeros((ne, ne))}
    rhs = np.zeros(ne)
    sp_e = prob.sp(e)
    for s in m.elements[e]:
        pts, w = prob.vol_quad(e, s)
        K, f = O.volume_block(sp_e[0], sp_e[1], pts, w, C, sp_e[2])
        blocks[e] += K
        rhs += f
    for fid in O._faces_of(m, e):
        face = m.faces[fid]
        nrm = prob.lateral_normal(face)
        if face.neighbor != BOUNDARY:
            side = 0 if face.owner == e else 1
            other = face.neighbor if side == 0 else face.owner
            sg, up = prob.sigma(face), prob.upwind(face)
            for pts, w in prob.lateral_quads(face):
                B = O.interior_blocks(prob.sp(face.owner), prob.sp(face.neighbor), pts, w, nrm, C,
                                      sg, up)
                blocks[e] += B[side][side]
                blocks.setdefault(other, np.zeros((ne, int(prob.n[other]))))
                blocks[other] += B[side][1 - side]
            continue
        tg = prob.lat_tag[fid]
        if tg == "dirichlet":
            sg = prob.sigma(face)
            wi = prob.lateral_sign(face) < 0.0
            for pts, w in prob.lateral_quads(face):
                K, f = O.dirichlet_block(sp_e, pts, w, nrm, C, sg, wi)
                blocks[e] += K
                rhs += f
        elif tg == "inflow":
            for pts, w in prob.lateral_quads(face):
                K, f = O.inflow_block(sp_e, pts, w, nrm, C)
                blocks[e] += K
                rhs += f
        elif tg == "neumann":
            for pts, w in prob.lateral_quads(face):
                rhs += O.neumann_load(sp_e, pts, w, C)
    # bottom facet: statically inflow, the time jump (spacetime.py:208-227, 355-362)
    nb = np.zeros(prob.d)
    nb[-1] = -1.0
    o = prob.order(e)
    rule = O.simplex_rule(prob.s, o)
    for s in m.elements[e]:
        sp_, sw = O.map_to_simplex(rule, m.base.vertices[m.base.simplices[s]])
        pts = np.concatenate([sp_, np.full((sp_.shape[0], 1), prob.t0)], axis=1)
        g = prob.previous_values(e, pts)
        K, f = O.inflow_block(sp_e, pts, sw, nb, C, g=g)
        blocks[e] += K
        rhs += f
    # top facet: statically outflow, no contribution
    return blocks, rhs


def assemble_slab(mesh, t0, t1, coeffs, specs, previous, quad_increment=2, penalty_constant=10.0,
                  coverable=None, row_elements=None, dirichlet_predicate=None, workers=1):
    """Oracle of ``assemble_slab`` (spacetime.py:391-413) with Approach 2:
    -> (row_ptr, col_idx, values, rhs[n_dofs]) for the rows of ``row_elements``."""
    prob = SlabProblem(mesh, t0, t1, coeffs, specs, previous, quad_increment, penalty_constant,
                       coverable, dirichlet_predicate)
    nel = len(specs)
    rows = np.arange(nel) if row_elements is None else np.sort(np.asarray(row_elements))
    pairs = [(int(i.owner), int(i.neighbor)) for i in mesh.interfaces]
    row_ptr, col_idx, nbs = O.block_pattern(prob.off, pairs, rows)
    results = _run(prob, rows, workers)
    values = np.zeros(col_idx.size)
    rhs = np.zeros(int(prob.off[-1]))
    pos = 0
    for e, (blocks, r) in zip(rows, results):
        e = int(e)
        ne = int(prob.n[e])
        rowblock = np.concatenate([blocks.get(j, np.zeros((ne, int(prob.n[j])))) for j in nbs[e]],
                                  axis=1)
        values[pos:pos + rowblock.size] = rowblock.ravel()
        pos += rowblock.size
        rhs[prob.off[e]:prob.off[e + 1]] = r
    return row_ptr, col_idx, values, rhs


_POOL = None


def _work(chunk):
    return [slab_element_rows(_POOL, int(e)) for e in chunk]


def _run(prob, rows, workers):
    global _POOL
    if workers <= 1 or len(rows) < 2 * workers:
        return [slab_element_rows(prob, int(e)) for e in rows]
    import multiprocessing as mp

    _POOL = prob
    chunks = np.array_split(np.asarray(rows), workers * 8)
    try:
        with mp.get_context("fork").Pool(workers) as pool:
            parts = pool.map(_work, chunks)
    finally:
        _POOL = None
    return [r for part in parts for r in part]
