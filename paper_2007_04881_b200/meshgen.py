"""Synthetic benchmark meshes.

* :func:`voronoi_mesh` -- bounded random-seed Voronoi tessellation of the unit
  square (cfg1/2/3/5): seeds ``default_rng(seed).uniform(0, 1, (n, 2))``,
  Morton-sorted so element ids are spatially coherent (contiguous id ranges =
  compact partitions), mirrored across the walls near the boundary so every
  cell is clipped exactly by the square, Voronoi vertices closer than
  ``1e-6 / sqrt(n)`` merged, every cell fan-triangulated counter-clockwise
  from its seed (positive orientation, so polydg's reorientation swap never
  fires), agglomeration map triangle -> cell.  Built from the ridge arrays
  with numpy only (no per-cell Python loop).
* :func:`kuhn_agglomerated_mesh` -- 3D: Kuhn tetrahedra of ``cube_grid(n)``,
  nearest-of-k random seeds by centroid, split into facet-connected
  components (polydg's agglomerate rejects disconnected elements,
  mesh.py:418-425) (cfg4).

These are test/benchmark inputs, outside the timed assembly path.
"""

from __future__ import annotations

import numpy as np

from .mesh import PolytopicMesh, SimplicialMesh, agglomerate


def morton_order(pts: np.ndarray, bits: int = 20) -> np.ndarray:
    q = np.clip((pts * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)

    def spread(v):
        v = v.astype(np.uint64)
        out = np.zeros_like(v)
        for b in range(bits):
            out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(2 * b)
        return out

    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1))
    return np.argsort(code, kind="stable")


def _union_find_roots(n: int, pairs: np.ndarray) -> np.ndarray:
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    if pairs.size == 0:
        return np.arange(n)
    g = coo_matrix((np.ones(pairs.shape[0]), (pairs[:, 0], pairs[:, 1])), shape=(n, n))
    _, lab = connected_components(g, directed=False)
    # representative = smallest member of each component
    rep = np.full(lab.max() + 1, n, np.int64)
    np.minimum.at(rep, lab, np.arange(n))
    return rep[lab]


def voronoi_simplicial(n: int, seed: int = 0):
    """-> (SimplicialMesh, agg_map) of the bounded Voronoi tessellation."""
    from scipy.spatial import Voronoi, cKDTree

    rng = np.random.default_rng(seed)
    seeds = rng.uniform(0.0, 1.0, (n, 2))
    seeds = seeds[morton_order(seeds)]
    band = min(0.5, 3.0 / np.sqrt(n))
    mir = [seeds]
    for axis, wall in ((0, 0.0), (0, 1.0), (1, 0.0), (1, 1.0)):
        sel = np.abs(seeds[:, axis] - wall) < band
        m = seeds[sel].copy()
        m[:, axis] = 2.0 * wall - m[:, axis]
        mir.append(m)
    allpts = np.concatenate(mir)
    vor = Voronoi(allpts)
    rp = vor.ridge_points
    rv = np.asarray(vor.ridge_vertices, dtype=np.int64)
    keep = (rp[:, 0] < n) | (rp[:, 1] < n)
    rp, rv = rp[keep], rv[keep]
    if np.any(rv < 0):
        raise RuntimeError("unbounded ridge next to an original cell; widen the mirror band")
    V = vor.vertices
    used = np.unique(rv)
    if np.any(V[used] < -1e-9) or np.any(V[used] > 1 + 1e-9):
        raise RuntimeError("Voronoi vertex of an original cell outside the unit square")
    # merge vertices closer than tol, clip the rest onto the square
    tol = 1e-6 / np.sqrt(n)
    Vu = np.clip(V[used], 0.0, 1.0)
    pairs = cKDTree(Vu).query_pairs(tol, output_type="ndarray")
    roots = _union_find_roots(used.size, pairs)
    remap = np.full(V.shape[0], -1, np.int64)
    remap[used] = roots
    rv = remap[rv]
    nondeg = rv[:, 0] != rv[:, 1]
    rp, rv = rp[nondeg], rv[nondeg]
    # compact vertex ids: Voronoi vertices first, then seeds
    vid = np.unique(rv)
    newv = np.full(used.size, -1, np.int64)
    newv[vid] = np.arange(vid.size)
    rv = newv[rv]
    verts = np.concatenate([Vu[vid], seeds])
    seed_vid = vid.size + np.arange(n)
    # one fan triangle per (original cell, ridge)
    cell = np.concatenate([rp[:, 0], rp[:, 1]])
    a = np.concatenate([rv[:, 0], rv[:, 1]])
    b = np.concatenate([rv[:, 1], rv[:, 0]])
    orig = cell < n
    cell, a, b = cell[orig], a[orig], b[orig]
    s = seed_vid[cell]
    P0, PA, PB = verts[s], verts[a], verts[b]
    cross = (PA[:, 0] - P0[:, 0]) * (PB[:, 1] - P0[:, 1]) - (PA[:, 1] - P0[:, 1]) * (PB[:, 0] - P0[:, 0])
    flip = cross < 0
    a2 = np.where(flip, b, a)
    b2 = np.where(flip, a, b)
    mid = 0.5 * (verts[a2] + verts[b2]) - P0
    ang = np.arctan2(mid[:, 1], mid[:, 0])
    order = np.lexsort((ang, cell))
    tris = np.stack([s, a2, b2], axis=1)[order]
    agg = cell[order]
    return SimplicialMesh(2, verts, tris), agg


def voronoi_mesh(n: int, seed: int = 0, device: bool = False) -> PolytopicMesh:
    """``device``: agglomerate on the GPU (meshprep.agglomerate_device, the
    same mesh bit for bit) -- used for the million-cell benchmark meshes."""
    base, agg = voronoi_simplicial(n, seed)
    if device:
        from .meshprep import agglomerate_device

        return agglomerate_device(base, agg, check_connected=False)
    return agglomerate(base, agg, check_connected=False)


def cube_grid_simplicial(n: int) -> SimplicialMesh:
    ax = np.linspace(0.0, 1.0, n + 1)
    g = np.stack(np.meshgrid(ax, ax, ax, indexing="ij"), axis=-1).reshape(-1, 3)
    idx = np.arange((n + 1) ** 3).reshape(n + 1, n + 1, n + 1)
    i, j, k = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    corner = np.stack([idx[i + a, j + b, k + c] for a in (0, 1) for b in (0, 1) for c in (0, 1)], axis=1)
    kuhn = np.array([(0, 1, 3, 7), (0, 1, 5, 7), (0, 2, 3, 7), (0, 2, 6, 7), (0, 4, 5, 7), (0, 4, 6, 7)])
    tets = corner[:, kuhn].reshape(-1, 4)
    return SimplicialMesh(3, g, tets)


def kuhn_agglomerated_mesh(n: int, k: int, seed: int = 4) -> PolytopicMesh:
    """3D polyhedral mesh: nearest-seed labels of Kuhn tets split into
    facet-connected components."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from scipy.spatial import cKDTree

    base = cube_grid_simplicial(n)
    cent = base.vertices[base.simplices].mean(axis=1)
    rng = np.random.default_rng(seed)
    sd = rng.uniform(0.0, 1.0, (k, 3))
    sd = sd[morton_order(sd[:, :2])]
    _, lab = cKDTree(sd).query(cent)
    ns = base.n_simplices
    loc = np.array([[j for j in range(4) if j != m] for m in range(4)])
    fac = np.sort(base.simplices[:, loc].reshape(ns * 4, 3), axis=1)
    key = (fac[:, 0] * (base.n_vertices + 1) + fac[:, 1]) * (base.n_vertices + 1) + fac[:, 2]
    order = np.argsort(key, kind="stable")
    ks = key[order]
    same = np.flatnonzero(ks[1:] == ks[:-1])
    s0, s1 = order[same] // 4, order[same + 1] // 4
    inside = lab[s0] == lab[s1]
    g = coo_matrix((np.ones(inside.sum()), (s0[inside], s1[inside])), shape=(ns, ns))
    _, comp = connected_components(g, directed=False)
    # renumber components in order of first appearance of the smallest simplex
    first = np.full(comp.max() + 1, ns, np.int64)
    np.minimum.at(first, comp, np.arange(ns))
    rank = np.empty_like(first)
    rank[np.argsort(first, kind="stable")] = np.arange(first.size)
    return agglomerate(base, rank[comp], check_connected=False)
