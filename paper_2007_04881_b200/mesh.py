"""Polytopic mesh data model, flattened to the device SoA layout.

The assembly kernels consume a :class:`FlatMesh`: plain contiguous arrays
(CSR offsets + index/coordinate tables) that are copied to HBM once and read
by every kernel.  Two routes produce the same arrays:

* :meth:`FlatMesh.from_polytopic` -- adapter for any polydg-style
  ``PolytopicMesh`` object (duck-typed: polydg's own class or this module's),
  replaying its element / face / interface order exactly;
* :func:`agglomerate` -- a vectorised re-implementation of polydg's
  ``agglomerate`` (``mesh.py:328-473``) that builds the flat arrays straight
  from ``(SimplicialMesh, agg_map)``; used for meshes of millions of
  elements where the object model does not scale.

Conventions that are part of parity (SURVEY.md §7 "Bit-faithful geometry
order") and that both routes keep:

* element simplices in ascending simplex id (``mesh.py:345``);
* a facet's vertex order is the local facet order of the LOWER simplex id
  sharing it (the stable lexsort at ``mesh.py:356-357`` puts it first;
  ``vids = facets[rows[0]]``, ``mesh.py:399``), even when the owner is the
  higher simplex;
* a face's normal is its first member facet's normal, oriented away from the
  owner-side simplex centroid (``mesh.py:403-404,440``);
* interior faces come first, grouped by interface in sorted ``(e0, e1)``
  order; boundary faces follow, grouped by element (``mesh.py:451-455``);
* co-hyperplanar facets of one pair merge greedily (``mesh.py:294-325``).
"""

from __future__ import annotations

import math
from collections.abc import Sequence
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

BOUNDARY = -1
NORMAL_TOL = 1e-9  # polydg mesh.py:28-29
PLANE_TOL = 1e-9


class MeshError(Exception):
    """Invalid mesh topology or geometry (polydg ``mesh.py:32``)."""


class MeshFormatError(MeshError):
    pass


class BoundaryTag(Enum):
    INTERIOR = "interior"
    DIRICHLET = "dirichlet"
    NEUMANN = "neumann"
    INFLOW = "inflow"
    OUTFLOW = "outflow"


#: device tag codes (include/pdg.h PDG_TAG_*)
TAG_CODE = {"interior": 0, "dirichlet": 1, "neumann": 2, "inflow": 3, "outflow": 4}
CODE_TAG = {v: BoundaryTag(k) for k, v in TAG_CODE.items()}


def tag_code(tag) -> int:
    """Code of this package's or polydg's BoundaryTag (compared by value)."""
    return TAG_CODE[getattr(tag, "value", tag)]


@dataclass
class SimplicialMesh:
    """Fine simplicial mesh, reoriented to positive volume (polydg ``mesh.py:48-104``)."""

    dim: int
    vertices: np.ndarray
    simplices: np.ndarray
    simplex_volumes: np.ndarray = field(init=False)

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise MeshError(f"mesh dimension must be 2 or 3, got {self.dim}")
        self.vertices = np.ascontiguousarray(self.vertices, dtype=float)
        self.simplices = np.ascontiguousarray(self.simplices, dtype=np.int64)
        nv = self.vertices.shape[0]
        if self.vertices.ndim != 2 or self.vertices.shape[1] != self.dim:
            raise MeshError("vertex array must be (nv, dim)")
        if self.simplices.ndim != 2 or self.simplices.shape[1] != self.dim + 1:
            raise MeshError("simplex array must be (ns, dim+1)")
        if self.simplices.size and (self.simplices.min() < 0 or self.simplices.max() >= nv):
            raise MeshError("simplex vertex index out of range")
        if _has_duplicate_rows(np.sort(self.simplices, axis=1), nv):
            raise MeshError("duplicate simplices in mesh")
        vols = self._signed_volumes()
        neg = vols < 0.0
        if neg.any():
            # swap the last two local vertices of negatively oriented simplices
            last = self.simplices[neg, -1].copy()
            self.simplices[neg, -1] = self.simplices[neg, -2]
            self.simplices[neg, -2] = last
            vols = np.abs(vols)
        span = self.vertices.max(axis=0) - self.vertices.min(axis=0)
        scale = float(np.prod(np.where(span > 0, span, 1.0)))
        bad = np.flatnonzero(vols <= 1e-14 * scale)
        if bad.size:
            raise MeshError(f"degenerate simplex {int(bad[0])} (volume {vols[bad[0]]:g})")
        self.simplex_volumes = vols

    def _signed_volumes(self) -> np.ndarray:
        v0 = self.vertices[self.simplices[:, 0]]
        edges = self.vertices[self.simplices[:, 1:]] - v0[:, None, :]
        return np.linalg.det(edges) / math.factorial(self.dim)

    @property
    def n_vertices(self) -> int:
        return self.vertices.shape[0]

    @property
    def n_simplices(self) -> int:
        return self.simplices.shape[0]


def _has_duplicate_rows(sorted_rows: np.ndarray, nv: int) -> bool:
    if sorted_rows.shape[0] < 2:
        return False
    keys = _row_keys(sorted_rows, nv)
    if keys is not None:
        keys = np.sort(keys)
        return bool(np.any(keys[1:] == keys[:-1]))
    u = np.unique(sorted_rows, axis=0)
    return u.shape[0] != sorted_rows.shape[0]


def _row_keys(rows: np.ndarray, nv: int):
    """Injective int64 key per row of small non-negative ints, or None."""
    k = rows.shape[1]
    if float(nv) ** k >= 2.0**62:
        return None
    key = np.zeros(rows.shape[0], dtype=np.int64)
    for j in range(k):
        key = key * np.int64(nv) + rows[:, j].astype(np.int64)
    return key


# ---------------------------------------------------------------------------
# flat (device) layout
# ---------------------------------------------------------------------------

@dataclass
class FlatMesh:
    """SoA polytopic mesh -- the layout the kernels read from HBM.

    int32 ids everywhere except CSR offsets (int64); coordinates float64.
    """

    dim: int
    vertices: np.ndarray            # f64 [nv, d]
    simplices: np.ndarray           # i32 [ns, d+1] reference (post-reorientation) order
    simplex_volumes: np.ndarray     # f64 [ns]
    elem_ptr: np.ndarray            # i64 [nel+1]
    elem_simplices: np.ndarray      # i32 [ns]   ascending within an element
    boxes: np.ndarray               # f64 [nel, 2, d]
    elem_volumes: np.ndarray        # f64 [nel]
    face_owner: np.ndarray          # i32 [nf]
    face_neighbor: np.ndarray       # i32 [nf]  (-1 boundary)
    face_tag: np.ndarray            # i8  [nf]  TAG_CODE
    face_normal: np.ndarray         # f64 [nf, d] outward from owner
    face_measure: np.ndarray        # f64 [nf]
    face_ptr: np.ndarray            # i64 [nf+1] -> facets
    facet_vertices: np.ndarray      # i32 [nfacet, d]
    facet_owner_simplex: np.ndarray     # i32 [nfacet]
    facet_neighbor_simplex: np.ndarray  # i32 [nfacet] (-1 boundary)
    facet_measures: np.ndarray      # f64 [nfacet]
    iface_owner: np.ndarray         # i32 [nif] (owner < neighbor, sorted)
    iface_neighbor: np.ndarray      # i32 [nif]
    iface_ptr: np.ndarray           # i64 [nif+1] -> iface_faces
    iface_faces: np.ndarray         # i32
    elem_bface_ptr: np.ndarray      # i64 [nel+1] -> elem_bfaces
    elem_bfaces: np.ndarray         # i32

    @property
    def n_vertices(self) -> int:
        return int(self.vertices.shape[0])

    @property
    def n_simplices(self) -> int:
        return int(self.simplices.shape[0])

    @property
    def n_elements(self) -> int:
        return int(self.elem_ptr.shape[0] - 1)

    @property
    def n_faces(self) -> int:
        return int(self.face_owner.shape[0])

    @property
    def n_facets(self) -> int:
        return int(self.facet_vertices.shape[0])

    @property
    def n_interfaces(self) -> int:
        return int(self.iface_owner.shape[0])

    def arrays(self) -> dict:
        return {k: v for k, v in self.__dict__.items() if isinstance(v, np.ndarray)}

    def nbytes(self) -> int:
        return sum(a.nbytes for a in self.arrays().values())

    def element_simplex_counts(self) -> np.ndarray:
        return np.diff(self.elem_ptr)

    # -- route 1: from a polydg-style PolytopicMesh -------------------------
    @classmethod
    def from_polytopic(cls, mesh) -> "FlatMesh":
        base = mesh.base
        d = int(base.dim)
        nel = len(mesh.elements)
        counts = np.array([len(s) for s in mesh.elements], dtype=np.int64)
        elem_ptr = np.zeros(nel + 1, np.int64)
        np.cumsum(counts, out=elem_ptr[1:])
        elem_simplices = (np.concatenate([np.asarray(s, np.int64) for s in mesh.elements])
                          if nel else np.zeros(0, np.int64))
        faces = mesh.faces
        nf = len(faces)
        fcount = np.array([f.vertex_ids.shape[0] for f in faces], dtype=np.int64)
        face_ptr = np.zeros(nf + 1, np.int64)
        np.cumsum(fcount, out=face_ptr[1:])
        cat = lambda xs, dt, shape: (np.concatenate(xs).astype(dt) if xs else np.zeros(shape, dt))
        facet_vertices = cat([np.asarray(f.vertex_ids).reshape(-1, d) for f in faces], np.int32, (0, d))
        fos = cat([np.asarray(f.owner_simplices).ravel() for f in faces], np.int32, (0,))
        fns = cat([np.asarray(f.neighbor_simplices).ravel() for f in faces], np.int32, (0,))
        fms = cat([np.asarray(f.facet_measures, float).ravel() for f in faces], np.float64, (0,))
        owner = np.array([f.owner for f in faces], np.int32)
        nbr = np.array([f.neighbor for f in faces], np.int32)
        tags = np.array([tag_code(f.tag) for f in faces], np.int8)
        normals = (np.stack([np.asarray(f.normal, float) for f in faces]) if nf
                   else np.zeros((0, d)))
        measures = np.array([float(f.measure) for f in faces], np.float64)
        ifs = mesh.interfaces
        iptr = np.zeros(len(ifs) + 1, np.int64)
        np.cumsum([len(i.face_ids) for i in ifs], out=iptr[1:])
        ifaces = cat([np.asarray(i.face_ids, np.int64) for i in ifs], np.int32, (0,))
        if not np.array_equal(ifaces, np.arange(ifaces.size)):
            # polydg emits the faces of each interface consecutively, interfaces
            # in sorted order, before all boundary faces (mesh.py:451-455); the
            # kernels address an interface's faces as the id range iface_ptr.
            raise NotImplementedError("interface faces must be the contiguous leading face ids")
        bfaces = np.flatnonzero(nbr == BOUNDARY)
        bowner = owner[bfaces]
        order = np.argsort(bowner, kind="stable")
        bcount = np.bincount(bowner, minlength=nel) if bfaces.size else np.zeros(nel, np.int64)
        bptr = np.zeros(nel + 1, np.int64)
        np.cumsum(bcount, out=bptr[1:])
        return cls(
            dim=d,
            vertices=np.ascontiguousarray(base.vertices, np.float64),
            simplices=np.ascontiguousarray(base.simplices, np.int32),
            simplex_volumes=np.ascontiguousarray(base.simplex_volumes, np.float64),
            elem_ptr=elem_ptr,
            elem_simplices=elem_simplices.astype(np.int32),
            boxes=np.ascontiguousarray(mesh.bounding_boxes, np.float64),
            elem_volumes=np.ascontiguousarray(mesh.element_volumes, np.float64),
            face_owner=owner, face_neighbor=nbr, face_tag=tags,
            face_normal=np.ascontiguousarray(normals, np.float64).reshape(nf, d),
            face_measure=measures, face_ptr=face_ptr,
            facet_vertices=np.ascontiguousarray(facet_vertices, np.int32),
            facet_owner_simplex=fos, facet_neighbor_simplex=fns, facet_measures=fms,
            iface_owner=np.array([i.owner for i in ifs], np.int32),
            iface_neighbor=np.array([i.neighbor for i in ifs], np.int32),
            iface_ptr=iptr, iface_faces=ifaces,
            elem_bface_ptr=bptr, elem_bfaces=bfaces[order].astype(np.int32),
        )


# ---------------------------------------------------------------------------
# object facade over a FlatMesh (what polydg-style callers and the oracle see)
# ---------------------------------------------------------------------------

class Face:
    """View of one face of a FlatMesh with polydg's ``Face`` attributes."""

    __slots__ = ("_m", "_f")

    def __init__(self, flat: FlatMesh, fid: int):
        self._m = flat
        self._f = int(fid)

    def _rows(self):
        a, b = self._m.face_ptr[self._f], self._m.face_ptr[self._f + 1]
        return slice(int(a), int(b))

    @property
    def vertex_ids(self):
        return self._m.facet_vertices[self._rows()].astype(np.int64)

    @property
    def normal(self):
        return self._m.face_normal[self._f]

    @property
    def owner(self) -> int:
        return int(self._m.face_owner[self._f])

    @property
    def neighbor(self) -> int:
        return int(self._m.face_neighbor[self._f])

    @property
    def owner_simplices(self):
        return self._m.facet_owner_simplex[self._rows()].astype(np.int64)

    @property
    def neighbor_simplices(self):
        return self._m.facet_neighbor_simplex[self._rows()].astype(np.int64)

    @property
    def facet_measures(self):
        return self._m.facet_measures[self._rows()]

    @property
    def measure(self) -> float:
        return float(self._m.face_measure[self._f])

    @property
    def tag(self) -> BoundaryTag:
        return CODE_TAG[int(self._m.face_tag[self._f])]

    @tag.setter
    def tag(self, value):
        self._m.face_tag[self._f] = tag_code(value)

    @property
    def is_boundary(self) -> bool:
        return self.neighbor == BOUNDARY

    @property
    def n_facets(self) -> int:
        r = self._rows()
        return r.stop - r.start

    def outward_normal(self, element: int):
        if element == self.owner:
            return self.normal
        if element == self.neighbor:
            return -self.normal
        raise MeshError(f"element {element} is not adjacent to this face")


@dataclass
class Interface:
    owner: int
    neighbor: int
    face_ids: list


class _LazySeq(Sequence):
    def __init__(self, n, make):
        self._n, self._make = n, make

    def __len__(self):
        return self._n

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._make(k) for k in range(*i.indices(self._n))]
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError(i)
        return self._make(i)


class PolytopicMesh:
    """Agglomerated mesh backed by a :class:`FlatMesh`.

    Exposes polydg's ``PolytopicMesh`` attributes (``mesh.py:153-188``) as
    lazy views so the same object feeds the device engine (flat arrays) and
    object-style callers such as the CPU oracle.
    """

    def __init__(self, base: SimplicialMesh, agg_map: np.ndarray, flat: FlatMesh):
        self.base = base
        self.agg_map = agg_map
        self.flat = flat

    @classmethod
    def from_flat(cls, flat: FlatMesh) -> "PolytopicMesh":
        """Object view of a FlatMesh (no validation: the arrays already are
        an agglomerated mesh, e.g. a cached workload mesh or a rank's sub-mesh)."""
        base = SimplicialMesh.__new__(SimplicialMesh)
        base.dim, base.vertices, base.simplex_volumes = flat.dim, flat.vertices, flat.simplex_volumes
        base.simplices = flat.simplices.astype(np.int64)
        agg = np.repeat(np.arange(flat.n_elements), np.diff(flat.elem_ptr))
        agg_full = np.empty_like(agg)
        agg_full[flat.elem_simplices] = agg
        return cls(base, agg_full, flat)

    @property
    def dim(self) -> int:
        return self.flat.dim

    @property
    def n_elements(self) -> int:
        return self.flat.n_elements

    @property
    def n_faces(self) -> int:
        return self.flat.n_faces

    @property
    def elements(self):
        f = self.flat
        return _LazySeq(f.n_elements, lambda e: f.elem_simplices[f.elem_ptr[e]:f.elem_ptr[e + 1]]
                        .astype(np.int64))

    @property
    def bounding_boxes(self):
        return self.flat.boxes

    @property
    def element_volumes(self):
        return self.flat.elem_volumes

    @property
    def faces(self):
        return _LazySeq(self.flat.n_faces, lambda i: Face(self.flat, i))

    @property
    def interfaces(self):
        f = self.flat
        return _LazySeq(f.n_interfaces, lambda i: Interface(
            int(f.iface_owner[i]), int(f.iface_neighbor[i]),
            [int(x) for x in f.iface_faces[f.iface_ptr[i]:f.iface_ptr[i + 1]]]))

    def boundary_face_ids(self):
        return [int(i) for i in np.flatnonzero(self.flat.face_neighbor == BOUNDARY)]

    def interior_face_ids(self):
        return [int(i) for i in np.flatnonzero(self.flat.face_neighbor != BOUNDARY)]

    def element_diameters(self):
        span = self.flat.boxes[:, 1, :] - self.flat.boxes[:, 0, :]
        return np.linalg.norm(span, axis=1)

    def facet_coordinates(self, face, row: int):
        return self.base.vertices[face.vertex_ids[row]]


def flat_of(mesh) -> FlatMesh:
    """FlatMesh of this package's PolytopicMesh (no copy) or of any
    polydg-style mesh object (adapter, cached on the object).

    The adapter is built once per polydg mesh and kept in ``mesh._pdg_flat``
    (so its HBM copy, ``_device_cache``, is reused too).  Face tags are the
    only field polydg mutates after construction (``classify_boundary_faces``,
    model.py:164-173): they are re-read on every call and written into the
    cached adapter in place, which ``DeviceMesh.refresh_tags`` then uploads."""
    if isinstance(mesh, FlatMesh):
        return mesh
    flat = getattr(mesh, "flat", None)
    if isinstance(flat, FlatMesh):
        return flat
    flat = getattr(mesh, "_pdg_flat", None)
    if isinstance(flat, FlatMesh) and flat.n_faces == len(mesh.faces):
        tags = np.fromiter((tag_code(f.tag) for f in mesh.faces), np.int8, len(mesh.faces))
        if not np.array_equal(tags, flat.face_tag):
            flat.face_tag[:] = tags
        return flat
    flat = FlatMesh.from_polytopic(mesh)
    try:
        object.__setattr__(mesh, "_pdg_flat", flat)
    except Exception:  # slotted / frozen objects: no cache
        pass
    return flat


# ---------------------------------------------------------------------------
# route 2: vectorised agglomeration
# ---------------------------------------------------------------------------

def _facet_local(d: int) -> np.ndarray:
    return np.array([[j for j in range(d + 1) if j != k] for k in range(d + 1)], dtype=np.int64)


def _normals_measures(coords: np.ndarray):
    """Unit normals (unoriented) and measures of facets ``coords[m, d, d]``
    (polydg ``mesh.py:265-275``)."""
    if coords.shape[1] == 2:
        t = coords[:, 1] - coords[:, 0]
        length = np.sqrt(t[:, 0] * t[:, 0] + t[:, 1] * t[:, 1])
        normal = np.stack([t[:, 1], -t[:, 0]], axis=1) / length[:, None]
        return normal, length
    c = np.cross(coords[:, 1] - coords[:, 0], coords[:, 2] - coords[:, 0])
    area2 = np.sqrt(np.einsum("ij,ij->i", c, c))
    return c / area2[:, None], 0.5 * area2


def _greedy_planes(members: np.ndarray, normals: np.ndarray, fverts: np.ndarray):
    """Split facet ids ``members`` into co-hyperplanar groups, greedily in
    order (the semantics of polydg ``_group_by_hyperplane``, mesh.py:294-325)."""
    groups = []  # [normal, point, lo, hi, list]
    for idx in members:
        n = normals[idx]
        v = fverts[idx]
        for g in groups:
            if np.max(np.abs(n - g[0])) > NORMAL_TOL:
                continue
            lo = np.minimum(g[2], v.min(axis=0))
            hi = np.maximum(g[3], v.max(axis=0))
            diam = float(np.linalg.norm(hi - lo)) or 1.0
            if np.abs((v - g[1]) @ g[0]).max() <= PLANE_TOL * diam:
                g[4].append(idx)
                g[2], g[3] = lo, hi
                break
        else:
            groups.append([n, v[0].copy(), v.min(axis=0), v.max(axis=0), [idx]])
    return [g[4] for g in groups]


def agglomerate(mesh: SimplicialMesh, agg_map, check_connected: bool = True) -> PolytopicMesh:
    """Group simplices into elements and extract faces, vectorised.

    Same result as polydg ``agglomerate`` (mesh.py:328-473) -- same element,
    face, facet and interface order and the same geometric conventions -- at
    numpy speed, so million-element meshes can be built.
    """
    agg = np.asarray(agg_map, dtype=np.int64)
    ns, d = mesh.n_simplices, mesh.dim
    if agg.shape != (ns,):
        raise MeshError("agglomeration map must have one entry per simplex")
    nel = int(agg.max()) + 1 if ns else 0
    if ns and (agg.min() < 0 or np.unique(agg).size != nel):
        raise MeshError("agglomeration map must be surjective onto 0..max")

    verts = mesh.vertices
    simp = mesh.simplices
    el_order = np.argsort(agg, kind="stable")
    el_count = np.bincount(agg, minlength=nel)
    elem_ptr = np.zeros(nel + 1, np.int64)
    np.cumsum(el_count, out=elem_ptr[1:])

    # facets: facet k of simplex s omits local vertex k; row = s*(d+1)+k
    nloc = d + 1
    facets = simp[:, _facet_local(d)].reshape(ns * nloc, d)
    keys = np.sort(facets, axis=1)
    key1 = _row_keys(keys, mesh.n_vertices)
    order = (np.argsort(key1, kind="stable") if key1 is not None
             else np.lexsort(keys.T[::-1]))
    ks = keys[order]
    new = np.ones(ks.shape[0], dtype=bool)
    new[1:] = np.any(ks[1:] != ks[:-1], axis=1)
    starts = np.flatnonzero(new)
    sizes = np.diff(np.append(starts, ks.shape[0]))
    if np.any(sizes > 2):
        raise MeshError("non-manifold facet shared by more than two simplices")
    r0 = order[starts]
    s0 = r0 // nloc
    pair = sizes == 2
    s1 = np.full(starts.shape[0], BOUNDARY, np.int64)
    s1[pair] = order[starts[pair] + 1] // nloc
    e0 = agg[s0]
    e1 = np.where(pair, agg[np.where(pair, s1, 0)], BOUNDARY)
    internal = pair & (e0 == e1)

    if check_connected and nel:
        from scipy.sparse import coo_matrix
        from scipy.sparse.csgraph import connected_components

        a, b = s0[internal], s1[internal]
        g = coo_matrix((np.ones(a.size), (a, b)), shape=(ns, ns))
        _, comp = connected_components(g, directed=False)
        first = comp[el_order[elem_ptr[:-1]]]
        bad = np.flatnonzero(comp[el_order] != np.repeat(first, el_count))
        if bad.size:
            e = int(agg[el_order[bad[0]]])
            raise MeshError(f"element {e} is not facet-connected; refine the agglomeration map")

    kept = ~internal
    r0k, s0k, s1k = r0[kept], s0[kept], s1[kept]
    e0k, e1k = e0[kept], e1[kept]
    pairk = s1k != BOUNDARY
    swap = pairk & (e0k > e1k)
    own_s = np.where(swap, s1k, s0k)
    nbr_s = np.where(swap, s0k, s1k)
    own_e = np.where(swap, e1k, e0k)
    nbr_e = np.where(swap, e0k, e1k)
    vids = facets[r0k]                       # lower simplex's local order
    coords = verts[vids]                     # [m, d, d]
    normal, measure = _normals_measures(coords)
    centroids = verts[simp[own_s]].mean(axis=1)
    fcent = coords.mean(axis=1)
    flip = np.einsum("ij,ij->i", normal, fcent - centroids) < 0.0
    normal[flip] *= -1.0
    nkept = vids.shape[0]

    # interfaces: interior kept facets sorted by (owner, neighbor), facet order kept
    inter = np.flatnonzero(pairk)
    ikey = own_e[inter] * np.int64(max(nel, 1)) + nbr_e[inter]
    io = inter[np.argsort(ikey, kind="stable")]
    iks = ikey[np.argsort(ikey, kind="stable")]
    inew = np.ones(io.size, dtype=bool)
    inew[1:] = iks[1:] != iks[:-1]
    istarts = np.flatnonzero(inew)
    isizes = np.diff(np.append(istarts, io.size))
    bnd = np.flatnonzero(~pairk)
    bo = bnd[np.argsort(own_e[bnd], kind="stable")]
    bks = own_e[bo]
    bnew = np.ones(bo.size, dtype=bool)
    bnew[1:] = bks[1:] != bks[:-1]
    bstarts = np.flatnonzero(bnew)
    bsizes = np.diff(np.append(bstarts, bo.size))

    # faces: singleton sets are one face each; larger sets are split greedily
    face_members = []   # list of arrays of kept-facet ids, in face order
    face_ifc = []
    multi_i = set(np.flatnonzero(isizes > 1).tolist())
    multi_b = set(np.flatnonzero(bsizes > 1).tolist())
    iface_face_count = np.ones(istarts.size, np.int64)
    if not multi_i and not multi_b:
        members_flat = np.concatenate([io, bo])
        face_len = np.ones(members_flat.size, np.int64)
    else:
        out_members, out_len = [], []
        for g, (a, n) in enumerate(zip(istarts, isizes)):
            if g in multi_i:
                groups = _greedy_planes(io[a:a + n], normal, coords)
                iface_face_count[g] = len(groups)
                for grp in groups:
                    out_members.extend(grp)
                    out_len.append(len(grp))
            else:
                out_members.append(int(io[a]))
                out_len.append(1)
        for g, (a, n) in enumerate(zip(bstarts, bsizes)):
            if g in multi_b:
                for grp in _greedy_planes(bo[a:a + n], normal, coords):
                    out_members.extend(grp)
                    out_len.append(len(grp))
            else:
                out_members.append(int(bo[a]))
                out_len.append(1)
        members_flat = np.asarray(out_members, np.int64)
        face_len = np.asarray(out_len, np.int64)

    nf = face_len.size
    face_ptr = np.zeros(nf + 1, np.int64)
    np.cumsum(face_len, out=face_ptr[1:])
    first = members_flat[face_ptr[:-1]]
    face_owner = own_e[first].astype(np.int32)
    face_nbr = np.where(pairk[first], nbr_e[first], BOUNDARY).astype(np.int32)
    fm = measure[members_flat]
    if np.all(face_len == 1):
        face_measure = fm.copy()
    else:
        face_measure = np.array([fm[face_ptr[i]:face_ptr[i + 1]].sum() for i in range(nf)])
    nif = istarts.size
    iface_ptr = np.zeros(nif + 1, np.int64)
    np.cumsum(iface_face_count, out=iface_ptr[1:])
    n_int_faces = int(iface_ptr[-1])
    b_owner = face_owner[n_int_faces:]
    bcount = np.bincount(b_owner, minlength=nel) if b_owner.size else np.zeros(nel, np.int64)
    bptr = np.zeros(nel + 1, np.int64)
    np.cumsum(bcount, out=bptr[1:])

    # boxes and volumes per element (simplices in ascending id)
    es = el_order
    pts_min = verts[simp[es]].min(axis=1)
    pts_max = verts[simp[es]].max(axis=1)
    boxes = np.empty((nel, 2, d))
    if nel:
        boxes[:, 0] = np.minimum.reduceat(pts_min, elem_ptr[:-1], axis=0)
        boxes[:, 1] = np.maximum.reduceat(pts_max, elem_ptr[:-1], axis=0)
    vols = np.add.reduceat(mesh.simplex_volumes[es], elem_ptr[:-1]) if nel else np.zeros(0)

    flat = FlatMesh(
        dim=d,
        vertices=np.ascontiguousarray(verts, np.float64),
        simplices=np.ascontiguousarray(simp, np.int32),
        simplex_volumes=np.ascontiguousarray(mesh.simplex_volumes, np.float64),
        elem_ptr=elem_ptr,
        elem_simplices=es.astype(np.int32),
        boxes=boxes,
        elem_volumes=np.ascontiguousarray(vols, np.float64),
        face_owner=face_owner,
        face_neighbor=face_nbr,
        face_tag=np.zeros(nf, np.int8),
        face_normal=np.ascontiguousarray(normal[first]),
        face_measure=np.ascontiguousarray(face_measure, np.float64),
        face_ptr=face_ptr,
        facet_vertices=np.ascontiguousarray(vids[members_flat], np.int32),
        facet_owner_simplex=own_s[members_flat].astype(np.int32),
        facet_neighbor_simplex=np.where(pairk[members_flat], nbr_s[members_flat],
                                        BOUNDARY).astype(np.int32),
        facet_measures=np.ascontiguousarray(fm, np.float64),
        iface_owner=own_e[io[istarts]].astype(np.int32),
        iface_neighbor=nbr_e[io[istarts]].astype(np.int32),
        iface_ptr=iface_ptr,
        iface_faces=np.arange(n_int_faces, dtype=np.int32),
        elem_bface_ptr=bptr,
        elem_bfaces=np.arange(n_int_faces, nf, dtype=np.int32),
    )
    return PolytopicMesh(mesh, agg, flat)


def identity_agglomeration(mesh: SimplicialMesh) -> PolytopicMesh:
    return agglomerate(mesh, np.arange(mesh.n_simplices, dtype=np.int64))
