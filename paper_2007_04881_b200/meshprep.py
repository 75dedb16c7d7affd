"""Mesh preprocessing on the device: polydg's ``agglomerate``
(mesh.py:328-473) as a sequence of sm_100a kernels and CUB sorts
(``csrc/pdg_agglomerate.cu``).  Produces the same ``PolytopicMesh`` as the
vectorised host version (``mesh.agglomerate``), bit for bit -- element,
face, facet and interface order, normals, measures, boxes, volumes -- in a
fraction of the time on million-element meshes."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .mesh import FlatMesh, MeshError, PolytopicMesh, SimplicialMesh

_OUT = ("elem_ptr", "elem_simplices", "boxes", "elem_volumes", "face_owner", "face_neighbor", "face_normal",
        "face_measure", "face_ptr", "facet_vertices", "facet_owner_simplex", "facet_neighbor_simplex",
        "facet_measures", "iface_owner", "iface_neighbor", "iface_ptr", "elem_bface_ptr")


def agglomerate_device(mesh: SimplicialMesh, agg_map, check_connected: bool = True, device=None) -> PolytopicMesh:
    """``agglomerate`` on the GPU; raises the same MeshError messages."""
    import torch

    from .assembly import _require_cuda

    dev = _require_cuda(device)
    lib = _lib.load()
    agg = np.asarray(agg_map, dtype=np.int64)
    ns, d = mesh.n_simplices, mesh.dim
    if agg.shape != (ns,):
        raise MeshError("agglomeration map must have one entry per simplex")
    if ns == 0:
        raise MeshError("empty mesh")
    nel = int(agg.max()) + 1
    nr = ns * (d + 1)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    verts = T(np.asarray(mesh.vertices, np.float64))
    simp = T(np.asarray(mesh.simplices, np.int32))
    svol = T(np.asarray(mesh.simplex_volumes, np.float64))
    tagg = T(agg)
    e = lambda n, dt: torch.empty(max(int(n), 1), dtype=dt, device=dev)
    i32, i64, f64 = torch.int32, torch.int64, torch.float64
    o = {"elem_ptr": e(nel + 1, i64), "elem_simplices": e(ns, i32), "boxes": e(nel * 2 * d, f64),
         "elem_volumes": e(nel, f64), "face_owner": e(nr, i32), "face_neighbor": e(nr, i32),
         "face_normal": e(nr * d, f64), "face_measure": e(nr, f64), "face_ptr": e(nr + 1, i64),
         "facet_vertices": e(nr * d, i32), "facet_owner_simplex": e(nr, i32), "facet_neighbor_simplex": e(nr, i32),
         "facet_measures": e(nr, f64), "iface_owner": e(nr, i32), "iface_neighbor": e(nr, i32),
         "iface_ptr": e(nr + 1, i64), "elem_bface_ptr": e(nel + 1, i64)}
    out = _lib.AggOut()
    for k in _OUT:
        setattr(out, k, _lib.ptr(o[k]))
    wsb = int(lib.pdg_agglomerate_workspace_bytes(d, ns, nel))
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    rc = lib.pdg_agglomerate(d, mesh.n_vertices, ns, _lib.ptr(verts), _lib.ptr(simp), _lib.ptr(svol),
                             _lib.ptr(tagg), nel, 1 if check_connected else 0, C.byref(out), _lib.ptr(ws), wsb,
                             _lib.stream_ptr(stream))
    if rc == _lib.PDG_ERR_INVALID:
        raise MeshError(lib.pdg_last_error().decode(errors="replace"))
    _lib.check(rc)
    nf, nk, nif, nfi = int(out.n_faces), int(out.n_facets), int(out.n_interfaces), int(out.n_interior_faces)
    h = lambda k, n: o[k][:n].cpu().numpy()
    flat = FlatMesh(
        dim=d,
        vertices=np.ascontiguousarray(mesh.vertices, np.float64),
        simplices=np.ascontiguousarray(mesh.simplices, np.int32),
        simplex_volumes=np.ascontiguousarray(mesh.simplex_volumes, np.float64),
        elem_ptr=h("elem_ptr", nel + 1),
        elem_simplices=h("elem_simplices", ns),
        boxes=h("boxes", nel * 2 * d).reshape(nel, 2, d),
        elem_volumes=h("elem_volumes", nel),
        face_owner=h("face_owner", nf),
        face_neighbor=h("face_neighbor", nf),
        face_tag=np.zeros(nf, np.int8),
        face_normal=h("face_normal", nf * d).reshape(nf, d),
        face_measure=h("face_measure", nf),
        face_ptr=h("face_ptr", nf + 1),
        facet_vertices=h("facet_vertices", nk * d).reshape(nk, d),
        facet_owner_simplex=h("facet_owner_simplex", nk),
        facet_neighbor_simplex=h("facet_neighbor_simplex", nk),
        facet_measures=h("facet_measures", nk),
        iface_owner=h("iface_owner", nif),
        iface_neighbor=h("iface_neighbor", nif),
        iface_ptr=h("iface_ptr", nif + 1),
        iface_faces=np.arange(nfi, dtype=np.int32),
        elem_bface_ptr=h("elem_bface_ptr", nel + 1),
        elem_bfaces=np.arange(nfi, nf, dtype=np.int32),
    )
    return PolytopicMesh(mesh, agg, flat)
