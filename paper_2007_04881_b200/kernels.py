"""Single-item public kernels of polydg, computed on the device.

polydg exports one function per kernel class for verification and for
callers that assemble by hand (``assembly.py:1139-1234``); they are also
what its hand-case tests call (``pkg/tests/test_assembly.py:97-227``).
Same names, arguments and return shapes here:

* ``interior_face_kernel(mesh, face, coeffs, spec_owner, spec_neighbor, sigma,
  quad_increment=2, include_gradient_terms=True, upwind_side=None)``
  -> ``(oo, on, no, nn)``;
* ``dirichlet_kernel(mesh, face, coeffs, spec, sigma, quad_increment=2,
  include_gradient_terms=True)`` -> ``(block, load)``;
* ``inflow_kernel(mesh, face, coeffs, spec, quad_increment=2)`` -> ``(block, load)``;
* ``neumann_outflow_kernel(mesh, face, coeffs, spec, quad_increment=2)`` -> ``load``;
* ``map_simplices`` / ``tabulate`` -- the device quadrature map and basis
  tabulation (``quadrature.py:118-136``, ``basis.py:129-164``);
* ``face_sigma`` -- the device penalty / flow-side pre-pass of a whole mesh
  (``assembly.py:596-626``, ``model.py:176-257``).

All of them run ``libpdg.so`` kernels (``pdg_face_blocks``,
``pdg_map_simplices``, ``pdg_tabulate``, ``pdg_face_prepass``); none has a
host implementation.  ``face`` may be a face object of the mesh (this
package's or polydg's) or a face id.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .basis import BasisSpec, family_name, num_basis
from .mesh import BOUNDARY, TAG_CODE, flat_of

_SIDE_OWNER, _SIDE_NEIGHBOR = 0, 1  # polydg assembly.py:50-51


def _face_id(mesh, face) -> int:
    if isinstance(face, (int, np.integer)):
        return int(face)
    fid = getattr(face, "_f", None)
    if fid is not None:
        return int(fid)
    for i, f in enumerate(mesh.faces):
        if f is face:
            return i
    raise ValueError("face does not belong to the mesh")


def _plan(mesh, coeffs, specs_by_element, quad_increment, include_gradient_terms=True):
    from .assembly import _UnitPlan

    flat = flat_of(mesh)
    base = specs_by_element.get("default")
    specs = [base] * flat.n_elements
    for e, s in specs_by_element.items():
        if e != "default":
            specs[e] = s
    plan = _UnitPlan(mesh, coeffs, specs, quad_increment)
    plan.params.include_gradient_terms = 1 if include_gradient_terms else 0
    return plan


def _run_items(plan, items):
    import torch

    n = len(items)
    nb = num_basis(int(plan.basis.max_degree), plan.dm.flat.dim)
    arr = (_lib.FaceItem * n)(*items)
    raw = np.frombuffer(bytes(arr), dtype=np.uint8)
    dev_items = torch.from_numpy(raw.copy()).to(plan.device)
    blocks = torch.empty(n * 4 * nb * nb, dtype=torch.float64, device=plan.device)
    loads = torch.empty(n * nb, dtype=torch.float64, device=plan.device)
    plan.flags.zero_()
    _lib.check(plan.lib.pdg_face_blocks(C.byref(plan.dm.struct), C.byref(plan.basis), C.byref(plan.coeffs),
                                        C.byref(plan.rules.struct), C.byref(plan.params), _lib.ptr(dev_items),
                                        n, _lib.ptr(blocks), _lib.ptr(loads), _lib.ptr(plan.flags),
                                        _lib.stream_ptr(plan.stream)))
    plan.stream.synchronize()
    from .assembly import _raise_flags

    _raise_flags(int(plan.flags.item()))
    return blocks.cpu().numpy().reshape(n, 2, 2, nb, nb), loads.cpu().numpy().reshape(n, nb)


def _flow_side(plan, fid: int) -> int:
    """Device flow classification of one face (pdg_face_prepass; straddling
    faces raise ClassificationError like polydg's _checked_flow_sign)."""
    import torch

    from .assembly import _raise_flags

    f = plan.dm.flat
    dev = plan.device
    sigma = torch.empty(max(f.n_faces, 1), dtype=torch.float64, device=dev)
    flow = torch.empty(max(f.n_faces, 1), dtype=torch.int8, device=dev)
    abar = torch.empty(max(f.n_elements, 1), dtype=torch.float64, device=dev)
    # polydg classifies the face whatever its tag (elemental_inflow_part,
    # model.py:176-191): the pre-pass sees every boundary face as Dirichlet
    tags = torch.from_numpy(np.where(f.face_neighbor == BOUNDARY, TAG_CODE["dirichlet"], TAG_CODE["interior"])
                            .astype(np.int8) if f.n_faces else np.zeros(1, np.int8)).to(dev)
    m = _lib.Mesh.from_buffer_copy(plan.dm.struct)
    m.face_tag = _lib.ptr(tags)
    plan.flags.zero_()
    _lib.check(plan.lib.pdg_frames_build(C.byref(m), C.byref(plan.basis), C.byref(plan.frames),
                                         _lib.ptr(plan.flags), _lib.stream_ptr(plan.stream)))
    _lib.check(plan.lib.pdg_face_prepass(C.byref(m), C.byref(plan.basis), C.byref(plan.coeffs),
                                         C.byref(plan.rules.struct), C.byref(plan.params), _lib.ptr(sigma),
                                         _lib.ptr(flow), _lib.ptr(abar), _lib.ptr(plan.flags),
                                         _lib.stream_ptr(plan.stream)))
    plan.stream.synchronize()
    _raise_flags(int(plan.flags.item()) & ~_lib.FLAG_NEG_DIFFUSION)
    return int(flow[fid].item())


def interior_face_kernel(mesh, face, coeffs, spec_owner, spec_neighbor, sigma, quad_increment=2,
                         include_gradient_terms=True, upwind_side=None):
    """Four dense blocks (oo, on, no, nn) integrated over all sub-faces
    (polydg ``assembly.py:1160-1188``)."""
    fid = _face_id(mesh, face)
    flat = flat_of(mesh)
    own, nbr = int(flat.face_owner[fid]), int(flat.face_neighbor[fid])
    if nbr == BOUNDARY:
        raise ValueError("interior_face_kernel needs an interior face")
    plan = _plan(mesh, coeffs, {"default": spec_owner, own: spec_owner, nbr: spec_neighbor}, quad_increment,
                 include_gradient_terms)
    if upwind_side is None:
        up = -1
        if plan.coeffs.has_advection:
            fl = _flow_side(plan, fid)  # 0: owner inflow, 1: neighbour inflow, -1: tangential
            up = _SIDE_OWNER if fl == 0 else (_SIDE_NEIGHBOR if fl == 1 else -1)
    else:
        up = int(upwind_side)
    B, _ = _run_items(plan, [_lib.FaceItem(fid, _lib.UNIT_INTERIOR, up, 0, float(sigma))])
    no, nn = spec_owner.n_funcs, spec_neighbor.n_funcs
    b = B[0]
    return (b[0, 0][:no, :no].copy(), b[0, 1][:no, :nn].copy(), b[1, 0][:nn, :no].copy(),
            b[1, 1][:nn, :nn].copy())


def dirichlet_kernel(mesh, face, coeffs, spec, sigma, quad_increment=2, include_gradient_terms=True):
    """Single-sided interior-penalty block and load of a Dirichlet face
    (polydg ``assembly.py:1190-1210``)."""
    fid = _face_id(mesh, face)
    own = int(flat_of(mesh).face_owner[fid])
    plan = _plan(mesh, coeffs, {"default": spec, own: spec}, quad_increment, include_gradient_terms)
    with_inflow = 0
    if plan.coeffs.has_advection:
        with_inflow = 1 if _flow_side(plan, fid) == 1 else 0
    B, L = _run_items(plan, [_lib.FaceItem(fid, _lib.UNIT_DIRICHLET, with_inflow, 0, float(sigma))])
    n = spec.n_funcs
    return B[0, 0, 0][:n, :n].copy(), L[0][:n].copy()


def inflow_kernel(mesh, face, coeffs, spec, quad_increment=2):
    """Weakly imposed upwind boundary term of a hyperbolic inflow face
    (polydg ``assembly.py:1212-1223``)."""
    fid = _face_id(mesh, face)
    own = int(flat_of(mesh).face_owner[fid])
    plan = _plan(mesh, coeffs, {"default": spec, own: spec}, quad_increment)
    if not plan.coeffs.has_advection:
        raise TypeError("inflow_kernel needs an advection field")
    B, L = _run_items(plan, [_lib.FaceItem(fid, _lib.UNIT_INFLOW, 0, 0, 0.0)])
    n = spec.n_funcs
    return B[0, 0, 0][:n, :n].copy(), L[0][:n].copy()


def neumann_outflow_kernel(mesh, face, coeffs, spec, quad_increment=2):
    """Load of a Neumann face; outflow (and any other tag) contributes
    nothing (polydg ``assembly.py:1225-1234``)."""
    fid = _face_id(mesh, face)
    flat = flat_of(mesh)
    n = spec.n_funcs
    if int(flat.face_tag[fid]) != TAG_CODE["neumann"]:
        return np.zeros(n)
    own = int(flat.face_owner[fid])
    plan = _plan(mesh, coeffs, {"default": spec, own: spec}, quad_increment)
    _, L = _run_items(plan, [_lib.FaceItem(fid, _lib.UNIT_NEUMANN, 0, 0, 0.0)])
    return L[0][:n].copy()


# ---------------------------------------------------------------------------
# quadrature map / tabulation / penalty pre-pass
# ---------------------------------------------------------------------------

def map_simplices(mesh, simplex_ids, order: int):
    """Mapped volume quadrature of simplices of ``mesh`` on the device
    (polydg ``map_to_simplex``, quadrature.py:118-136) ->
    (points [n, nq, d], weights [n, nq])."""
    import torch

    from .assembly import DeviceRules, _raise_flags, _require_cuda, device_mesh

    dm = device_mesh(mesh)
    d = dm.flat.dim
    dev = _require_cuda(None)
    rules = DeviceRules(d, [int(order)], [], dev)
    ids = torch.from_numpy(np.ascontiguousarray(np.asarray(simplex_ids, np.int32))).to(dev)
    n = int(ids.numel())
    nq = _rule_points(d, int(order))
    pts = torch.empty(max(n * nq * d, 1), dtype=torch.float64, device=dev)
    wts = torch.empty(max(n * nq, 1), dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    _lib.check(_lib.load().pdg_map_simplices(C.byref(dm.struct), C.byref(rules.struct), int(order), _lib.ptr(ids),
                                             n, _lib.ptr(pts), _lib.ptr(wts), _lib.ptr(flags),
                                             _lib.stream_ptr(stream)))
    stream.synchronize()
    _raise_flags(int(flags.item()))
    return pts[: n * nq * d].cpu().numpy().reshape(n, nq, d), wts[: n * nq].cpu().numpy().reshape(n, nq)


def _rule_points(d: int, order: int) -> int:
    from .quadrature import points_per_axis

    return points_per_axis(order) ** d


def tabulate(spec: BasisSpec, pts):
    """Basis values (n, nq) and gradients (n, d, nq) of ``spec`` at physical
    points ``pts`` (nq, d), on the device (polydg ``basis.tabulate``,
    basis.py:129-164)."""
    import torch

    from .assembly import _require_cuda

    pts = np.ascontiguousarray(np.asarray(pts, np.float64))
    nq, d = pts.shape
    box = np.asarray(spec.box, np.float64).reshape(2, d)
    p = int(spec.degree)
    if family_name(spec.family) != "P":
        raise NotImplementedError("device tabulation implements family P")
    dev = _require_cuda(None)
    lib = _lib.load()
    m = _lib.Mesh()
    m.dim = d
    t_deg = torch.tensor([p], dtype=torch.int32, device=dev)
    t_box = torch.from_numpy(box.reshape(1, 2, d).copy()).to(dev)
    t_dof = torch.tensor([0, num_basis(p, d)], dtype=torch.int64, device=dev)
    b = _lib.Basis()
    b.max_degree = p
    b.degree, b.box, b.dof_offset = _lib.ptr(t_deg), _lib.ptr(t_box), _lib.ptr(t_dof)
    nb = num_basis(p, d)
    t_pts = torch.from_numpy(pts).to(dev)
    vals = torch.empty(max(nq * nb, 1), dtype=torch.float64, device=dev)
    grads = torch.empty(max(nq * d * nb, 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    _lib.check(lib.pdg_tabulate(C.byref(m), C.byref(b), 0, _lib.ptr(t_pts), nq, _lib.ptr(vals), _lib.ptr(grads),
                                _lib.stream_ptr(stream)))
    stream.synchronize()
    v = vals[: nq * nb].cpu().numpy().reshape(nq, nb).T.copy()
    g = grads[: nq * d * nb].cpu().numpy().reshape(nq, d, nb).transpose(2, 1, 0).copy()
    return v, g


def eval_coefficients(coeffs, pts):
    """Every coefficient field at ``pts`` (nq, d) on the device (bytecode
    interpreter, numpy-identical trigonometry) -> dict of arrays:
    ``diffusion`` (nq, d, d), ``advection`` (nq, d), ``reaction``, ``source``,
    ``dirichlet``, ``neumann`` (nq,)."""
    import torch

    from .assembly import _require_cuda
    from .model import compile_coeffs

    pts = np.ascontiguousarray(np.asarray(pts, np.float64))
    nq, d = pts.shape
    dev = _require_cuda(None)
    cs = _lib.coeffs_struct(compile_coeffs(coeffs, d))
    K = d * d + d + 4
    t_pts = torch.from_numpy(pts).to(dev)
    out = torch.empty(max(nq * K, 1), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    _lib.check(_lib.load().pdg_eval_coeffs(d, C.byref(cs), _lib.ptr(t_pts), nq, _lib.ptr(out),
                                           _lib.stream_ptr(stream)))
    stream.synchronize()
    o = out[: nq * K].cpu().numpy().reshape(nq, K)
    return {"diffusion": o[:, : d * d].reshape(nq, d, d), "advection": o[:, d * d: d * d + d],
            "reaction": o[:, d * d + d], "source": o[:, d * d + d + 1],
            "dirichlet": o[:, d * d + d + 2], "neumann": o[:, d * d + d + 3]}


def face_sigma(mesh, coeffs, specs, config=None):
    """Penalty sigma and flow side of every face from the device pre-pass
    (polydg ``MeshGeometry.face_sigma`` / ``upwind_side`` / ``dirichlet_inflow``,
    assembly.py:596-626) -> (sigma [n_faces], flow [n_faces]); flow: interior
    0 = owner inflow, 1 = neighbour inflow, -1 = none; boundary 1 = owner inflow.
    As in polydg's work plan, sigma and flow are formed only where the
    assembly reads them (interior and Dirichlet faces); other faces hold 0."""
    import torch

    from .assembly import AssemblyConfig, SipgPlan

    plan = SipgPlan(mesh, coeffs, specs, config or AssemblyConfig())
    with torch.cuda.stream(plan.stream):
        plan._frames()
        plan._face_prepass()
    plan.stream.synchronize()
    from .assembly import _raise_flags

    _raise_flags(int(plan.t["flags"].item()) & ~_lib.FLAG_NEG_DIFFUSION)
    nf = plan.flat.n_faces
    return plan.t["sigma"][:nf].cpu().numpy(), plan.t["flow"][:nf].cpu().numpy()
