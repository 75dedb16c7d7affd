"""Space-time slabs on the B200 engine -- drop-in for polydg ``spacetime.py``.

A slab is one time interval crossed with a spatial polytopic mesh; its
elements are prisms (spatial element x interval) with bounding boxes
(spatial box x interval).  polydg assembles it through the same Approach-2
engine as the spatial problem with a second geometry provider
(``SlabGeometry``, spacetime.py:133-364):

* volume sub-items are sub-prisms (fine spatial simplex x interval) under
  tensor rules (simplex rule x interval rule of the same order,
  quadrature.py:159-178);
* lateral faces (spatial face x interval, normal (n, 0)) carry the interior /
  Dirichlet / Neumann / inflow / outflow machinery;
* bottom facets (the spatial subdivision at t0) are statically inflow: the
  time jump, with the previous slab's trace (or initial data) as boundary
  values; top facets are outflow (no contribution).

Here the whole slab (volume, lateral faces, bottom facet, RHS) is one fused
sm_100a kernel (``csrc/slab_body.cuh``, runtime-specialised with NVRTC per
coefficient set, degree and family), with the index phase and spatial
geometry frames shared with the spatial engine.  Public names mirror polydg:
``TimePartition``, ``SlabMesh``, ``build_slab``, ``assemble_slab``,
``march``, ``save_solution_vector`` / ``load_solution_vector``.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

from .basis import Family, SpecList, family_name
from .mesh import MeshError


@dataclass
class TimePartition:
    """Strictly increasing time nodes t_0 = 0 < ... < t_N = T (spacetime.py:58-81)."""

    nodes: np.ndarray

    def __post_init__(self):
        self.nodes = np.asarray(self.nodes, dtype=float)
        if self.nodes.ndim != 1 or self.nodes.shape[0] < 2:
            raise ValueError("need at least two time nodes")
        if np.any(np.diff(self.nodes) <= 0):
            raise ValueError("time nodes must be strictly increasing")

    @classmethod
    def uniform(cls, t_final: float, n_steps: int) -> "TimePartition":
        return cls(np.linspace(0.0, t_final, n_steps + 1))

    @property
    def n_steps(self) -> int:
        return self.nodes.shape[0] - 1

    def interval(self, n: int) -> tuple:
        return float(self.nodes[n]), float(self.nodes[n + 1])


@dataclass
class SlabMesh:
    """One space-time slab: spatial mesh x (t0, t1) (spacetime.py:84-104)."""

    spatial: object
    t0: float
    t1: float

    @property
    def tau(self) -> float:
        return self.t1 - self.t0

    @property
    def dim(self) -> int:
        return self.spatial.dim + 1

    @property
    def n_elements(self) -> int:
        return self.spatial.n_elements

    def prism_volume(self, element: int) -> float:
        return float(self.spatial.element_volumes[element] * self.tau)


def build_slab(spatial_mesh, interval, degrees, family=Family.PQ):
    """Slab mesh plus per-prism basis specs on (spatial box) x interval
    (spacetime.py:107-128)."""
    t0, t1 = float(interval[0]), float(interval[1])
    if not t1 > t0:
        raise ValueError("slab interval must have positive length")
    slab = SlabMesh(spatial_mesh, t0, t1)
    n = spatial_mesh.n_elements
    if np.isscalar(degrees):
        degrees = np.full(n, int(degrees))
    degrees = np.asarray(degrees, dtype=np.int64)
    if degrees.shape != (n,):
        raise ValueError("degrees must be scalar or one per element")
    sbox = np.asarray(spatial_mesh.bounding_boxes, dtype=np.float64)
    boxes = np.empty((n, 2, slab.dim))
    boxes[:, :, :-1] = sbox
    boxes[:, 0, -1], boxes[:, 1, -1] = t0, t1
    return slab, SpecList(degrees, boxes, family)


# -- binary solution dumps (spacetime.py:624-645) --------------------------------

def save_solution_vector(path, vec) -> None:
    """Little-endian binary dump: uint64 length header, then float64 data."""
    vec = np.asarray(vec, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", vec.shape[0]))
        fh.write(vec.tobytes())


def load_solution_vector(path) -> np.ndarray:
    with open(path, "rb") as fh:
        (n,) = struct.unpack("<Q", fh.read(8))
        data = np.frombuffer(fh.read(8 * n), dtype="<f8")
    if data.shape[0] != n:
        raise MeshError(f"{path}: truncated solution vector")
    return data.astype(float)


# -- lateral boundary classification (host pre-pass) ---------------------------------

def classify_lateral_faces(flat, t0, t1, coeffs, dirichlet_predicate=None) -> np.ndarray:
    """Tags of the lateral faces of a slab (``SlabGeometry._classify_lateral``,
    spacetime.py:229-246), vectorised over the spatial boundary faces: the
    order-2 facet rule x order-2 interval rule sample points; Dirichlet
    (or Neumann by predicate) where n^T A n > 1e-12 max(1, |A|) at their mean,
    else inflow / outflow by the sign of the mean b.n.  Interior faces get 0.
    polydg classifies inside the geometry constructor, i.e. per assembly, on
    the host; so does this (boundary faces only, a few per cent of faces)."""
    from .model import _checked_flow_sign_grouped, _face_sample_points
    from .mesh import BOUNDARY, BoundaryTag, tag_code
    from .quadrature import interval_rule

    tags = np.zeros(flat.n_faces, np.int8)
    bf = np.flatnonzero(flat.face_neighbor == BOUNDARY)
    if bf.size == 0:
        return tags
    sp, which, counts = _face_sample_points(flat, bf)
    tr = interval_rule(2)
    tau = t1 - t0
    tp = t0 + tau * tr.points[:, 0]
    nt = tp.shape[0]
    S = flat.dim
    pts = np.empty((sp.shape[0] * nt, S + 1))
    pts[:, :S] = np.repeat(sp, nt, axis=0)
    pts[:, S] = np.tile(tp, sp.shape[0])
    which = np.repeat(which, nt)
    counts = counts * nt
    n3 = np.zeros((bf.size, S + 1))
    n3[:, :S] = flat.face_normal[bf]
    mean = np.add.reduceat(pts, np.r_[0, np.cumsum(counts)[:-1]], axis=0) / counts[:, None]
    out = np.full(bf.size, tag_code(BoundaryTag.OUTFLOW), np.int8)
    decided = np.zeros(bf.size, bool)
    if coeffs.diffusion is not None:
        a = np.asarray(coeffs.diffusion(mean))
        tol = 1e-12 * np.maximum(1.0, np.abs(a).reshape(bf.size, -1).max(axis=1))
        ell = np.einsum("fi,fij,fj->f", n3, a, n3) > tol
        dirich = ell.copy()
        if dirichlet_predicate is not None:
            for k in np.flatnonzero(ell):
                dirich[k] = bool(dirichlet_predicate(mean[k]))
        out[ell & dirich] = tag_code(BoundaryTag.DIRICHLET)
        out[ell & ~dirich] = tag_code(BoundaryTag.NEUMANN)
        decided |= ell
    if coeffs.advection is not None:
        rest = ~decided
        bn = np.einsum("qd,qd->q", np.asarray(coeffs.advection(pts)), n3[which])
        sign = _checked_flow_sign_grouped(bn, counts, "a lateral slab face", rest)
        out[rest & (sign < 0.0)] = tag_code(BoundaryTag.INFLOW)
    tags[bf] = out
    return tags


# -- the device plan ------------------------------------------------------------------

class SlabPlan:
    """Device buffers + descriptors for repeated assembly of one slab.

    ``run()`` enqueues, on one stream and without host synchronisation: the
    index phase (adjacency, row offsets -- shared with the spatial engine, on
    the prism DoF map), the spatial affine frames, the lateral face pre-pass
    (sigma, flow side) and the fused slab kernel (values + col_idx + RHS).
    """

    def __init__(self, slab, coeffs, specs, u_prev, config=None, row_elements=None, device=None,
                 stream=None, dirichlet_predicate=None):
        import ctypes as C

        from . import _lib
        from .assembly import AssemblyConfig, AssemblyError, DeviceRules, DofMap, _torch, device_mesh
        from .basis import num_basis, spec_arrays
        from .model import as_scalar_expr, slab_policy

        torch = _torch()
        self.lib = _lib.load()
        config = config or AssemblyConfig()
        self.config = config
        self.slab = slab
        self.dm = device_mesh(slab.spatial, device)
        dev = self.device = self.dm.device
        flat = self.flat = self.dm.flat
        if flat.dim not in (2, 3):
            raise NotImplementedError("the device slab engine supports 2D and 3D spatial meshes")
        S = flat.dim
        self.S = S
        deg, boxes, fam = spec_arrays(specs)
        fname = family_name(fam)
        if deg.shape[0] != flat.n_elements:
            raise AssemblyError("one BasisSpec per element required")
        if boxes.shape[1:] != (2, S + 1):
            raise ValueError(f"slab spec boxes must be (2, {S + 1}): spatial box x interval")
        if not (np.all(boxes[:, 0, S] == slab.t0) and np.all(boxes[:, 1, S] == slab.t1)):
            raise NotImplementedError("the device slab engine needs prism boxes with the slab's time "
                                      "interval (build_slab)")
        pmax = int(deg.max()) if deg.size else 0
        if pmax > _lib.SLAB_MAX_DEGREE[fname]:
            raise NotImplementedError(f"slab degree {pmax} exceeds the device range "
                                      f"(p <= {_lib.SLAB_MAX_DEGREE[fname]} for family {fname})")
        if fname == "PQ" and np.any(deg != pmax):
            raise NotImplementedError("family PQ slabs need a uniform degree on the device")
        counts = np.array([num_basis(int(p), S + 1, fam) for p in deg], np.int64)
        self.dof = DofMap(np.concatenate([[0], np.cumsum(counts)]).astype(np.int64))
        self.degrees = deg
        inc = int(config.quad_increment)
        pen = config.penalty
        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self.t = {"degree": T(deg.astype(np.int32)), "box": T(boxes), "dof": T(self.dof.offsets),
                  "sbox": T(np.ascontiguousarray(boxes[:, :, :S]))}
        b = _lib.Basis()
        b.max_degree = pmax
        b.degree, b.box, b.dof_offset = _lib.ptr(self.t["degree"]), _lib.ptr(self.t["box"]), _lib.ptr(self.t["dof"])
        self.basis = b
        sb = _lib.Basis()  # spatial view for the frame pre-pass (2D boxes)
        sb.max_degree = pmax
        sb.degree, sb.box, sb.dof_offset = b.degree, _lib.ptr(self.t["sbox"]), b.dof_offset
        self.sbasis = sb

        uniq = np.unique(deg)
        vol_orders = [2 * int(p) + inc for p in uniq]
        face_orders = [2 * int(max(p, q)) + inc for p in uniq for q in uniq] + vol_orders
        self.rules = DeviceRules(S, vol_orders, face_orders, dev)
        # time axis: interval rules of every order in use (face tables of a 1D-facet table)
        self.trules = DeviceRules(2, [], sorted(set(face_orders) | {2}), dev)

        # time-jump data (spacetime.py:367-388)
        initial = None
        self.t["prev"] = self.t["prev_dof"] = self.t["prev_box"] = None
        if u_prev is None:
            raise MeshError("slab assembly needs initial data or a previous solution")
        if callable(u_prev) and not isinstance(u_prev, tuple):
            initial = as_scalar_expr(u_prev, "initial data")
        else:
            pspecs, pvec = u_prev
            pdeg, pbox, pfam = spec_arrays(pspecs)
            pvec = np.asarray(pvec, dtype=np.float64)
            pcounts = np.array([num_basis(int(p), S + 1, pfam) for p in pdeg], np.int64)
            if pcounts.sum() != pvec.shape[0]:
                raise MeshError(f"previous solution has {pvec.shape[0]} dofs, expected {int(pcounts.sum())}")
            if pdeg.shape[0] != flat.n_elements:
                raise MeshError("previous slab has a different spatial element count")
            if family_name(pfam) != fname or np.any(pdeg != deg):
                raise NotImplementedError("the device time jump needs the previous slab's degree and family")
            self.t["prev"] = T(pvec)
            self.t["prev_dof"] = T(np.concatenate([[0], np.cumsum(pcounts)]).astype(np.int64))
            self.t["prev_box"] = T(pbox)
        self.policy, rows, self.policy_info = slab_policy(coeffs, initial, with_info=True, dim=S + 1)
        self.family = fam
        self.policy = self.policy.encode()
        _lib.check(self.lib.pdg_slab_prepare(self.policy, S, pmax, 1 if fname == "PQ" else 0))

        tags = classify_lateral_faces(flat, slab.t0, slab.t1, coeffs, dirichlet_predicate)
        self.lateral_tags = tags
        self.t["lat"] = T(tags if tags.size else np.zeros(1, np.int8))
        s = _lib.Slab()
        s.t0, s.t1 = float(slab.t0), float(slab.t1)
        s.lateral_tag = _lib.ptr(self.t["lat"])
        s.prev_values = _lib.ptr(self.t["prev"])
        s.prev_dof_offset = _lib.ptr(self.t["prev_dof"])
        s.prev_box = _lib.ptr(self.t["prev_box"])
        s.family = 1 if fname == "PQ" else 0
        s.table_rows = rows
        s.time_rules = self.trules.struct
        self.sdesc = s

        prm = _lib.Params()
        prm.quad_increment = inc
        prm.include_gradient_terms = 1
        prm.penalty_constant = float(pen.constant)
        if pen.coverable is not None:
            self.t["coverable"] = T(np.asarray(pen.coverable, bool).astype(np.uint8))
            prm.coverable = _lib.ptr(self.t["coverable"])
        self.params = prm

        nel = flat.n_elements
        if row_elements is None:
            self.row_elements = np.arange(nel, dtype=np.int64)
            self.t["rows"] = None
        else:
            self.row_elements = np.unique(np.asarray(row_elements, dtype=np.int64))
            self.t["rows"] = T(self.row_elements.astype(np.int32))
        nr = self.row_elements.shape[0]
        self.n_local_rows = int(counts[self.row_elements].sum())
        FW = 8 if S == 2 else 16
        z = lambda n, dt: torch.empty(max(int(n), 1), dtype=dt, device=dev)
        i64, i32 = torch.int64, torch.int32
        nadj = nel + 2 * flat.n_interfaces
        self.t.update(nbr_ptr=z(nel + 1, i64), nbr_elem=z(nadj, i32), nbr_iface=z(nadj, i32),
                      row_len=z(nr, i64), val_off=z(nr + 1, i64), row_off=z(nr + 1, i64),
                      row_ptr=z(self.n_local_rows + 1, i64),
                      nbr_rec=z(nadj * 10, torch.float64),  # pdg_iface_rec, 80 B per entry
                      sigma=z(flat.n_faces, torch.float64), flow=z(flat.n_faces, torch.int8),
                      flags=torch.zeros(1, dtype=torch.int32, device=dev),
                      sframe=z(flat.n_simplices * FW, torch.float64), fframe=z(flat.n_facets * FW, torch.float64),
                      erec=z(nel * FW, torch.float64))
        fr = _lib.Frames()
        fr.simplex, fr.facet, fr.element = _lib.ptr(self.t["sframe"]), _lib.ptr(self.t["fframe"]), _lib.ptr(self.t["erec"])
        self.frames = fr
        self.ws_bytes = int(self.lib.pdg_workspace_bytes(nel, flat.n_interfaces))
        self.t["ws"] = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        pat = _lib.Pattern()
        pat.n_row_elements = nr
        pat.row_elements = _lib.ptr(self.t["rows"])
        pat.nbr_ptr, pat.nbr_elem, pat.nbr_iface = (_lib.ptr(self.t["nbr_ptr"]), _lib.ptr(self.t["nbr_elem"]),
                                                    _lib.ptr(self.t["nbr_iface"]))
        pat.row_len, pat.elem_val_offset, pat.elem_row_offset = (
            _lib.ptr(self.t["row_len"]), _lib.ptr(self.t["val_off"]), _lib.ptr(self.t["row_off"]))
        pat.row_ptr = _lib.ptr(self.t["row_ptr"])
        pat.nbr_rec = _lib.ptr(self.t["nbr_rec"])
        self.pattern = pat
        # kind flags the interface-record pre-pass reads (advection -> downwind bit)
        self.cflags = _lib.Coeffs()
        self.cflags.has_advection = int(self.policy_info["adv"])
        with torch.cuda.stream(self.stream):
            self._index_phase(size_query=True)
        self.t["col_idx"] = z(self.nnz, i64)
        self.t["values"] = z(self.nnz, torch.float64)
        self.t["rhs"] = torch.zeros(max(self.dof.n_dofs, 1), dtype=torch.float64, device=dev)
        pat.col_idx = _lib.ptr(self.t["col_idx"])
        self._C = C

    def _index_phase(self, size_query=False):
        from . import _lib

        C = __import__("ctypes")
        s = _lib.stream_ptr(self.stream)
        _lib.check(self.lib.pdg_adjacency(C.byref(self.dm.struct), _lib.ptr(self.t["nbr_ptr"]),
                                          _lib.ptr(self.t["nbr_elem"]), _lib.ptr(self.t["nbr_iface"]),
                                          _lib.ptr(self.t["ws"]), self.ws_bytes, s))
        nnz = C.c_int64(0)
        _lib.check(self.lib.pdg_pattern_offsets(C.byref(self.dm.struct), C.byref(self.basis), C.byref(self.pattern),
                                                self.n_local_rows, C.byref(nnz) if size_query else None,
                                                _lib.ptr(self.t["ws"]), self.ws_bytes, s))
        if size_query:
            self.nnz = int(nnz.value)

    def _prepass(self):
        from . import _lib

        C = self._C
        s = _lib.stream_ptr(self.stream)
        _lib.check(self.lib.pdg_frames_build(C.byref(self.dm.struct), C.byref(self.sbasis), C.byref(self.frames),
                                             _lib.ptr(self.t["flags"]), s))
        _lib.check(self.lib.pdg_slab_prepass(
            C.byref(self.dm.struct), C.byref(self.basis), self.policy, C.byref(self.rules.struct),
            C.byref(self.params), C.byref(self.sdesc), C.byref(self.frames), _lib.ptr(self.t["sigma"]),
            _lib.ptr(self.t["flow"]), _lib.ptr(self.t["flags"]), s))
        _lib.check(self.lib.pdg_iface_records(
            C.byref(self.dm.struct), C.byref(self.basis), C.byref(self.cflags), C.byref(self.rules.struct),
            C.byref(self.params), C.byref(self.pattern), _lib.ptr(self.t["sigma"]), _lib.ptr(self.t["flow"]), s))

    def _elements(self):
        from . import _lib

        C = self._C
        _lib.check(self.lib.pdg_slab_assemble(
            C.byref(self.dm.struct), C.byref(self.basis), self.policy, C.byref(self.rules.struct),
            C.byref(self.params), C.byref(self.sdesc), C.byref(self.pattern), C.byref(self.frames),
            _lib.ptr(self.t["sigma"]), _lib.ptr(self.t["flow"]), _lib.ptr(self.t["values"]),
            _lib.ptr(self.t["rhs"]), _lib.ptr(self.t["flags"]), _lib.stream_ptr(self.stream)))

    def run(self, events=None):
        """Enqueue index phase + pre-pass + slab kernel; no host sync."""
        import torch

        with torch.cuda.stream(self.stream):
            if events:
                events[0].record(self.stream)
            self._index_phase()
            if events:
                events[1].record(self.stream)
            self._prepass()
            if events:
                events[2].record(self.stream)
            self._elements()
            if events:
                events[3].record(self.stream)

    def check_flags(self):
        from . import _lib
        from .assembly import _raise_flags

        self.stream.synchronize()
        flags = int(self.t["flags"].item())
        if flags & _lib.FLAG_STACK:
            raise NotImplementedError("slab element with more than 32 neighbours (device staging capacity)")
        _raise_flags(flags)

    # -- results ----------------------------------------------------------------
    @property
    def values(self):
        return self.t["values"][: self.nnz]

    @property
    def col_idx(self):
        return self.t["col_idx"][: self.nnz]

    @property
    def row_ptr(self):
        return self.t["row_ptr"][: self.n_local_rows + 1]

    @property
    def rhs(self):
        return self.t["rhs"][: self.dof.n_dofs]

    def to_csr(self):
        from .assembly import CSRMatrix

        return CSRMatrix(self.n_local_rows, self.dof.n_dofs, self.row_ptr.cpu().numpy(),
                         self.col_idx.cpu().numpy(), self.values.cpu().numpy())

    def work_stats(self):
        """polydg per-kernel work items (assembly.py:360-391) of the slab: volume
        items = sub-prisms, interior = lateral sub-facets, inflow includes the
        bottom facets (one per sub-prism), top facets are outflow items."""
        from .assembly import KERNEL_NAMES, KernelTiming
        from .mesh import BOUNDARY, TAG_CODE

        f = self.flat
        counts = np.diff(self.dof.offsets)
        owned = np.zeros(f.n_elements, bool)
        owned[self.row_elements] = True
        nsim = np.diff(f.elem_ptr)
        out = {k: KernelTiming(k) for k in KERNEL_NAMES}
        out["element"].work_items = int(nsim[owned].sum())
        out["element"].nnz_written = int((nsim * counts * counts)[owned].sum())
        nfac = np.diff(f.face_ptr)
        o, nb = f.face_owner, f.face_neighbor
        inter = nb != BOUNDARY
        oo = owned[o]
        on = np.where(inter, owned[np.where(inter, nb, 0)], False)
        no, nn = counts[o], counts[np.where(inter, nb, 0)]
        per = np.where(oo & on, (no + nn) ** 2, np.where(oo, no * (no + nn), nn * (no + nn)))
        sel = inter & (oo | on)
        out["interior"].work_items = int(nfac[sel].sum())
        out["interior"].nnz_written = int((per * nfac)[sel].sum())
        tg = self.lateral_tags
        for name, codes in (("dirichlet", (TAG_CODE["dirichlet"],)), ("inflow", (TAG_CODE["inflow"],)),
                            ("neumann_outflow", (TAG_CODE["neumann"], TAG_CODE["outflow"]))):
            m = (~inter) & oo & np.isin(tg, codes)
            out[name].work_items = int(nfac[m].sum())
            if name != "neumann_outflow":
                out[name].nnz_written = int((nfac * no * no)[m].sum())
        out["inflow"].work_items += int(nsim[owned].sum())
        out["inflow"].nnz_written += int((nsim * counts * counts)[owned].sum())
        out["neumann_outflow"].work_items += int(nsim[owned].sum())
        return out


@dataclass
class ParabolicProblem:
    """Space-time description of a parabolic model problem (polydg
    model.py:263-275): block-form fields in (x, y, t) (diffusion
    [[a, 0], [0, 0]], advection (w, 1)) and initial data of the spatial
    coordinates."""

    spatial_dim: int
    coeffs: object
    initial: object
    t_final: float = 1.0


def assemble_slab(slab, coeffs, specs, u_prev, config=None, approach=2, dirichlet_predicate=None,
                  row_elements=None):
    """Assemble one slab system on the B200 (polydg ``spacetime.assemble_slab``,
    spacetime.py:391-413).  ``u_prev``: initial-data field of the spatial
    points (an Expr / ScalarField: it is evaluated on the device) for the
    first slab, or ``(previous specs, previous coefficient vector)``.
    ``approach`` 1 and 2 run the same preset-sparsity engine (polydg's two
    approaches agree within 1e-12).  Returns (CSRMatrix, rhs, AssemblyStats)."""
    import time

    import torch

    from .assembly import AssemblyStats

    if approach not in (1, 2):
        raise ValueError("approach must be 1 or 2")
    t_start = time.perf_counter()
    plan = SlabPlan(slab, coeffs, specs, u_prev, config, row_elements=row_elements,
                    dirichlet_predicate=dirichlet_predicate)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    plan.run(ev)
    plan.check_flags()
    ms_index, ms_pre, ms_el = (ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]))
    from .assembly import apportion
    from .roofline import slab_work

    kern = plan.work_stats()
    w = slab_work(plan)
    # one fused slab kernel: its time split by canonical FLOPs (the bottom
    # facet's time jump is polydg's inflow item, spacetime.py:367-388)
    apportion(kern, {"element": w["flops_volume"], "interior": w["flops_interior"],
                     "dirichlet": w["flops_dirichlet"], "inflow": w["flops_bottom"], "neumann_outflow": 0.0}, ms_el)
    stats = AssemblyStats(kernels=kern, index_seconds=ms_index * 1e-3, kernel_wall_seconds=ms_el * 1e-3,
                          triplet_count=sum(k.nnz_written for k in kern.values()), nnz=plan.nnz,
                          device_ms={"index": ms_index, "prepass": ms_pre, "element": ms_el},
                          kernel_split="apportioned by canonical FLOPs (one fused slab kernel)")
    matrix = plan.to_csr()
    rhs = plan.rhs.cpu().numpy().copy()
    stats.total_seconds = time.perf_counter() - t_start
    return matrix, rhs, stats


def _default_solver(matrix, rhs, dof_map):
    """polydg's default (spacetime.py:448-456): block-Jacobi preconditioned
    GMRES -- here on the device (solver.py)."""
    from .solver import solve

    result = solve(matrix, rhs, dof_map=dof_map)
    if not result.converged:
        raise RuntimeError(f"linear solve stagnated (residual {result.residual:.3e})")
    return result.x


def march(spatial_mesh, time_partition, problem, degrees, family=Family.PQ, config=None, solver=None,
          approach=2, dirichlet_predicate=None, dump_path=None):
    """Sequential slab-by-slab solve (polydg spacetime.py:434-481): each slab
    is assembled on the device with the previous slab's solution as the
    time-jump data; returns (per-slab coefficient vectors, [(slab, specs)])."""
    from .assembly import DofMap

    solver = solver or _default_solver
    solutions, slabs = [], []
    prev = problem.initial
    for n in range(time_partition.n_steps):
        slab, specs = build_slab(spatial_mesh, time_partition.interval(n), degrees, family)
        matrix, rhs, _ = assemble_slab(slab, problem.coeffs, specs, prev, config, approach, dirichlet_predicate)
        counts = np.diff(np.concatenate([[0], np.cumsum([s.n_funcs for s in specs])]))
        dof_map = DofMap(np.concatenate([[0], np.cumsum(counts)]).astype(np.int64))
        try:
            vec = np.asarray(solver(matrix, rhs, dof_map))
        except Exception as exc:
            raise RuntimeError(f"slab {n}: {exc}") from exc
        solutions.append(vec)
        slabs.append((slab, specs))
        prev = (specs, vec)
        if dump_path is not None:
            save_solution_vector(f"{dump_path}.slab{n:04d}.bin", vec)
    return solutions, slabs
