"""Approach 1 (stage-and-sort) on the B200 -- polydg ``assemble_approach1``
(assembly.py:158-174, 977-1087), the paper's first approach.

Every work item of polydg's plan -- volume sub-simplex, interior sub-facet,
boundary sub-facet (assembly.py:665-728) -- is one warp of
``pdg_a1_emit`` (csrc/approach1_body.cuh) that writes its dense local blocks
into its triplet stripe (widths of ``_item_stripe_width``, assembly.py:733-745;
unused slots keep the sentinel), then ``pdg_triplets_to_csr`` sorts the
triplets (stable radix sort) and merges duplicates (reduce-by-key) into the
CSR -- the index phase the paper times against Approach 2's preset pattern
(PAPER.md:601).  Items are in polydg's order for uniform-degree meshes
(volume by element, interior by face, then Dirichlet / inflow / Neumann by
face), so duplicates merge in the same order.
"""

from __future__ import annotations

import ctypes as C
import time
from typing import Optional

import numpy as np

from . import _lib
from .assembly import (
    AssemblyConfig,
    AssemblyStats,
    CSRMatrix,
    KERNEL_NAMES,
    KernelTiming,
    SipgPlan,
    _check_classified,
    _torch,
)
from .mesh import BOUNDARY, TAG_CODE


class Approach1Plan:
    """Device buffers of one stage-and-sort assembly (reuses a SipgPlan for
    the mesh, basis, rules, coefficients, frames and the face pre-pass)."""

    def __init__(self, mesh, coeffs, specs, config: Optional[AssemblyConfig] = None, device=None, stream=None):
        torch = _torch()
        self.base = SipgPlan(mesh, coeffs, specs, config, device=device, stream=stream, allocate_csr=False)
        b = self.base
        if b.jit_source is None:
            raise NotImplementedError("Approach 1 needs the runtime-specialised (NVRTC) kernels")
        f = b.flat
        dev = b.device
        counts = np.diff(b.dof.offsets)
        deg = b.degrees
        nsim = np.diff(f.elem_ptr)
        # -- work items in polydg's order (uniform degree: build_work_plan's order)
        vol_el = np.repeat(np.arange(f.n_elements, dtype=np.int32), nsim)
        nfac = np.diff(f.face_ptr)
        o, nb = f.face_owner.astype(np.int64), f.face_neighbor.astype(np.int64)
        inter = nb != BOUNDARY
        tag = f.face_tag
        groups = [np.flatnonzero(inter)]
        for name in ("dirichlet", "inflow", "neumann"):
            groups.append(np.flatnonzero((~inter) & (tag == TAG_CODE[name])))
        faces, rows, widths, loads = [], [], [], []
        for gi, fs in enumerate(groups):
            if fs.size:
                key = np.lexsort((fs, deg[o[fs]] if gi else np.maximum(deg[o[fs]], deg[np.where(inter, nb, 0)[fs]])))
                fs = fs[key]
            rep = nfac[fs]
            ff = np.repeat(fs, rep)
            first = np.repeat(f.face_ptr[fs], rep)
            within = np.arange(ff.size) - np.repeat(np.cumsum(rep) - rep, rep)
            faces.append(ff)
            rows.append(first + within)
            no = counts[o[ff]]
            if gi == 0:
                nn = counts[nb[ff]]
                widths.append(4 * np.maximum(no, nn) ** 2)
                loads.append(np.zeros(ff.size, np.int64))
            elif gi < 3:
                widths.append(no * no)
                loads.append(no)
            else:
                widths.append(np.zeros(ff.size, np.int64))
                loads.append(no)
        if vol_el.size and np.any(deg != deg[0]):
            order = np.lexsort((np.arange(vol_el.size), deg[vol_el]))
            if np.any(order != np.arange(order.size)):
                raise NotImplementedError("per-element degrees: Approach 1 on the device keeps element "
                                          "order for volume items (use assemble_approach2)")
        vw = counts[vol_el] ** 2
        vl = counts[vol_el]
        face = np.concatenate(faces).astype(np.int32) if faces else np.zeros(0, np.int32)
        frow = np.concatenate(rows).astype(np.int64) if rows else np.zeros(0, np.int64)
        width = np.concatenate([vw] + widths).astype(np.int64)
        load = np.concatenate([vl] + loads).astype(np.int64)
        self.stripe = np.concatenate([[0], np.cumsum(width)]).astype(np.int64)
        self.lstripe = np.concatenate([[0], np.cumsum(load)]).astype(np.int64)
        self.n_volume, self.n_interior = int(vol_el.size), int(faces[0].size)
        self.n_boundary = int(face.size - self.n_interior)
        self.n_triplets = int(self.stripe[-1])
        self.n_loads = int(self.lstripe[-1])
        # triplets actually written (the rest are sentinel padding)
        ii = face[: self.n_interior].astype(np.int64)
        no_i, nn_i = counts[o[ii]], counts[nb[ii]]
        self.n_written = int(self.n_triplets - np.sum(4 * np.maximum(no_i, nn_i) ** 2 - (no_i + nn_i) ** 2))
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        z = lambda n, dt: torch.empty(max(int(n), 1), dtype=dt, device=dev)
        self.t = {"vol_el": T(vol_el if vol_el.size else np.zeros(1, np.int32)),
                  "face": T(face if face.size else np.zeros(1, np.int32)),
                  "frow": T(frow if frow.size else np.zeros(1, np.int64)),
                  "stripe": T(self.stripe), "lstripe": T(self.lstripe),
                  "keys": z(self.n_triplets, torch.int64), "vals": z(self.n_triplets, torch.float64),
                  "lkeys": z(self.n_loads, torch.int64), "lvals": z(self.n_loads, torch.float64),
                  "row_ptr": z(b.dof.n_dofs + 1, torch.int64), "col_idx": z(self.n_triplets, torch.int64),
                  "values": z(self.n_triplets, torch.float64), "rhs": z(b.dof.n_dofs, torch.float64),
                  "nnz": torch.zeros(1, dtype=torch.int64, device=dev)}
        ws = int(b.lib.pdg_triplets_workspace_bytes(max(self.n_triplets, self.n_loads)))
        self.ws_bytes = ws
        self.t["ws"] = torch.empty(ws, dtype=torch.uint8, device=dev)
        it = _lib.A1Items()
        it.n_volume, it.n_interior, it.n_boundary = self.n_volume, self.n_interior, self.n_boundary
        it.n_cols = b.dof.n_dofs
        it.volume_element = _lib.ptr(self.t["vol_el"])
        it.face, it.facet_row = _lib.ptr(self.t["face"]), _lib.ptr(self.t["frow"])
        it.stripe_offset, it.load_offset = _lib.ptr(self.t["stripe"]), _lib.ptr(self.t["lstripe"])
        self.items = it
        self.stream = b.stream

    def _prepass(self):
        self.base._frames()
        self.base._face_prepass()

    def _emit(self):
        b = self.base
        s = _lib.stream_ptr(self.stream)
        self.t["keys"].fill_(-1)  # sentinel stripes (assembly.py:158-174)
        _lib.check(b.lib.pdg_a1_emit(C.byref(b.dm.struct), C.byref(b.basis), C.byref(b.coeffs), b.jit_source,
                                     C.byref(b.rules.struct), C.byref(b.params), C.byref(b.frames),
                                     _lib.ptr(b.t["sigma"]), _lib.ptr(b.t["flow"]), C.byref(self.items),
                                     _lib.ptr(self.t["keys"]), _lib.ptr(self.t["vals"]), _lib.ptr(self.t["lkeys"]),
                                     _lib.ptr(self.t["lvals"]), _lib.ptr(b.t["flags"]), s))

    def _merge(self):
        b = self.base
        s = _lib.stream_ptr(self.stream)
        n = b.dof.n_dofs
        _lib.check(b.lib.pdg_triplets_to_csr(_lib.ptr(self.t["keys"]), _lib.ptr(self.t["vals"]), self.n_triplets,
                                             n, n, _lib.ptr(self.t["row_ptr"]), _lib.ptr(self.t["col_idx"]),
                                             _lib.ptr(self.t["values"]), _lib.ptr(self.t["nnz"]),
                                             _lib.ptr(self.t["ws"]), self.ws_bytes, s))
        _lib.check(b.lib.pdg_triplets_to_vector(_lib.ptr(self.t["lkeys"]), _lib.ptr(self.t["lvals"]), self.n_loads,
                                                n, _lib.ptr(self.t["rhs"]), _lib.ptr(self.t["ws"]), self.ws_bytes, s))

    def run(self, events=None):
        """Enqueue frames + face pre-pass, item emission (the kernels), then
        sort + merge (the index phase); no host sync.  ``events``: 4 CUDA
        events recorded at the phase boundaries."""
        torch = _torch()
        with torch.cuda.stream(self.stream):
            if events:
                events[0].record(self.stream)
            self._prepass()
            if events:
                events[1].record(self.stream)
            self._emit()
            if events:
                events[2].record(self.stream)
            self._merge()
            if events:
                events[3].record(self.stream)

    def check_flags(self):
        self.base.check_flags()

    def to_csr(self) -> CSRMatrix:
        nnz = int(self.t["nnz"].item())
        n = self.base.dof.n_dofs
        return CSRMatrix(n, n, self.t["row_ptr"][: n + 1].cpu().numpy(), self.t["col_idx"][:nnz].cpu().numpy(),
                         self.t["values"][:nnz].cpu().numpy())

    @property
    def rhs(self):
        return self.t["rhs"][: self.base.dof.n_dofs]

    # HostIO / bench view (the CSR as produced by the merge)
    @property
    def dm(self):
        return self.base.dm

    @property
    def dof(self):
        return self.base.dof

    @property
    def nnz(self) -> int:
        """Entries of the merged CSR (device count of the last merge; one sync
        the first time it is read)."""
        if not getattr(self, "_nnz", 0):
            self.stream.synchronize()
            self._nnz = int(self.t["nnz"].item())
        return self._nnz

    @property
    def row_ptr(self):
        return self.t["row_ptr"][: self.base.dof.n_dofs + 1]

    @property
    def col_idx(self):
        return self.t["col_idx"][: self.nnz]

    @property
    def values(self):
        return self.t["values"][: self.nnz]


def assemble_approach1_device(mesh, coeffs, specs, config: Optional[AssemblyConfig] = None):
    """Stage-and-sort assembly on the B200 (polydg ``assemble_approach1``,
    assembly.py:1036-1045) -> (CSRMatrix, rhs, AssemblyStats)."""
    torch = _torch()
    t0 = time.perf_counter()
    _check_classified(mesh)
    plan = Approach1Plan(mesh, coeffs, specs, config)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    plan.run(ev)
    plan.check_flags()
    ms_pre, ms_k, ms_idx = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])
    matrix = plan.to_csr()
    rhs = plan.rhs.cpu().numpy().copy()
    # polydg A1 timers: index = triplets_to_csr (sort + merge), kernel wall =
    # the emission kernels; the pre-pass (sigma / flow side) is plan work
    from .assembly import apportion
    from .roofline import assembly_work

    kern = plan.base.work_stats()
    w = assembly_work(plan.base)
    apportion(kern, {"element": w["flops_volume"], "interior": w["flops_interior"],
                     "dirichlet": w["flops_dirichlet"], "inflow": w["flops_inflow"],
                     "neumann_outflow": w["flops_neumann"]}, ms_k)
    stats = AssemblyStats(kernels=kern, index_seconds=ms_idx * 1e-3, kernel_wall_seconds=ms_k * 1e-3,
                          total_seconds=time.perf_counter() - t0, triplet_count=plan.n_written, nnz=matrix.nnz,
                          device_ms={"prepass": ms_pre, "emit": ms_k, "sort_merge": ms_idx},
                          kernel_split="apportioned by canonical FLOPs (one fused emission kernel)")
    return matrix, rhs, stats


__all__ = ["Approach1Plan", "assemble_approach1_device", "KERNEL_NAMES", "KernelTiming"]
