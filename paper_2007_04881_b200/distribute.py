"""Row-partitioned (multi-GPU) assembly -- polydg ``distribute.py`` semantics.

Assembly is communication-free (polydg ``distribute.py:1-12``):
each part owns the rows of its elements and computes, with the same element
kernel, its volumes, its boundary faces and BOTH traces of every face that
touches it -- cut faces are evaluated once per side and emit only the owned
rows (``_SIDE_OWNER/_SIDE_NEIGHBOR``, polydg ``assembly.py:685-696``).  Because
the device kernel is already element-centric (one writer per row), a part's
rows are bit-identical to the same rows of the monolithic assembly.

Partitioning: polydg's greedy graph bisection (``distribute.py:75-184``) is
replaced by contiguous element ranges (element ids are spatially coherent,
e.g. Morton-ordered Voronoi seeds) cut at prefix sums of polydg's cost model
``quadrature_cost_weights`` (``distribute.py:63-72``).  Any other
element->part map can be supplied as a :class:`Partition`.

One process per GPU; ``torch.distributed`` (NCCL) is used only to gather the
row blocks on rank 0 for verification (``gather_and_verify``) -- never on the
assembly path.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .assembly import AssemblyConfig, AssemblyError, CSRMatrix, DofMap, assemble_device
from .basis import spec_arrays
from .mesh import flat_of
from .quadrature import points_per_axis


class PartitionError(ValueError):
    pass


@dataclass
class Partition:
    """Element-to-part map (polydg ``distribute.py:39-60``)."""

    n_parts: int
    part_of: np.ndarray
    owned: list
    cut_interfaces: np.ndarray
    weights: np.ndarray

    def validate(self, mesh) -> None:
        flat = flat_of(mesh)
        if self.part_of.shape != (flat.n_elements,):
            raise PartitionError("partition map has wrong length")
        for p in range(self.n_parts):
            if self.owned[p].size == 0:
                raise PartitionError(f"part {p} owns no elements")
        po = self.part_of
        cut = np.flatnonzero(po[flat.iface_owner] != po[flat.iface_neighbor])
        if not np.array_equal(np.sort(cut), np.sort(np.asarray(self.cut_interfaces))):
            raise PartitionError("cut-interface list inconsistent with the map")


def quadrature_cost_weights(mesh, specs, quad_increment: int = 2) -> np.ndarray:
    """simplices x quadrature points x n_basis^2 per element (polydg ``distribute.py:63-72``)."""
    flat = flat_of(mesh)
    d = flat.dim
    deg, _, fam = spec_arrays(specs)
    dm = DofMap.from_specs(specs)
    n = np.diff(dm.offsets)
    orders = 2 * deg + quad_increment  # family P: total degree = degree
    nq = np.array([points_per_axis(int(o)) ** d for o in orders], dtype=np.float64)
    return np.diff(flat.elem_ptr).astype(np.float64) * nq * n * n


def partition_from_map(mesh, part_of, weights=None) -> Partition:
    flat = flat_of(mesh)
    part_of = np.asarray(part_of, dtype=np.int64)
    n_parts = int(part_of.max()) + 1 if part_of.size else 0
    w = np.ones(flat.n_elements) if weights is None else np.asarray(weights, float)
    owned = [np.flatnonzero(part_of == p) for p in range(n_parts)]
    cut = np.flatnonzero(part_of[flat.iface_owner] != part_of[flat.iface_neighbor])
    totals = np.array([w[o].sum() for o in owned])
    p = Partition(n_parts, part_of, owned, cut, totals)
    p.validate(mesh)
    return p


def contiguous_partition(mesh, n_parts: int, weights: Optional[np.ndarray] = None) -> Partition:
    """Contiguous element ranges with balanced weight prefix sums."""
    flat = flat_of(mesh)
    nel = flat.n_elements
    if n_parts < 1:
        raise PartitionError("n_parts must be >= 1")
    if n_parts > nel:
        raise PartitionError(f"cannot split {nel} elements into {n_parts} parts")
    w = np.ones(nel) if weights is None else np.asarray(weights, dtype=float)
    cum = np.cumsum(w)
    targets = cum[-1] * np.arange(1, n_parts) / n_parts
    cuts = np.searchsorted(cum, targets, side="left") + 1
    cuts = np.clip(cuts, np.arange(1, n_parts), nel - np.arange(n_parts - 1, 0, -1))
    # strictly increasing, every part non-empty: forward pass cuts[k] >= cuts[k-1] + 1,
    # backward pass cuts[k] <= nel - (n_parts - 1 - k)
    for k in range(1, cuts.size):
        cuts[k] = max(cuts[k], cuts[k - 1] + 1)
    for k in range(cuts.size - 1, -1, -1):
        cuts[k] = min(cuts[k], nel - (n_parts - 1 - k), cuts[k + 1] - 1 if k + 1 < cuts.size else nel)
    part_of = np.zeros(nel, dtype=np.int64)
    for c in cuts:
        part_of[c:] += 1
    return partition_from_map(mesh, part_of, w)


@dataclass
class PartialMatrix:
    """Rows owned by one part, global columns (polydg ``distribute.py:187-197``)."""

    part: int
    row_ranges: list
    matrix: CSRMatrix

    @property
    def n_rows(self) -> int:
        return self.matrix.n_rows


def _row_ranges(dof: DofMap, own: np.ndarray):
    starts = dof.offsets[own]
    stops = dof.offsets[own + 1]
    ranges = []
    for a, b in zip(starts.tolist(), stops.tolist()):
        if ranges and ranges[-1][1] == a:
            ranges[-1] = (ranges[-1][0], b)
        else:
            ranges.append((a, b))
    return ranges


def _ragged(ptr: np.ndarray, sel: np.ndarray):
    """(flat indices of the ranges ptr[sel[i]]:ptr[sel[i]+1] concatenated, counts)."""
    a, b = ptr[sel], ptr[sel + 1]
    cnt = (b - a).astype(np.int64)
    tot = int(cnt.sum())
    idx = np.repeat(a - np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt) + np.arange(tot, dtype=np.int64)
    return idx, cnt


@dataclass
class LocalProblem:
    """One rank's share of a row-partitioned assembly: its owned elements plus
    their one-ring face neighbours (the halo), relabelled monotonically.

    ``flat`` is a complete FlatMesh of those elements (whole simplices,
    vertices, the faces touching an owned element, the interfaces through
    them), so the rank's index phase, pre-pass and element kernel touch
    nothing else -- the paper's "each GPU creates the sparsity pattern of
    its allocated subdivision".  Because a row depends
    only on its element and the face neighbours (patch oracle)
    and the relabelling preserves order, the owned rows are bit-identical
    to the same rows of the whole-mesh assembly; ``col_dof`` (the GLOBAL
    first DoF of every local element) makes the kernels emit global column
    indices (pdg_pattern.col_dof)."""

    flat: object                 # FlatMesh of owned + halo elements
    elements: np.ndarray         # local -> global element id (ascending)
    owned_local: np.ndarray      # local ids of the owned elements (ascending)
    col_dof: np.ndarray          # int64 [n_local]: global DoF offset of each local element
    specs: object                # SpecList of the local elements
    config: AssemblyConfig       # penalty coverability sliced to the local elements
    n_dofs_global: int


def submesh(flat, owned: np.ndarray):
    """(local FlatMesh, local->global element ids, local ids of ``owned``) of
    ``owned`` + its face neighbours, every id relabelled monotonically (element,
    simplex, vertex order preserved; faces in their original order; interfaces
    stay sorted by (owner, neighbour))."""
    from .mesh import FlatMesh

    nel = flat.n_elements
    owned = np.unique(np.asarray(owned, np.int64))
    own = np.zeros(nel, bool)
    own[owned] = True
    io, inb = flat.iface_owner.astype(np.int64), flat.iface_neighbor.astype(np.int64)
    ik = np.flatnonzero(own[io] | own[inb])
    K = np.unique(np.concatenate([owned, io[ik], inb[ik]]))
    newid = np.full(nel, -1, np.int64)
    newid[K] = np.arange(K.size)
    # simplices (whole elements) and vertices
    sidx, scnt = _ragged(flat.elem_ptr, K)
    sim_g = flat.elem_simplices[sidx].astype(np.int64)
    sim_sorted = np.sort(sim_g)
    newsim = np.full(flat.n_simplices, -1, np.int64)
    newsim[sim_sorted] = np.arange(sim_sorted.size)
    sv = flat.simplices[sim_sorted].astype(np.int64)
    vg = np.unique(sv)
    newv = np.full(flat.n_vertices, -1, np.int64)
    newv[vg] = np.arange(vg.size)
    elem_ptr = np.zeros(K.size + 1, np.int64)
    np.cumsum(scnt, out=elem_ptr[1:])
    # faces: every face of an interface through an owned element, then the
    # owned elements' boundary faces (original order)
    fidx, fcnt_if = _ragged(flat.iface_ptr, ik)
    fi = flat.iface_faces[fidx].astype(np.int64)
    bf = np.flatnonzero((flat.face_neighbor == -1) & own[flat.face_owner])
    kf = np.concatenate([fi, bf])
    nb = flat.face_neighbor[kf].astype(np.int64)
    face_neighbor = np.where(nb >= 0, newid[np.maximum(nb, 0)], -1).astype(np.int32)
    face_owner = newid[flat.face_owner[kf]].astype(np.int32)
    ridx, rcnt = _ragged(flat.face_ptr, kf)
    face_ptr = np.zeros(kf.size + 1, np.int64)
    np.cumsum(rcnt, out=face_ptr[1:])
    fns = flat.facet_neighbor_simplex[ridx].astype(np.int64)
    iface_ptr = np.zeros(ik.size + 1, np.int64)
    np.cumsum(fcnt_if, out=iface_ptr[1:])
    bown = face_owner[fi.size:].astype(np.int64)
    order = np.argsort(bown, kind="stable")
    bptr = np.zeros(K.size + 1, np.int64)
    np.cumsum(np.bincount(bown, minlength=K.size), out=bptr[1:])
    local = FlatMesh(
        dim=flat.dim,
        vertices=np.ascontiguousarray(flat.vertices[vg]),
        simplices=newv[sv].astype(np.int32),
        simplex_volumes=np.ascontiguousarray(flat.simplex_volumes[sim_sorted]),
        elem_ptr=elem_ptr,
        elem_simplices=newsim[sim_g].astype(np.int32),
        boxes=np.ascontiguousarray(flat.boxes[K]),
        elem_volumes=np.ascontiguousarray(flat.elem_volumes[K]),
        face_owner=face_owner, face_neighbor=face_neighbor,
        face_tag=np.ascontiguousarray(flat.face_tag[kf]),
        face_normal=np.ascontiguousarray(flat.face_normal[kf]),
        face_measure=np.ascontiguousarray(flat.face_measure[kf]),
        face_ptr=face_ptr,
        facet_vertices=newv[flat.facet_vertices[ridx]].astype(np.int32),
        facet_owner_simplex=newsim[flat.facet_owner_simplex[ridx]].astype(np.int32),
        facet_neighbor_simplex=np.where(fns >= 0, newsim[np.maximum(fns, 0)], -1).astype(np.int32),
        facet_measures=np.ascontiguousarray(flat.facet_measures[ridx]),
        iface_owner=newid[io[ik]].astype(np.int32),
        iface_neighbor=newid[inb[ik]].astype(np.int32),
        iface_ptr=iface_ptr,
        iface_faces=np.arange(fi.size, dtype=np.int32),
        elem_bface_ptr=bptr,
        elem_bfaces=(fi.size + order).astype(np.int32),
    )
    return local, K, newid[owned]


def local_problem(mesh, partition: Partition, part_id: int, specs,
                  config: Optional[AssemblyConfig] = None) -> LocalProblem:
    """The sub-mesh, specs and global column map of one part (host
    preprocessing, outside the timed assembly)."""
    from dataclasses import replace

    from .basis import SpecList, spec_arrays

    if not 0 <= part_id < partition.n_parts:
        raise PartitionError(f"part {part_id} out of range")
    flat = flat_of(mesh)
    config = config or AssemblyConfig()
    local, K, own_local = submesh(flat, partition.owned[part_id])
    deg, boxes, fam = spec_arrays(specs)
    dof = DofMap.from_specs(specs)
    pen = config.penalty
    if pen.coverable is not None:
        pen = replace(pen, coverable=np.asarray(pen.coverable, bool)[K])
    return LocalProblem(local, K, own_local, dof.offsets[K].astype(np.int64), SpecList(deg[K], boxes[K], fam),
                        replace(config, penalty=pen), dof.n_dofs)


def assemble_partition_device(mesh, partition: Partition, part_id: int, coeffs, specs,
                              config: Optional[AssemblyConfig] = None, device=None, local: bool = True):
    """Device-resident rows of one part (the per-GPU call of the N-GPU run).

    ``local=True`` (default): the rank's sub-mesh only (owned + halo,
    ``local_problem``) with global columns; the result's ``plan.rhs`` is
    indexed by LOCAL DoFs (``DeviceAssembly.local``).  ``local=False``: the
    whole mesh with a row subset (every rank pays the whole-mesh index /
    pre-pass work; kept as the cross-check)."""
    from .assembly import _check_classified

    if not 0 <= part_id < partition.n_parts:
        raise PartitionError(f"part {part_id} out of range")
    _check_classified(mesh)
    if not local:
        return assemble_device(mesh, coeffs, specs, config, row_elements=partition.owned[part_id],
                               device=device)
    lp = local_problem(mesh, partition, part_id, specs, config)
    res = assemble_device(lp.flat, coeffs, lp.specs, lp.config, row_elements=lp.owned_local, device=device,
                          col_dof=lp.col_dof)
    res.local = lp
    return res


def assemble_partition(mesh, partition: Partition, part_id: int, coeffs, specs,
                       config: Optional[AssemblyConfig] = None):
    """polydg ``assemble_partition`` (distribute.py:200-232) ->
    (PartialMatrix, load over owned rows, AssemblyStats)."""
    res = assemble_partition_device(mesh, partition, part_id, coeffs, specs, config)
    plan, lp = res.plan, res.local
    ranges = _row_ranges(DofMap.from_specs(specs), partition.owned[part_id])
    loc_ranges = _row_ranges(plan.dof, lp.owned_local)
    own_rows = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in loc_ranges])
    rhs = plan.rhs.cpu().numpy()
    m = plan.to_csr()
    m.n_cols = lp.n_dofs_global
    return PartialMatrix(part_id, ranges, m), rhs[own_rows], res.stats


def gather_and_verify(partials, n_dofs: int) -> CSRMatrix:
    """Stack row-distributed partials; every row covered exactly once
    (polydg ``distribute.py:235-266``)."""
    coverage = np.zeros(n_dofs, dtype=np.int64)
    for pm in partials:
        for a, b in pm.row_ranges:
            coverage[a:b] += 1
    if (coverage != 1).any():
        bad = int(np.flatnonzero(coverage != 1)[0])
        raise AssemblyError(f"row {bad} covered {coverage[bad]} times")
    # global row -> (partial, local row)
    src_part = np.empty(n_dofs, np.int64)
    src_row = np.empty(n_dofs, np.int64)
    for k, pm in enumerate(partials):
        loc = 0
        for a, b in pm.row_ranges:
            src_part[a:b] = k
            src_row[a:b] = np.arange(loc, loc + (b - a))
            loc += b - a
    lens = np.empty(n_dofs, np.int64)
    for k, pm in enumerate(partials):
        sel = src_part == k
        lens[sel] = np.diff(pm.matrix.row_ptr)[src_row[sel]]
    row_ptr = np.zeros(n_dofs + 1, np.int64)
    np.cumsum(lens, out=row_ptr[1:])
    col_idx = np.empty(row_ptr[-1], np.int64)
    values = np.empty(row_ptr[-1])
    for k, pm in enumerate(partials):
        rows = np.flatnonzero(src_part == k)
        if rows.size == 0:
            continue
        lr = src_row[rows]
        s = pm.matrix.row_ptr[lr]
        e = pm.matrix.row_ptr[lr + 1]
        # gather index lists segment-wise (vectorised ragged copy)
        ln = e - s
        dst = np.repeat(row_ptr[rows], ln) + (np.arange(ln.sum()) - np.repeat(np.cumsum(ln) - ln, ln))
        srcidx = np.repeat(s, ln) + (np.arange(ln.sum()) - np.repeat(np.cumsum(ln) - ln, ln))
        col_idx[dst] = pm.matrix.col_idx[srcidx]
        values[dst] = pm.matrix.values[srcidx]
    return CSRMatrix(n_dofs, n_dofs, row_ptr, col_idx, values)


def gather_load(partial_loads, partials, n_dofs: int) -> np.ndarray:
    out = np.zeros(n_dofs)
    for load, pm in zip(partial_loads, partials):
        loc = 0
        for a, b in pm.row_ranges:
            out[a:b] = load[loc: loc + (b - a)]
            loc += b - a
    return out


def _rank_rows(plan, lp):
    """The four tensors one rank contributes: local row_ptr, col_idx (global
    columns), values, and the RHS of its owned rows (owned-element order)."""
    import torch

    off = plan.dof.offsets
    own = lp.owned_local if lp is not None else plan.row_elements
    idx = np.concatenate([np.arange(off[e], off[e + 1], dtype=np.int64) for e in own]) if len(own) else \
        np.zeros(0, np.int64)
    rhs = plan.rhs.index_select(0, torch.from_numpy(idx).to(plan.rhs.device))
    return {"row_ptr": plan.row_ptr, "col_idx": plan.col_idx, "values": plan.values, "rhs": rhs}


def gather_verify_partition(plan, lp, partition: Partition, mesh, coeffs, specs,
                            config: Optional[AssemblyConfig] = None, group=None,
                            chunk_bytes: int = 1 << 28) -> Optional[dict]:
    """The verification gather of the N-GPU run (north star: "a single NCCL
    gather over NVLink runs only to collect the CSR rows for verification").

    Every rank sends its rows (row_ptr, col_idx, values, owned RHS) to rank 0
    point-to-point in ``chunk_bytes`` pieces (NCCL on GPUs; gloo moves the
    chunks through host memory).  Rank 0 re-assembles each part's rows on the
    WHOLE mesh (the row-subset path, one part at a time, so its HBM holds one
    part, not the matrix) and compares every chunk bit for bit
    (``torch.equal``) -- the rows of an N-GPU run must equal the 1-GPU rows.
    Returns {"verified", "bytes", "seconds", "mismatch"} on rank 0, None elsewhere."""
    import time

    import torch
    import torch.distributed as dist

    from .assembly import SipgPlan

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    gloo = dist.get_backend(group) == "gloo"
    mine = _rank_rows(plan, lp)
    names = ("row_ptr", "col_idx", "values", "rhs")
    dev = plan.values.device
    sizes = torch.tensor([mine[n].numel() for n in names], dtype=torch.int64,
                         device="cpu" if gloo else dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    if rank != 0:
        for n in names:
            t = mine[n]
            step = max(1, chunk_bytes // t.element_size())
            for a in range(0, t.numel(), step):
                c = t[a:a + step].contiguous()
                dist.send(c.cpu() if gloo else c, dst=0, group=group)
        return None
    t0 = time.perf_counter()
    moved, bad = 0, []
    cfg = config or AssemblyConfig()
    for r in range(world):
        ref_plan = SipgPlan(mesh, coeffs, specs, cfg, row_elements=partition.owned[r], device=dev)
        ref_plan.run()
        ref_plan.check_flags()
        ref = _rank_rows(ref_plan, None)
        for k, n in enumerate(names):
            cnt = int(all_sizes[r][k])
            same = cnt == ref[n].numel()
            if not same:
                bad.append(f"part {r} {n}: {cnt} entries, monolithic {ref[n].numel()}")
            if r == 0:
                if same and not torch.equal(mine[n], ref[n]):
                    bad.append(f"part 0 {n}")
                continue
            step = max(1, chunk_bytes // ref[n].element_size())
            for a in range(0, cnt, step):  # always drain the sender (no deadlock on a mismatch)
                m = min(step, cnt - a)
                buf = torch.empty(m, dtype=ref[n].dtype, device="cpu" if gloo else dev)
                dist.recv(buf, src=r, group=group)
                moved += m * buf.element_size()
                if same and not torch.equal(buf.to(dev), ref[n][a:a + m]):
                    bad.append(f"part {r} {n} chunk at {a}")
        del ref, ref_plan
        torch.cuda.empty_cache()
    return {"verified": not bad, "bytes": moved, "seconds": time.perf_counter() - t0, "mismatch": bad[:8]}


def nccl_gather_rows(partial_values, partial_col_idx, partial_row_ptr, group=None):
    """Gather every rank's row block on rank 0 over torch.distributed (NCCL
    on GPUs, gloo on CPU) -- the verification collective; not on the
    assembly path.  Returns the list of (row_ptr, col_idx, values) on rank 0,
    None elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = partial_values.device
    sizes = torch.tensor([partial_values.numel(), partial_row_ptr.numel()], dtype=torch.int64,
                         device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    # point-to-point to rank 0 (gather semantics)
    if rank == 0:
        out = [(partial_row_ptr, partial_col_idx, partial_values)]
        for r in range(1, world):
            nv, nr = (int(x) for x in all_sizes[r].tolist())
            bufs = (torch.empty(nr, dtype=torch.int64, device=dev),
                    torch.empty(nv, dtype=torch.int64, device=dev),
                    torch.empty(nv, dtype=torch.float64, device=dev))
            for b in bufs:
                dist.recv(b, src=r, group=group)
            out.append(bufs)
        return out
    for b in (partial_row_ptr, partial_col_idx, partial_values):
        dist.send(b, dst=0, group=group)
    return None
