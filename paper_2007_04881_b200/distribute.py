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


def assemble_partition_device(mesh, partition: Partition, part_id: int, coeffs, specs,
                              config: Optional[AssemblyConfig] = None, device=None):
    """Device-resident rows of one part (the per-GPU call of the N-GPU run)."""
    if not 0 <= part_id < partition.n_parts:
        raise PartitionError(f"part {part_id} out of range")
    from .assembly import _check_classified

    _check_classified(mesh)
    return assemble_device(mesh, coeffs, specs, config, row_elements=partition.owned[part_id],
                           device=device)


def assemble_partition(mesh, partition: Partition, part_id: int, coeffs, specs,
                       config: Optional[AssemblyConfig] = None):
    """polydg ``assemble_partition`` (distribute.py:200-232) ->
    (PartialMatrix, load over owned rows, AssemblyStats)."""
    res = assemble_partition_device(mesh, partition, part_id, coeffs, specs, config)
    plan = res.plan
    own = plan.row_elements
    ranges = _row_ranges(plan.dof, own)
    own_rows = np.concatenate([np.arange(a, b, dtype=np.int64) for a, b in ranges])
    rhs = plan.rhs.cpu().numpy()
    return PartialMatrix(part_id, ranges, plan.to_csr()), rhs[own_rows], res.stats


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
