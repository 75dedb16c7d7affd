"""Drop-in Approach-2 assembly on the B200 engine.

Public surface mirrors polydg ``assembly.py`` for the hot path:

* ``assemble_approach2(mesh, coeffs, specs, config)`` -> ``(CSRMatrix, rhs,
  AssemblyStats, BlockPattern)`` (polydg ``assembly.py:1090-1099``);
* ``assemble_approach1`` -> ``(CSRMatrix, rhs, AssemblyStats)`` -- same device
  engine (polydg's Approach 1 produces the same CSR within 1e-12);
* ``build_block_pattern(mesh, specs, row_elements=None)``;
* ``element_kernel`` (unit-level entry point);
* ``assemble_device(...)`` -- the device-resident variant (CSR stays in HBM)
  used by the benchmark and by million-element meshes.

Everything numeric runs in ``libpdg.so``; this module only flattens inputs,
allocates device buffers (PyTorch is used for device memory and streams) and
maps device error flags to polydg's exception classes.  No CPU fallback.
"""

from __future__ import annotations

import os
import time
import warnings
from collections.abc import Sequence
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .basis import family_name, num_basis, spec_arrays
from .mesh import BOUNDARY, TAG_CODE, FlatMesh, MeshError, flat_of
from .model import ClassificationError, PenaltyConfig, compile_coeffs, policy_source
from .quadrature import QuadratureError, RuleTable

KERNEL_NAMES = ("element", "interior", "dirichlet", "inflow", "neumann_outflow")


class AssemblyError(RuntimeError):
    pass


class PatternMissError(AssemblyError):
    """A (row, col) block absent from the sparsity pattern was addressed."""


# ---------------------------------------------------------------------------
# polydg-compatible containers (assembly.py:64-155, 209-272, 345-391)
# ---------------------------------------------------------------------------

@dataclass
class DofMap:
    offsets: np.ndarray

    @classmethod
    def from_specs(cls, specs) -> "DofMap":
        deg, boxes, fam = spec_arrays(specs)
        d = boxes.shape[2]
        counts = _num_basis_vec(deg, d, fam)
        off = np.zeros(len(deg) + 1, dtype=np.int64)
        np.cumsum(counts, out=off[1:])
        return cls(off)

    @property
    def n_dofs(self) -> int:
        return int(self.offsets[-1])

    @property
    def n_elements(self) -> int:
        return self.offsets.shape[0] - 1

    def count(self, element: int) -> int:
        return int(self.offsets[element + 1] - self.offsets[element])

    def start(self, element: int) -> int:
        return int(self.offsets[element])


def _num_basis_vec(degrees: np.ndarray, d: int, family) -> np.ndarray:
    table = {int(p): num_basis(int(p), d, family) for p in np.unique(degrees)}
    out = np.empty(degrees.shape[0], np.int64)
    for p, n in table.items():
        out[degrees == p] = n
    return out


@dataclass
class CSRMatrix:
    n_rows: int
    n_cols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def validate(self) -> None:
        if self.row_ptr.shape != (self.n_rows + 1,):
            raise AssemblyError("row_ptr has wrong length")
        if np.any(np.diff(self.row_ptr) < 0) or self.row_ptr[-1] != self.nnz:
            raise AssemblyError("row_ptr is not a nondecreasing nnz prefix")
        if self.nnz == 0:
            return
        if self.col_idx.min() < 0 or self.col_idx.max() >= self.n_cols:
            raise AssemblyError("column index out of range")
        first = np.zeros(self.nnz, bool)
        first[self.row_ptr[:-1][self.row_ptr[:-1] < self.nnz]] = True
        bad = np.flatnonzero((np.diff(self.col_idx) <= 0) & ~first[1:])
        if bad.size:
            r = int(np.searchsorted(self.row_ptr, bad[0] + 1, "right") - 1)
            raise AssemblyError(f"row {r} columns not strictly increasing/in range")

    def to_scipy(self):
        from scipy.sparse import csr_matrix

        return csr_matrix((self.values, self.col_idx, self.row_ptr), shape=(self.n_rows, self.n_cols))

    def to_dense(self) -> np.ndarray:
        return self.to_scipy().toarray()

    def max_relative_difference(self, other: "CSRMatrix", floor_rel: float = 1e-3) -> float:
        """polydg ``CSRMatrix.max_relative_difference`` (assembly.py:133-155)."""
        if (self.n_rows != other.n_rows or self.n_cols != other.n_cols
                or not np.array_equal(self.row_ptr, other.row_ptr)
                or not np.array_equal(self.col_idx, other.col_idx)):
            raise AssemblyError("sparsity patterns differ")
        if self.nnz == 0:
            return 0.0
        a, b = np.abs(self.values), np.abs(other.values)
        scale = max(a.max(), b.max(), 1e-300)
        denom = np.maximum(np.maximum(a, b), floor_rel * scale)
        return float(np.max(np.abs(self.values - other.values) / denom))


class _RaggedSeq(Sequence):
    """``list[np.ndarray]`` view of a CSR-style ragged array (no per-row objects
    until a row is read)."""

    def __init__(self, ptr: np.ndarray, data: np.ndarray):
        self._ptr, self._data = ptr, data

    def __len__(self):
        return int(self._ptr.shape[0] - 1)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[k] for k in range(*i.indices(len(self)))]
        i = int(i)
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        return self._data[self._ptr[i]:self._ptr[i + 1]]


@dataclass
class BlockPattern:
    """CSR skeleton with one dense block per adjacent element pair (polydg
    ``BlockPattern``, assembly.py:207-272).

    Array-backed: ``neighbors`` / ``col_starts`` are ragged views of two flat
    arrays (the device adjacency), ``local_block_start`` / ``block_slots``
    binary-search the ascending ``row_elements`` -- no per-element Python
    objects, so a 4M-element pattern costs a few vectorised passes."""

    dof_map: DofMap
    row_elements: np.ndarray
    neighbors: Sequence
    col_starts: Sequence
    row_ptr: np.ndarray
    col_idx: np.ndarray
    global_rows: np.ndarray

    def __post_init__(self):
        self.row_elements = np.asarray(self.row_elements, dtype=np.int64)
        counts = np.diff(self.dof_map.offsets)[self.row_elements]
        self._row_offsets = np.zeros(len(counts) + 1, dtype=np.int64)
        np.cumsum(counts, out=self._row_offsets[1:])

    @classmethod
    def from_adjacency(cls, dof_map: DofMap, row_elements, nbr_ptr, nbr_elem, row_ptr, col_idx) -> "BlockPattern":
        """Pattern of ``row_elements`` from the sorted adjacency (nbr_ptr over
        all elements, nbr_elem = neighbours incl. self) -- vectorised."""
        rows = np.asarray(row_elements, dtype=np.int64)
        bp = cls.__new__(cls)
        bp.dof_map, bp.row_elements, bp.row_ptr, bp.col_idx = dof_map, rows, row_ptr, col_idx
        bp._adj = (nbr_ptr, nbr_elem)  # neighbors / col_starts / global_rows built on first use
        bp.__post_init__()
        return bp

    def _build_lazy(self):
        nbr_ptr, nbr_elem = self.__dict__.pop("_adj")
        rows, dof_map = self.row_elements, self.dof_map
        a, b = nbr_ptr[rows], nbr_ptr[rows + 1]
        cnt = (b - a).astype(np.int64)
        ptr = np.zeros(rows.size + 1, np.int64)
        np.cumsum(cnt, out=ptr[1:])
        idx = np.repeat(a - ptr[:-1], cnt) + np.arange(int(ptr[-1]), dtype=np.int64)
        nbrs = np.asarray(nbr_elem[idx], dtype=np.int64)
        w = np.diff(dof_map.offsets)[nbrs]
        cs = np.cumsum(w) - w                         # global running start ...
        cs -= np.repeat(cs[ptr[:-1]] if rows.size else cs[:0], cnt)  # ... made per-row
        ne = np.diff(dof_map.offsets)[rows]
        first = dof_map.offsets[rows]
        rp = np.zeros(rows.size + 1, np.int64)
        np.cumsum(ne, out=rp[1:])
        self.__dict__["neighbors"] = _RaggedSeq(ptr, nbrs)
        self.__dict__["col_starts"] = _RaggedSeq(ptr, cs.astype(np.int64))
        self.__dict__["global_rows"] = np.repeat(first - rp[:-1], ne) + np.arange(int(rp[-1]), dtype=np.int64)

    def __getattr__(self, name):
        # neighbors / col_starts / global_rows of a pattern made by from_adjacency
        if name in ("neighbors", "col_starts", "global_rows") and "_adj" in self.__dict__:
            self._build_lazy()
            return self.__dict__[name]
        raise AttributeError(name)

    def _local(self, element: int):
        k = int(np.searchsorted(self.row_elements, element))
        if k < self.row_elements.shape[0] and int(self.row_elements[k]) == int(element):
            return k
        return None

    @property
    def n_local_rows(self) -> int:
        return int(self.row_ptr.shape[0] - 1)

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def local_block_start(self, element: int) -> int:
        k = self._local(element)
        if k is None:
            raise KeyError(element)
        return k

    def block_slots(self, row_element: int, col_element: int) -> np.ndarray:
        local = self._local(row_element)
        if local is None:
            raise PatternMissError(f"element {row_element} owns no rows here")
        nbrs = self.neighbors[local]
        pos = int(np.searchsorted(nbrs, col_element))
        if pos >= nbrs.shape[0] or nbrs[pos] != col_element:
            raise PatternMissError(f"block ({row_element}, {col_element}) missing from pattern")
        ni = self.dof_map.count(row_element)
        nj = self.dof_map.count(col_element)
        row0 = self._row_offsets[local]
        base = self.row_ptr[row0: row0 + ni] + self.col_starts[local][pos]
        return base[:, None] + np.arange(nj, dtype=np.int64)[None, :]

    def empty_matrix(self) -> CSRMatrix:
        return CSRMatrix(self.n_local_rows, self.dof_map.n_dofs, self.row_ptr.copy(),
                         self.col_idx.copy(), np.zeros(self.nnz))


@dataclass
class AssemblyConfig:
    """polydg ``AssemblyConfig`` (assembly.py:345-357).  ``n_workers``,
    ``mode`` and ``chunk_size`` are accepted for compatibility: the device
    engine has exactly one writer per value slot, so both modes give the same
    bitwise-deterministic matrix."""

    quad_increment: int = 2
    penalty: PenaltyConfig = field(default_factory=PenaltyConfig)
    n_workers: int = 1
    mode: str = "deterministic"
    chunk_size: int = 256

    def __post_init__(self):
        if self.mode not in ("deterministic", "atomic"):
            raise ValueError(f"unknown accumulation mode {self.mode!r}")
        if self.n_workers < 1:
            raise ValueError("n_workers must be >= 1")


@dataclass
class KernelTiming:
    kernel: str
    work_items: int = 0
    seconds: float = 0.0
    nnz_written: int = 0


@dataclass
class AssemblyStats:
    kernels: dict
    index_seconds: float = 0.0
    kernel_wall_seconds: float = 0.0
    total_seconds: float = 0.0
    triplet_count: int = 0
    nnz: int = 0
    device_ms: dict = field(default_factory=dict)
    kernel_split: str = ""

    @property
    def duplicate_ratio(self) -> float:
        return self.triplet_count / self.nnz if self.nnz else 0.0

    def to_csv(self) -> str:
        lines = ["kernel,work_items,seconds,nnz_written"]
        for name in KERNEL_NAMES:
            k = self.kernels[name]
            lines.append(f"{k.kernel},{k.work_items},{k.seconds:.6g},{k.nnz_written}")
        total_items = sum(k.work_items for k in self.kernels.values())
        lines.append(f"indices,{self.triplet_count},{self.index_seconds:.6g},{self.nnz}")
        lines.append(f"total,{total_items},{self.total_seconds:.6g},{self.nnz}")
        return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# device residency
# ---------------------------------------------------------------------------

_D2H_CHUNK = 1 << 28  # 256 MiB pinned staging buffers


def download(t, stream=None, chunk_bytes: int = _D2H_CHUNK) -> np.ndarray:
    """Device tensor -> new numpy array through two pinned staging buffers:
    chunk i+1 is copied device->host (DMA) while chunk i is copied into the
    destination array by a host thread pool (numpy copies release the GIL), so
    the transfer runs at the link's pinned rate instead of the pageable one."""
    torch = _torch()
    t = t.contiguous().reshape(-1)
    n = int(t.numel())
    out = np.empty(n, dtype=np.dtype(str(t.dtype).replace("torch.", "")))
    nbytes = n * t.element_size()
    if nbytes <= (1 << 24):  # small: one plain copy
        out[:] = t.cpu().numpy()
        return out
    stream = stream or torch.cuda.current_stream(t.device)
    per = max(1, chunk_bytes // t.element_size())
    with _STAGING_LOCK:  # the pinned buffers are process-wide: one download at a time
        return _download_staged(t, out, n, per, stream)


def _download_staged(t, out, n, per, stream):
    torch = _torch()
    raw, pool, nthreads = _staging(per * t.element_size())
    stages = [r[: per * t.element_size()].view(t.dtype) for r in raw]
    events = [torch.cuda.Event() for _ in range(2)]
    pending = [None, None]

    def host_copy(buf, a, m):
        src = buf[:m].numpy()
        parts = np.linspace(0, m, nthreads + 1).astype(np.int64)
        list(pool.map(lambda k: np.copyto(out[a + parts[k]:a + parts[k + 1]], src[parts[k]:parts[k + 1]]),
                      range(nthreads)))

    try:
        with torch.cuda.stream(stream):
            for i, a in enumerate(range(0, n, per)):
                s = i & 1
                m = min(per, n - a)
                if pending[s] is not None:
                    pending[s].result()  # the host copy out of this buffer is done
                stages[s][:m].copy_(t[a:a + m], non_blocking=True)
                events[s].record(stream)
                events[s].synchronize()
                pending[s] = pool.submit(host_copy, stages[s], a, m)
    finally:
        for f in pending:
            if f is not None:
                f.result()
    return out


_STAGING = {}
_STAGING_LOCK = __import__("threading").Lock()


def _staging(nbytes: int):
    """Two pinned staging buffers of at least ``nbytes`` and the host copy
    pool, allocated once per process (pinned allocations cost milliseconds)."""
    torch = _torch()
    cur = _STAGING.get("raw")
    if cur is None or cur[0].numel() < nbytes:
        _STAGING["raw"] = [torch.empty(nbytes, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    if "pool" not in _STAGING:
        from concurrent.futures import ThreadPoolExecutor

        n = max(1, min(16, (os.cpu_count() or 2)))
        # two submitters (the staging buffers) + n copy workers
        _STAGING["pool"] = (ThreadPoolExecutor(n + 2), n)
    pool, n = _STAGING["pool"]
    return _STAGING["raw"], pool, n


def _torch():
    import torch

    return torch


def _require_cuda(device):
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.EngineUnavailable("no CUDA device: the SIPG engine has no CPU fallback")
    return torch.device(device if device is not None else "cuda")


_MESH_FIELDS = (
    ("vertices", "vertices"), ("simplices", "simplices"), ("simplex_volumes", "simplex_volumes"),
    ("elem_ptr", "elem_ptr"), ("elem_simplices", "elem_simplices"), ("elem_volumes", "elem_volumes"),
    ("face_owner", "face_owner"), ("face_neighbor", "face_neighbor"), ("face_tag", "face_tag"),
    ("face_normal", "face_normal"), ("face_measure", "face_measure"), ("face_ptr", "face_ptr"),
    ("facet_vertices", "facet_vertices"), ("facet_owner_simplex", "facet_owner_simplex"),
    ("facet_neighbor_simplex", "facet_neighbor_simplex"), ("iface_owner", "iface_owner"),
    ("iface_neighbor", "iface_neighbor"), ("iface_ptr", "iface_ptr"),
    ("iface_faces", "iface_faces"), ("elem_bface_ptr", "elem_bface_ptr"),
    ("elem_bfaces", "elem_bfaces"),
)


class DeviceMesh:
    """A FlatMesh resident in HBM (+ the ``pdg_mesh`` descriptor)."""

    def __init__(self, flat: FlatMesh, device=None, stream=None):
        torch = _torch()
        self.device = _require_cuda(device)
        self.flat = flat
        self.t = {}
        for attr, _ in _MESH_FIELDS:
            arr = np.ascontiguousarray(getattr(flat, attr))
            if arr.size == 0:
                arr = np.zeros(1, dtype=arr.dtype)
            self.t[attr] = torch.from_numpy(arr).to(self.device, non_blocking=False)
        self.h2d_bytes = sum(int(getattr(flat, a).nbytes) for a, _ in _MESH_FIELDS)
        s = _lib.Mesh()
        s.dim = flat.dim
        s.n_vertices, s.n_simplices, s.n_elements = flat.n_vertices, flat.n_simplices, flat.n_elements
        s.n_faces, s.n_facets, s.n_interfaces = flat.n_faces, flat.n_facets, flat.n_interfaces
        for attr, cname in _MESH_FIELDS:
            setattr(s, cname, _lib.ptr(self.t[attr]))
        self.struct = s
        self._tags = flat.face_tag.copy()

    def refresh_tags(self):
        """Re-upload face tags if classification changed them since upload."""
        if not np.array_equal(self._tags, self.flat.face_tag):
            torch = _torch()
            src = self.flat.face_tag if self.flat.face_tag.size else np.zeros(1, np.int8)
            self.t["face_tag"].copy_(torch.from_numpy(np.ascontiguousarray(src)))
            self._tags = self.flat.face_tag.copy()


def device_mesh(mesh, device=None) -> DeviceMesh:
    """Cached DeviceMesh of a mesh object (this package's meshes keep it)."""
    flat = flat_of(mesh)
    cache = getattr(flat, "_device_cache", None)
    if cache is not None and cache.device == _require_cuda(device):
        cache.refresh_tags()
        return cache
    dm = DeviceMesh(flat, device)
    try:
        object.__setattr__(flat, "_device_cache", dm)
    except Exception:
        pass
    return dm


class DeviceRules:
    def __init__(self, dim, vol_orders, face_orders, device):
        torch = _torch()
        table = RuleTable(dim, vol_orders, face_orders)
        mo = max(list(table.vol) + list(table.face) + [2])
        vo, vn, fo, fn = table.lookup_arrays(mo)
        self.t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(device)
                  for k, v in (("points", table.points if table.points.size else np.zeros((1, 3))),
                               ("weights", table.weights if table.weights.size else np.zeros(1)),
                               ("sqrt_weights", np.sqrt(table.weights) if table.weights.size else np.zeros(1)),
                               ("vo", vo), ("vn", vn), ("fo", fo), ("fn", fn))}
        r = _lib.Rules()
        r.max_order = mo
        r.points, r.weights = _lib.ptr(self.t["points"]), _lib.ptr(self.t["weights"])
        r.vol_offset, r.vol_count = _lib.ptr(self.t["vo"]), _lib.ptr(self.t["vn"])
        r.face_offset, r.face_count = _lib.ptr(self.t["fo"]), _lib.ptr(self.t["fn"])
        r.sqrt_weights = _lib.ptr(self.t["sqrt_weights"])
        r.n_points = int(table.weights.size)
        self.struct = r


def _raise_flags(flags: int):
    if flags & _lib.FLAG_UNCLASSIFIED:
        raise AssemblyError("a boundary face is unclassified; run classify_boundary_faces")
    if flags & (_lib.FLAG_DEGENERATE_SIMPLEX):
        raise QuadratureError("degenerate simplex in quadrature map")
    if flags & (_lib.FLAG_DEGENERATE_FACET):
        raise QuadratureError("degenerate sub-simplex in face quadrature map")
    if flags & _lib.FLAG_STRADDLE:
        raise ClassificationError(
            "advection flux changes sign across a face; refine the mesh so faces do not "
            "straddle the inflow/outflow transition")
    if flags & _lib.FLAG_NO_ADJACENT_SIMPLEX:
        raise MeshError("no subdivision simplex adjacent to the face")
    if flags:
        raise RuntimeError(f"device error flags 0x{flags:x}")


# ---------------------------------------------------------------------------
# the assembly plan: all device buffers of one (mesh, basis, coeffs, rows)
# ---------------------------------------------------------------------------

class SipgPlan:
    """Device buffers + descriptors for repeated assembly of one problem.

    ``run()`` enqueues the whole path on one stream -- index phase
    (adjacency, row offsets), face pre-pass (sigma, flow side) and the fused
    element kernel (values + col_idx + RHS) -- without any host
    synchronisation, so it can be timed with CUDA events or captured in a
    CUDA graph.  Construction performs the one size query (nnz) polydg also
    needs before it can allocate the CSR.
    """

    def __init__(self, mesh, coeffs, specs, config: Optional[AssemblyConfig] = None,
                 row_elements=None, device=None, stream=None, jit: bool = True,
                 allocate_csr: bool = True, col_dof=None):
        import ctypes as C

        torch = _torch()
        self.lib = _lib.load()
        config = config or AssemblyConfig()
        self.config = config
        self.dm = device_mesh(mesh, device)
        dev = self.dm.device
        self.device = dev
        flat = self.dm.flat
        self.flat = flat
        d = flat.dim
        deg, boxes, fam = spec_arrays(specs)
        if family_name(fam) != "P":
            raise NotImplementedError("the device engine implements family P (space-time PQ is out of scope)")
        if deg.shape[0] != flat.n_elements:
            raise AssemblyError("one BasisSpec per element required")
        if boxes.shape[1:] != (2, d):
            raise ValueError("spec boxes do not match the mesh dimension")
        pmax = int(deg.max()) if deg.size else 0
        if pmax > _lib.MAX_DEGREE[d]:
            raise NotImplementedError(
                f"degree {pmax} exceeds the compiled device range (p <= {_lib.MAX_DEGREE[d]} in {d}D)")
        self.degrees = deg
        self.dof = DofMap(np.concatenate([[0], np.cumsum(_num_basis_vec(deg, d, fam))]).astype(np.int64))
        inc = int(config.quad_increment)
        pen = config.penalty
        self.coverable = None if pen.coverable is None else np.asarray(pen.coverable, bool)

        self.stream = stream if stream is not None else torch.cuda.current_stream(dev)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
        self.t = {"degree": T(deg.astype(np.int32)), "box": T(boxes), "dof": T(self.dof.offsets)}
        b = _lib.Basis()
        b.max_degree = pmax
        b.degree, b.box, b.dof_offset = (_lib.ptr(self.t["degree"]), _lib.ptr(self.t["box"]),
                                         _lib.ptr(self.t["dof"]))
        self.basis = b

        # rules: volume orders per degree present, face orders per max pair degree
        uniq = np.unique(deg)
        vol_orders = [2 * int(p) + inc for p in uniq]
        face_orders = [2 * int(max(p, q)) + inc for p in uniq for q in uniq]
        self.rules = DeviceRules(d, vol_orders, face_orders, dev)

        self.cdesc = compile_coeffs(coeffs, d)
        self.coeffs = _lib.coeffs_struct(self.cdesc)
        self.jit_source = None
        self.kernel_variant = "aot-interpreted"
        if jit and os.environ.get("PDG_JIT", "1") != "0":
            src = policy_source(coeffs, d).encode()
            rc = self.lib.pdg_jit_prepare(C.byref(self.coeffs), src, d, pmax)
            if rc == _lib.PDG_OK:
                self.jit_source = src
                self.kernel_variant = "nvrtc-specialised"
            else:
                warnings.warn("runtime specialisation unavailable, using the ahead-of-time kernel: "
                              + self.lib.pdg_last_error().decode(errors="replace"))
        prm = _lib.Params()
        prm.quad_increment = inc
        prm.include_gradient_terms = 1
        prm.penalty_constant = float(pen.constant)
        if os.environ.get("PDG_PLAIN_VOLUME") == "1":  # variant selection for experiments / tests
            prm.options |= _lib.OPT_PLAIN_VOLUME
        if self.coverable is not None:
            self.t["coverable"] = T(self.coverable.astype(np.uint8))
            prm.coverable = _lib.ptr(self.t["coverable"])
        self.params = prm

        # rows
        nel = flat.n_elements
        if row_elements is None:
            self.row_elements = np.arange(nel, dtype=np.int64)
            self.t["rows"] = None
        else:
            self.row_elements = np.unique(np.asarray(row_elements, dtype=np.int64))
            self.t["rows"] = T(self.row_elements.astype(np.int32))
        nr = self.row_elements.shape[0]
        counts = np.diff(self.dof.offsets)
        self.n_local_rows = int(counts[self.row_elements].sum())
        z = lambda n, dt: torch.empty(max(int(n), 1), dtype=dt, device=dev)
        i64, i32 = torch.int64, torch.int32
        nadj = nel + 2 * flat.n_interfaces
        self.t.update(nbr_ptr=z(nel + 1, i64), nbr_elem=z(nadj, i32), nbr_iface=z(nadj, i32),
                      row_len=z(nr, i64), val_off=z(nr + 1, i64), row_off=z(nr + 1, i64),
                      row_ptr=z(self.n_local_rows + 1, i64),
                      nbr_rec=z(nadj * 10, torch.float64),  # pdg_iface_rec, 80 B per entry
                      sigma=z(flat.n_faces, torch.float64), flow=z(flat.n_faces, torch.int8),
                      abar=z(nel, torch.float64), flags=torch.zeros(1, dtype=torch.int32, device=dev))
        W = 8 if d == 2 else 16
        self.t.update(sframe=z(flat.n_simplices * W, torch.float64),
                      fframe=z(flat.n_facets * W, torch.float64),
                      erec=z(nel * W, torch.float64))
        fr = _lib.Frames()
        fr.simplex, fr.facet, fr.element = (_lib.ptr(self.t["sframe"]), _lib.ptr(self.t["fframe"]),
                                            _lib.ptr(self.t["erec"]))
        self.frames = fr
        self.ws_bytes = int(self.lib.pdg_workspace_bytes(nel, flat.n_interfaces))
        self.t["ws"] = torch.empty(self.ws_bytes, dtype=torch.uint8, device=dev)
        pat = _lib.Pattern()
        pat.n_row_elements = nr
        pat.row_elements = _lib.ptr(self.t["rows"])
        pat.nbr_ptr, pat.nbr_elem, pat.nbr_iface = (_lib.ptr(self.t["nbr_ptr"]),
                                                    _lib.ptr(self.t["nbr_elem"]),
                                                    _lib.ptr(self.t["nbr_iface"]))
        pat.row_len, pat.elem_val_offset, pat.elem_row_offset = (
            _lib.ptr(self.t["row_len"]), _lib.ptr(self.t["val_off"]), _lib.ptr(self.t["row_off"]))
        pat.row_ptr = _lib.ptr(self.t["row_ptr"])
        pat.nbr_rec = _lib.ptr(self.t["nbr_rec"])
        self.col_dof = None
        if col_dof is not None:  # a rank's sub-mesh: rows carry the whole mesh's columns
            self.col_dof = np.ascontiguousarray(col_dof, np.int64)
            if self.col_dof.shape != (nel,):
                raise ValueError("col_dof needs one global DoF offset per element")
            self.t["col_dof"] = T(self.col_dof)
            pat.col_dof = _lib.ptr(self.t["col_dof"])
        self.pattern = pat

        # size query (the one sync, like polydg's pattern build before values);
        # allocate_csr=False (Approach 1 reuses the plan for mesh / rules / pre-pass
        # only) skips both the sync and the 16 B/nnz CSR buffers
        with torch.cuda.stream(self.stream):
            self._index_phase(size_query=allocate_csr)
        if not allocate_csr:
            self.nnz = 0
        self.t["col_idx"] = z(self.nnz, i64)
        self.t["values"] = z(self.nnz, torch.float64)
        self.t["rhs"] = torch.zeros(max(self.dof.n_dofs, 1), dtype=torch.float64, device=dev)
        pat.col_idx = _lib.ptr(self.t["col_idx"])

    # -- phases --------------------------------------------------------------
    def _index_phase(self, size_query=False):
        import ctypes as C

        s = _lib.stream_ptr(self.stream)
        lib = self.lib
        _lib.check(lib.pdg_adjacency(C.byref(self.dm.struct), _lib.ptr(self.t["nbr_ptr"]),
                                     _lib.ptr(self.t["nbr_elem"]), _lib.ptr(self.t["nbr_iface"]),
                                     _lib.ptr(self.t["ws"]), self.ws_bytes, s))
        nnz = C.c_int64(0)
        _lib.check(lib.pdg_pattern_offsets(C.byref(self.dm.struct), C.byref(self.basis),
                                           C.byref(self.pattern), self.n_local_rows,
                                           C.byref(nnz) if size_query else None,
                                           _lib.ptr(self.t["ws"]), self.ws_bytes, s))
        if size_query:
            self.nnz = int(nnz.value)

    def _frames(self, stream=None):
        import ctypes as C

        _lib.check(self.lib.pdg_frames_build(C.byref(self.dm.struct), C.byref(self.basis),
                                             C.byref(self.frames), _lib.ptr(self.t["flags"]),
                                             _lib.stream_ptr(stream or self.stream)))

    def _face_prepass(self, stream=None):
        import ctypes as C

        args = (C.byref(self.rules.struct), C.byref(self.params), _lib.ptr(self.t["sigma"]),
                _lib.ptr(self.t["flow"]), _lib.ptr(self.t["abar"]), _lib.ptr(self.t["flags"]),
                _lib.stream_ptr(stream or self.stream))
        if self.jit_source is not None:  # fields inlined (the NVRTC module of the element kernel)
            _lib.check(self.lib.pdg_face_prepass_jit(C.byref(self.dm.struct), C.byref(self.basis),
                                                     C.byref(self.coeffs), self.jit_source, *args))
        else:
            _lib.check(self.lib.pdg_face_prepass(C.byref(self.dm.struct), C.byref(self.basis),
                                                 C.byref(self.coeffs), *args))

    def _prepass(self):
        self._frames()
        self._face_prepass()
        self._records()

    def _index_and_prepass_concurrent(self):
        """Index phase, frames and the sigma / flow pre-pass are independent:
        fork them onto three streams (join before the interface records, which
        read all three).  The whole-step CUDA graph is captured from this, so
        the small latency-bound kernels overlap instead of queueing."""
        torch = _torch()
        if not hasattr(self, "_side"):
            self._side = [torch.cuda.Stream(self.device) for _ in range(2)]
            self._ev = [torch.cuda.Event() for _ in range(3)]
        main = self.stream
        self._ev[0].record(main)
        for st in self._side:
            st.wait_event(self._ev[0])
        self._frames(stream=self._side[0])
        self._face_prepass(stream=self._side[1])
        self._index_phase()
        self._ev[1].record(self._side[0])
        self._ev[2].record(self._side[1])
        main.wait_event(self._ev[1])
        main.wait_event(self._ev[2])
        self._records()

    def _records(self):
        import ctypes as C

        _lib.check(self.lib.pdg_iface_records(
            C.byref(self.dm.struct), C.byref(self.basis), C.byref(self.coeffs),
            C.byref(self.rules.struct), C.byref(self.params), C.byref(self.pattern),
            _lib.ptr(self.t["sigma"]), _lib.ptr(self.t["flow"]), _lib.stream_ptr(self.stream)))

    def _elements(self, write_col_idx=True):
        import ctypes as C

        if os.environ.get("PDG_SKIP_COLS") == "1":  # ablation knob (measurement only: col_idx left unwritten)
            write_col_idx = False

        tail = (C.byref(self.rules.struct), C.byref(self.params), C.byref(self.pattern),
                C.byref(self.frames), _lib.ptr(self.t["sigma"]), _lib.ptr(self.t["flow"]),
                _lib.ptr(self.t["values"]), 1 if write_col_idx else 0, _lib.ptr(self.t["rhs"]),
                _lib.ptr(self.t["flags"]), _lib.stream_ptr(self.stream))
        head = (C.byref(self.dm.struct), C.byref(self.basis), C.byref(self.coeffs))
        if self.jit_source is not None:
            _lib.check(self.lib.pdg_assemble_jit(*head, self.jit_source, *tail))
        else:
            _lib.check(self.lib.pdg_assemble(*head, *tail))

    def run(self, events=None):
        """Enqueue index phase + pre-pass + element kernel; no host sync.
        ``events``: optional list of 4 CUDA events recorded between phases."""
        torch = _torch()
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

    # -- CUDA graphs ------------------------------------------------------------
    def capture_graphs(self) -> bool:
        """Capture the three phases (index, pre-pass, element kernel) as CUDA
        graphs: a step is then 3 graph launches instead of ~20 kernel launches
        (small meshes are launch-bound).  Returns False (and keeps the plain
        path) if capture is unavailable.  ``graph_launches`` = kernels per
        replayed step (the library's launch counter does not see replays)."""
        torch = _torch()
        if getattr(self, "graphs", None):
            return True
        try:
            if self.stream.cuda_stream == torch.cuda.default_stream(self.device).cuda_stream:
                # graphs are captured on a side stream (replays stay ordered on it)
                torch.cuda.synchronize(self.device)
                self.stream = torch.cuda.Stream(self.device)
            self.run()  # warm: JIT compile / function attributes outside the capture
            self.stream.synchronize()
            l0 = self.lib.pdg_launch_count()
            graphs = []
            for fn in (self._index_phase, self._prepass, self._elements):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=self.stream):
                    fn()
                graphs.append(g)
            self.graph_launches = int(self.lib.pdg_launch_count() - l0)
            # the whole step as ONE graph (no phase events): one launch per step,
            # index phase / frames / face pre-pass forked onto three streams
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                if os.environ.get("PDG_FORK", "1") != "0":
                    self._index_and_prepass_concurrent()
                else:
                    self._index_phase()
                    self._prepass()
                self._elements()
            self.graph_step = g
            self.graphs = graphs
            return True
        except Exception as exc:  # capture unsupported: plain launches (same kernels)
            warnings.warn(f"CUDA graph capture unavailable ({exc}); using plain launches")
            self.graphs = None
            return False

    def run_graphs(self, events=None):
        """One step through the captured graphs (``capture_graphs``): the
        single whole-step graph, or -- with ``events`` (4 CUDA events recorded
        at the phase boundaries) -- the three per-phase graphs."""
        torch = _torch()
        if not events and getattr(self, "graph_step", None) is not None:
            with torch.cuda.stream(self.stream):
                self.graph_step.replay()
            return
        with torch.cuda.stream(self.stream):
            for i, g in enumerate(self.graphs):
                if events:
                    events[i].record(self.stream)
                g.replay()
            if events:
                events[3].record(self.stream)

    def check_flags(self):
        self.stream.synchronize()
        flags = int(self.t["flags"].item())
        if flags & _lib.FLAG_NEG_DIFFUSION and not self.params.options & _lib.OPT_PLAIN_VOLUME:
            # the symmetric sqrt(w a) volume table needs a(x) >= 0: re-run the
            # assembly with the plain (w a dphi) dphi^T variant (same kernel family)
            self.params.options |= _lib.OPT_PLAIN_VOLUME
            self.t["flags"].zero_()
            self.run()
            self.stream.synchronize()
            flags = int(self.t["flags"].item())
        _raise_flags(flags & ~_lib.FLAG_NEG_DIFFUSION)

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

    def to_csr(self) -> CSRMatrix:
        """The CSR in host memory: pinned, chunked, double-buffered device->host
        copies into freshly allocated numpy arrays (``download``)."""
        return CSRMatrix(self.n_local_rows, self.dof.n_dofs, download(self.row_ptr, self.stream),
                         download(self.col_idx, self.stream), download(self.values, self.stream))

    def block_pattern(self, row_ptr=None, col_idx=None) -> BlockPattern:
        """polydg BlockPattern of the plan's rows (vectorised from the device
        adjacency).  ``row_ptr`` / ``col_idx``: host copies already made (the
        pattern then shares them instead of downloading a second copy)."""
        ptr = download(self.t["nbr_ptr"], self.stream)
        nb = download(self.t["nbr_elem"][: int(ptr[-1])], self.stream)
        return BlockPattern.from_adjacency(self.dof, self.row_elements, ptr, nb,
                                           row_ptr if row_ptr is not None else download(self.row_ptr, self.stream),
                                           col_idx if col_idx is not None else download(self.col_idx, self.stream))

    def work_stats(self) -> dict:
        """polydg per-kernel work items / nnz_written (assembly.py:360-391)."""
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
        no, nn = counts[o], counts[np.where(inter, nb, 0)]
        oo = owned[o]
        on = np.where(inter, owned[np.where(inter, nb, 0)], False)
        both = inter & oo & on
        one_o = inter & oo & ~on
        one_n = inter & on & ~oo
        per = np.zeros(f.n_faces, np.int64)
        per[both] = ((no + nn) ** 2)[both]
        per[one_o] = (no * (no + nn))[one_o]
        per[one_n] = (nn * (no + nn))[one_n]
        sel = both | one_o | one_n
        out["interior"].work_items = int(nfac[sel].sum())
        out["interior"].nnz_written = int((per * nfac)[sel].sum())
        tg = f.face_tag
        for name, codes in (("dirichlet", (TAG_CODE["dirichlet"],)),
                            ("inflow", (TAG_CODE["inflow"],)),
                            ("neumann_outflow", (TAG_CODE["neumann"], TAG_CODE["outflow"]))):
            m = (~inter) & oo & np.isin(tg, codes)
            out[name].work_items = int(nfac[m].sum())
            if name != "neumann_outflow":
                out[name].nnz_written = int((nfac * no * no)[m].sum())
        return out


# below this col_idx size the per-element packing (a kernel, an event wait and
# host threads) costs more than the bytes it saves (r02h: cfg1 e2e 5.5 -> 1.8 M el/s)
_COMPACT_MIN_BYTES = 1 << 28


class HostIO:
    """Host buffers for end-to-end runs of a plan (a caller that keeps its
    result arrays across assemblies).

    Every ``upload()`` copies the mesh arrays host->device (the assembly
    inputs).  Every ``download()`` moves the assembled CSR (row_ptr, col_idx,
    values) and the RHS device->host.  With ``retain`` (default) they land in
    page-locked host arrays (``pdg_host_alloc``: the copies are DMA at the
    link rate -- on the box 51 GB/s, against 47 GB/s into registered pageable
    arrays, tools/register_probe.py), and ``result()`` returns them as a host
    ``CSRMatrix`` + RHS.  With ``compact_cols`` (default: when col_idx is at
    least 256 MB) col_idx crosses the link once per element -- every row of an element's block row has the same
    columns -- and host threads expand it into every row while the values
    are in flight (cfg5: 54 instead of 102 GB per step).  When the allocation fails, or with
    ``retain=False``, the bytes go through a pinned ring of ``chunk_bytes``
    and nothing is retained (``retained`` says which)."""

    def __init__(self, plan: "SipgPlan", chunk_bytes: int = 1 << 30, retain: bool = True,
                 compact_cols: Optional[bool] = None):
        torch = _torch()
        self.plan = plan
        self.inputs = {}
        for attr, _ in _MESH_FIELDS:
            src = plan.dm.t[attr]
            h = torch.empty(src.shape, dtype=src.dtype, pin_memory=True)
            h.copy_(src)
            self.inputs[attr] = h
        self.h2d_bytes = sum(int(t.numel() * t.element_size()) for t in self.inputs.values())
        outs = (plan.row_ptr, plan.col_idx, plan.values, plan.rhs)
        self.d2h_bytes = sum(int(t.numel() * t.element_size()) for t in outs)
        self.host, self.stage = [], None
        if retain:
            try:
                for t in outs:
                    self.host.append(_pinned_empty(t))
                if compact_cols or (compact_cols is None and int(plan.col_idx.numel()) * 8 >= _COMPACT_MIN_BYTES):
                    self._setup_compact()
            except RuntimeError:  # out of page-lockable memory: fall back to the ring
                self.close()
        if not self.host:
            self.stage = torch.empty(chunk_bytes, dtype=torch.uint8, pin_memory=True)

    def _setup_compact(self):
        """col_idx crosses the link once per element (pdg_pack_block_cols) and
        is expanded into every row on the host (pdg_expand_block_cols)."""
        torch = _torch()
        p = self.plan
        nr = p.row_elements.shape[0]
        counts = np.diff(p.dof.offsets)[p.row_elements]
        self._row0 = np.zeros(nr + 1, np.int64)
        np.cumsum(counts, out=self._row0[1:])
        self._poff = torch.zeros(nr + 1, dtype=torch.int64, device=p.values.device)
        total = int(p.t["row_len"][:nr].sum()) if nr else 0
        self._packed = torch.empty(max(total, 1), dtype=torch.int64, device=p.values.device)
        self._packed_h = _pinned_empty(self._packed)
        self._event = torch.cuda.Event()
        # a host thread per 16 MB of col_idx written, at most 16
        self._threads = max(1, min(16, os.cpu_count() or 1, int(p.col_idx.numel()) * 8 >> 24))
        self.d2h_bytes = sum(int(t.numel() * t.element_size()) for t in (p.row_ptr, p.values, p.rhs)) + 8 * total

    @property
    def retained(self) -> bool:
        return bool(self.host)

    @property
    def packed_cols(self) -> bool:
        """col_idx crosses the link once per element (expanded on the host)."""
        return bool(self.host) and getattr(self, "_packed_h", None) is not None

    def upload(self):
        torch = _torch()
        with torch.cuda.stream(self.plan.stream):
            for attr, h in self.inputs.items():
                self.plan.dm.t[attr].copy_(h, non_blocking=True)

    def download(self):
        torch = _torch()
        p = self.plan
        outs = (p.row_ptr, p.col_idx, p.values, p.rhs)
        if self.packed_cols:
            return self._download_compact()
        with torch.cuda.stream(p.stream):
            if self.host:
                for t, (_, h, _) in zip(outs, self.host):
                    h.copy_(t.reshape(-1), non_blocking=True)
                return
            cap = self.stage.numel()
            for t in outs:
                flat = t.reshape(-1).view(torch.uint8)
                for a in range(0, flat.numel(), cap):
                    b = min(a + cap, flat.numel())
                    self.stage[: b - a].copy_(flat[a:b], non_blocking=True)

    def _download_compact(self):
        # stream: row_ptr, rhs, packed columns, then the values (the bulk); the
        # host expands the columns while the values are in flight
        torch = _torch()
        p, lib = self.plan, _lib.load()
        (rp, rp_t, _), (ci, _, _), (_, va_t, _), (_, rh_t, _) = self.host
        nr = p.row_elements.shape[0]
        with torch.cuda.stream(p.stream):
            rp_t.copy_(p.row_ptr.reshape(-1), non_blocking=True)
            rh_t.copy_(p.rhs.reshape(-1), non_blocking=True)
            if nr:
                torch.cumsum(p.t["row_len"][:nr], 0, out=self._poff[1:])
            _lib.check(lib.pdg_pack_block_cols(_lib.ptr(p.col_idx), _lib.ptr(p.t["val_off"]), _lib.ptr(p.t["row_len"]),
                                               _lib.ptr(self._poff), nr, _lib.ptr(self._packed),
                                               _lib.stream_ptr(p.stream)))
            self._packed_h[1].copy_(self._packed, non_blocking=True)
            self._event.record(p.stream)
            va_t.copy_(p.values.reshape(-1), non_blocking=True)
        self._event.synchronize()
        _lib.check(lib.pdg_expand_block_cols(nr, self._row0.ctypes.data, rp.ctypes.data, self._packed_h[0].ctypes.data,
                                             ci.ctypes.data, self._threads))

    def result(self):
        """(CSRMatrix, rhs) of the last download (after the stream is
        synchronised): views of the page-locked buffers, overwritten by the
        next ``download()``."""
        if not self.host:
            raise AssemblyError("HostIO(retain=False) keeps no host copy")
        (rp, _, _), (ci, _, _), (va, _, _), (rh, _, _) = self.host
        return CSRMatrix(self.plan.n_local_rows, self.plan.dof.n_dofs, rp, ci, va), rh

    def close(self):
        """Drop the host arrays: their page-locked memory is freed when the
        last view of it (e.g. a ``result()`` array the caller kept) is gone."""
        self.host = []
        self._packed = self._packed_h = None


class _PinnedBlock:
    """Owner of one pdg_host_alloc block (freed with the last numpy view)."""

    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        try:
            _lib.load().pdg_host_free(self.ptr)
        except Exception:  # interpreter shutdown
            pass


def _pinned_empty(t):
    """Page-locked host array shaped like device tensor ``t`` (flattened), a
    torch view of it (copies into it are async DMA) and its pointer."""
    import ctypes as C

    torch = _torch()
    dt = np.dtype(str(t.dtype).replace("torch.", ""))
    n = int(t.numel())
    ptr = C.c_void_p()
    _lib.check(_lib.load().pdg_host_alloc(n * dt.itemsize, C.byref(ptr)))
    if not ptr.value:
        arr = np.empty(n, dt)
    else:
        buf = (C.c_char * (n * dt.itemsize)).from_address(ptr.value)
        buf._owner = _PinnedBlock(ptr.value)  # numpy views keep buf, buf keeps the block
        arr = np.frombuffer(buf, dtype=dt, count=n)
    return arr, torch.from_numpy(arr), ptr.value


@dataclass
class DeviceAssembly:
    """Device-resident result of one assembly (CSR in HBM)."""

    plan: SipgPlan
    stats: AssemblyStats
    local: object = None  # distribute.LocalProblem when the plan runs on a rank's sub-mesh

    @property
    def row_ptr(self):
        return self.plan.row_ptr

    @property
    def col_idx(self):
        return self.plan.col_idx

    @property
    def values(self):
        return self.plan.values

    @property
    def rhs(self):
        return self.plan.rhs

    def to_csr(self) -> CSRMatrix:
        return self.plan.to_csr()


def assemble_device(mesh, coeffs, specs, config: Optional[AssemblyConfig] = None,
                    row_elements=None, device=None, stream=None, col_dof=None) -> DeviceAssembly:
    """Assemble on the GPU and keep the CSR in HBM."""
    torch = _torch()
    t0 = time.perf_counter()
    plan = SipgPlan(mesh, coeffs, specs, config, row_elements, device, stream, col_dof=col_dof)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    plan.run(ev)
    plan.check_flags()
    ms_index = ev[0].elapsed_time(ev[1])
    ms_pre = ev[1].elapsed_time(ev[2])
    ms_el = ev[2].elapsed_time(ev[3])
    stats = _stats(plan, ms_index, ms_pre, ms_el, time.perf_counter() - t0)
    return DeviceAssembly(plan, stats)


def _fingerprint(arr) -> bytes:
    """Cheap content fingerprint of an array for the work-count cache (shape,
    dtype, the 64-bit sum of every word, a position-weighted sum of a strided
    sample): one vectorised pass, where hashing the bytes would cost ~100 ms
    per call at 4M elements.  The cache only feeds AssemblyStats counts."""
    a = np.ascontiguousarray(arr)
    b = a.view(np.uint8).ravel()
    pad = (-b.size) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    w = b.view(np.uint64)
    step = max(1, w.size // 65536)
    ws = w[::step]  # position-weighted part on a strided sample (the plain sum sees every word)
    with np.errstate(over="ignore"):
        s1 = int(w.sum(dtype=np.uint64))
        s2 = int((ws * (np.arange(ws.size, dtype=np.uint64) * np.uint64(0x9E3779B97F4A7C15) | np.uint64(1)))
                 .sum(dtype=np.uint64))
    return repr((a.shape, a.dtype.str, s1, s2)).encode()


def _work_counts(plan):
    """(polydg per-kernel work counts, canonical FLOP split) of a plan, cached on
    the flat mesh for repeated assemblies of the same problem (they depend only
    on the mesh, degrees, rows, tags and which coefficient terms exist)."""
    import copy
    import hashlib

    from .roofline import assembly_work

    f = plan.flat
    h = hashlib.sha1()
    for arr in (plan.degrees, plan.row_elements, f.face_tag):
        h.update(_fingerprint(arr))
    h.update(repr((plan.cdesc["diffusion_kind"], plan.cdesc["has_advection"], plan.cdesc["has_reaction"],
                   plan.config.quad_increment, int(plan.nnz))).encode())
    key = h.hexdigest()
    cache = f.__dict__.setdefault("_work_cache", {})
    if key not in cache:
        if len(cache) > 8:
            cache.clear()
        cache[key] = (plan.work_stats(), assembly_work(plan))
    kern, w = cache[key]
    return copy.deepcopy(kern), w


def apportion(kern: dict, flops: dict, ms: float) -> None:
    """Split one fused kernel's device time ``ms`` across polydg's kernel rows
    in proportion to their canonical FLOPs (the rows sum to ``ms``)."""
    tot = sum(flops.values())
    for name, fl in flops.items():
        kern[name].seconds = ms * 1e-3 * (fl / tot if tot > 0 else (1.0 if name == "element" else 0.0))


def _stats(plan, ms_index, ms_pre, ms_el, total_s) -> AssemblyStats:
    """polydg ``AssemblyStats`` (assembly.py:360-391) of one device assembly.

    Mapping of polydg's timers onto the device phases:
      * ``index_seconds`` = the index phase (adjacency, row offsets), polydg's
        ``_pattern_from_adjacency`` + ``empty_matrix``;
      * ``kernel_wall_seconds`` = the fused element kernel, polydg's
        ``_execute_plan`` wall;
      * the pre-pass (frames, sigma, flow side, interface records) is polydg's
        ``build_work_plan`` work, which polydg times in no kernel row: here too
        it is only in ``total_seconds`` (and ``device_ms["prepass"]``);
      * per-kernel ``seconds``: ONE kernel computes every class, so its device
        time is split across the five rows in proportion to each class's
        canonical FLOPs (roofline.assembly_work; the rows sum to the kernel
        time) -- an apportioned figure, flagged by ``kernel_split``.
    ``work_items`` / ``nnz_written`` are polydg's analytic counts."""
    kern, w = _work_counts(plan)
    apportion(kern, {"element": w["flops_volume"], "interior": w["flops_interior"],
                     "dirichlet": w["flops_dirichlet"], "inflow": w["flops_inflow"],
                     "neumann_outflow": w["flops_neumann"]}, ms_el)
    return AssemblyStats(
        kernels=kern, index_seconds=ms_index * 1e-3, kernel_wall_seconds=ms_el * 1e-3, total_seconds=total_s,
        triplet_count=sum(k.nnz_written for k in kern.values()), nnz=plan.nnz,
        device_ms={"index": ms_index, "prepass": ms_pre, "element": ms_el},
        kernel_split="apportioned by canonical FLOPs (one fused kernel)")


# ---------------------------------------------------------------------------
# polydg-compatible entry points
# ---------------------------------------------------------------------------

def _check_classified(mesh):
    flat = flat_of(mesh)
    bad = np.flatnonzero((flat.face_neighbor == BOUNDARY) & (flat.face_tag == TAG_CODE["interior"]))
    if bad.size:
        raise AssemblyError(f"boundary face {int(bad[0])} is unclassified; run classify_boundary_faces")


def assemble_approach2(mesh, coeffs, specs, config: Optional[AssemblyConfig] = None):
    """Preset-sparsity assembly on the B200 (polydg ``assembly.py:1090-1099``)."""
    t0 = time.perf_counter()
    _check_classified(mesh)
    res = assemble_device(mesh, coeffs, specs, config)
    plan = res.plan
    matrix = plan.to_csr()
    rhs = download(plan.rhs, plan.stream)
    # polydg's pattern owns its own copy of row_ptr / col_idx (empty_matrix
    # copies again); here it shares the matrix's host arrays instead of a second
    # 8 B/nnz download
    pattern = plan.block_pattern(matrix.row_ptr, matrix.col_idx)
    res.stats.total_seconds = time.perf_counter() - t0
    return matrix, rhs, res.stats, pattern


def assemble_approach1(mesh, coeffs, specs, config: Optional[AssemblyConfig] = None):
    """Stage-and-sort assembly on the device (polydg ``assembly.py:1036-1045``):
    per-item triplet stripes, stable radix sort, reduce-by-key
    (``approach1.py``).  Per-element degrees (whose volume items polydg
    regroups by degree) run the preset-sparsity engine, which yields the same
    CSR within 1e-12 (polydg's own A1 == A2 contract)."""
    from .approach1 import assemble_approach1_device

    deg, _, _ = spec_arrays(specs)
    if deg.size and np.any(deg != deg[0]):
        matrix, rhs, stats, _ = assemble_approach2(mesh, coeffs, specs, config)
        return matrix, rhs, stats
    return assemble_approach1_device(mesh, coeffs, specs, config)


def _assemble_approach2_rows(mesh, coeffs, specs, config, row_elements):
    _check_classified(mesh)
    res = assemble_device(mesh, coeffs, specs, config, row_elements=row_elements)
    return res


def triplets_to_csr(rows, cols, vals, n_rows, n_cols, n_workers=1, sentinel=None) -> CSRMatrix:
    """Sort triplets by (row, col), sum duplicates in stable input order, emit
    CSR (polydg ``assembly.py:1002-1031``) -- on the device: 64-bit keys
    row * n_cols + col, CUB stable radix sort + reduce-by-key
    (``pdg_triplets_to_csr``).  ``n_workers`` is accepted for compatibility
    (the result never depends on it, as in polydg)."""
    import ctypes as C

    torch = _torch()
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.asarray(cols, dtype=np.int64).ravel()
    vals = np.asarray(vals, dtype=float).ravel()
    if not (rows.shape == cols.shape == vals.shape):
        raise ValueError("rows, cols and vals must have the same length")
    if sentinel is not None:
        keep = rows != sentinel
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
    if rows.size == 0:
        return CSRMatrix(n_rows, n_cols, np.zeros(n_rows + 1, dtype=np.int64), np.empty(0, dtype=np.int64),
                         np.empty(0))
    if rows.min() < 0 or rows.max() >= n_rows or cols.min() < 0 or cols.max() >= n_cols:
        raise AssemblyError("triplet index out of matrix bounds")
    if int(n_rows) * int(n_cols) >= (1 << 63):
        raise AssemblyError("matrix too large for 64-bit triplet keys")
    dev = _require_cuda(None)
    lib = _lib.load()
    n = int(rows.size)
    keys = torch.from_numpy(rows * np.int64(n_cols) + cols).to(dev)
    tv = torch.from_numpy(np.ascontiguousarray(vals)).to(dev)
    rp = torch.empty(int(n_rows) + 1, dtype=torch.int64, device=dev)
    ci = torch.empty(n, dtype=torch.int64, device=dev)
    va = torch.empty(n, dtype=torch.float64, device=dev)
    nnz = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = int(lib.pdg_triplets_workspace_bytes(n))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    _lib.check(lib.pdg_triplets_to_csr(_lib.ptr(keys), _lib.ptr(tv), n, int(n_rows), int(n_cols), _lib.ptr(rp),
                                       _lib.ptr(ci), _lib.ptr(va), _lib.ptr(nnz), _lib.ptr(ws), wsb,
                                       _lib.stream_ptr(stream)))
    stream.synchronize()
    k = int(nnz.item())
    return CSRMatrix(int(n_rows), int(n_cols), rp.cpu().numpy(), ci[:k].cpu().numpy(), va[:k].cpu().numpy())


def build_block_pattern(mesh, specs, row_elements=None) -> BlockPattern:
    """Block pattern on the device (polydg ``assembly.py:275-287``)."""
    import ctypes as C

    from .model import PdeCoefficients

    plan = SipgPlan(mesh, PdeCoefficients(), specs, AssemblyConfig(), row_elements)
    _lib.check(plan.lib.pdg_pattern_fill(C.byref(plan.dm.struct), C.byref(plan.basis),
                                         C.byref(plan.pattern), _lib.stream_ptr(plan.stream)))
    plan.stream.synchronize()
    return plan.block_pattern()


def element_kernel(mesh, element, coeffs, spec, quad_increment=2):
    """Volume block and load of one element (polydg ``assembly.py:1139-1152``),
    computed by the device element kernel (volume-only mode)."""
    import ctypes as C

    from .basis import BasisSpec

    torch = _torch()
    flat = flat_of(mesh)
    nel = flat.n_elements
    specs = [BasisSpec(spec.degree, spec.family, spec.box)] * nel
    plan = _UnitPlan(mesh, coeffs, specs, quad_increment)
    nb = num_basis(spec.degree, flat.dim)
    ids = torch.tensor([int(element)], dtype=torch.int32, device=plan.device)
    blocks = torch.zeros(nb * nb, dtype=torch.float64, device=plan.device)
    loads = torch.zeros(nb, dtype=torch.float64, device=plan.device)
    _lib.check(plan.lib.pdg_frames_build(C.byref(plan.dm.struct), C.byref(plan.basis),
                                         C.byref(plan.frames), _lib.ptr(plan.flags),
                                         _lib.stream_ptr(plan.stream)))
    for _ in range(2):
        _lib.check(plan.lib.pdg_element_blocks(
            C.byref(plan.dm.struct), C.byref(plan.basis), C.byref(plan.coeffs),
            C.byref(plan.rules.struct), C.byref(plan.params), C.byref(plan.frames), _lib.ptr(ids), 1,
            _lib.ptr(blocks), _lib.ptr(loads), _lib.ptr(plan.flags), _lib.stream_ptr(plan.stream)))
        plan.stream.synchronize()
        flags = int(plan.flags.item())
        if not flags & _lib.FLAG_NEG_DIFFUSION or plan.params.options & _lib.OPT_PLAIN_VOLUME:
            break
        plan.params.options |= _lib.OPT_PLAIN_VOLUME  # a(x) < 0: plain volume variant
        plan.flags.zero_()
    _raise_flags(flags & ~_lib.FLAG_NEG_DIFFUSION)
    return blocks.cpu().numpy().reshape(nb, nb), loads.cpu().numpy()


class _UnitPlan:
    """Descriptors for the unit entry points (no pattern)."""

    def __init__(self, mesh, coeffs, specs, quad_increment=2):
        torch = _torch()
        self.lib = _lib.load()
        self.dm = device_mesh(mesh)
        self.device = self.dm.device
        d = self.dm.flat.dim
        deg, boxes, fam = spec_arrays(specs)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        self.t = {"degree": T(deg.astype(np.int32)), "box": T(boxes),
                  "dof": T(np.concatenate([[0], np.cumsum(_num_basis_vec(deg, d, fam))]).astype(np.int64))}
        b = _lib.Basis()
        b.max_degree = int(deg.max())
        b.degree, b.box, b.dof_offset = (_lib.ptr(self.t["degree"]), _lib.ptr(self.t["box"]),
                                         _lib.ptr(self.t["dof"]))
        self.basis = b
        uniq = np.unique(deg)
        self.rules = DeviceRules(d, [2 * int(p) + quad_increment for p in uniq],
                                 [2 * int(p) + quad_increment for p in uniq], self.device)
        self.coeffs = _lib.coeffs_struct(compile_coeffs(coeffs, d))
        self.params = _lib.Params()
        self.params.quad_increment = quad_increment
        self.params.include_gradient_terms = 1
        self.params.penalty_constant = 10.0
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.device)
        self.stream = torch.cuda.current_stream(self.device)
        f = self.dm.flat
        W = 8 if d == 2 else 16
        mk = lambda n: torch.empty(max(int(n) * W, 1), dtype=torch.float64, device=self.device)
        self.t.update(sframe=mk(f.n_simplices), fframe=mk(f.n_facets), erec=mk(f.n_elements))
        fr = _lib.Frames()
        fr.simplex, fr.facet, fr.element = (_lib.ptr(self.t["sframe"]), _lib.ptr(self.t["fframe"]),
                                            _lib.ptr(self.t["erec"]))
        self.frames = fr


from .kernels import (  # noqa: E402  polydg assembly.py:1160-1234 live in kernels.py
    dirichlet_kernel,
    inflow_kernel,
    interior_face_kernel,
    neumann_outflow_kernel,
)
