"""Consumers of the assembled system on the device -- polydg
``solver.py`` (restarted GMRES with element-block Jacobi preconditioning)
and the Matrix Market IO of ``assembly.py:177-204``.

The matrix-vector product and the preconditioner are hand-written kernels
(``csrc/pdg_solver.cu``): the element-block SpMV reads each element's column
list once (the assembled CSR repeats it on every row of the element) and the
block-Jacobi setup inverts every diagonal block in shared memory.  The
Krylov loop (right-preconditioned restarted GMRES, modified Gram-Schmidt)
runs on device vectors; torch supplies the BLAS-1 plumbing.  Same contract
as polydg: the reported residual is recomputed explicitly, relative to
||rhs||; ``converged`` = residual <= 10 tol; non-convergence is reported,
not raised.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib


class SolverError(RuntimeError):
    pass


@dataclass
class SolveResult:
    x: np.ndarray
    residual: float
    iterations: int
    converged: bool


class DeviceSystem:
    """The assembled CSR + DoF map resident on the GPU (from a plan, a
    DeviceAssembly, or uploaded from a host CSRMatrix)."""

    def __init__(self, matrix, dof_offsets, device=None, stream=None):
        import torch

        from .assembly import _require_cuda

        self.device = _require_cuda(device)
        self.lib = _lib.load()
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        T = lambda a: a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a)).to(self.device)
        self.row_ptr, self.col_idx, self.values = T(matrix.row_ptr), T(matrix.col_idx), T(matrix.values)
        self.dof = T(np.asarray(dof_offsets, np.int64))
        self.n = int(matrix.n_rows)
        if int(matrix.n_rows) != int(matrix.n_cols):
            raise SolverError("solve needs a square matrix")
        self.n_elements = int(self.dof.shape[0] - 1)
        self.flags = torch.zeros(1, dtype=torch.int32, device=self.device)

    def matvec(self, x, out=None):
        import torch

        y = out if out is not None else torch.empty(self.n, dtype=torch.float64, device=self.device)
        _lib.check(self.lib.pdg_spmv_blocked(_lib.ptr(self.dof), self.n_elements, _lib.ptr(self.row_ptr),
                                             _lib.ptr(self.col_idx), _lib.ptr(self.values), _lib.ptr(x), _lib.ptr(y),
                                             _lib.ptr(self.flags), _lib.stream_ptr(self.stream)))
        return y


def _host_diagonal_blocks(matrix, offsets) -> list:
    """Dense diagonal blocks of any host CSR (polydg ``_extract_diagonal_blocks``,
    solver.py:30-44): entries outside the stored pattern are zero."""
    rp, ci, va = np.asarray(matrix.row_ptr), np.asarray(matrix.col_idx), np.asarray(matrix.values)
    rows = np.repeat(np.arange(rp.size - 1, dtype=np.int64), np.diff(rp))
    elem = np.searchsorted(offsets, rows, "right") - 1
    keep = (ci >= offsets[elem]) & (ci < offsets[elem + 1])
    blocks = [np.zeros((int(offsets[e + 1] - offsets[e]),) * 2) for e in range(offsets.size - 1)]
    for r, c, v, e in zip(rows[keep].tolist(), ci[keep].tolist(), va[keep].tolist(), elem[keep].tolist()):
        blocks[e][r - offsets[e], c - offsets[e]] = v
    return blocks


class BlockJacobiPreconditioner:
    """Action of the inverse element-block diagonal (polydg solver.py:47-70).

    Block-structured CSRs (the assembled pattern) are inverted on the device.
    Otherwise (``host`` = the host CSR) the dense diagonal blocks are extracted
    on the host, as polydg does for any CSR.  Point Jacobi (1x1 blocks)
    substitutes 1.0 for a zero or missing diagonal entry (polydg solver.py:102-104)."""

    def __init__(self, system: DeviceSystem, offsets=None, host=None):
        import torch

        self.sys = system
        offs = np.asarray(offsets if offsets is not None else system.dof.cpu().numpy(), np.int64)
        self.dof = torch.from_numpy(offs).to(system.device)
        self.n_blocks = int(offs.size - 1)
        counts = np.diff(offs)
        off = np.concatenate([[0], np.cumsum(counts * counts)]).astype(np.int64)
        self.inv_off = torch.from_numpy(off).to(system.device)
        point = bool(counts.size == 0 or counts.max() == 1)
        if host is None:
            self.inv = torch.empty(max(int(off[-1]), 1), dtype=torch.float64, device=system.device)
            mx = int(counts.max()) if counts.size else 1
            system.flags.zero_()
            _lib.check(system.lib.pdg_block_jacobi_setup(
                _lib.ptr(self.dof), self.n_blocks, mx, _lib.ptr(system.row_ptr), _lib.ptr(system.col_idx),
                _lib.ptr(system.values), _lib.ptr(self.inv_off), _lib.ptr(self.inv), _lib.ptr(system.flags),
                _lib.stream_ptr(system.stream)))
            system.stream.synchronize()
            fl = int(system.flags.item())
            system.flags.zero_()
            if fl and point:  # zero / missing diagonal entries: 1/d with d -> 1.0
                d = _device_diagonal(system)
                self.inv = torch.where(d != 0, 1.0 / torch.where(d != 0, d, 1.0), 1.0)
                return
            if fl & 4:
                raise SolverError("singular diagonal block")
            if fl & 2:
                raise SolverError("matrix has no diagonal block for some element")
            return
        blocks = _host_diagonal_blocks(host, offs)
        if point:
            dg = np.array([b[0, 0] for b in blocks])
            inv = [np.array([[1.0 / v if v != 0 else 1.0]]) for v in dg]
        else:
            inv = []
            for b in blocks:
                try:
                    inv.append(np.linalg.inv(b))
                except np.linalg.LinAlgError as exc:
                    raise SolverError(f"singular diagonal block (size {b.shape[0]}): {exc}")
        flat = np.concatenate([i.ravel() for i in inv]) if inv else np.zeros(1)
        self.inv = torch.from_numpy(np.ascontiguousarray(flat)).to(system.device)

    def apply(self, r, out=None):
        import torch

        z = out if out is not None else torch.empty_like(r)
        s = self.sys
        _lib.check(s.lib.pdg_block_jacobi_apply(_lib.ptr(self.dof), self.n_blocks, _lib.ptr(self.inv_off),
                                                _lib.ptr(self.inv), _lib.ptr(r), _lib.ptr(z),
                                                _lib.stream_ptr(s.stream)))
        return z


def _device_diagonal(system):
    """Diagonal of the device CSR (0 where no entry is stored)."""
    import torch

    rp = system.row_ptr
    n = system.n
    lens = rp[1:] - rp[:-1]
    rows = torch.repeat_interleave(torch.arange(n, device=system.device), lens)
    hit = system.col_idx == rows
    d = torch.zeros(n, dtype=torch.float64, device=system.device)
    d.index_put_((rows[hit],), system.values[hit], accumulate=True)
    return d


def gmres_device(system: DeviceSystem, b, precond=None, tol=1e-10, restart=150, max_iter=2000):
    """Right-preconditioned restarted GMRES on device vectors -> (x, iterations)."""
    import torch

    dev = system.device
    n = system.n
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    bnorm = float(torch.linalg.vector_norm(b))
    it = 0
    M = (lambda v: precond.apply(v)) if precond is not None else (lambda v: v.clone())
    with torch.cuda.stream(system.stream):
        while it < max_iter:
            r = b - system.matvec(x)
            beta = float(torch.linalg.vector_norm(r))
            if beta <= tol * bnorm:
                break
            m = min(restart, max_iter - it)
            V = torch.empty((m + 1, n), dtype=torch.float64, device=dev)
            Z = torch.empty((m, n), dtype=torch.float64, device=dev)
            H = np.zeros((m + 1, m))
            V[0] = r / beta
            g = np.zeros(m + 1)
            g[0] = beta
            cs, sn = np.zeros(m), np.zeros(m)
            k_done = 0
            for k in range(m):
                Z[k] = M(V[k])
                w = system.matvec(Z[k])
                h = V[: k + 1] @ w                      # classical GS, twice (re-orthogonalised)
                w = w - h @ V[: k + 1]
                h2 = V[: k + 1] @ w
                w = w - h2 @ V[: k + 1]
                hk = (h + h2).cpu().numpy()
                hn = float(torch.linalg.vector_norm(w))
                H[: k + 1, k] = hk
                H[k + 1, k] = hn
                if hn > 0:
                    V[k + 1] = w / hn
                # Givens rotations on the new column
                for j in range(k):
                    t = cs[j] * H[j, k] + sn[j] * H[j + 1, k]
                    H[j + 1, k] = -sn[j] * H[j, k] + cs[j] * H[j + 1, k]
                    H[j, k] = t
                den = np.hypot(H[k, k], H[k + 1, k])
                cs[k], sn[k] = (1.0, 0.0) if den == 0 else (H[k, k] / den, H[k + 1, k] / den)
                H[k, k] = cs[k] * H[k, k] + sn[k] * H[k + 1, k]
                H[k + 1, k] = 0.0
                g[k + 1] = -sn[k] * g[k]
                g[k] = cs[k] * g[k]
                it += 1
                k_done = k + 1
                if abs(g[k + 1]) <= tol * bnorm or hn == 0:
                    break
            y = np.linalg.solve(np.triu(H[:k_done, :k_done]), g[:k_done]) if k_done else np.zeros(0)
            x = x + torch.from_numpy(y).to(dev) @ Z[:k_done]
            if abs(g[k_done]) <= tol * bnorm:
                break
    return x, it


def _block_structured(matrix, offsets) -> bool:
    """Every row of each DoF block has the same column list (the assembled
    pattern's structure, assembly.py:316-324) -- what the blocked SpMV needs."""
    rp = np.asarray(matrix.row_ptr)
    ci = np.asarray(matrix.col_idx)
    lens = np.diff(rp)
    first = np.repeat(offsets[:-1], np.diff(offsets))          # first row of each row's block
    if not np.array_equal(lens, lens[first]):
        return False
    k = np.arange(ci.size) - np.repeat(rp[:-1], lens)          # position within the row
    rows = np.repeat(np.arange(lens.size), lens)
    return bool(np.array_equal(ci, ci[rp[first[rows]] + k]))


def solve(matrix, rhs, tol: float = 1e-10, max_iter: int = 2000, restart: int = 150, dof_map=None,
          device=None) -> SolveResult:
    """Solve matrix x = rhs on the GPU by block-Jacobi preconditioned restarted
    GMRES (polydg ``solver.solve``, solver.py:73-118).  ``matrix``: a host
    CSRMatrix, or a plan / DeviceAssembly whose CSR is already in HBM.
    Without a ``dof_map`` the preconditioner is point Jacobi (1x1 blocks)."""
    import torch

    if tol <= 0.0:
        raise SolverError("tolerance must be positive")
    plan = getattr(matrix, "plan", None) or (matrix if hasattr(matrix, "dm") else None)
    if plan is not None:
        csr = _PlanCSR(plan)
        offsets = np.asarray(dof_map.offsets if dof_map is not None else plan.dof.offsets, np.int64)
        pre_offsets, host = offsets, None
    else:
        csr = matrix
        if matrix.n_rows != matrix.n_cols:
            raise SolverError("solve needs a square matrix")
        offsets = (np.asarray(dof_map.offsets, np.int64) if dof_map is not None
                   else np.arange(matrix.n_rows + 1, dtype=np.int64))
        pre_offsets, host = offsets, None
        if dof_map is not None and not _block_structured(matrix, offsets):
            # a CSR without the assembled block structure: the SpMV runs on row
            # blocks, the preconditioner keeps the element blocks (host extraction)
            offsets = np.arange(matrix.n_rows + 1, dtype=np.int64)
            host = matrix
    sys_ = DeviceSystem(csr, offsets, device)
    b = torch.as_tensor(np.asarray(rhs, dtype=np.float64)).to(sys_.device)
    bnorm = float(torch.linalg.vector_norm(b))
    if bnorm == 0.0:
        return SolveResult(np.zeros(sys_.n), 0.0, 0, True)
    pre = BlockJacobiPreconditioner(sys_, pre_offsets, host)
    x, iters = gmres_device(sys_, b, pre, tol, restart, max_iter)
    res = float(torch.linalg.vector_norm(b - sys_.matvec(x))) / bnorm
    sys_.stream.synchronize()
    return SolveResult(x.cpu().numpy(), res, iters, res <= tol * 10.0)


class _PlanCSR:
    def __init__(self, plan):
        self.row_ptr, self.col_idx, self.values = plan.row_ptr, plan.col_idx, plan.values
        self.n_rows = self.n_cols = plan.dof.n_dofs


# -- Matrix Market IO (assembly.py:177-204) ------------------------------------------------

def write_matrix_market(path, matrix) -> None:
    """Coordinate Matrix Market, 17 significant digits (exact round-trip)."""
    rows = np.repeat(np.arange(matrix.n_rows, dtype=np.int64), np.diff(matrix.row_ptr))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{matrix.n_rows} {matrix.n_cols} {matrix.nnz}\n")
        body = np.char.add(np.char.add(np.char.add((rows + 1).astype(str), " "),
                                       np.char.add((np.asarray(matrix.col_idx) + 1).astype(str), " ")),
                           np.array([f"{v:.17g}" for v in np.asarray(matrix.values)], dtype=str))
        if body.size:
            fh.write("\n".join(body.tolist()) + "\n")


def read_matrix_market(path):
    from .assembly import AssemblyError, CSRMatrix

    with open(path, "r", encoding="utf-8") as fh:
        header = fh.readline()
        if "matrix coordinate real general" not in header:
            raise AssemblyError(f"{path}: unsupported Matrix Market header")
        line = fh.readline()
        while line.startswith("%"):
            line = fh.readline()
        n_rows, n_cols, nnz = (int(t) for t in line.split())
        data = np.loadtxt(fh, dtype=str, ndmin=2) if nnz else np.zeros((0, 3), str)
    rows = data[:, 0].astype(np.int64) - 1
    cols = data[:, 1].astype(np.int64) - 1
    vals = data[:, 2].astype(np.float64)
    key = rows * np.int64(max(n_cols, 1)) + cols
    order = np.argsort(key, kind="stable")
    ks, vs = key[order], vals[order]
    starts = np.flatnonzero(np.concatenate([[True], ks[1:] != ks[:-1]])) if ks.size else np.zeros(0, np.int64)
    sums = np.add.reduceat(vs, starts) if ks.size else np.zeros(0)
    uk = ks[starts] if ks.size else np.zeros(0, np.int64)
    row_ptr = np.zeros(n_rows + 1, np.int64)
    np.cumsum(np.bincount(uk // max(n_cols, 1), minlength=n_rows), out=row_ptr[1:])
    return CSRMatrix(n_rows, n_cols, row_ptr, (uk % max(n_cols, 1)).astype(np.int64), sums)
