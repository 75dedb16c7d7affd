"""Reference-domain quadrature tables for the device kernels.

The device maps the reference rule onto every sub-simplex itself
(``x = v0 + xi @ E``, ``w = w_hat * |det E|``); the host only builds the small
reference tables once per (dim, order) and uploads them, exactly like the
paper keeps its reference rule in constant memory.

The tables follow polydg's conical-product construction point for point,
because the rules are not symmetric under vertex permutation and parity with
the CPU path depends on the point order:

* ``simplex_rule``  -- polydg ``quadrature.py:69-94``: ``(order+2)//2``
  Gauss-Jacobi points per collapsed axis, axis j with weight (1-t)^j,
  tensor grid flattened C-order, unfolded ``x_i = xi_i * prod_{j>i}(1-xi_j)``.
* ``interval_rule`` -- polydg ``quadrature.py:97-103``.

Gauss-Jacobi roots come from ``scipy.special`` (the same call polydg makes,
``quadrature.py:59-66``) so the reference points are bit-identical.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

MAX_ORDER = 40

SIMPLEX = "simplex"
INTERVAL = "interval"


class QuadratureError(ValueError):
    """Degenerate geometry or unsupported rule (polydg ``quadrature.py:26``)."""


@dataclass(frozen=True)
class QuadratureRule:
    domain: str
    dim: int
    order: int
    points: np.ndarray
    weights: np.ndarray

    @property
    def n_points(self) -> int:
        return int(self.weights.shape[0])


def _check_order(order: int) -> None:
    if order < 0:
        raise QuadratureError(f"quadrature order must be nonnegative, got {order}")
    if order > MAX_ORDER:
        raise QuadratureError(f"quadrature order {order} exceeds the supported cap {MAX_ORDER}")


def _jacobi01(npts: int, alpha: int):
    """Gauss rule for f(t)(1-t)^alpha on (0,1) (polydg ``quadrature.py:59-66``)."""
    from scipy.special import roots_jacobi, roots_legendre

    if alpha == 0:
        x, w = roots_legendre(npts)
    else:
        x, w = roots_jacobi(npts, alpha, 0.0)
    return 0.5 * (x + 1.0), w * 0.5 ** (alpha + 1)


def points_per_axis(order: int) -> int:
    return (order + 2) // 2


@lru_cache(maxsize=None)
def simplex_rule(d: int, order: int) -> QuadratureRule:
    if d not in (1, 2, 3):
        raise QuadratureError(f"simplex rules support d in {{1, 2, 3}}, got {d}")
    _check_order(order)
    m = points_per_axis(order)
    axes = [_jacobi01(m, j) for j in range(d)]
    # C-order tensor grid: the last collapsed axis varies fastest.
    t_grid = np.stack(np.meshgrid(*(a[0] for a in axes), indexing="ij"), axis=-1).reshape(-1, d)
    w_grid = np.stack(np.meshgrid(*(a[1] for a in axes), indexing="ij"), axis=-1).reshape(-1, d)
    weights = np.ones(t_grid.shape[0])
    for j in range(d):
        weights *= w_grid[:, j]
    points = t_grid.copy()
    for i in range(d):
        for j in range(i + 1, d):
            points[:, i] *= 1.0 - t_grid[:, j]
    points.setflags(write=False)
    weights.setflags(write=False)
    return QuadratureRule(SIMPLEX, d, order, points, weights)


@lru_cache(maxsize=None)
def interval_rule(order: int) -> QuadratureRule:
    _check_order(order)
    t, w = _jacobi01(points_per_axis(order), 0)
    pts = t[:, None].copy()
    pts.setflags(write=False)
    w = w.copy()
    w.setflags(write=False)
    return QuadratureRule(INTERVAL, 1, order, pts, w)


def face_rule(dim: int, order: int) -> QuadratureRule:
    """Rule on one sub-facet: an interval in 2D, a triangle in 3D
    (polydg ``assembly.py:582-590``)."""
    return interval_rule(order) if dim == 2 else simplex_rule(dim - 1, order)


CLASSIFY_ORDER = 2  # polydg model.py:26 -- flow-side sample rule order


class RuleTable:
    """All reference rules one assembly needs, packed for upload.

    ``order -> (offset, n_points)`` for volume rules (dim-simplex) and face
    rules (interval / triangle); points are stored padded to 3 coordinates.
    """

    def __init__(self, dim: int, orders_volume, orders_face):
        self.dim = dim
        pts, wts = [], []
        self.vol = {}
        self.face = {}
        off = 0
        for kind, orders, fn in (
            ("vol", sorted(set(orders_volume)), lambda o: simplex_rule(dim, o)),
            ("face", sorted(set(orders_face) | {CLASSIFY_ORDER}), lambda o: face_rule(dim, o)),
        ):
            table = self.vol if kind == "vol" else self.face
            for o in orders:
                r = fn(o)
                p3 = np.zeros((r.n_points, 3))
                p3[:, : r.points.shape[1]] = r.points
                pts.append(p3)
                wts.append(np.asarray(r.weights, dtype=np.float64))
                table[o] = (off, r.n_points)
                off += r.n_points
        self.points = np.ascontiguousarray(np.concatenate(pts)) if pts else np.zeros((0, 3))
        self.weights = np.ascontiguousarray(np.concatenate(wts)) if wts else np.zeros(0)

    def lookup_arrays(self, max_order: int):
        """Dense ``order -> offset`` / ``order -> n_points`` arrays (-1 = absent)."""
        vo = np.full(max_order + 1, -1, np.int32)
        vn = np.zeros(max_order + 1, np.int32)
        fo = np.full(max_order + 1, -1, np.int32)
        fn = np.zeros(max_order + 1, np.int32)
        for o, (a, n) in self.vol.items():
            if o <= max_order:
                vo[o], vn[o] = a, n
        for o, (a, n) in self.face.items():
            if o <= max_order:
                fo[o], fn[o] = a, n
        return vo, vn, fo, fn
