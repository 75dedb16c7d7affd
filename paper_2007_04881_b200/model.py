"""PDE coefficients as device-evaluable expressions.

polydg passes coefficients as vectorised numpy callables
(``PdeCoefficients``, polydg ``model.py:38-55``).  A GPU cannot call Python,
so here every field is an :class:`Expr` -- a small expression tree that is

* callable on an ``(n, d)`` numpy point array exactly like polydg's fields
  (so the same object feeds the CPU oracle / the reference), and
* compiled to a stack bytecode that the kernels interpret per quadrature
  point (``csrc/sipg_device.cuh`` ``eval_prog``).

polydg's own builders (``constant_scalar`` / ``constant_vector`` /
``constant_tensor`` / ``isotropic_diffusion``, polydg ``model.py:90-113``)
are recognised from their closures and converted.  Any other opaque Python
callable is rejected with ``NotImplementedError``: there is no CPU fallback.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional, Sequence

import numpy as np

from .mesh import BOUNDARY, BoundaryTag, FlatMesh, MeshError, flat_of, tag_code
from .quadrature import CLASSIFY_ORDER, face_rule


class ClassificationError(MeshError):
    """A face straddles the inflow/outflow transition (polydg ``model.py:29``)."""


# ---------------------------------------------------------------------------
# expression trees
# ---------------------------------------------------------------------------

# opcodes: must match csrc/sipg_device.cuh
OP_CONST, OP_COORD, OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_NEG = range(7)
OP_SIN, OP_COS, OP_EXP, OP_LOG, OP_SQRT, OP_POW, OP_ABS, OP_TANH = range(7, 15)

_BINARY = {OP_ADD: np.add, OP_SUB: np.subtract, OP_MUL: np.multiply, OP_DIV: np.divide,
           OP_POW: np.power}
_UNARY = {OP_NEG: np.negative, OP_SIN: np.sin, OP_COS: np.cos, OP_EXP: np.exp, OP_LOG: np.log,
          OP_SQRT: np.sqrt, OP_ABS: np.abs, OP_TANH: np.tanh}


def _as_expr(v) -> "Expr":
    return v if isinstance(v, Expr) else Expr(OP_CONST, value=float(v))


class Expr:
    """Scalar field of the point coordinates; ``expr(points) -> (n,)``."""

    __slots__ = ("op", "args", "value")

    def __init__(self, op: int, args=(), value=0.0):
        self.op = op
        self.args = tuple(args)
        self.value = value

    # numpy evaluation (the oracle / reference side) ---------------------
    def _eval(self, pts: np.ndarray) -> np.ndarray:
        if self.op == OP_CONST:
            return np.full(pts.shape[0], self.value)
        if self.op == OP_COORD:
            return pts[:, int(self.value)]
        if self.op == OP_POW and self.args[1].op == OP_CONST:
            # scalar exponent: numpy's fast paths (x**2 -> square), as user code would
            return self.args[0]._eval(pts) ** float(self.args[1].value)
        if self.op in _BINARY:
            return _BINARY[self.op](self.args[0]._eval(pts), self.args[1]._eval(pts))
        return _UNARY[self.op](self.args[0]._eval(pts))

    def __call__(self, points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        return np.asarray(self._eval(pts), dtype=float)

    # algebra -------------------------------------------------------------
    def __add__(self, o):
        return Expr(OP_ADD, (self, _as_expr(o)))

    def __radd__(self, o):
        return Expr(OP_ADD, (_as_expr(o), self))

    def __sub__(self, o):
        return Expr(OP_SUB, (self, _as_expr(o)))

    def __rsub__(self, o):
        return Expr(OP_SUB, (_as_expr(o), self))

    def __mul__(self, o):
        return Expr(OP_MUL, (self, _as_expr(o)))

    def __rmul__(self, o):
        return Expr(OP_MUL, (_as_expr(o), self))

    def __truediv__(self, o):
        return Expr(OP_DIV, (self, _as_expr(o)))

    def __rtruediv__(self, o):
        return Expr(OP_DIV, (_as_expr(o), self))

    def __pow__(self, o):
        return Expr(OP_POW, (self, _as_expr(o)))

    def __neg__(self):
        return Expr(OP_NEG, (self,))

    @property
    def is_constant(self) -> bool:
        return self.op == OP_CONST

    def compile(self, code: list, consts: list) -> None:
        """Post-order bytecode: op | (arg << 8)."""
        if self.op == OP_CONST:
            code.append(OP_CONST | (len(consts) << 8))
            consts.append(float(self.value))
        elif self.op == OP_COORD:
            code.append(OP_COORD | (int(self.value) << 8))
        else:
            for a in self.args:
                a.compile(code, consts)
            code.append(self.op)

    def depth(self) -> int:
        if not self.args:
            return 1
        return max(a.depth() + i for i, a in enumerate(self.args))

    def __repr__(self):
        if self.op == OP_CONST:
            return repr(self.value)
        if self.op == OP_COORD:
            return "xyz"[int(self.value)]
        names = {OP_ADD: "+", OP_SUB: "-", OP_MUL: "*", OP_DIV: "/", OP_POW: "**"}
        if self.op in names:
            return f"({self.args[0]!r} {names[self.op]} {self.args[1]!r})"
        fn = {OP_NEG: "-", OP_SIN: "sin", OP_COS: "cos", OP_EXP: "exp", OP_LOG: "log",
              OP_SQRT: "sqrt", OP_ABS: "abs", OP_TANH: "tanh"}[self.op]
        return f"{fn}({self.args[0]!r})"


def const(v: float) -> Expr:
    return Expr(OP_CONST, value=float(v))


def coord(k: int) -> Expr:
    return Expr(OP_COORD, value=int(k))


X, Y, Z = coord(0), coord(1), coord(2)


def _unary(op):
    def f(e):
        return Expr(op, (_as_expr(e),))
    return f


sin, cos, exp, log, sqrt = (_unary(o) for o in (OP_SIN, OP_COS, OP_EXP, OP_LOG, OP_SQRT))
fabs, tanh = _unary(OP_ABS), _unary(OP_TANH)


class ScalarField:
    """``(n, d) -> (n,)`` field wrapping one Expr."""

    def __init__(self, expr):
        self.expr = _as_expr(expr)

    def __call__(self, points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        return self.expr(pts)


class VectorField:
    """``(n, d) -> (n, d)`` field, one Expr per component."""

    def __init__(self, components: Sequence):
        self.components = [_as_expr(c) for c in components]

    def __call__(self, points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        return np.stack([c(pts) for c in self.components], axis=1)


class TensorField:
    """``(n, d) -> (n, d, d)`` field: ``scalar * I`` (isotropic) or a full
    row-major matrix of Exprs."""

    def __init__(self, dim: int, scalar=None, entries: Optional[Sequence] = None):
        self.dim = dim
        if (scalar is None) == (entries is None):
            raise ValueError("give exactly one of scalar / entries")
        self.scalar = None if scalar is None else _as_expr(scalar)
        self.entries = None if entries is None else [_as_expr(e) for e in entries]
        if self.entries is not None and len(self.entries) != dim * dim:
            raise ValueError("tensor needs dim*dim entries")

    @property
    def isotropic(self) -> bool:
        return self.scalar is not None

    def __call__(self, points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        n, d = pts.shape[0], self.dim
        if self.isotropic:
            out = np.zeros((n, d, d))
            a = self.scalar(pts)
            for k in range(d):
                out[:, k, k] = a
            return out
        return np.stack([e(pts) for e in self.entries], axis=1).reshape(n, d, d)


# polydg-compatible builders (polydg model.py:90-113) -----------------------

def constant_scalar(value: float) -> ScalarField:
    return ScalarField(const(value))


def constant_vector(values) -> VectorField:
    return VectorField([const(v) for v in np.asarray(values, dtype=float)])


def constant_tensor(matrix) -> TensorField:
    mat = np.atleast_2d(np.asarray(matrix, dtype=float))
    d = mat.shape[0]
    return TensorField(d, entries=[const(v) for v in mat.ravel()])


def isotropic_diffusion(value: float, dim: int) -> TensorField:
    # polydg builds constant_tensor(eye * value); keep the full constant matrix
    # so n^T A n is formed from the same entries.
    return constant_tensor(np.eye(dim) * value)


def scalar_diffusion(a, dim: int) -> TensorField:
    """``a(x) * I`` with a variable scalar ``a``."""
    return TensorField(dim, scalar=a)


# ---------------------------------------------------------------------------
# polydg-compatible containers
# ---------------------------------------------------------------------------

@dataclass
class PdeCoefficients:
    """Fields of -div(A grad u) + b.grad u + c u = f (polydg ``model.py:38-55``)."""

    diffusion: Optional[Callable] = None
    advection: Optional[Callable] = None
    reaction: Optional[Callable] = None
    source: Optional[Callable] = None
    dirichlet_data: Optional[Callable] = None
    neumann_data: Optional[Callable] = None
    exact_solution: Optional[Callable] = None
    exact_gradient: Optional[Callable] = None
    energy_weight: Optional[Callable] = None


@dataclass
class PenaltyConfig:
    """Penalty constant + coverability flags (polydg ``model.py:58-74``)."""

    constant: float = 10.0
    coverable: Optional[np.ndarray] = None

    def __post_init__(self):
        if self.constant <= 0.0:
            raise ValueError("penalty constant must be positive")

    def is_coverable(self, element: int) -> bool:
        return bool(self.coverable is not None and self.coverable[element])


@dataclass
class PenaltySideData:
    """Per-side penalty inputs (polydg ``model.py:77-87``)."""

    volume: float
    degree: int
    a_bar: float
    max_adjacent_volume: float
    cov_cap: float


def penalty_side_data(mesh, element: int, face, degree: int, volume_points, coeffs,
                      config: PenaltyConfig) -> PenaltySideData:
    """Per-side penalty inputs (polydg ``model.py:196-235``): ``a_bar`` =
    max over ``volume_points`` of n.A(x)n with the face normal, evaluated by
    the device coefficient kernel (``pdg_eval_coeffs``); the largest
    subdivision simplex of ``element`` touching the face; the coverability
    cap p^(2(d-1))."""
    from .kernels import _face_id, eval_coefficients
    from .mesh import BOUNDARY, MeshError, flat_of

    flat = flat_of(mesh)
    fid = _face_id(mesh, face)
    n = np.asarray(flat.face_normal[fid], float)
    if coeffs.diffusion is None:
        a_bar = 0.0
    else:
        a = eval_coefficients(coeffs, np.asarray(volume_points, float))["diffusion"]
        a_bar = float(np.einsum("i,qij,j->q", n, a, n).max())
    rows = slice(int(flat.face_ptr[fid]), int(flat.face_ptr[fid + 1]))
    if element == int(flat.face_owner[fid]):
        adj = flat.facet_owner_simplex[rows]
    elif element == int(flat.face_neighbor[fid]):
        adj = flat.facet_neighbor_simplex[rows]
    else:
        raise MeshError("element is not adjacent to the face")
    adj = adj[adj != BOUNDARY]
    if adj.size == 0:
        raise MeshError("no subdivision simplex adjacent to the face")
    max_adj = float(flat.simplex_volumes[adj].max())
    d = flat.dim
    cov_cap = float(degree ** (2 * (d - 1))) if config.is_coverable(element) else np.inf
    return PenaltySideData(volume=float(flat.elem_volumes[element]), degree=int(degree), a_bar=a_bar,
                           max_adjacent_volume=max_adj, cov_cap=cov_cap)


def penalty_sigma(face, owner_data: PenaltySideData, neighbor_data: Optional[PenaltySideData],
                  config: PenaltyConfig) -> float:
    """sigma = C max_k min(|k| / sup|K^F|, cov_cap) a_bar p^2 |F| / |k|, over the
    owner only on Dirichlet faces (polydg ``model.py:238-257``).  The assembly
    path computes the same value for every face on the device
    (``kernels.face_sigma``, csrc/prepass_body.cuh)."""
    from .mesh import MeshError

    sides = [owner_data] if neighbor_data is None else [owner_data, neighbor_data]
    best = 0.0
    for s in sides:
        if s.max_adjacent_volume <= 0.0:
            raise MeshError("penalty data has no adjacent subdivision simplex")
        ratio = min(s.volume / s.max_adjacent_volume, s.cov_cap)
        best = max(best, ratio * s.a_bar * s.degree ** 2 * float(face.measure) / s.volume)
    return config.constant * best


# ---------------------------------------------------------------------------
# conversion of arbitrary coefficient objects into device descriptors
# ---------------------------------------------------------------------------

def _closure_vars(fn) -> dict:
    code = getattr(fn, "__code__", None)
    cells = getattr(fn, "__closure__", None) or ()
    if code is None:
        return {}
    return {name: c.cell_contents for name, c in zip(code.co_freevars, cells)}


def _builder_name(fn) -> str:
    qn = getattr(fn, "__qualname__", "")
    return qn.split(".<locals>")[0] if ".<locals>" in qn else ""


def as_scalar_expr(field, what: str) -> Optional[Expr]:
    if field is None:
        return None
    if isinstance(field, Expr):
        return field
    if isinstance(field, ScalarField):
        return field.expr
    if isinstance(field, (int, float)):
        return const(field)
    if _builder_name(field) == "constant_scalar":
        return const(_closure_vars(field)["value"])
    raise NotImplementedError(
        f"{what}: opaque Python callable {field!r} cannot run on the device; "
        "express it with paper_2007_04881_b200.model (Expr / ScalarField)")


def as_vector_exprs(field, dim: int, what: str) -> Optional[list]:
    if field is None:
        return None
    if isinstance(field, VectorField):
        comps = field.components
    elif _builder_name(field) == "constant_vector":
        comps = [const(v) for v in np.asarray(_closure_vars(field)["vec"], float)]
    else:
        raise NotImplementedError(
            f"{what}: opaque Python callable {field!r} cannot run on the device; "
            "use paper_2007_04881_b200.model.VectorField")
    if len(comps) != dim:
        raise ValueError(f"{what} has {len(comps)} components, mesh dim is {dim}")
    return comps


def as_tensor(field, dim: int, what: str):
    """-> None | ("iso", Expr) | ("full", [Expr]*d*d)."""
    if field is None:
        return None
    if isinstance(field, TensorField):
        if field.dim != dim:
            raise ValueError(f"{what} is {field.dim}-dimensional, mesh dim is {dim}")
        return ("iso", field.scalar) if field.isotropic else ("full", field.entries)
    if _builder_name(field) == "constant_tensor":
        mat = np.atleast_2d(np.asarray(_closure_vars(field)["mat"], float))
        if mat.shape != (dim, dim):
            raise ValueError(f"{what} has shape {mat.shape}, mesh dim is {dim}")
        return ("full", [const(v) for v in mat.ravel()])
    raise NotImplementedError(
        f"{what}: opaque Python callable {field!r} cannot run on the device; "
        "use paper_2007_04881_b200.model.TensorField")


# ---------------------------------------------------------------------------
# boundary classification (host pre-pass the caller runs before assembly)
# ---------------------------------------------------------------------------

def _face_sample_points(flat: FlatMesh, faces: np.ndarray):
    """Order-2 sample points of every sub-facet of ``faces`` (polydg
    ``model.py:118-125``) -> (points [m, d], face index per point)."""
    d = flat.dim
    rule = face_rule(d, CLASSIFY_ORDER)
    counts = flat.face_ptr[faces + 1] - flat.face_ptr[faces]
    rows = np.concatenate([np.arange(a, b) for a, b in
                           zip(flat.face_ptr[faces], flat.face_ptr[faces + 1])]) \
        if faces.size else np.zeros(0, np.int64)
    coords = flat.vertices[flat.facet_vertices[rows]]          # [r, d, d]
    edges = coords[:, 1:] - coords[:, :1]
    pts = coords[:, None, 0, :] + np.einsum("qk,rkd->rqd", rule.points, edges)
    owner_face = np.repeat(np.arange(faces.size), counts * rule.n_points)
    return pts.reshape(-1, d), owner_face, counts * rule.n_points


def classify_boundary_faces(mesh, coeffs, dirichlet_predicate=None):
    """Tag every boundary face (polydg ``model.py:138-173``), vectorised.

    Works on this package's meshes (tags written into the flat arrays); for
    polydg's own mesh objects use polydg's classifier.
    """
    flat = flat_of(mesh)
    if not hasattr(mesh, "flat"):
        raise TypeError("classify_boundary_faces needs this package's PolytopicMesh; "
                        "classify polydg meshes with polydg.model.classify_boundary_faces")
    bf = np.flatnonzero(flat.face_neighbor == BOUNDARY)
    if bf.size == 0:
        return mesh
    pts, which, counts = _face_sample_points(flat, bf)
    normals = flat.face_normal[bf]
    mean = np.add.reduceat(pts, np.r_[0, np.cumsum(counts)[:-1]], axis=0) / counts[:, None]
    tags = np.full(bf.size, tag_code(BoundaryTag.OUTFLOW), np.int8)
    decided = np.zeros(bf.size, bool)
    if coeffs.diffusion is not None:
        a = coeffs.diffusion(mean)
        tau = 1e-12 * np.maximum(1.0, np.abs(a).reshape(bf.size, -1).max(axis=1))
        nan = np.einsum("fi,fij,fj->f", normals, a, normals)
        ell = nan > tau
        dirich = ell.copy()
        if dirichlet_predicate is not None:
            for k in np.flatnonzero(ell):
                dirich[k] = bool(dirichlet_predicate(mean[k]))
        tags[ell & dirich] = tag_code(BoundaryTag.DIRICHLET)
        tags[ell & ~dirich] = tag_code(BoundaryTag.NEUMANN)
        decided |= ell
    if coeffs.advection is not None:
        rest = ~decided
        bn = np.einsum("qd,qd->q", coeffs.advection(pts), normals[which])
        sign = _checked_flow_sign_grouped(bn, counts, "a boundary face", rest)
        tags[rest & (sign < 0.0)] = tag_code(BoundaryTag.INFLOW)
    flat.face_tag[bf] = tags
    return mesh


def _checked_flow_sign_grouped(bn, counts, where, check=None):
    """Per-group mean of b.n with polydg's straddle check (``model.py:128-135``)
    applied to the groups selected by ``check``."""
    starts = np.r_[0, np.cumsum(counts)[:-1]]
    mx = np.maximum.reduceat(np.abs(bn), starts)
    lo = np.minimum.reduceat(bn, starts)
    hi = np.maximum.reduceat(bn, starts)
    tol = 1e-10 * np.maximum(1.0, mx)
    straddle = (lo < -tol) & (hi > tol)
    if check is not None:
        straddle &= check
    if np.any(straddle):
        raise ClassificationError(
            f"advection flux changes sign across {where}; refine the mesh so "
            "faces do not straddle the inflow/outflow transition")
    return np.add.reduceat(bn, starts) / counts


# ---------------------------------------------------------------------------
# device descriptor (filled into include/pdg.h ``pdg_coeffs``)
# ---------------------------------------------------------------------------

MAX_CODE, MAX_CONST, MAX_STACK = 448, 96, 8


def compile_coeffs(coeffs, dim: int) -> dict:
    """Lower a coefficient object to bytecode programs + kind flags.

    Raises NotImplementedError for anything the device cannot evaluate
    (opaque callables); there is no host fallback.
    """
    code: list = []
    consts: list = []

    def prog(expr: Expr, what: str):
        if expr.depth() > MAX_STACK:
            raise NotImplementedError(f"{what}: expression deeper than {MAX_STACK}")
        off = len(code)
        expr.compile(code, consts)
        return (off, len(code) - off, int(expr.is_constant),
                float(expr.value) if expr.is_constant else 0.0)

    desc = {"diffusion_kind": 0, "diffusion_symmetric": 1, "diffusion": [], "advection": []}
    ten = as_tensor(coeffs.diffusion, dim, "diffusion")
    if ten is not None:
        kind, val = ten
        if kind == "full" and all(e.is_constant for e in val):
            m = np.array([e.value for e in val]).reshape(dim, dim)
            if np.all(m == np.diag(np.diag(m))) and np.all(np.diag(m) == m[0, 0]):
                kind, val = "iso", const(m[0, 0])
        if kind == "iso":
            desc["diffusion_kind"] = 1
            desc["diffusion"] = [prog(val, "diffusion")]
        else:
            desc["diffusion_kind"] = 2
            desc["diffusion"] = [prog(e, f"diffusion[{k}]") for k, e in enumerate(val)]
            sym = all(repr(val[i * dim + j]) == repr(val[j * dim + i])
                      for i in range(dim) for j in range(dim))
            desc["diffusion_symmetric"] = int(sym)
    adv = as_vector_exprs(coeffs.advection, dim, "advection")
    desc["has_advection"] = int(adv is not None)
    if adv is not None:
        desc["advection"] = [prog(e, f"advection[{k}]") for k, e in enumerate(adv)]
    for name, field_name in (("reaction", "reaction"), ("source", "source"),
                             ("dirichlet", "dirichlet_data"), ("neumann", "neumann_data")):
        ex = as_scalar_expr(getattr(coeffs, field_name), field_name)
        desc["has_" + name] = int(ex is not None)
        desc[name] = None if ex is None else prog(ex, field_name)
    if len(code) > MAX_CODE or len(consts) > MAX_CONST:
        raise NotImplementedError("coefficient programs exceed the device program capacity")
    desc["code"], desc["consts"] = code, consts
    return desc


# ---------------------------------------------------------------------------
# runtime-specialised policy (CUDA source for pdg_assemble_jit)
# ---------------------------------------------------------------------------

_CFN = {OP_SIN: "sin", OP_COS: "cos", OP_EXP: "exp", OP_LOG: "log", OP_SQRT: "sqrt",
        OP_ABS: "fabs", OP_TANH: "tanh"}
_COP = {OP_ADD: "+", OP_SUB: "-", OP_MUL: "*", OP_DIV: "/"}


def cuda_expr(e: Expr, sinpi: bool = True) -> str:
    """C expression with the same operation order as the numpy evaluation.

    ``sinpi``: sin/cos of (k*pi)*u are emitted as pdg_sinpi/pdg_cospi(k*u) -- the
    same value up to the rounding of k*pi*u (<= 1 ulp of the argument),
    without the pi/2 argument reduction of sin/cos.  Off = the reference's
    own sin(fl(k*pi*u)), bit-for-bit in the argument: needed where data is
    evaluated on a boundary that is a zero of the field (sin(fl(pi)) =
    1.2e-16, not 0) and a large penalty amplifies it (slab Dirichlet data)."""
    rec = lambda x: cuda_expr(x, sinpi)
    if e.op == OP_CONST:
        v = float(e.value)
        if not np.isfinite(v):
            raise NotImplementedError("non-finite constant in a coefficient")
        return f"({v!r})"
    if e.op == OP_COORD:
        return f"x[{int(e.value)}]"
    if sinpi and e.op in (OP_SIN, OP_COS) and e.args[0].op == OP_MUL:
        a, b = e.args[0].args
        for c, u in ((a, b), (b, a)):
            if c.op == OP_CONST:
                k = _pi_multiple(float(c.value))
                if k is not None:
                    fn = "pdg_sinpi" if e.op == OP_SIN else "pdg_cospi"  # sipg_device.cuh
                    arg = rec(u) if k == 1 else f"({float(k)!r} * {rec(u)})"
                    return f"{fn}({arg})"
    if e.op in _COP:
        return f"({rec(e.args[0])} {_COP[e.op]} {rec(e.args[1])})"
    if e.op == OP_POW:
        base, ex = e.args
        if ex.op == OP_CONST and float(ex.value) == 2.0:  # numpy squares exactly
            b = rec(base)
            return f"({b} * {b})"
        return f"pow({rec(base)}, {rec(ex)})"
    if e.op == OP_NEG:
        return f"(-{rec(e.args[0])})"
    return f"{_CFN[e.op]}({rec(e.args[0])})"


def policy_source(coeffs, dim: int, initial=None) -> str:
    """CUDA source of the coefficient policy class ``JitCoef`` consumed by
    ``assemble_body`` (csrc/assemble_body.cuh, see InterpCoef for the
    interface) and ``slab_body`` (csrc/slab_body.cuh: additionally the
    compile-time zero pattern of A and b, and the slab's initial data
    ``u0`` of the spatial coordinates)."""
    return _policy(coeffs, dim, initial)[0]


def slab_policy(coeffs, initial=None, with_info=False, dim=3):
    """(policy source, shared-memory table rows[, info]) of a space-time slab
    (coordinates (x, y, t)); the rows follow ``slab_rows`` in slab_body.cuh."""
    src, info = _policy(coeffs, dim, initial, sinpi=False)
    kind, diag, n_act = info["kind"], info["diag"], info["n_active"]
    vol = 0 if kind == 0 else (n_act if diag else 2 * dim)
    has_vr = info["adv"] or info["reac"]
    vol += 2 if has_vr else (1 if info["src"] else 0)
    return (src, max(vol, 4), info) if with_info else (src, max(vol, 4))


def _is_zero(e) -> bool:
    return e is not None and e.is_constant and float(e.value) == 0.0


def _policy(coeffs, dim: int, initial=None, sinpi: bool = True):
    # sinpi lowering only for the volume fields (A, c, f: a 1-ulp argument
    # difference is invisible there).  Fields evaluated on faces -- the
    # Dirichlet / Neumann data, the advection field that decides inflow /
    # upwinding, the initial data -- keep the reference's sin(fl(k*pi)*u):
    # on a boundary that is a zero of the field (polydg's manufactured
    # solutions, model.py:312-358) sin(fl(pi)) = 1.2e-16, not 0, and the
    # penalty amplifies the difference to ~1e-11 of the element's RHS.
    cuda_expr_ = lambda e: cuda_expr(e, sinpi)
    exact_ = lambda e: cuda_expr(e, False)
    ten = as_tensor(coeffs.diffusion, dim, "diffusion")
    kind, ent = 0, None
    if ten is not None:
        k, val = ten
        if k == "full" and all(e.is_constant for e in val):
            m = np.array([e.value for e in val]).reshape(dim, dim)
            if np.all(m == np.diag(np.diag(m))) and np.all(np.diag(m) == m[0, 0]):
                k, val = "iso", const(m[0, 0])
        kind, ent = (1, val) if k == "iso" else (2, val)
    adv = as_vector_exprs(coeffs.advection, dim, "advection")
    sc = {n: as_scalar_expr(getattr(coeffs, f), f) for n, f in
          (("c", "reaction"), ("f", "source"), ("gD", "dirichlet_data"), ("gN", "neumann_data"))}
    u0 = as_scalar_expr(initial, "initial data") if initial is not None else None
    b = lambda v: "true" if v else "false"
    # zero pattern of A (entry identically 0) and b
    if kind == 0:
        nz = [[False] * dim for _ in range(dim)]
    elif kind == 1:
        nz = [[i == j and not _is_zero(ent) for j in range(dim)] for i in range(dim)]
    else:
        nz = [[not _is_zero(ent[i * dim + j]) for j in range(dim)] for i in range(dim)]
    diag = all(not nz[i][j] for i in range(dim) for j in range(dim) if i != j)
    a_const = kind == 0 or (ent.is_constant if kind == 1 else all(e.is_constant for e in ent))
    bnz = [adv is not None and not _is_zero(c) for c in (adv or [None] * dim)]
    out = ["struct JitCoef {",
           f"  __device__ static constexpr int diff_kind() {{ return {kind}; }}",
           f"  __device__ static constexpr bool has_adv() {{ return {b(adv is not None)}; }}",
           f"  __device__ static constexpr bool has_reac() {{ return {b(sc['c'] is not None)}; }}",
           f"  __device__ static constexpr bool has_src() {{ return {b(sc['f'] is not None)}; }}",
           f"  __device__ static constexpr bool has_dir() {{ return {b(sc['gD'] is not None)}; }}",
           f"  __device__ static constexpr bool has_neu() {{ return {b(sc['gN'] is not None)}; }}",
           f"  __device__ static constexpr bool has_u0() {{ return {b(u0 is not None)}; }}",
           f"  __device__ static constexpr bool a_diag() {{ return {b(diag)}; }}",
           f"  __device__ static constexpr bool a_const() {{ return {b(a_const)}; }}"]
    nzc = " ".join(f"case {i * dim + j}: return true;" for i in range(dim) for j in range(dim)
                   if nz[i][j])
    out.append(f"  __device__ static constexpr bool a_nz(int i, int j) "
               f"{{ switch (i * {dim} + j) {{ {nzc} default: break; }} return false; }}")
    bzc = " ".join(f"case {i}: return true;" for i in range(dim) if bnz[i])
    out.append(f"  __device__ static constexpr bool b_nz(int i) "
               f"{{ switch (i) {{ {bzc} default: break; }} return false; }}")
    iso = cuda_expr_(ent) if kind == 1 else "1.0"
    out.append(f"  __device__ double a_iso(const double* x) const {{ return {iso}; }}")
    cases = ""
    if kind == 2:
        cases = " ".join(f"case {k}: return {cuda_expr_(e)};" for k, e in enumerate(ent))
    elif kind == 1:  # the slab kernel reads A entrywise
        cases = " ".join(f"case {i * dim + i}: return {iso};" for i in range(dim))
    out.append(f"  __device__ double a_ij(int i, int j, const double* x) const "
               f"{{ switch (i * {dim} + j) {{ {cases} default: break; }} return 0.0; }}")
    cases = ""
    if adv is not None:
        cases = " ".join(f"case {k}: return {exact_(e)};" for k, e in enumerate(adv))
    out.append(f"  __device__ double b_i(int i, const double* x) const "
               f"{{ switch (i) {{ {cases} default: break; }} return 0.0; }}")
    for n in ("c", "f", "gD", "gN"):
        lower = cuda_expr_ if n in ("c", "f") else exact_
        body = lower(sc[n]) if sc[n] is not None else "0.0"
        out.append(f"  __device__ double {n}(const double* x) const {{ return {body}; }}")
    out.append(f"  __device__ double u0(const double* x) const "
               f"{{ return {exact_(u0) if u0 is not None else '0.0'}; }}")
    out.append("};")
    info = dict(kind=kind, diag=diag, n_active=sum(nz[i][i] for i in range(dim)),
                adv=adv is not None, reac=sc["c"] is not None, src=sc["f"] is not None,
                adv_spatial=any(bnz[: dim - 1]))
    return "\n".join(out), info


def _pi_multiple(v: float):
    """k if v == k * float(pi) exactly for a small integer k, else None."""
    k = round(v / math.pi)
    if k != 0 and abs(k) <= 64 and float(k) * math.pi == v:
        return int(k)
    return None


