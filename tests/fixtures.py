"""Deterministic test meshes (the shapes of the reference suite's fixtures,
``pkg/tests/meshes.py``, rebuilt on this package's mesh types) plus
coefficient sets used by the parity tests."""

from __future__ import annotations

import itertools

import numpy as np

from paper_2007_04881_b200 import model as M
from paper_2007_04881_b200.mesh import SimplicialMesh, agglomerate

# the 6 Kuhn tetrahedra of a cube: monotone lattice paths 0 -> 7
KUHN = [(0, 1, 3, 7), (0, 1, 5, 7), (0, 2, 3, 7), (0, 2, 6, 7), (0, 4, 5, 7), (0, 4, 6, 7)]


def square_grid(n: int) -> SimplicialMesh:
    """n x n cells on (0,1)^2, each split (a,b,c),(a,c,d) along its diagonal."""
    ax = np.linspace(0.0, 1.0, n + 1)
    V = np.array([(x, y) for x in ax for y in ax])
    idx = np.arange((n + 1) ** 2).reshape(n + 1, n + 1)
    tris = []
    for i, j in itertools.product(range(n), range(n)):
        a, b, c, d = idx[i, j], idx[i + 1, j], idx[i + 1, j + 1], idx[i, j + 1]
        tris += [(a, b, c), (a, c, d)]
    return SimplicialMesh(2, V, np.array(tris, dtype=np.int64))


def cube_grid(n: int) -> SimplicialMesh:
    ax = np.linspace(0.0, 1.0, n + 1)
    V = np.array([(x, y, z) for x in ax for y in ax for z in ax])
    idx = np.arange((n + 1) ** 3).reshape(n + 1, n + 1, n + 1)
    tets = []
    for i, j, k in itertools.product(range(n), range(n), range(n)):
        corner = [idx[i + a, j + b, k + c] for a in (0, 1) for b in (0, 1) for c in (0, 1)]
        tets += [tuple(corner[v] for v in t) for t in KUHN]
    return SimplicialMesh(3, V, np.array(tets, dtype=np.int64))


def square_blocks(n: int, block: int) -> np.ndarray:
    nb = n // block
    cell = np.array([(i // block) * nb + (j // block) for i in range(n) for j in range(n)])
    return np.repeat(cell, 2)


def cube_blocks(n: int, block: int) -> np.ndarray:
    nb = n // block
    cell = np.array([((i // block) * nb + (j // block)) * nb + (k // block)
                     for i in range(n) for j in range(n) for k in range(n)])
    return np.repeat(cell, 6)


def facet_neighbours(mesh: SimplicialMesh):
    d = mesh.dim
    nbr = [[] for _ in range(mesh.n_simplices)]
    seen = {}
    for s, simp in enumerate(mesh.simplices):
        for k in range(d + 1):
            key = tuple(sorted(int(v) for m, v in enumerate(simp) if m != k))
            if key in seen:
                o = seen.pop(key)
                nbr[s].append(o)
                nbr[o].append(s)
            else:
                seen[key] = s
    return nbr


def grown_clusters(mesh: SimplicialMesh, k: int, seed: int = 0) -> np.ndarray:
    """k facet-connected clusters grown breadth-first from spread seeds."""
    nbr = facet_neighbours(mesh)
    ns = mesh.n_simplices
    rng = np.random.default_rng(seed)
    lab = np.full(ns, -1, np.int64)
    seeds = rng.choice(ns, size=k, replace=False)
    fronts = [[int(s)] for s in seeds]
    for c, s in enumerate(seeds):
        lab[s] = c
    while (lab < 0).any():
        grew = False
        for c in range(k):
            nxt = []
            for s in fronts[c]:
                for t in nbr[s]:
                    if lab[t] < 0:
                        lab[t] = c
                        nxt.append(t)
                        grew = True
            fronts[c] = nxt
        if not grew:
            break
    # relabel to 0..k-1 in order of first appearance (surjective, connected)
    _, first = np.unique(lab, return_index=True)
    order = np.argsort(first)
    remap = np.empty(k, np.int64)
    remap[np.unique(lab)[order]] = np.arange(k)
    return remap[lab]


def zigzag(n_segments: int = 3):
    """Two polygons on [0,2]x[0,1] separated by a zig-zag polyline: one
    interface made of several planar faces."""
    mid = ([(1.0, 0.0), (1.2, 0.5), (1.0, 1.0)] if n_segments == 2
           else [(1.0, 0.0), (1.2, 1.0 / 3.0), (0.95, 2.0 / 3.0), (1.0, 1.0)])
    V = np.array(mid + [(0.0, 0.0), (0.0, 1.0), (2.0, 0.0), (2.0, 1.0)])
    m = len(mid)
    L0, L1, R0, R1 = m, m + 1, m + 2, m + 3
    tris, agg = [], []
    for k in range(m - 1):
        tris += [(L0, k, k + 1), (R0, k + 1, k)]
        agg += [0, 1]
    tris += [(L0, m - 1, L1), (R0, R1, m - 1)]
    agg += [0, 1]
    return agglomerate(SimplicialMesh(2, V, np.array(tris)), np.array(agg))


def two_squares():
    V = np.array([[0.0, 0.0], [1.0, 0.0], [2.0, 0.0], [0.0, 1.0], [1.0, 1.0], [2.0, 1.0]])
    T = np.array([[0, 1, 4], [0, 4, 3], [1, 2, 5], [1, 5, 4]])
    return agglomerate(SimplicialMesh(2, V, T), np.array([0, 0, 1, 1]))


def one_square():
    V = np.array([[0.0, 0.0], [1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    return agglomerate(SimplicialMesh(2, V, np.array([[0, 1, 2], [0, 2, 3]])), np.array([0, 0]))


# ---- coefficient sets (all device-expressible, all numpy-callable) ---------

X, Y, Z = M.X, M.Y, M.Z


def generic(dim):
    """The reference suite's cross-oracle problem (test_assembly.py:364-376)."""
    b = [1.0 + X] + [M.const(1.0)] * (dim - 1)
    return M.PdeCoefficients(
        diffusion=M.isotropic_diffusion(0.7, dim),
        advection=M.VectorField(b),
        reaction=M.constant_scalar(2.0),
        source=M.ScalarField(M.cos(X) + Y),
        dirichlet_data=M.ScalarField(X * 0.3 + 1.0),
    )


def poisson_sine(dim):
    pi = np.pi
    f = dim * pi ** 2 * M.sin(pi * X) * M.sin(pi * Y)
    if dim == 3:
        f = f * M.sin(pi * Z)
    return M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, dim), source=M.ScalarField(f),
                             dirichlet_data=M.constant_scalar(0.0))


def variable_diffusion(dim):
    pi = np.pi
    a = 1.0 + 0.5 * M.sin(2 * pi * X) * M.cos(2 * pi * Y)
    return M.PdeCoefficients(diffusion=M.scalar_diffusion(a, dim), source=M.constant_scalar(1.0),
                             dirichlet_data=M.constant_scalar(0.0))


def adr(dim):
    b = [1.0 + X, 1.0 + Y] + ([1.0 + Z] if dim == 3 else [])
    c = 3.0 + X * Y if dim == 2 else 3.0 + X * Y * Z
    return M.PdeCoefficients(diffusion=M.isotropic_diffusion(0.01, dim), advection=M.VectorField(b),
                             reaction=M.ScalarField(c), source=M.constant_scalar(1.0),
                             dirichlet_data=M.constant_scalar(0.0))


def advdiff3d(dim=3):
    """polydg ``advection_diffusion_3d_problem`` (model.py:312-358): A = 0.01 I,
    b = 1 + x, c = 3 + xyz, u = sin(pi x) sin(pi y) sin(pi z) as Dirichlet data
    (zero on the cube's faces only up to sin(fl(pi)) = 1.2e-16), f manufactured."""
    pi = np.pi
    sx, sy, sz = M.sin(pi * X), M.sin(pi * Y), M.sin(pi * Z)
    cx, cy, cz = M.cos(pi * X), M.cos(pi * Y), M.cos(pi * Z)
    u = sx * sy * sz
    grad = [pi * cx * sy * sz, pi * sx * cy * sz, pi * sx * sy * cz]
    b = [1.0 + X, 1.0 + Y, 1.0 + Z]
    conv = b[0] * grad[0] + b[1] * grad[1] + b[2] * grad[2]
    c = 3.0 + X * Y * Z
    f = 0.01 * 3.0 * pi ** 2 * u + conv + c * u
    return M.PdeCoefficients(diffusion=M.isotropic_diffusion(0.01, 3), advection=M.VectorField(b),
                             reaction=M.ScalarField(c), source=M.ScalarField(f),
                             dirichlet_data=M.ScalarField(u))


def sine_dirichlet(dim=2):
    """2D analogue: ADR with Dirichlet data sin(pi x) sin(pi y) (vanishing on
    the unit square's boundary up to rounding) and a variable source."""
    pi = np.pi
    u = M.sin(pi * X) * M.sin(pi * Y)
    return M.PdeCoefficients(diffusion=M.isotropic_diffusion(0.01, 2), advection=M.VectorField([1.0 + X, 1.0 + Y]),
                             reaction=M.ScalarField(3.0 + X * Y), source=M.ScalarField(2.0 * pi ** 2 * u + 1.0),
                             dirichlet_data=M.ScalarField(u))


def anisotropic(dim):
    """Full variable symmetric tensor + Neumann data (exercises the FULL path)."""
    if dim == 2:
        ent = [1.0 + 0.2 * X, 0.1 * Y, 0.1 * Y, 0.8 + 0.0 * X]
    else:
        ent = [1.0 + 0.2 * X, 0.1 * Y, 0.0 * X, 0.1 * Y, 0.8 + 0.0 * X, 0.05 * Z, 0.0 * X, 0.05 * Z,
               1.2 + 0.0 * X]
    return M.PdeCoefficients(diffusion=M.TensorField(dim, entries=ent),
                             reaction=M.constant_scalar(0.5),
                             source=M.ScalarField(M.exp(X) * Y),
                             dirichlet_data=M.ScalarField(X + Y),
                             neumann_data=M.ScalarField(1.0 + X))


def hyperbolic(dim):
    """No diffusion: pure advection-reaction, inflow/outflow boundary tags."""
    b = [M.const(1.0), M.const(0.5)] + ([M.const(0.25)] if dim == 3 else [])
    return M.PdeCoefficients(advection=M.VectorField(b), reaction=M.constant_scalar(1.0),
                             source=M.ScalarField(1.0 + X), dirichlet_data=M.ScalarField(Y))


# ---- space-time slab coefficient sets (coordinates (x, y, t), time last) ----
# the block form of polydg's parabolic problems (model.py:263-303):
# diffusion [[a, 0], [0, 0]], advection (w, 1)

T = M.Z


def slab_heat():
    """polydg parabolic_sine_problem (model.py:277-303): u = sin(pi x) sin(pi y) (1 - t)."""
    pi = np.pi
    s = M.sin(pi * X) * M.sin(pi * Y)
    coeffs = M.PdeCoefficients(
        diffusion=M.constant_tensor(np.diag([1.0, 1.0, 0.0])),
        advection=M.constant_vector([0.0, 0.0, 1.0]),
        reaction=M.constant_scalar(1.0),
        source=M.ScalarField(s * ((2.0 * pi ** 2 + 1.0) * (1.0 - T) - 1.0)),
        dirichlet_data=M.ScalarField(s * (1.0 - T)))
    return coeffs, M.ScalarField(s)


def slab_adv_heat():
    """Variable spatial diffusion, oblique transport (lateral upwinding and
    inflow Dirichlet faces), Neumann data on x >= 0.5."""
    a = 0.1 * (1.0 + 0.5 * X)
    z = 0.0 * X
    coeffs = M.PdeCoefficients(
        diffusion=M.TensorField(3, entries=[a, z, z, z, a, z, z, z, z]),
        advection=M.constant_vector([0.5, 0.25, 1.0]),
        source=M.ScalarField(1.0 + T * X),
        dirichlet_data=M.ScalarField(X + T),
        neumann_data=M.ScalarField(1.0 + Y))
    return coeffs, M.ScalarField(X * Y)


def slab_transport():
    """No diffusion: lateral boundary faces are inflow / outflow."""
    coeffs = M.PdeCoefficients(
        advection=M.constant_vector([1.0, 0.5, 1.0]),
        reaction=M.constant_scalar(0.5),
        source=M.ScalarField(X + T),
        dirichlet_data=M.ScalarField(Y))
    return coeffs, M.ScalarField(1.0 + X)


def slab_predicate(name):
    """Dirichlet/Neumann split of the lateral boundary (None = all Dirichlet)."""
    if name == "slab_adv_heat":
        return lambda p: bool(p[0] < 0.5)
    return None


def slab_heat3d():
    """3+1D heat problem (spacetime over a 3D mesh): u = sin sin sin (1 - t)."""
    pi = np.pi
    W = M.coord(3)
    s = M.sin(pi * X) * M.sin(pi * Y) * M.sin(pi * Z)
    coeffs = M.PdeCoefficients(
        diffusion=M.constant_tensor(np.diag([1.0, 1.0, 1.0, 0.0])),
        advection=M.constant_vector([0.0, 0.0, 0.0, 1.0]),
        reaction=M.constant_scalar(1.0),
        source=M.ScalarField(s * ((3.0 * pi ** 2 + 1.0) * (1.0 - W) - 1.0)),
        dirichlet_data=M.ScalarField(s * (1.0 - W)))
    return coeffs, M.ScalarField(s)
