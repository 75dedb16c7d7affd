"""Generate golden CSR/RHS fixtures by running the REAL reference (polydg,
read-only at /root/reference) in the build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Each fixture stores the fine mesh + agglomeration map, the degree, the name of
a coefficient case (defined identically here with polydg builders / numpy
lambdas and in tests/fixtures.py with this package's Expr fields), and the
reference's ``assemble_approach2`` output.  The GPU box has no reference
checkout; the committed .npz files are what pins the oracle there.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.append("/root/reference/pkg/src")

import fixtures as F  # noqa: E402
from polydg import assembly as RA, basis as RB, mesh as RM, model as Rm  # noqa: E402


def ref_coeffs(name: str, dim: int):
    """polydg-style callables equal to fixtures.<name>(dim)."""
    pi = np.pi
    if name == "generic":
        def b_field(p):
            out = np.ones((p.shape[0], dim))
            out[:, 0] = 1.0 + p[:, 0]
            return out
        return Rm.PdeCoefficients(diffusion=Rm.isotropic_diffusion(0.7, dim), advection=b_field,
                                  reaction=Rm.constant_scalar(2.0),
                                  source=lambda p: np.cos(p[:, 0]) + p[:, 1],
                                  dirichlet_data=lambda p: p[:, 0] * 0.3 + 1.0)
    if name == "poisson_sine":
        def f(p):
            v = dim * pi ** 2 * np.sin(pi * p[:, 0]) * np.sin(pi * p[:, 1])
            return v * np.sin(pi * p[:, 2]) if dim == 3 else v
        return Rm.PdeCoefficients(diffusion=Rm.isotropic_diffusion(1.0, dim), source=f,
                                  dirichlet_data=Rm.constant_scalar(0.0))
    if name == "variable_diffusion":
        def A(p):
            a = 1.0 + 0.5 * np.sin(2 * pi * p[:, 0]) * np.cos(2 * pi * p[:, 1])
            out = np.zeros((p.shape[0], dim, dim))
            for k in range(dim):
                out[:, k, k] = a
            return out
        return Rm.PdeCoefficients(diffusion=A, source=Rm.constant_scalar(1.0),
                                  dirichlet_data=Rm.constant_scalar(0.0))
    if name == "adr":
        def b(p):
            return 1.0 + p[:, :dim]
        def c(p):
            return 3.0 + (p[:, 0] * p[:, 1] if dim == 2 else p[:, 0] * p[:, 1] * p[:, 2])
        return Rm.PdeCoefficients(diffusion=Rm.isotropic_diffusion(0.01, dim), advection=b, reaction=c,
                                  source=Rm.constant_scalar(1.0), dirichlet_data=Rm.constant_scalar(0.0))
    if name == "hyperbolic":
        vec = [1.0, 0.5] + ([0.25] if dim == 3 else [])
        return Rm.PdeCoefficients(advection=Rm.constant_vector(vec), reaction=Rm.constant_scalar(1.0),
                                  source=lambda p: 1.0 + p[:, 0], dirichlet_data=lambda p: p[:, 1])
    if name == "advdiff3d":  # the reference's own named problem, unmodified
        return Rm.advection_diffusion_3d_problem()
    if name == "sine_dirichlet":
        def u(p):
            return np.sin(pi * p[:, 0]) * np.sin(pi * p[:, 1])
        return Rm.PdeCoefficients(diffusion=Rm.isotropic_diffusion(0.01, 2), advection=lambda p: 1.0 + p[:, :2],
                                  reaction=lambda p: 3.0 + p[:, 0] * p[:, 1],
                                  source=lambda p: 2.0 * pi ** 2 * u(p) + 1.0, dirichlet_data=u)
    raise KeyError(name)


def cases():
    """(name, base SimplicialMesh of this package, agg map, degree, coeff case)."""
    g10 = F.square_grid(10)
    g6 = F.square_grid(6)
    c3 = F.cube_grid(3)
    from paper_2007_04881_b200.meshgen import voronoi_simplicial

    vb, va = voronoi_simplicial(120, seed=7)
    v1k, a1k = voronoi_simplicial(1000, seed=0)  # the cfg1 mesh (problems.WORKLOADS["cfg1"])
    c4 = F.cube_grid(4)
    return [
        ("cfg1_voronoi1000_poisson_p1", v1k, a1k, 1, "poisson_sine"),
        ("cube4_advdiff3d_p2", c4, F.grown_clusters(c4, 30, seed=5), 2, "advdiff3d"),
        ("voronoi120_sinedir_p3", vb, va, 3, "sine_dirichlet"),
        ("clusters10_generic_p2", g10, F.grown_clusters(g10, 23, seed=2), 2, "generic"),
        ("clusters6_poisson_p3", g6, F.grown_clusters(g6, 7, seed=1), 3, "poisson_sine"),
        ("blocks8_vardiff_p2", F.square_grid(8), F.square_blocks(8, 2), 2, "variable_diffusion"),
        ("voronoi120_adr_p2", vb, va, 2, "adr"),
        ("voronoi120_poisson_p4", vb, va, 4, "poisson_sine"),
        ("clusters10_hyperbolic_p1", g10, F.grown_clusters(g10, 23, seed=2), 1, "hyperbolic"),
        ("cube3_generic_p1", c3, F.grown_clusters(c3, 11, seed=3), 1, "generic"),
        ("cube3_adr_p2", c3, F.grown_clusters(c3, 11, seed=3), 2, "adr"),
    ]


def main(only=None):
    for name, base, agg, p, cname in cases():
        if only and name not in only:
            continue
        pm = RM.agglomerate(RM.SimplicialMesh(base.dim, base.vertices, base.simplices), agg)
        C = ref_coeffs(cname, base.dim)
        Rm.classify_boundary_faces(pm, C)
        specs = RB.build_basis(pm, p)
        m, rhs, _, _ = RA.assemble_approach2(pm, C, specs)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), vertices=base.vertices,
                            simplices=base.simplices, agg=np.asarray(agg), degree=p, coeffs=cname,
                            row_ptr=m.row_ptr, col_idx=m.col_idx, values=m.values, rhs=rhs)
        print(name, pm.n_elements, m.nnz)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
