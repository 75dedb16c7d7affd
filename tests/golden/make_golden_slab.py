"""Generate golden space-time slab fixtures by running the REAL reference
(polydg ``spacetime.assemble_slab``, read-only at /root/reference) in the
build container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_slab.py

Each fixture stores the spatial fine mesh + agglomeration map, the slab
interval, degree and family, the coefficient case (defined identically here
with numpy callables and in tests/fixtures.py with this package's Expr
fields), the time-jump data (initial-data callable, or a previous slab's
coefficient vector) and the reference's Approach-2 CSR + RHS.
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
from polydg import assembly as RA, basis as RB, mesh as RM, model as Rm, spacetime as RS  # noqa: E402


def ref_slab_coeffs(name):
    """polydg-style callables equal to fixtures.<name>() -> (coeffs, initial)."""
    pi = np.pi
    if name == "slab_heat":
        def u(p):
            return np.sin(pi * p[:, 0]) * np.sin(pi * p[:, 1]) * (1.0 - p[:, 2])

        def f(p):
            s = np.sin(pi * p[:, 0]) * np.sin(pi * p[:, 1])
            return s * ((2.0 * pi ** 2 + 1.0) * (1.0 - p[:, 2]) - 1.0)

        C = Rm.PdeCoefficients(diffusion=Rm.constant_tensor(np.diag([1.0, 1.0, 0.0])),
                               advection=Rm.constant_vector([0.0, 0.0, 1.0]),
                               reaction=Rm.constant_scalar(1.0), source=f, dirichlet_data=u)
        return C, lambda xy: np.sin(pi * xy[:, 0]) * np.sin(pi * xy[:, 1])
    if name == "slab_adv_heat":
        def A(p):
            a = 0.1 * (1.0 + 0.5 * p[:, 0])
            out = np.zeros((p.shape[0], 3, 3))
            out[:, 0, 0] = a
            out[:, 1, 1] = a
            return out

        C = Rm.PdeCoefficients(diffusion=A, advection=Rm.constant_vector([0.5, 0.25, 1.0]),
                               source=lambda p: 1.0 + p[:, 2] * p[:, 0],
                               dirichlet_data=lambda p: p[:, 0] + p[:, 2],
                               neumann_data=lambda p: 1.0 + p[:, 1])
        return C, lambda xy: xy[:, 0] * xy[:, 1]
    if name == "slab_heat3d":
        def u(p):
            return np.sin(pi * p[:, 0]) * np.sin(pi * p[:, 1]) * np.sin(pi * p[:, 2]) * (1.0 - p[:, 3])

        def f(p):
            s = np.sin(pi * p[:, 0]) * np.sin(pi * p[:, 1]) * np.sin(pi * p[:, 2])
            return s * ((3.0 * pi ** 2 + 1.0) * (1.0 - p[:, 3]) - 1.0)

        C = Rm.PdeCoefficients(diffusion=Rm.constant_tensor(np.diag([1.0, 1.0, 1.0, 0.0])),
                               advection=Rm.constant_vector([0.0, 0.0, 0.0, 1.0]),
                               reaction=Rm.constant_scalar(1.0), source=f, dirichlet_data=u)
        return C, lambda x: np.sin(pi * x[:, 0]) * np.sin(pi * x[:, 1]) * np.sin(pi * x[:, 2])
    if name == "slab_transport":
        C = Rm.PdeCoefficients(advection=Rm.constant_vector([1.0, 0.5, 1.0]),
                               reaction=Rm.constant_scalar(0.5),
                               source=lambda p: p[:, 0] + p[:, 2],
                               dirichlet_data=lambda p: p[:, 1])
        return C, lambda xy: 1.0 + xy[:, 0]
    raise KeyError(name)


def cases():
    """(name, base mesh, agg, (t0, t1), degree, family, coeff case, previous)
    previous: None = the case's initial data, else (t0_prev, t1_prev, seed)
    of a previous slab of the same degree/family with a random vector."""
    g10 = F.square_grid(10)
    g6 = F.square_grid(6)
    from paper_2007_04881_b200.meshgen import voronoi_simplicial

    vb, va = voronoi_simplicial(60, seed=5)
    c10 = F.grown_clusters(g10, 23, seed=2)
    return [
        ("slab_heat_pq1", g10, c10, (0.0, 0.25), 1, "PQ", "slab_heat", None),
        ("slab_heat_pq2_prev", g10, c10, (0.25, 0.5), 2, "PQ", "slab_heat", (0.0, 0.25, 11)),
        ("slab_advheat_pq2", vb, va, (0.1, 0.3), 2, "PQ", "slab_adv_heat", None),
        ("slab_transport_p2_prev", g10, c10, (0.5, 1.0), 2, "P", "slab_transport", (0.0, 0.5, 12)),
        ("slab_heat_pq3", g6, F.grown_clusters(g6, 7, seed=1), (0.0, 0.2), 3, "PQ", "slab_heat", None),
        ("slab_advheat_p1", g10, c10, (0.0, 0.1), 1, "P", "slab_adv_heat", None),
        ("slab_3d_heat_pq1", F.cube_grid(2), F.cube_blocks(2, 1), (0.0, 0.2), 1, "PQ", "slab_heat3d", None),
        ("slab_3d_heat_p2_prev", F.cube_grid(2), F.grown_clusters(F.cube_grid(2), 5, seed=1), (0.2, 0.4), 2, "P",
         "slab_heat3d", (0.0, 0.2, 13)),
    ]


def main():
    for name, base, agg, (t0, t1), p, fam, cname, prev in cases():
        pm = RM.agglomerate(RM.SimplicialMesh(base.dim, base.vertices, base.simplices), agg)
        C, initial = ref_slab_coeffs(cname)
        family = RB.Family(fam)
        slab, specs = RS.build_slab(pm, (t0, t1), p, family)
        extra = {}
        if prev is None:
            u_prev = initial
        else:
            tp0, tp1, seed = prev
            _, pspecs = RS.build_slab(pm, (tp0, tp1), p, family)
            n = sum(s.n_funcs for s in pspecs)
            vec = np.random.default_rng(seed).standard_normal(n)
            u_prev = (pspecs, vec)
            extra = dict(prev_t0=tp0, prev_t1=tp1, prev_vec=vec)
        pred = F.slab_predicate(cname)
        m, rhs, _ = RS.assemble_slab(slab, C, specs, u_prev, RA.AssemblyConfig(), approach=2,
                                     dirichlet_predicate=pred)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), vertices=base.vertices,
                            simplices=base.simplices, agg=np.asarray(agg), degree=p, family=fam,
                            t0=t0, t1=t1, coeffs=cname, row_ptr=m.row_ptr, col_idx=m.col_idx,
                            values=m.values, rhs=rhs, **extra)
        print(name, pm.n_elements, m.nnz)


if __name__ == "__main__":
    main()
