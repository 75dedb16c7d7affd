"""Error behaviour of the device paths (polydg's exception classes):
unclassified boundary faces, flux straddling an interior face, unsupported
slab inputs, the library refusing to run without its extension."""

import numpy as np
import pytest

import fixtures as F
import paper_2007_04881_b200.model as M
from paper_2007_04881_b200 import build_basis, classify_boundary_faces
from paper_2007_04881_b200.mesh import agglomerate


@pytest.mark.gpu
def test_unclassified_boundary_raises_assembly_error():
    from paper_2007_04881_b200 import AssemblyError, assemble_approach2
    from paper_2007_04881_b200.assembly import SipgPlan

    pm = agglomerate(F.square_grid(4), F.square_blocks(4, 2))
    C = F.poisson_sine(2)
    specs = build_basis(pm, 1)
    with pytest.raises(AssemblyError, match="unclassified"):
        assemble_approach2(pm, C, specs)
    plan = SipgPlan(pm, C, specs)  # below the host check: the device flag
    plan.run()
    with pytest.raises(AssemblyError):
        plan.check_flags()


@pytest.mark.gpu
def test_straddling_interior_face_raises_classification_error():
    from paper_2007_04881_b200 import ClassificationError, assemble_approach2

    g = F.square_grid(3)
    pm = agglomerate(g, np.arange(g.n_simplices))
    C = M.PdeCoefficients(diffusion=M.isotropic_diffusion(1.0, 2),
                          advection=M.VectorField([M.X - 0.5, M.const(0.0)]),
                          source=M.constant_scalar(1.0), dirichlet_data=M.constant_scalar(0.0))
    classify_boundary_faces(pm, C)
    with pytest.raises(ClassificationError):
        assemble_approach2(pm, C, build_basis(pm, 1))


@pytest.mark.gpu
def test_slab_unsupported_inputs():
    from paper_2007_04881_b200 import Family
    from paper_2007_04881_b200.spacetime import assemble_slab, build_slab

    coeffs, initial = F.slab_heat()
    pm = agglomerate(F.square_grid(4), F.square_blocks(4, 2))
    slab, specs = build_slab(pm, (0.0, 0.1), np.array([1, 2, 1, 1]), Family.PQ)
    with pytest.raises(NotImplementedError):  # PQ needs a uniform degree on the device
        assemble_slab(slab, coeffs, specs, initial)
    slab, specs = build_slab(pm, (0.0, 0.1), 1, Family.PQ)
    with pytest.raises(NotImplementedError):  # opaque callable initial data
        assemble_slab(slab, coeffs, specs, lambda xy: xy[:, 0])


def test_no_cpu_fallback_without_a_gpu(monkeypatch):
    """On a host without CUDA the engine refuses instead of computing on the CPU."""
    import torch

    from paper_2007_04881_b200 import _lib, assemble_approach2

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    pm = agglomerate(F.square_grid(4), F.square_blocks(4, 2))
    C = F.poisson_sine(2)
    classify_boundary_faces(pm, C)
    with pytest.raises(_lib.EngineUnavailable):
        assemble_approach2(pm, C, build_basis(pm, 1))


@pytest.mark.gpu
def test_cuda_graph_replay_bitwise_equal_to_plain_launches():
    """The bench's CUDA-graph step (3 graph launches) reproduces the plain
    launches bit for bit."""
    from paper_2007_04881_b200.assembly import SipgPlan

    pm = agglomerate(F.square_grid(10), F.grown_clusters(F.square_grid(10), 23, seed=2))
    C = F.adr(2)
    classify_boundary_faces(pm, C)
    plan = SipgPlan(pm, C, build_basis(pm, 3))
    plan.run()
    plan.check_flags()
    v0, r0, c0 = plan.values.clone(), plan.rhs.clone(), plan.col_idx.clone()
    assert plan.capture_graphs()
    plan.t["values"].zero_()
    plan.t["rhs"].zero_()
    plan.t["col_idx"].zero_()
    for _ in range(3):
        plan.run_graphs()
    plan.check_flags()
    assert plan.graph_launches > 0
    assert bool((plan.values == v0).all()) and bool((plan.rhs == r0).all()) and bool((plan.col_idx == c0).all())
