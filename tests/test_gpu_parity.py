"""GPU parity: the CUDA engine (through libpdg.so) against the CPU oracle.

Indices bit-exact, values <= 1e-12 relative in max-norm per block, RHS
<= 1e-12 relative per element.  Every case runs the full
device path: index phase, face pre-pass, fused element kernel.
"""

import numpy as np
import pytest

import fixtures as F
from compare import REL_TOL, assert_parity
from oracle import sipg as oracle
from paper_2007_04881_b200 import (
    AssemblyConfig,
    PenaltyConfig,
    assemble_approach2,
    assemble_device,
    build_basis,
    build_block_pattern,
    classify_boundary_faces,
    element_kernel,
)
from paper_2007_04881_b200.mesh import agglomerate, identity_agglomeration

pytestmark = pytest.mark.gpu


def _run(pm, coeffs, p, predicate=None, config=None):
    classify_boundary_faces(pm, coeffs, predicate)
    specs = build_basis(pm, p)
    cfg = config or AssemblyConfig()
    m, rhs, stats, pattern = assemble_approach2(pm, coeffs, specs, cfg)
    ref = oracle.assemble(pm, coeffs, specs, cfg.quad_increment, cfg.penalty.constant,
                          cfg.penalty.coverable)
    be, re = assert_parity(m, rhs, ref, pattern.dof_map.offsets)
    return m, rhs, stats, be, re


def _mesh(name):
    if name == "blocks8":
        return agglomerate(F.square_grid(8), F.square_blocks(8, 2))
    if name == "clusters6":
        g = F.square_grid(6)
        return agglomerate(g, F.grown_clusters(g, 7, seed=1))
    if name == "zigzag":
        return F.zigzag(3)
    if name == "cube":
        return agglomerate(F.cube_grid(2), F.cube_blocks(2, 2))
    if name == "identity4":
        return identity_agglomeration(F.square_grid(4))
    if name == "clusters10":
        g = F.square_grid(10)
        return agglomerate(g, F.grown_clusters(g, 23, seed=2))
    if name == "cube3":
        g = F.cube_grid(3)
        return agglomerate(g, F.grown_clusters(g, 11, seed=3))
    raise KeyError(name)


@pytest.mark.parametrize("name,p", [("blocks8", 1), ("clusters6", 2), ("zigzag", 2), ("cube", 1),
                                    ("identity4", 1), ("cube3", 2), ("clusters10", 3)])
def test_cross_oracle_generic(name, p):
    """The reference suite's cross-oracle cases (test_assembly.py:349-389)."""
    pm = _mesh(name)
    _run(pm, F.generic(pm.dim), p)


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4, 5, 6])
def test_poisson_degrees_2d(p):
    pm = _mesh("clusters10")
    _run(pm, F.poisson_sine(2), p)


@pytest.mark.parametrize("p", [0, 1, 2, 3, 4])
def test_poisson_degrees_3d(p):
    pm = _mesh("cube3")
    _run(pm, F.poisson_sine(3), p)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_variable_diffusion(p):
    _run(_mesh("clusters10"), F.variable_diffusion(2), p)


@pytest.mark.parametrize("name,p", [("clusters10", 2), ("clusters10", 3), ("clusters10", 4), ("clusters10", 5),
                                    ("clusters10", 6), ("cube3", 2), ("cube3", 3), ("cube3", 4)])
def test_advection_diffusion_reaction(name, p):
    """Upwinded faces (assembly.py:455-462) at every degree of the cfg3 sweep (2D)
    and up to the compiled 3D maximum."""
    pm = _mesh(name)
    _run(pm, F.adr(pm.dim), p)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6])
def test_sine_dirichlet_data_2d(p):
    """Dirichlet data that vanishes on the boundary only up to sin(fl(pi)):
    the face fields must be evaluated as the reference does (no sinpi)."""
    _run(_mesh("clusters10"), F.sine_dirichlet(2), p)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_reference_advdiff3d_problem(p):
    """polydg's own advection_diffusion_3d_problem (model.py:312-358)."""
    _run(_mesh("cube3"), F.advdiff3d(3), p)


@pytest.mark.parametrize("name,p", [("clusters10", 2), ("cube3", 1)])
def test_anisotropic_tensor_with_neumann(name, p):
    pm = _mesh(name)
    # Dirichlet on the x < 0.5 half of the boundary, Neumann elsewhere
    _run(pm, F.anisotropic(pm.dim), p, predicate=lambda x: x[0] < 0.5)


@pytest.mark.parametrize("name,p", [("clusters10", 2), ("clusters10", 3), ("cube3", 1), ("cube3", 2)])
def test_hyperbolic_inflow_outflow(name, p):
    pm = _mesh(name)
    _run(pm, F.hyperbolic(pm.dim), p)


def test_sign_changing_diffusion_reruns_plain_volume():
    """a(x) < 0 somewhere: the sqrt(w a) volume table cannot hold it, the
    device flags it and the plan re-runs the plain variant (same result)."""
    import paper_2007_04881_b200.model as M

    coeffs = M.PdeCoefficients(diffusion=M.scalar_diffusion(F.X - 0.3, 2), source=M.constant_scalar(1.0),
                               dirichlet_data=M.constant_scalar(0.0))
    _run(_mesh("clusters10"), coeffs, 3)


@pytest.mark.parametrize("env", [{"PDG_JIT": "0"}, {"PDG_PLAIN_VOLUME": "1"},
                                 {"PDG_JIT": "0", "PDG_PLAIN_VOLUME": "1"},
                                 {"PDG_JIT_DEFINES": "-DPDG_BULK=1"},
                                 {"PDG_JIT_MINBLOCKS": "1"},
                                 {"PDG_JIT_DEFINES": "-DPDG_PAD_ZERO=1 -DPDG_VOL_FULL=0 -DPDG_REG_CAPPED=0"}])
@pytest.mark.parametrize("case", ["vardiff", "adr", "aniso3d"])
def test_kernel_variants(monkeypatch, env, case):
    """The ahead-of-time (bytecode-interpreted) kernels, the plain volume
    variant, the opt-in bulk-copy (TMA) staging, the wide-register build and
    the padding / unrolling switches match the oracle like the default
    NVRTC-specialised kernel."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    if case == "vardiff":
        _run(_mesh("clusters10"), F.variable_diffusion(2), 3)
    elif case == "adr":
        _run(_mesh("clusters10"), F.adr(2), 2)
    else:
        pm = _mesh("cube3")
        _run(pm, F.anisotropic(3), 1, predicate=lambda x: x[0] < 0.5)


def test_variable_degree():
    """Per-element degrees (reference test_assembly.py:440-450)."""
    pm = agglomerate(F.square_grid(4), F.square_blocks(4, 2))
    coeffs = F.generic(2)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, np.array([1, 2, 2, 3]))
    m, rhs, _, pattern = assemble_approach2(pm, coeffs, specs)
    ref = oracle.assemble(pm, coeffs, specs)
    assert_parity(m, rhs, ref, pattern.dof_map.offsets)


def test_coverable_penalty_and_constant():
    pm = _mesh("clusters10")
    cov = np.zeros(pm.n_elements, bool)
    cov[::2] = True
    cfg = AssemblyConfig(quad_increment=3, penalty=PenaltyConfig(constant=7.5, coverable=cov))
    _run(pm, F.variable_diffusion(2), 2, config=cfg)


def test_partition_rows_bit_identical_to_monolithic():
    """Row-partitioned assembly (one-sided cut faces) reproduces the
    monolithic rows bit for bit."""
    pm = _mesh("clusters10")
    coeffs = F.adr(2)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 3)
    full = assemble_device(pm, coeffs, specs)
    vals = full.values.cpu().numpy()
    rp = full.row_ptr.cpu().numpy()
    rhs = full.rhs.cpu().numpy()
    off = full.plan.dof.offsets
    rng = np.random.default_rng(0)
    part_of = rng.integers(0, 3, pm.n_elements)
    for part in range(3):
        own = np.flatnonzero(part_of == part)
        res = assemble_device(pm, coeffs, specs, row_elements=own)
        prp = res.row_ptr.cpu().numpy()
        pv = res.values.cpu().numpy()
        prhs = res.rhs.cpu().numpy()
        r = 0
        for e in own:
            ne = off[e + 1] - off[e]
            g0 = off[e]
            a, b = rp[g0], rp[g0 + ne]
            assert np.array_equal(pv[prp[r]:prp[r + ne]], vals[a:b])
            assert np.array_equal(prhs[g0:g0 + ne], rhs[g0:g0 + ne])
            r += ne


@pytest.mark.parametrize("n_parts", [2, 5])
def test_assemble_partition_and_gather_equal_monolithic(n_parts):
    """polydg's partition API end to end (distribute.py:200-276): every part's
    sub-mesh assembly (owned + halo, global columns) stacked by
    gather_and_verify / gather_load == assemble_approach2, bit for bit."""
    from paper_2007_04881_b200 import (assemble_partition, contiguous_partition, gather_and_verify, gather_load,
                                       quadrature_cost_weights)

    pm = _mesh("clusters10")
    coeffs = F.adr(2)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 3)
    m, rhs, _, pattern = assemble_approach2(pm, coeffs, specs)
    part = contiguous_partition(pm, n_parts, quadrature_cost_weights(pm, specs))
    partials, loads = [], []
    for r in range(n_parts):
        pmat, load, stats = assemble_partition(pm, part, r, coeffs, specs)
        assert pmat.matrix.n_cols == m.n_cols
        assert stats.kernel_wall_seconds > 0
        partials.append(pmat)
        loads.append(load)
    full = gather_and_verify(partials, pattern.dof_map.n_dofs)
    assert np.array_equal(full.row_ptr, m.row_ptr)
    assert np.array_equal(full.col_idx, m.col_idx)
    assert np.array_equal(full.values, m.values)
    assert np.array_equal(gather_load(loads, partials, pattern.dof_map.n_dofs), rhs)


def test_stats_rows_sum_to_the_kernel_time():
    """AssemblyStats (assembly.py:360-391): index = index phase, kernel wall =
    the fused kernel, per-kernel rows apportioned and summing to it."""
    pm = _mesh("clusters10")
    coeffs = F.anisotropic(2)
    classify_boundary_faces(pm, coeffs, lambda x: x[0] < 0.5)
    specs = build_basis(pm, 2)
    _, _, stats, _ = assemble_approach2(pm, coeffs, specs)
    tot = sum(k.seconds for k in stats.kernels.values())
    assert abs(tot - stats.kernel_wall_seconds) <= 1e-9 + 1e-9 * tot
    assert stats.kernels["element"].seconds > 0 and stats.kernels["interior"].seconds > 0
    assert stats.kernels["dirichlet"].seconds > 0 and stats.kernels["neumann_outflow"].seconds > 0
    assert abs(stats.kernel_wall_seconds - stats.device_ms["element"] * 1e-3) < 1e-12
    assert stats.index_seconds > 0 and stats.total_seconds >= stats.kernel_wall_seconds
    assert "apportioned" in stats.kernel_split
    assert stats.to_csv().count("\n") == 8


def test_bitwise_determinism():
    pm = _mesh("cube3")
    coeffs = F.adr(3)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 2)
    a = assemble_device(pm, coeffs, specs)
    va, ra = a.values.cpu().numpy().copy(), a.rhs.cpu().numpy().copy()
    b = assemble_device(pm, coeffs, specs)
    assert np.array_equal(va, b.values.cpu().numpy())
    assert np.array_equal(ra, b.rhs.cpu().numpy())


def test_block_pattern_matches_oracle():
    pm = _mesh("clusters10")
    degrees = 1 + (np.arange(pm.n_elements) % 3)
    specs = build_basis(pm, degrees)
    pat = build_block_pattern(pm, specs)
    off = pat.dof_map.offsets
    rp, ci, _ = oracle.block_pattern(off, [(i.owner, i.neighbor) for i in pm.interfaces],
                                     np.arange(pm.n_elements))
    assert np.array_equal(pat.row_ptr, rp)
    assert np.array_equal(pat.col_idx, ci)
    rows = np.array([3, 7, 11])
    sub = build_block_pattern(pm, specs, row_elements=rows)
    rp2, ci2, _ = oracle.block_pattern(off, [(i.owner, i.neighbor) for i in pm.interfaces], rows)
    assert np.array_equal(sub.row_ptr, rp2)
    assert np.array_equal(sub.col_idx, ci2)


@pytest.mark.parametrize("p", [0, 1, 2, 3])
def test_element_kernel_unit(p):
    pm = _mesh("clusters6")
    coeffs = F.adr(2)
    specs = build_basis(pm, p)
    for e in (0, 3, 6):
        K, f = element_kernel(pm, e, coeffs, specs[e])
        Kr, fr = oracle.element_kernel(pm, e, coeffs, specs[e])
        assert np.abs(K - Kr).max() <= REL_TOL * np.abs(Kr).max()
        assert np.abs(f - fr).max() <= REL_TOL * max(np.abs(fr).max(), 1e-300)


def test_element_kernel_mass_identity_on_box():
    """reference test_assembly.py:64-69: mass = I on a box-filling element."""
    pm = F.one_square()
    coeffs = F.M.PdeCoefficients(reaction=F.M.constant_scalar(1.0))
    for p in range(4):
        spec = build_basis(pm, p)[0]
        K, _ = element_kernel(pm, 0, coeffs, spec)
        np.testing.assert_allclose(K, np.eye(spec.n_funcs), atol=1e-12)


def test_pinned_chunked_download_and_block_slots_on_assembled_matrix():
    """download() (pinned double-buffered D2H into numpy) is exact for odd
    chunkings; the pattern's block_slots address the assembled values."""
    import torch

    from paper_2007_04881_b200.assembly import download

    t = torch.randn(3_000_001, dtype=torch.float64, device="cuda")
    for ch in (1 << 20, 3 << 19, 1 << 30):
        assert np.array_equal(download(t, chunk_bytes=ch), t.cpu().numpy())
    ti = torch.randint(0, 1 << 40, (2_500_003,), dtype=torch.int64, device="cuda")
    assert np.array_equal(download(ti, chunk_bytes=1 << 20), ti.cpu().numpy())
    pm = _mesh("clusters10")
    coeffs = F.generic(2)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 2)
    m, _, _, pattern = assemble_approach2(pm, coeffs, specs)
    dense = m.to_dense()
    off = pattern.dof_map.offsets
    for k, e in enumerate(pattern.row_elements[:12]):
        for j in pattern.neighbors[k]:
            sl = pattern.block_slots(int(e), int(j))
            assert np.array_equal(m.values[sl], dense[off[e]:off[e + 1], off[j]:off[j + 1]])


def test_hostio_retained_host_csr_matches_assembly():
    """HostIO (the bench's e2e leg): uploads the mesh, downloads into
    page-locked host arrays, and result() is the assembled CSR + RHS; close()
    drops them (result raises; arrays the caller kept stay valid)."""
    import torch

    from paper_2007_04881_b200.assembly import AssemblyError, HostIO, SipgPlan

    pm = _mesh("clusters10")
    coeffs = F.generic(2)
    classify_boundary_faces(pm, coeffs)
    specs = build_basis(pm, 3)
    m, rhs, _, _ = assemble_approach2(pm, coeffs, specs)
    plan = SipgPlan(pm, coeffs, specs)
    io = HostIO(plan, compact_cols=True)  # (auto mode packs only CSRs of >= 256 MB)
    assert io.retained
    for _ in range(2):
        io.upload()
        plan.run()
        io.download()
    torch.cuda.synchronize()
    mh, rh = io.result()
    assert mh.n_rows == m.n_rows and mh.n_cols == m.n_cols
    assert np.array_equal(mh.row_ptr, m.row_ptr) and np.array_equal(mh.col_idx, m.col_idx)
    assert np.array_equal(mh.values, m.values) and np.array_equal(rh, rhs)
    io.close()
    with pytest.raises(AssemblyError):
        io.result()
    # the page-locked memory lives as long as a view of it
    assert np.array_equal(mh.values, m.values) and np.array_equal(rh, rhs)
    del mh, rh
    full = HostIO(plan, compact_cols=False)  # every row of col_idx over the link
    full.upload(); plan.run(); full.download()
    torch.cuda.synchronize()
    mf, rf = full.result()
    assert np.array_equal(mf.col_idx, m.col_idx) and np.array_equal(mf.values, m.values)
    assert full.d2h_bytes > io.d2h_bytes
    del mf, rf
    full.close()
    ring = HostIO(plan, retain=False)
    assert not ring.retained
    ring.upload(); plan.run(); ring.download()
    torch.cuda.synchronize()
