"""B200-native fp64 SIPG assembly on polytopic meshes (arXiv 2007.04881).

Drop-in for polydg's Approach-2 assembly path: same entry points and
containers, computed by hand-written sm_100a kernels in ``libpdg.so``
(C ABI: ``include/pdg.h``).  See DESIGN.md.
"""

from .basis import BasisSpec, Family, SpecList, build_basis, num_basis
from .mesh import (
    BOUNDARY,
    BoundaryTag,
    FlatMesh,
    MeshError,
    PolytopicMesh,
    SimplicialMesh,
    agglomerate,
    identity_agglomeration,
)
from .model import (
    ClassificationError,
    PdeCoefficients,
    PenaltyConfig,
    PenaltySideData,
    ScalarField,
    TensorField,
    VectorField,
    classify_boundary_faces,
    constant_scalar,
    constant_tensor,
    constant_vector,
    isotropic_diffusion,
    penalty_side_data,
    penalty_sigma,
    scalar_diffusion,
)
from .quadrature import QuadratureError
from .assembly import (
    AssemblyConfig,
    AssemblyError,
    AssemblyStats,
    BlockPattern,
    CSRMatrix,
    DofMap,
    KernelTiming,
    PatternMissError,
    SipgPlan,
    assemble_approach1,
    assemble_approach2,
    assemble_device,
    build_block_pattern,
    dirichlet_kernel,
    element_kernel,
    inflow_kernel,
    interior_face_kernel,
    neumann_outflow_kernel,
    triplets_to_csr,
)
from .kernels import eval_coefficients, face_sigma, map_simplices, tabulate
from .distribute import (
    PartialMatrix,
    Partition,
    PartitionError,
    assemble_partition,
    contiguous_partition,
    gather_and_verify,
    gather_load,
    partition_from_map,
    quadrature_cost_weights,
)

from .spacetime import (
    ParabolicProblem,
    SlabMesh,
    SlabPlan,
    TimePartition,
    assemble_slab,
    build_slab,
    load_solution_vector,
    march,
    save_solution_vector,
)
from .solver import SolveResult, SolverError, read_matrix_market, solve, write_matrix_market

__all__ = [n for n in dir() if not n.startswith("_")]
__version__ = "0.1.0"
