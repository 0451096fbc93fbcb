"""B200-native tangent-stiffness assembly for the epfem reference
(arXiv:1805.04155 elastoplastic FEM): constitutive update + K = B^T W D B into
a fixed CSR pattern, hand-written CUDA for sm_100a behind a C-ABI
(include/epfem_gpu.h).  See DESIGN.md.
"""
from .api import (  # noqa: F401
    AssemblyCache, Context, CsrMatrix, DPMode, DruckerPragerEval, DruckerPragerParams,
    ElasticEval, Error, IntegrationState, MaterialField, Mesh, TangentEngine, VonMisesEval,
    VonMisesParams, assemble_elastic_stiffness, assemble_tangent_packed,
    assemble_tangent_stiffness, build_assembly_cache, constitutive_dp, constitutive_elastic,
    constitutive_vm, default_context, dp_parameters, elastic_moduli, evaluate_constitutive,
    internal_forces, unpack_D, uniform_drucker_prager, uniform_elastic, uniform_von_mises,
)
from .mesh import ElementType, StructuredMesh, structured_mesh  # noqa: F401
from .solver import (  # noqa: F401
    LinearSolver, NewtonResult, NewtonSettings, NonConvergenceError, SolveInfo, SolveSettings, SolverError,
    energy_norm, newton_solve, restricted_solve,
)
