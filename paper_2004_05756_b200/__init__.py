"""B200-native FE-evaluation hot path of the ROM-accelerated SIMP topology optimizer
(arXiv 2004.05756; reference package ``romtopt``).

Drop-in mirror of the reference's hot-path public API (reference __init__.py:9-49):
mesh/element definitions, the Helmholtz filter, the full-order solver and the reduced-order
model.  Compute runs in ``libtopo_b200.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/topo_b200.h``); there is no CPU fallback.
"""

from .fem import (
    IndefiniteMatrixError,
    StructuredMesh,
    assemble,
    build_mesh,
    build_mesh_3d,
    elasticity_element_matrix,
    element_mass_matrix,
    helmholtz_element_matrices,
    hex8_element_matrix,
)
from .filtering import LENGTH_SCALE_FACTOR, ConeFilter, FilterResult, HelmholtzFilter
from .hdm import (
    ComplianceObjective,
    HdmSolution,
    HdmSolver,
    MaterialModel,
    Objective,
    StaleSolutionError,
    psi_digest,
)
from ._lib import NotConvergedError
from .rom import (
    BasisMismatchError,
    DegenerateBasisError,
    ErrorReport,
    ReducedBasis,
    RomModel,
    RomSolution,
    SnapshotWindow,
    gram_schmidt,
    pod,
)
from .mma import MmaConfig, MmaOptimizer
from .stats import RunStats
from .subproblem import SubproblemResult, TrustRegionSubproblem

__version__ = "0.1.0"
