"""B200-native MG-PCG hot path of arxiv 2001.01655 (topology-optimisation
multigrid study), behind the reference package's interface (``topomg``).

Host side is Python mirroring the reference's call interface; the compute is
hand-written fp64 CUDA for sm_100a in ``lib/libtopomg_b200.so`` (C ABI declared
in ``include/topomg_b200.h``).  There is no CPU fallback: importing the compute
entry points without the built library raises ImportError.
"""

from . import _lib
from .krylov import SolveConfig, SolveRecord, cg_solve, fgmres_solve, gmres_solve, pcg_solve, solve
from .material import SimpLaw
from .mesh import (BoundaryConditions, StiffnessOperator, StructuredMesh, assemble_stiffness,
                   build_mesh, element_stiffness, rigid_body_modes)
from .multigrid import (AdaptiveHybridController, MgHierarchy, SmootherConfig, adapt_after_solve, build_gmg,
                        build_hybrid, build_sa_amg, gmg_level_dims, make_smoother, smooth)
from .optimization import SolverHarness, compliance_and_sensitivity, element_strain_energies

__version__ = "0.1.0"

__all__ = [
    "SolveConfig", "SolveRecord", "cg_solve", "pcg_solve", "solve", "gmres_solve", "fgmres_solve", "SimpLaw", "BoundaryConditions",
    "StiffnessOperator", "StructuredMesh", "assemble_stiffness", "build_mesh", "element_stiffness",
    "rigid_body_modes", "MgHierarchy", "SmootherConfig", "build_gmg", "build_hybrid", "build_sa_amg",
    "gmg_level_dims", "make_smoother", "smooth", "AdaptiveHybridController", "adapt_after_solve",
    "SolverHarness", "compliance_and_sensitivity", "element_strain_energies",
]
