"""paper_2308_06085_b200: B200-native matrix-free CSLP-preconditioned Krylov
solver for the 3D heterogeneous Helmholtz equation.

Drop-in for the operator / preconditioner / solve entry points of the
reference package `helmfree` (arxiv 2308.06085).  The compute path is the
native library paper_2308_06085_b200/_lib/libhelmfree_b200.so (sm_100a);
there is no CPU fallback.
"""

from .grid import (BlockExtent, Grid3, HaloField, coarsen, full_extent, make_grid)
from .operators import (Dirichlet, OperatorSpec, Sommerfeld, StencilOperator, apply_operator)
from .multigrid import MGConfig, build_hierarchy, mg_precondition
from .krylov import ConvergenceReport, SolverConfig, Solver, run_solver

__version__ = "0.1.0"

__all__ = ["BlockExtent", "Grid3", "HaloField", "coarsen", "full_extent", "make_grid",
           "Dirichlet", "OperatorSpec", "Sommerfeld", "StencilOperator", "apply_operator",
           "MGConfig", "build_hierarchy", "mg_precondition", "ConvergenceReport",
           "SolverConfig", "Solver", "run_solver"]
