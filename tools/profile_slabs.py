"""Warm-up + profiled native-slab Bi-CGSTAB iterations at 513^3 (for ncu launch lists).

    PROF_SLABS=2 PROF_MAXIT=4 python tools/profile_slabs.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_06085_b200 import problems  # noqa: E402
from paper_2308_06085_b200.dist import NativeSlabSolver  # noqa: E402
from paper_2308_06085_b200.krylov import SolverConfig  # noqa: E402
from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition  # noqa: E402

n = int(os.environ.get("PROF_N", 513))
ns = int(os.environ.get("PROF_SLABS", 1))
p = problems.wedge3_problem(n)
spec, b = problems.build_problem(p)
ext = slab_partition(p.grid, ns)
S = NativeSlabSolver(p.grid, ext, np.ascontiguousarray(spec.k_field), p.bc, LocalSlabComm(ns))
parts = [b[e.lo1 - 1:e.hi1] for e in ext]
_, rep = S.solve(parts, SolverConfig(method="bicgstab", tol=1e-6, maxit=int(os.environ.get("PROF_MAXIT", 4)), check_every=4))
torch.cuda.synchronize()
print("iterations", rep.iterations)
