"""Diagnostic: native vs oracle Bi-CGSTAB residual histories."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2308_06085_b200 import problems  # noqa: E402
from paper_2308_06085_b200.krylov import Solver, SolverConfig  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402

for n, kv in [(65, 40.0)]:
    p = problems.point_source_cube(n, kv, "sommerfeld")
    spec, b = problems.build_problem(p)
    k = np.full(p.grid.shape, kv)
    A = StencilOperator(spec, p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, k), MGConfig())
    S = Solver(A, hier)
    for ce in (4, 1):
        x, rep = S.solve(b, SolverConfig(method="bicgstab", tol=1e-6, maxit=400, check_every=ce))
        print("native check_every", ce, rep.iterations, rep.matvec_count)
    xo, ro = O.solve(k, b, p.grid.h, bc="sommerfeld", method="bicgstab", tol=1e-6, maxit=400)
    h, ho = np.array(rep.residual_history), np.array(ro["residual_history"])
    m = min(len(h), len(ho))
    for i in range(m):
        print(i, h[i], ho[i], abs(h[i] / ho[i] - 1))
    # same iteration through the public pieces: one manual step
