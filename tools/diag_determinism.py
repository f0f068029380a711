"""Run the same solves several times; iteration counts and solutions must be
bit-identical (deterministic reductions, no races)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06085_b200 import problems  # noqa: E402
from paper_2308_06085_b200.krylov import Solver, SolverConfig  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402

for n, kv in [(65, 40.0), (129, 80.0)]:
    p = problems.point_source_cube(n, kv, "sommerfeld")
    spec, b = problems.build_problem(p)
    A = StencilOperator(spec, p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
    S = Solver(A, hier)
    ref = None
    for t in range(4):
        x, rep = S.solve(b, SolverConfig(method="bicgstab", tol=1e-6, maxit=400, check_every=1 + t))
        x = x.cpu().numpy()
        same = ref is None or np.array_equal(x, ref)
        ref = x if ref is None else ref
        print(n, "run", t, "iterations", rep.iterations, "bitwise-identical", same, flush=True)
