"""One warm-up + one profiled 129^3 CSLP-Bi-CGSTAB solve (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200.krylov import Solver, SolverConfig  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402

p, spec, b = bench._problem()
A = StencilOperator(spec, p.grid)
hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
S = Solver(A, hier)
bd = torch.as_tensor(b).cuda()
cfg = SolverConfig(method="bicgstab", tol=1e-6, maxit=int(os.environ.get("PROF_MAXIT", 400)))
for _ in range(int(os.environ.get("PROF_SOLVES", 2))):
    x, rep = S.solve(bd, cfg)
torch.cuda.synchronize()
print("iterations", rep.iterations, "launches", rep.kernel_launches)
