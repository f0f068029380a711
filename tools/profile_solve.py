"""Warm-up + profiled CSLP-Bi-CGSTAB solve(s) of a bench workload (for ncu).

    PROF_CONFIG=c2 PROF_MAXIT=2 PROF_SOLVES=1 python tools/profile_solve.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200.krylov import SolverConfig  # noqa: E402

from paper_2308_06085_b200 import _native  # noqa: E402

for kv in os.environ.get("HF_PROF_OPTS", "").split(","):       # e.g. HF_PROF_OPTS=no_wide=1
    if "=" in kv:
        _native.set_option(kv.split("=")[0], int(kv.split("=")[1]))
cfgname = os.environ.get("PROF_CONFIG", "c2")
p, spec, b = bench._problem(cfgname)
A, hier, S = bench._solver_for(p, spec)
bd = torch.as_tensor(b).cuda()
cfg = SolverConfig(method="bicgstab", tol=1e-6, maxit=int(os.environ.get("PROF_MAXIT", 400)))
for _ in range(int(os.environ.get("PROF_SOLVES", 2))):
    x, rep = S.solve(bd, cfg)
torch.cuda.synchronize()
print("iterations", rep.iterations, "launches", rep.kernel_launches)
