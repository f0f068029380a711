"""A/B of kernel-variant option sets on the bench workload: ms per Bi-CGSTAB
iteration of the 513^3 wedge (fixed budget of 50 iterations, 3 timed solves
after 1 warm-up), every variant in one process on one box.  AB_N sets the grid
side, AB_MEDIUM the medium (wedge | const | random: n x n x (n+1)/2).

    python tools/ab_iter.py "no_wide=1" "" "wide_p4=1"
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200 import _native  # noqa: E402
from paper_2308_06085_b200.krylov import SolverConfig  # noqa: E402

n = int(os.environ.get("AB_N", 513))
iters = int(os.environ.get("AB_ITERS", 50))
medium = os.environ.get("AB_MEDIUM", "wedge")     # wedge | const | random
from paper_2308_06085_b200 import problems  # noqa: E402
if medium == "const":
    p = problems.point_source_cube(n, 80.0 * (n - 1) / 128, "sommerfeld")
elif medium == "random":
    p = problems.random_medium_problem((n, n, (n + 1) // 2))
else:
    p = problems.wedge3_problem(n)
spec, b_host = problems.build_problem(p)
b = torch.as_tensor(b_host).cuda()
x = torch.empty_like(b)
cfg = SolverConfig(method="bicgstab", tol=1e-6, maxit=iters, check_every=4)
for variant in sys.argv[1:] or [""]:
    opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in variant.split(",") if "=" in kv}
    with _native.options(**opts):
        A, H, S = bench._solver_for(p, spec)
        S.solve(b, cfg, x=x)
        ms = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            _, rep = S.solve(b, cfg, x=x)
            e.record()
            torch.cuda.synchronize()
            ms.append(s.elapsed_time(e) / rep.iterations)
        print(json.dumps({"variant": variant or "default", "grid": list(p.grid.shape), "medium": medium, "ms_per_iteration": [round(m, 3) for m in ms],
                          "iterations": rep.iterations, "relres": rep.final_relres}), flush=True)
        del A, H, S
    torch.cuda.empty_cache()
