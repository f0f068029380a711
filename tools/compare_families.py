"""Converged configs[2]-type solves (three-layer wedge, seeded shadow vector) with the
wide sweep family (default) and with the tiled family (no_wide): iteration counts, final
residuals and the distance between the two solutions.

    python tools/compare_families.py [n]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200 import _native, problems  # noqa: E402
from paper_2308_06085_b200.krylov import SolverConfig  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 257
p = problems.wedge3_problem(n)
spec, b_host = problems.build_problem(p)
b = torch.as_tensor(b_host).cuda()
cfg = SolverConfig(method="bicgstab", tol=1e-8, maxit=6000, shadow="random", check_every=16)
out = {}
xs = {}
for label, opts in (("wide", {}), ("tiled", dict(no_wide=1))):
    with _native.options(**opts):
        A, H, S = bench._solver_for(p, spec)
        x, rep = S.solve(b, cfg)
        torch.cuda.synchronize()
        r = b - A.apply(x)
        out[label] = {"iterations": rep.iterations, "converged": bool(rep.converged), "final_relres": rep.final_relres,
                      "true_relres": float(torch.linalg.vector_norm(r) / torch.linalg.vector_norm(b)),
                      "solve_s": round(rep.wall_time, 3)}
        xs[label] = x.clone()
        del A, H, S
d = float(torch.linalg.vector_norm(xs["wide"] - xs["tiled"]) / torch.linalg.vector_norm(xs["tiled"]))
print(json.dumps({"grid": n, "problem": "three-layer wedge, seeded shadow, tol 1e-8", **out,
                  "rel_l2_between_solutions": d}))
