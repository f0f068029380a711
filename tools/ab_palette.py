"""A/B of the palette layout on the 513^3 wedge: alternating 40-iteration
device-timed solves with and without it (same process, same box)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200 import _native  # noqa: E402
from paper_2308_06085_b200.krylov import SolverConfig  # noqa: E402

p, spec, b_host = bench._problem("c2")
b = torch.as_tensor(b_host).cuda()
solvers = {}
for name, off in (("palette", 0), ("no_palette", 1)):
    with _native.options(no_palette=off):
        solvers[name] = bench._solver_for(p, spec)
cfg = SolverConfig(method="bicgstab", tol=1e-6, maxit=40)
res = {k: [] for k in solvers}
for rep in range(4):
    for name, (A, H, S) in solvers.items():
        x = torch.empty_like(b)
        S.solve(b, cfg, x=x)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        _, r = S.solve(b, cfg, x=x)
        s1.record()
        torch.cuda.synchronize()
        res[name].append(s0.elapsed_time(s1) / r.iterations)
for k, v in res.items():
    print(k, " ".join(f"{t:.3f}" for t in v), "ms/it; min", f"{min(v):.3f}")
