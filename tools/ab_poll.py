"""A/B of the host poll interval of the device-resident Bi-CGSTAB (check_every)
and of the conditional-graph solve, on the bench workload (129^3), timed as
bench.py times a step (L2 flushed, CUDA events).

    python tools/ab_poll.py [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200.krylov import Solver, SolverConfig  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
p, spec, b_host = bench._problem("c1")
A = StencilOperator(spec, p.grid)
hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
solver = Solver(A, hier)
b = torch.as_tensor(b_host).cuda()
x = torch.empty_like(b)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")


def run(every):
    cfg = SolverConfig(method="bicgstab", tol=bench.TOL, maxit=400, check_every=every)
    for _ in range(3):
        solver.solve(b, cfg, x=x)
    ts = []
    for _ in range(reps):
        flush.fill_(1.0)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _, rep = solver.solve(b, cfg, x=x)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts)), rep.iterations


for rnd in range(2):
    for every in (4, 2, 8, 16, 32):
        ms, it = run(every)
        print(f"round {rnd} check_every {every:3d}: {ms:.3f} ms, {it} iterations, "
              f"{ms / it * 1e3:.1f} us per iteration", flush=True)
