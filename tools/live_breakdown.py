"""Live (un-serialised, warm-L2) per-kernel time breakdown of the 129^3 solve
through CUPTI (torch.profiler), plus the idle share of the step: wall time of
the solve minus the summed kernel time.

    python tools/live_breakdown.py [out.txt]
"""
import os
import sys
from collections import defaultdict

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
cfg = SolverConfig(method="bicgstab", tol=1e-6, maxit=400)
for _ in range(2):
    S.solve(bd, cfg)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    x, rep = S.solve(bd, cfg)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = defaultdict(lambda: [0, 0.0])
t0, t1 = min(e.time_range.start for e in ev), max(e.time_range.end for e in ev)
busy = 0.0
for e in ev:
    d = e.time_range.end - e.time_range.start
    agg[e.name][0] += 1
    agg[e.name][1] += d
    busy += d
it = rep.iterations
lines = [f"iterations {it}  span {t1 - t0:.0f} us  kernel-busy {busy:.0f} us  "
         f"idle {(t1 - t0 - busy) / (t1 - t0):.1%}  per-iteration span {(t1 - t0) / it:.1f} us"]
lines.append(f"{'kernel':90s} {'n':>6s} {'mean us':>8s} {'us/iter':>8s} {'share':>6s}")
for name, (n, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{name[:90]:90s} {n:6d} {tot / n:8.2f} {tot / it:8.2f} {tot / busy:6.3f}")
text = "\n".join(lines)
print(text)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        f.write(text + "\n")
