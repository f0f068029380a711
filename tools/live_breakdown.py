"""Live (un-serialised, warm-L2) per-kernel time breakdown of the 129^3 solve
through CUPTI (torch.profiler), split by launch grid (= level), plus the idle
share of the step: wall time of the solve minus the summed kernel time.

    python tools/live_breakdown.py [out.txt] [--n 129]
"""
import json
import os
import sys
import tempfile
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200 import problems  # noqa: E402
from paper_2308_06085_b200.krylov import Solver, SolverConfig  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402

n = int(sys.argv[sys.argv.index("--n") + 1]) if "--n" in sys.argv else 129
p = problems.point_source_cube(n, 80.0 * (n - 1) / 128, "sommerfeld")
spec, b = problems.build_problem(p)
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
fd, path = tempfile.mkstemp(suffix=".json")
os.close(fd)
prof.export_chrome_trace(path)
with open(path) as f:
    tr = json.load(f)
os.unlink(path)
ev = [e for e in tr["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
agg = defaultdict(lambda: [0, 0.0])
t0 = min(e["ts"] for e in ev)
t1 = max(e["ts"] + e["dur"] for e in ev)
busy = 0.0
for e in ev:
    name = e["name"].split("(")[0].replace("void ", "")[:60]
    g = e.get("args", {}).get("grid")
    key = f"{name} {tuple(g) if g else ''}"
    agg[key][0] += 1
    agg[key][1] += e["dur"]
    busy += e["dur"]
it = rep.iterations
lines = [f"grid {n}^3  iterations {it}  span {t1 - t0:.0f} us  kernel-busy {busy:.0f} us  "
         f"idle {(t1 - t0 - busy) / (t1 - t0):.1%}  per-iteration span {(t1 - t0) / it:.1f} us"]
lines.append(f"{'kernel (grid)':80s} {'n':>6s} {'mean us':>8s} {'us/iter':>8s} {'share':>6s}")
for name, (cnt, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append(f"{name[:80]:80s} {cnt:6d} {tot / cnt:8.2f} {tot / it:8.2f} {tot / busy:6.3f}")
text = "\n".join(lines)
print(text)
if len(sys.argv) > 1 and not sys.argv[1].startswith("--"):
    with open(sys.argv[1], "w") as f:
        f.write(text + "\n")
