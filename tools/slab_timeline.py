"""CUPTI timeline (torch.profiler) of the native slab graph at 513^3: busy vs
span per iteration and the largest gaps between consecutive GPU activities.

    PROF_SLABS=1 python tools/slab_timeline.py
"""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_06085_b200 import problems  # noqa: E402
from paper_2308_06085_b200.dist import NativeSlabSolver  # noqa: E402
from paper_2308_06085_b200.krylov import SolverConfig  # noqa: E402
from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition  # noqa: E402

n = int(os.environ.get("PROF_N", 513))
ns = int(os.environ.get("PROF_SLABS", 1))
p = problems.wedge3_problem(n)
spec, b = problems.build_problem(p)
cfg = SolverConfig(method="bicgstab", tol=1e-6, maxit=8, check_every=4)
if ns == 0:                                   # the single-slab solver, for comparison
    import bench
    A, H, S1 = bench._solver_for(p, spec)
    bd = torch.as_tensor(b).cuda()

    class _S:
        def solve(self, parts, cfg):
            return S1.solve(bd, cfg)
    S, parts = _S(), None
else:
    ext = slab_partition(p.grid, ns)
    S = NativeSlabSolver(p.grid, ext, np.ascontiguousarray(spec.k_field), p.bc, LocalSlabComm(ns))
    parts = [b[e.lo1 - 1:e.hi1] for e in ext]
S.solve(parts, cfg)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    _, rep = S.solve(parts, cfg)
    torch.cuda.synchronize()
fd, path = tempfile.mkstemp(suffix=".json")
os.close(fd)
prof.export_chrome_trace(path)
tr = json.load(open(path))
os.unlink(path)
ev = sorted((e for e in tr["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")),
            key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
busy = sum(e["dur"] for e in ev)
print(f"slabs {ns}  iterations {rep.iterations}  activities {len(ev)}  span {t1 - t0:.0f} us  busy {busy:.0f} us  "
      f"per iteration: span {(t1 - t0) / rep.iterations:.0f} us, busy {busy / rep.iterations:.0f} us, "
      f"{len(ev) / rep.iterations:.0f} activities")
import collections
agg = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    g = e.get("args", {}).get("grid")
    agg[e["name"].split("(")[0].replace("void hf::", "")[:44] + f" {tuple(g) if g else ''}"][0] += 1
    agg[e["name"].split("(")[0].replace("void hf::", "")[:44] + f" {tuple(g) if g else ''}"][1] += e["dur"]
for k_, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"  {k_:70s} n {v[0]:4d}  mean {v[1] / v[0]:9.1f} us  per iteration {v[1] / rep.iterations:9.1f} us")
gaps = []
end = ev[0]["ts"] + ev[0]["dur"]
for a, c in zip(ev, ev[1:]):
    g = c["ts"] - end
    gaps.append((g, a["name"][:50], c["name"][:50], a["dur"]))
    end = max(end, c["ts"] + c["dur"])
tot = sum(max(g[0], 0) for g in gaps)
print(f"sum of gaps {tot:.0f} us; histogram:")
for lo, hi in ((0, 2), (2, 5), (5, 10), (10, 20), (20, 50), (50, 1e9)):
    sel = [g for g in gaps if lo <= g[0] < hi]
    print(f"  gap {lo:>3}-{hi if hi < 1e9 else 'inf':>4} us: {len(sel):5d}  sum {sum(g[0] for g in sel):8.0f} us")
import collections
by = collections.defaultdict(lambda: [0, 0.0])
for g, a, c, d in gaps:
    if g > 0:
        by[(a.split('<')[0].replace('void hf::', ''), c.split('<')[0].replace('void hf::', ''))][0] += 1
        by[(a.split('<')[0].replace('void hf::', ''), c.split('<')[0].replace('void hf::', ''))][1] += g
for k_, v in sorted(by.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"  {v[1]:8.0f} us in {v[0]:4d} gaps  after {k_[0][:40]:40s} before {k_[1][:40]}")
