"""Virtual slabs on one GPU (LOCAL transport): ms per Bi-CGSTAB iteration of the
native slab graph at 513^3 for 1 / 2 / 4 / 8 slabs of the decomposition, all in
one process -- the per-GPU kernels of an N-GPU run launched back to back (no
NVLink, no concurrency: an upper bound of N x the per-rank compute time, and a
check that the slab path's sub-slab launches cost little against the
single-slab solver).

    python tools/ab_slabs.py [n] [option=1,...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2308_06085_b200 import _native, problems  # noqa: E402
from paper_2308_06085_b200.dist import NativeSlabSolver  # noqa: E402
from paper_2308_06085_b200.krylov import SolverConfig  # noqa: E402
from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
opts = {kv.split("=")[0]: int(kv.split("=")[1]) for kv in (sys.argv[2] if len(sys.argv) > 2 else "").split(",") if "=" in kv}
p = problems.wedge3_problem(n)
spec, b = problems.build_problem(p)
k = np.ascontiguousarray(spec.k_field)
iters = 24
with _native.options(**opts):
    for ns in (1, 2, 4, 8):
        ext = slab_partition(p.grid, ns)
        S = NativeSlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(ns))
        parts = [torch.as_tensor(np.ascontiguousarray(b[e.lo1 - 1:e.hi1])).cuda() for e in ext]   # resident
        cfg = SolverConfig(method="bicgstab", tol=1e-6, maxit=iters, check_every=4)
        S.solve(parts, cfg)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _, rep = S.solve(parts, cfg)
        e.record()
        torch.cuda.synchronize()
        print(json.dumps({"grid": n, "slabs": ns, "options": opts, "iterations": rep.iterations,
                          "ms_per_iteration": round(s.elapsed_time(e) / rep.iterations, 3),
                          "relres": rep.final_relres}), flush=True)
        del S
        torch.cuda.empty_cache()
