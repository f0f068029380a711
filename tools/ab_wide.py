"""A/B of the wide-plane sweep family (hf_wide.cu) against the tiled k_stencil
kernels on the finest level of the 513^3 wedge: live CUDA-event kernel table
per variant.

    python tools/ab_wide.py [n] [const]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import bench  # noqa: E402
from paper_2308_06085_b200 import _native, problems  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
const = "const" in sys.argv[2:]
p = problems.point_source_cube(n, 80.0 * (n - 1) / 128, "sommerfeld") if const else problems.wedge3_problem(n)
spec, b = problems.build_problem(p)
hbm, _ = bench._peaks()
names = ("helmholtz_matvec", "jacobi_postsmooth", "presmooth_residual")
for label, opts in (("tiled", dict(no_wide=1)), ("wide_p2", {}), ("wide_p4", dict(wide_p4=1))):
    with _native.options(**opts):
        A, H, S = bench._solver_for(p, spec)
        t = bench.kernel_table(A, H, S, n ** 3, 1.0)
    print(json.dumps({"variant": label, "grid": n, "medium": "const" if const else "wedge",
                      **{k: {"ms": t[k]["ms"], "frac": round(t[k]["gbs"] / hbm, 3)} for k in names if k in t}}))
    del A, H, S
