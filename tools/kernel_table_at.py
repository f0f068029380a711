"""Live CUDA-event kernel table (bench.kernel_table) on a larger cube.

    python tools/kernel_table_at.py 513 [wedge]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200 import problems  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 513
p = (problems.wedge3_problem(n) if "wedge" in sys.argv[2:]
     else problems.point_source_cube(n, 80.0 * (n - 1) / 128, "sommerfeld"))
spec, b = problems.build_problem(p)
A, H, S = bench._solver_for(p, spec)
hbm, kind = bench._peaks()
t = bench.kernel_table(A, H, S, n ** 3, 1.0)
for k, v in t.items():
    v["frac"] = round(v["gbs"] / hbm, 4)
    v.pop("share", None)
print(json.dumps({"grid": n, "medium": "wedge" if "wedge" in sys.argv[2:] else "const",
                  "peak_gbs": hbm, "kernels": t}))
