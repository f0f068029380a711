"""Each solve-path kernel of bench.kernel_table launched a few times on the
129^3 hierarchy (ncu target: -k regex:<kernel> -c <n>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402

p, spec, b = bench._problem()
A = StencilOperator(spec, p.grid)
H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
t = bench.kernel_table(A, H, p.grid.num_vertices, 1.0, reps=int(os.environ.get("PROF_REPS", 2)))
print({k: v["ms"] for k, v in t.items()})
