"""A few V-cycles of the 129^3 hierarchy (ncu target for the cycle kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec  # noqa: E402

p, spec, b = bench._problem()
H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
r = torch.as_tensor(b).cuda()
z = torch.empty_like(r)
for _ in range(int(os.environ.get("PROF_CYCLES", 3))):
    mg_precondition(H, r, out=z)
torch.cuda.synchronize()
print("ok")
