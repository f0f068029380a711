"""One launch each of the wide-plane (513^3 wedge) level kernels, for ncu:
the tiled fused down + restriction (k_down_restrict), the tiled fused up-sweep
(MODE_UP), the split presmooth+residual and the Jacobi sweep.

    ncu --set full -k regex:k_down_restrict -c 1 python tools/prof_wide.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200 import _native  # noqa: E402

n = int(os.environ.get("PROF_N", 513))
from paper_2308_06085_b200 import problems  # noqa: E402
p = problems.wedge3_problem(n)
spec, b = problems.build_problem(p)
A, H, S = bench._solver_for(p, spec)
L = _native.load()
_native.set_stream_from_torch()
sh = H.levels[0].extent.shape
csh = H.levels[1].extent.shape
r = lambda s: torch.randn(s, dtype=torch.complex128, device="cuda")
bb, u, t, bc, ec = r(sh), r(sh), r(sh), r(csh), r(csh)
for _ in range(2):
    _native.check(L.hf_level_down_restrict(H._h, 0, bb.data_ptr(), bc.data_ptr()))
    _native.check(L.hf_level_down1(H._h, 0, bb.data_ptr(), u.data_ptr()))
    _native.check(L.hf_level_smooth(H._h, 0, t.data_ptr(), bb.data_ptr(), u.data_ptr()))
    with _native.options(fuse_up=1):
        _native.check(L.hf_level_up(H._h, 0, bb.data_ptr(), ec.data_ptr(), u.data_ptr()))
torch.cuda.synchronize()
print("ok")
