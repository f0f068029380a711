"""One launch each of the 513^3 wedge finest-level kernels the solve runs, in
the order of tools/gpu_evidence3.sh's kernel list (pre-smoothing + residual
sweep, restriction, fused up-sweep, matvec, matvec with t^H t / t^H s, the
Bi-CGSTAB p / s / x,r updates, then the split correction + Jacobi pair of the
slab path), for ncu --set full."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2308_06085_b200 import _native, problems  # noqa: E402

for kv in os.environ.get("HF_PROF_OPTS", "").split(","):       # e.g. HF_PROF_OPTS=wide_p2=1,no_wide=0
    if "=" in kv:
        _native.set_option(kv.split("=")[0], int(kv.split("=")[1]))
p = problems.wedge3_problem(int(os.environ.get("PROF_N", 513)))
spec, b = problems.build_problem(p)
A, H, S = bench._solver_for(p, spec)
L = _native.load()
_native.set_stream_from_torch()
sh, csh = H.levels[0].extent.shape, H.levels[1].extent.shape
r = lambda s: torch.randn(s, dtype=torch.complex128, device="cuda")
bb, u, t, bc, ec = r(sh), r(sh), r(sh), r(csh), r(csh)
ms = ctypes.c_float()
A_h = A._h
for _ in range(int(os.environ.get("PROF_PASSES", 2))):
    _native.check(L.hf_level_down1(H._h, 0, bb.data_ptr(), u.data_ptr()))             # presmooth_residual
    _native.check(L.hf_restrict_fw(H._h, 0, u.data_ptr(), bc.data_ptr()))             # restrict_fw
    _native.check(L.hf_level_up(H._h, 0, bb.data_ptr(), ec.data_ptr(), u.data_ptr())) # up_fused
    _native.check(L.hf_operator_apply(A_h, u.data_ptr(), t.data_ptr()))               # helmholtz_matvec
    _native.check(L.hf_solver_bench_vec(S._h, 4, 1, ctypes.byref(ms)))                # matvec_dot2
    _native.check(L.hf_solver_bench_vec(S._h, 0, 1, ctypes.byref(ms)))                # bcg_p_update
    _native.check(L.hf_solver_bench_vec(S._h, 1, 1, ctypes.byref(ms)))                # bcg_s_update
    _native.check(L.hf_solver_bench_vec(S._h, 3, 1, ctypes.byref(ms)))                # bcg_xr_update (sparse)
    # the split up-sweep pair (slab path)
    _native.check(L.hf_level_correct(H._h, 0, bb.data_ptr(), ec.data_ptr(), t.data_ptr()))
    _native.check(L.hf_level_smooth(H._h, 0, t.data_ptr(), bb.data_ptr(), u.data_ptr()))
torch.cuda.synchronize()
print("ok")
