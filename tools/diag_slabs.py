"""Diagnostic: slab pieces vs single-slab native results."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2308_06085_b200 import _native, problems  # noqa: E402
from paper_2308_06085_b200.dist import SlabSolver  # noqa: E402
from paper_2308_06085_b200.grid import HaloField  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator  # noqa: E402
from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition  # noqa: E402

p = problems.point_source_cube(65, 40.0, "sommerfeld")
spec, b = problems.build_problem(p)
k = np.full(p.grid.shape, 40.0)
A = StencilOperator(spec, p.grid)
H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, k), MGConfig())
ext = slab_partition(p.grid, 2)
S = SlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(2))
rng = np.random.default_rng(0)
u = rng.standard_normal(p.grid.shape) + 1j * rng.standard_normal(p.grid.shape)
ud = torch.as_tensor(u).cuda()
src = [HaloField(e) for e in ext]
for f, e in zip(src, ext):
    f.owned.copy_(ud[e.lo1 - 1:e.hi1])
rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())
# apply
v1 = A.apply(ud).cpu().numpy()
vs = [torch.empty(e.shape, dtype=torch.complex128, device="cuda") for e in ext]
S.apply_A(src, vs)
print("apply", rel(np.concatenate([x.cpu().numpy() for x in vs]), v1))
# per-level down1 on level 0
L = _native.load()
r1 = torch.empty_like(ud)
_native.check(L.hf_level_down1(H._h, 0, ud.data_ptr(), r1.data_ptr()))
S._halo(src)
rs = []
for i, e in enumerate(ext):
    out = torch.empty(e.shape, dtype=torch.complex128, device="cuda")
    _native.check(L.hf_level_down1(S.H[i], 0, src[i].owned.data_ptr(), out.data_ptr()))
    rs.append(out.cpu().numpy())
print("down1 L0", rel(np.concatenate(rs), r1.cpu().numpy()))
for i in range(2):
    e = ext[i]
    print("  slab", i, rel(rs[i], r1.cpu().numpy()[e.lo1 - 1:e.hi1]))
# full cycle
z1 = mg_precondition(H, ud).cpu().numpy()
dst = [HaloField(e) for e in ext]
S.precondition(src, dst)
zs = np.concatenate([d.owned.cpu().numpy() for d in dst])
print("cycle", rel(zs, z1))
for i in range(2):
    e = ext[i]
    d = np.abs(zs[e.lo1 - 1:e.hi1] - z1[e.lo1 - 1:e.hi1]).max(axis=(1, 2))
    print("  slab", i, "max err per plane (first/last 3):", d[:3], d[-3:])
print("levels", [[ (lv.lo1, lv.hi1) for lv in S.levels[r]] for r in range(2)])
