"""Multi-slab path on one GPU (virtual ranks over LocalSlabComm): every slab
runs the native kernels on its own planes with ghost planes filled by the
halo exchange; the coarsest level is gathered.  Results must match the
single-slab native solve (reduction order is the only difference)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _single(p, k):
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    spec, b = problems.build_problem(p)
    A = StencilOperator(spec, p.grid)
    H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, k), MGConfig())
    x, rep = Solver(A, H).solve(b, SolverConfig(method="bicgstab"))
    return b, x.cpu().numpy(), rep, H


def _slabs(p, k, b, nslabs):
    from paper_2308_06085_b200.dist import SlabSolver
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    ext = slab_partition(p.grid, nslabs)
    S = SlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(nslabs))
    xs, rep = S.solve([b[e.lo1 - 1:e.hi1] for e in ext])
    return np.concatenate([x.cpu().numpy() for x in xs], 0), rep, S, ext


@pytest.mark.parametrize("nslabs", [2, 3])
def test_slab_bicgstab_matches_single(nslabs):
    from paper_2308_06085_b200 import problems
    p = problems.point_source_cube(65, 40.0, "sommerfeld")
    k = np.full(p.grid.shape, 40.0)
    b, x1, r1, _ = _single(p, k)
    xs, rs, _, _ = _slabs(p, k, b, nslabs)
    assert rs.converged and abs(rs.iterations - r1.iterations) <= 1
    assert np.linalg.norm(xs - x1) / np.linalg.norm(x1) < 1e-8


def test_slab_precondition_matches_single_heterogeneous():
    """Varying medium (staged D^-1 ghost planes), 4 slabs, one V-cycle."""
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.grid import HaloField, full_extent
    from paper_2308_06085_b200.multigrid import mg_precondition
    p = problems.wedge3_problem(65)
    k = p.medium.k_field(p.grid, full_extent(p.grid))
    b, x1, r1, H = _single(p, k)
    from paper_2308_06085_b200.dist import SlabSolver
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    ext = slab_partition(p.grid, 4)
    S = SlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(4))
    rng = np.random.default_rng(3)
    r = rng.standard_normal(p.grid.shape) + 1j * rng.standard_normal(p.grid.shape)
    z1 = mg_precondition(H, r).cpu().numpy()
    src = [HaloField(e) for e in ext]
    dst = [HaloField(e) for e in ext]
    for f, e in zip(src, ext):
        f.owned.copy_(torch.as_tensor(r[e.lo1 - 1:e.hi1]))
    S.precondition(src, dst)
    zs = np.concatenate([d.owned.cpu().numpy() for d in dst], 0)
    assert np.abs(zs - z1).max() / np.abs(z1).max() < 1e-12
    xs, rs, _, _ = _slabs(p, k, b, 4)
    assert rs.converged and abs(rs.iterations - r1.iterations) <= 1
    assert np.linalg.norm(xs - x1) / np.linalg.norm(x1) < 1e-8


@pytest.mark.parametrize("nslabs", [1, 2, 3])
def test_slab_device_bicgstab_matches_single(nslabs):
    """Device-resident slab Bi-CGSTAB (hf_bcg_*: scalars on the device, partial
    sums added over slabs) against the single-slab graph solve."""
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.dist import SlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    p = problems.point_source_cube(65, 40.0, "sommerfeld")
    k = np.full(p.grid.shape, 40.0)
    b, x1, r1, _ = _single(p, k)
    ext = slab_partition(p.grid, nslabs)
    S = SlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(nslabs))
    xs, rs = S.solve_device([b[e.lo1 - 1:e.hi1] for e in ext], SolverConfig(method="bicgstab"))
    xs = np.concatenate([x.cpu().numpy() for x in xs], 0)
    assert rs.converged and abs(rs.iterations - r1.iterations) <= 1, (rs.iterations, r1.iterations)
    assert np.linalg.norm(xs - x1) / np.linalg.norm(x1) < 1e-8
    assert len(rs.residual_history) == rs.iterations


_NCCL_CHILD = r'''
import os, sys, json
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2308_06085_b200 import problems
from paper_2308_06085_b200.dist import SlabSolver
from paper_2308_06085_b200.krylov import SolverConfig
from paper_2308_06085_b200.partition import TorchSlabComm, slab_partition
os.environ["MASTER_ADDR"] = "127.0.0.1"
os.environ["MASTER_PORT"] = sys.argv[1]
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
p = problems.point_source_cube(65, 40.0, "sommerfeld")
spec, b = problems.build_problem(p)
e = slab_partition(p.grid, 1)[0]
S = SlabSolver(p.grid, [e], spec.k_field, p.bc, TorchSlabComm())
xs, rep = S.solve_device([b], SolverConfig(method="bicgstab"))
np.save(sys.argv[2], xs[0].cpu().numpy())
print(json.dumps({"iterations": rep.iterations, "converged": rep.converged}))
dist.destroy_process_group()
'''


def test_nccl_comm_device_solve_world1(tmp_path):
    """The N > 1 bench path (TorchSlabComm over NCCL, device all-reduce of the
    Bi-CGSTAB partial sums) on a one-rank NCCL group matches the single-slab
    graph solve."""
    import json
    import os
    import socket
    import subprocess
    import sys
    from paper_2308_06085_b200 import problems
    p = problems.point_source_cube(65, 40.0, "sommerfeld")
    k = np.full(p.grid.shape, 40.0)
    b, x1, r1, _ = _single(p, k)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = tmp_path / "x.npy"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = subprocess.run([sys.executable, "-c", _NCCL_CHILD, str(port), str(out)], cwd=root,
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    rep = json.loads(res.stdout.strip().splitlines()[-1])
    assert rep["converged"] and abs(rep["iterations"] - r1.iterations) <= 1
    xs = np.load(out)
    assert np.linalg.norm(xs - x1) / np.linalg.norm(x1) < 1e-8
