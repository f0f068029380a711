"""The native multi-slab driver (hf_slab_*, dist.NativeSlabSolver): one
Bi-CGSTAB iteration over i1 slabs -- slab V(1,1) cycle, halo exchanges,
coarsest gather, inner-product all-reduces, scalar update -- replayed as one
CUDA graph.

LOCAL transport: all slabs of the decomposition in this process (virtual
ranks on one GPU, halos as device copies) against the single-slab solve and
the Python-driven slab path (same kernels, same reduction order).  NCCL
transport: a one-rank NCCL group (the only multi-rank configuration one GPU
allows), so the NCCL communicator, all-reduce and all-gather run inside the
captured graph; N > 1 ranks need N GPUs (bench.py --gpus N)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _problem(kind):
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.grid import full_extent
    p = problems.wedge3_problem(65) if kind == "wedge" else problems.point_source_cube(65, 40.0)
    spec, b = problems.build_problem(p)
    return p, np.ascontiguousarray(spec.k_field), b


def _single(p, k, b, shadow="rhs"):
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, Sommerfeld, StencilOperator
    A = StencilOperator(OperatorSpec("helmholtz", 1.0, 0.0, Sommerfeld(), k), p.grid)
    H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, Sommerfeld(), k), MGConfig())
    x, rep = Solver(A, H).solve(b, SolverConfig(method="bicgstab", shadow=shadow))
    return x.cpu().numpy(), rep


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("kind", ["cube", "wedge"])
@pytest.mark.parametrize("nslabs", [1, 2, 3, 4])
def test_native_slabs_match_single(kind, nslabs):
    from paper_2308_06085_b200.dist import NativeSlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    p, k, b = _problem(kind)
    x1, r1 = _single(p, k, b)
    ext = slab_partition(p.grid, nslabs)
    S = NativeSlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(nslabs))
    xs, rep = S.solve([b[e.lo1 - 1:e.hi1] for e in ext], SolverConfig(method="bicgstab"))
    x = np.concatenate([t.cpu().numpy() for t in xs], 0)
    assert rep.converged and abs(rep.iterations - r1.iterations) <= 1
    assert _rel(x, x1) < 1e-8
    assert rep.kernel_launches > 0
    # a second solve replays the captured graph: identical result
    xs2, rep2 = S.solve([b[e.lo1 - 1:e.hi1] for e in ext], SolverConfig(method="bicgstab"))
    assert rep2.iterations == rep.iterations
    assert np.array_equal(np.concatenate([t.cpu().numpy() for t in xs2], 0), x)


@pytest.mark.parametrize("kind,nslabs", [("cube", 2), ("wedge", 3), ("wedge", 4), ("cube", 5)])
def test_native_slabs_wide_family(kind, nslabs, hfopt):
    """The wide-plane sweep family (hf_wide.cu) on slabs: interior slab faces read
    the ghost planes, only the global end planes are mirrored, one-plane
    sub-slabs (the matvec's face planes), and the fused up-sweep launched as an
    interior range overlapping the exchange of the coarse correction plus two
    face ranges that read its ghost planes -- `force_wide` routes the 65^3
    levels through it; against the single-slab solve of the default kernels."""
    from paper_2308_06085_b200.dist import NativeSlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    p, k, b = _problem(kind)
    x1, r1 = _single(p, k, b)
    hfopt("force_wide", 1)
    hfopt("no_dr", 1)
    ext = slab_partition(p.grid, nslabs)
    S = NativeSlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(nslabs))
    xs, rep = S.solve([b[e.lo1 - 1:e.hi1] for e in ext], SolverConfig(method="bicgstab"))
    x = np.concatenate([t.cpu().numpy() for t in xs], 0)
    assert rep.converged and abs(rep.iterations - r1.iterations) <= 1
    assert _rel(x, x1) < 1e-8


def test_native_slabs_match_python_slab_driver():
    """Same decomposition through the Python-driven device path
    (SlabSolver.solve_device): same kernels; the native matvec sums its
    interior and face planes separately (overlapped halo), so rounding only."""
    from paper_2308_06085_b200.dist import NativeSlabSolver, SlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    p, k, b = _problem("wedge")
    ext = slab_partition(p.grid, 3)
    parts = [b[e.lo1 - 1:e.hi1] for e in ext]
    xn, rn = NativeSlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(3)).solve(parts)
    xp, rp = SlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(3)).solve_device(parts)
    assert abs(rn.iterations - rp.iterations) <= 1
    x1 = np.concatenate([t.cpu().numpy() for t in xn], 0)
    x2 = np.concatenate([t.cpu().numpy() for t in xp], 0)
    assert _rel(x1, x2) < 1e-9


def test_native_slabs_random_shadow_layout_independent():
    """The seeded shadow vector is drawn by global vertex index: 1 and 3 slabs
    run the same recurrences."""
    from paper_2308_06085_b200.dist import NativeSlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    p, k, b = _problem("wedge")
    x1, r1 = _single(p, k, b, shadow="random")
    ext = slab_partition(p.grid, 3)
    xs, rep = NativeSlabSolver(p.grid, ext, k, p.bc, LocalSlabComm(3)).solve(
        [b[e.lo1 - 1:e.hi1] for e in ext], SolverConfig(method="bicgstab", shadow="random"))
    assert abs(rep.iterations - r1.iterations) <= 1
    assert _rel(np.concatenate([t.cpu().numpy() for t in xs], 0), x1) < 1e-8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_native_slabs_nccl_one_rank():
    import torch.distributed as dist

    from paper_2308_06085_b200.dist import NativeSlabSolver
    from paper_2308_06085_b200.grid import full_extent
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import TorchSlabComm
    p, k, b = _problem("wedge")
    x1, r1 = _single(p, k, b)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        S = NativeSlabSolver(p.grid, [full_extent(p.grid)], k, p.bc, TorchSlabComm())
        xs, rep = S.solve([b], SolverConfig(method="bicgstab"))
        assert rep.converged and abs(rep.iterations - r1.iterations) <= 1
        assert _rel(xs[0].cpu().numpy(), x1) < 1e-8
        del S
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nslabs", [2, 3])
def test_native_slabs_wide_planes(nslabs):
    """Planes wider than 255 vertices: the slab cycle runs the split
    pre-smoothing / restriction pair with both halos overlapped, and the
    65 x 17 x 145 coarsest grid (no exact factorisation) runs the device GMRES
    fallback."""
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.dist import NativeSlabSolver
    from paper_2308_06085_b200.grid import make_grid
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    grid = make_grid(33, 65, 289, 1.0 / 288)
    rng = np.random.default_rng(5)
    k = rng.uniform(40.0, 60.0, grid.shape)
    b = np.zeros(grid.shape, complex)
    b[16, 32, 144] = 1.0 / grid.h ** 3

    class P:
        pass
    P.grid = grid
    x1, r1 = _single(P, k, b)
    ext = slab_partition(grid, nslabs)
    from paper_2308_06085_b200.operators import Sommerfeld
    xs, rep = NativeSlabSolver(grid, ext, k, Sommerfeld(), LocalSlabComm(nslabs)).solve(
        [b[e.lo1 - 1:e.hi1] for e in ext], SolverConfig(method="bicgstab"))
    assert rep.converged and abs(rep.iterations - r1.iterations) <= 1
    assert _rel(np.concatenate([t.cpu().numpy() for t in xs], 0), x1) < 1e-8
