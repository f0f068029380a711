"""Parity of the native CUDA path with the C oracle (which is pinned to the
reference by tests/test_oracle.py).  Tolerances: complex128 kernels agree to
1e-12 relative (reduction order / FMA only); solves agree on the iteration
count within +-1 and on the solution within 1e-8 relative L2 (north_star)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _kfield(shape, seed=0, lo=3.0, hi=8.0):
    rng = np.random.default_rng(seed)
    return rng.uniform(lo, hi, shape)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.fixture(scope="module")
def hf():
    import paper_2308_06085_b200 as pkg
    from paper_2308_06085_b200 import _native
    _native.load()
    return pkg


GRIDS = [(5, 5, 5), (7, 7, 7), (9, 9, 9), (5, 7, 9), (17, 17, 17), (33, 17, 9)]


@pytest.mark.parametrize("dims", GRIDS)
@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
@pytest.mark.parametrize("kind", ["helmholtz", "cslp"])
def test_apply_matches_oracle(hf, oracle, dims, bc, kind):
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld, StencilOperator
    h = 0.125
    k = _kfield(dims, 1)
    u = _rand(dims, 2)
    spec = OperatorSpec(kind, 1.0, -0.5, Dirichlet(1.0) if bc == "dirichlet" else Sommerfeld(), k)
    grid = hf.make_grid(*dims, h)
    got = StencilOperator(spec, grid).apply(u).cpu().numpy()
    want = oracle.apply(k, u, h, spec.shift, bc)
    assert _rel(got, want) < 1e-12


def test_constant_k_fast_path(hf, oracle):
    from paper_2308_06085_b200.operators import OperatorSpec, Sommerfeld, StencilOperator
    dims, h = (17, 9, 33), 1 / 16
    k = np.full(dims, 7.5)
    u = _rand(dims, 3)
    spec = OperatorSpec("cslp", 1.0, -0.5, Sommerfeld(), k)
    got = StencilOperator(spec, hf.make_grid(*dims, h)).apply(u).cpu().numpy()
    assert _rel(got, oracle.apply(k, u, h, spec.shift, "sommerfeld")) < 1e-12


def _pair(hf, oracle, n, bc, k, beta2=-0.5, **cfg):
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld
    grid = hf.make_grid(*n, 1.0 / (n[0] - 1))
    spec = OperatorSpec("cslp", 1.0, beta2, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), k)
    mg = MGConfig(**cfg)
    hier = build_hierarchy(grid, None, spec, mg)
    oh = oracle.Hierarchy(k, grid.h, beta2=beta2, bc=bc, nu1=mg.nu1, nu2=mg.nu2, omega=mg.omega,
                          cycle=mg.cycle, threshold=mg.coarsest_threshold,
                          threshold_cmp=mg.threshold_cmp)
    return hier, oh


@pytest.mark.parametrize("dims,h,kc", [((17, 17, 17), 1 / 16, 80.0), ((9, 17, 5), 1 / 8, 7.5),
                                       ((17, 17, 17), 1 / 16, 40.0)])
def test_coarsest_fast_diagonalisation(hf, oracle, dims, h, kc, hfopt):
    """Constant-k Sommerfeld coarsest solve (separable, k_fdm_*) is exact: the
    true residual through the oracle's operator is at round-off and it agrees
    with the dense-inverse path (HF_COARSEST_DENSE) to 1e-12."""
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, coarsest_solve
    from paper_2308_06085_b200.operators import OperatorSpec, Sommerfeld
    grid = hf.make_grid(*dims, h)
    spec = OperatorSpec("cslp", 1.0, -0.5, Sommerfeld(), np.full(dims, kc))
    b = _rand(dims, 21)
    hier = build_hierarchy(grid, None, spec, MGConfig(coarsest_threshold=64))
    assert len(hier.levels) == 1 and hier.coarsest_kind == "separable"
    x = coarsest_solve(hier, b).cpu().numpy()
    r = b - oracle.apply(np.full(dims, kc), x, h, spec.shift, "sommerfeld")
    assert np.linalg.norm(r) / np.linalg.norm(b) < 1e-12
    hfopt("coarsest_dense", 1)
    dense = build_hierarchy(grid, None, spec, MGConfig(coarsest_threshold=64))
    assert dense.coarsest_kind == "symmetric"
    xd = coarsest_solve(dense, b).cpu().numpy()
    assert _rel(x, xd) < 1e-12


@pytest.mark.parametrize("dims,bc,kind,mg", [
    ((65, 65, 65), "sommerfeld", "const", {}),
    ((129, 65, 97), "sommerfeld", "const", {}),
    ((65, 33, 49), "dirichlet", "const", {}),
    ((65, 65, 65), "sommerfeld", "field", {}),
    ((65, 49, 33), "dirichlet", "field", {}),
    ((65, 65, 65), "sommerfeld", "const", {"nu1": 0}),
])
def test_fused_up_matches_split(hf, dims, bc, kind, mg, hfopt):
    """Prolongation + correction produced inside the post-smoothing sweep
    (MODE_UP) matches the split correction + Jacobi kernels (same arithmetic;
    FMA contraction may differ between the kernels)."""
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld
    grid = hf.make_grid(*dims, 1.0 / (dims[0] - 1))
    k = np.full(dims, 30.0) if kind == "const" else _kfield(dims, 11, 20, 35)
    spec = OperatorSpec("cslp", 1.0, -0.5, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), k)
    r = torch.as_tensor(_rand(dims, 41)).cuda()
    hier = build_hierarchy(grid, None, spec, MGConfig(**mg))
    hfopt("fuse_up", 1)
    fused = mg_precondition(hier, r).cpu().numpy()        # tiled MODE_UP
    hfopt("flat_up", 1)
    flat = mg_precondition(hier, r).cpu().numpy()         # flat MODE_UP (opt-in)
    hfopt("flat_up", 0)
    hfopt("no_fuse", 1)
    split = mg_precondition(hier, r).cpu().numpy()
    assert _rel(fused, split) < 1e-13
    assert _rel(flat, split) < 1e-13


@pytest.mark.parametrize("dims,bc,kind", [
    ((129, 129, 129), "sommerfeld", "const"),
    ((65, 65, 65), "sommerfeld", "const"),
    ((129, 65, 97), "sommerfeld", "const"),
    ((65, 33, 49), "dirichlet", "const"),
    ((65, 65, 65), "sommerfeld", "field"),
    ((65, 49, 33), "dirichlet", "field"),
    ((33, 17, 65), "sommerfeld", "field"),
])
@pytest.mark.parametrize("variant", ["flat", "tiled"])
def test_fused_down_restrict_matches_split(hf, dims, bc, kind, variant, hfopt):
    """Pre-smoothing + residual + full weighting in one kernel (k_flat_dr, or
    the tiled k_down_restrict used on wide planes) matches the split down1 +
    restriction kernels on every level of the cycle (same arithmetic; only
    FMA contraction may differ)."""
    if variant == "tiled":
        hfopt("no_flat_dr", 1)
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld
    grid = hf.make_grid(*dims, 1.0 / (dims[0] - 1))
    k = np.full(dims, 30.0) if kind == "const" else _kfield(dims, 12, 20, 35)
    spec = OperatorSpec("cslp", 1.0, -0.5, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), k)
    r = torch.as_tensor(_rand(dims, 43)).cuda()
    hier = build_hierarchy(grid, None, spec, MGConfig())
    hfopt("tiled_dr", 1)
    fused = mg_precondition(hier, r).cpu().numpy()
    hfopt("no_dr", 1)
    split = mg_precondition(hier, r).cpu().numpy()
    assert _rel(fused, split) < 1e-13


@pytest.mark.parametrize("n,kind", [(129, "wedge"), (129, "const"), (65, "wedge")])
def test_flat_kernels_match_tiled(hf, n, kind, hfopt):
    """The flat bulk-copy kernels (k_flat_stencil, k_flat_dr, k_corr_flat) and
    the 2-D tiled cp.async kernels compute the same V-cycle and operator at
    BASELINE-like sizes, varying medium included (rounding-level differences
    only)."""
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    p = problems.wedge3_problem(n) if kind == "wedge" else problems.point_source_cube(n, 80.0 * (n - 1) / 128)
    spec, _ = problems.build_problem(p)
    r = torch.as_tensor(_rand(p.grid.shape, 47)).cuda()
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
    A = StencilOperator(spec, p.grid)
    z_flat = mg_precondition(hier, r).cpu().numpy()
    v_flat = A.apply(r).cpu().numpy()
    hfopt("no_flat", 1)
    hfopt("no_dr", 1)
    z_tile = mg_precondition(hier, r).cpu().numpy()
    v_tile = A.apply(r).cpu().numpy()
    assert _rel(z_flat, z_tile) < 1e-12
    assert _rel(v_flat, v_tile) < 1e-13


@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
def test_transfers_and_smoother(hf, oracle, bc):
    from paper_2308_06085_b200.multigrid import jacobi_smooth, prolong_tl, restrict_fw
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld, StencilOperator
    n = (17, 17, 17)
    k = _kfield(n, 4)
    hier, oh = _pair(hf, oracle, n, bc, k, coarsest_threshold=5)
    assert [lv.grid.shape for lv in hier.levels] == oh.shapes
    r = _rand(n, 5)
    got = restrict_fw(r, hier.levels[0], hier.levels[1]).cpu().numpy()
    assert _rel(got, oh.restrict(0, r)) < 1e-14
    e = _rand(oh.shapes[1], 6)
    got = prolong_tl(e, hier.levels[1], hier.levels[0]).cpu().numpy()
    assert _rel(got, oh.prolong(0, e)) < 1e-15
    spec = OperatorSpec("cslp", 1.0, -0.5, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), k)
    op = StencilOperator(spec, hf.make_grid(*n, 1 / 16))
    u0, b = _rand(n, 7), _rand(n, 8)
    u = torch.as_tensor(u0).cuda()
    jacobi_smooth(op, u, b, 0.8, 2)
    assert _rel(u.cpu().numpy(), oh.jacobi(0, u0, b, 0.8, 2)) < 1e-12
    u = torch.zeros(n, dtype=torch.complex128, device="cuda")
    jacobi_smooth(op, u, b, 0.8, 1, assume_zero=True)
    assert _rel(u.cpu().numpy(), oh.jacobi(0, np.zeros(n), b, 0.8, 1, assume_zero=True)) < 1e-13


@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
@pytest.mark.parametrize("cfg", [dict(), dict(cycle="F"), dict(nu1=2, nu2=1), dict(nu1=0, nu2=1),
                                 dict(threshold_cmp="ge")])
def test_cycle_matches_oracle(hf, oracle, bc, cfg):
    from paper_2308_06085_b200.multigrid import mg_precondition
    n = (33, 33, 33)
    k = _kfield(n, 9, 15, 25)
    hier, oh = _pair(hf, oracle, n, bc, k, **cfg)
    r = _rand(n, 10)
    got = mg_precondition(hier, r).cpu().numpy()
    want = oh.precondition(r)
    # coarsest: exact LU here vs GMRES to 1e-11 in the reference
    assert _rel(got, want) < 1e-9


@pytest.mark.parametrize("n,bc,kind", [((17, 17, 193), "sommerfeld", "const"),
                                        ((9, 9, 161), "dirichlet", "field"),
                                        ((9, 17, 255), "sommerfeld", "field")])
def test_wide_plane_flat_kernels_match_oracle(hf, oracle, n, bc, kind, hfopt):
    """Planes 154..255 vertices wide: the flat kernels' five-points-per-thread
    fused down-sweep (k_flat_dr RPT 5) and the widest flat ranges, against the
    oracle's V-cycle, and the fused down-sweep against the split pair."""
    from paper_2308_06085_b200.multigrid import mg_precondition
    k = np.full(n, 9.0) if kind == "const" else _kfield(n, 21, 6, 12)
    hier, oh = _pair(hf, oracle, n, bc, k)
    r = _rand(n, 22)
    got = mg_precondition(hier, r).cpu().numpy()
    assert _rel(got, oh.precondition(r)) < 1e-9
    hfopt("no_dr", 1)
    split = mg_precondition(hier, r).cpu().numpy()
    assert _rel(got, split) < 1e-13


def _solve_pair(hf, oracle, pspec, k_full, method="bicgstab", beta2=-0.5, tol=1e-6, maxit=400,
                **mg):
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    spec, b = problems.build_problem(pspec)
    A = StencilOperator(spec, pspec.grid)
    hier = build_hierarchy(pspec.grid, None, OperatorSpec("cslp", 1.0, beta2, spec.bc, k_full),
                           MGConfig(**mg))
    x, rep = Solver(A, hier).solve(b, SolverConfig(method=method, tol=tol, maxit=maxit))
    bc = "dirichlet" if type(spec.bc).__name__ == "Dirichlet" else "sommerfeld"
    xo, ro = oracle.solve(k_full, b, pspec.grid.h, bc=bc, method=method, tol=tol, maxit=maxit,
                          beta2=beta2, **{k_: v for k_, v in mg.items() if k_ != "coarsest_method"})
    return x.cpu().numpy(), rep, xo, ro


@pytest.mark.parametrize("n,k,bc", [(33, 20.0, "dirichlet"), (33, 20.0, "sommerfeld"),
                                    (65, 40.0, "sommerfeld")])
def test_bicgstab_point_source(hf, oracle, n, k, bc):
    from paper_2308_06085_b200 import problems
    p = problems.point_source_cube(n, k, bc)
    x, rep, xo, ro = _solve_pair(hf, oracle, p, np.full(p.grid.shape, k))
    assert rep.converged and ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert abs(rep.matvec_count - ro["matvec_count"]) <= 2
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-8
    np.testing.assert_allclose(rep.residual_history[:5], ro["residual_history"][:5], rtol=1e-7)


def test_bicgstab_heterogeneous_wedge(hf, oracle):
    from paper_2308_06085_b200 import problems
    p = problems.wedge3_problem(41)
    k = p.medium.k_field(p.grid, hf.full_extent(p.grid))
    x, rep, xo, ro = _solve_pair(hf, oracle, p, k)
    assert rep.converged and ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-8


def test_bicgstab_noncubic_layered_wedge(hf, oracle):
    """The reference's own two-interface wedge builder (problems.wedge_problem)
    on a non-cubic 33 x 33 x 49 grid (h = 20 m, 5 Hz, kh <= 0.42)."""
    from paper_2308_06085_b200 import problems
    p = problems.wedge_problem(shape=(33, 33, 49), domain=((0.0, 640.0), (0.0, 640.0), (-960.0, 0.0)),
                               frequency=5.0, source_at=(320.0, 320.0, 0.0))
    k = p.medium.k_field(p.grid, hf.full_extent(p.grid))
    x, rep, xo, ro = _solve_pair(hf, oracle, p, k)
    assert rep.converged and ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-8


def test_solve_host_buffers(hf, oracle):
    """hf_solve_host (the e2e entry point) returns the same answer as hf_solve."""
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    p = problems.point_source_cube(33, 20.0, "sommerfeld")
    spec, b = problems.build_problem(p)
    A = StencilOperator(spec, p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
    S = Solver(A, hier)
    cfg = SolverConfig(method="bicgstab")
    xd, r1 = S.solve(b, cfg)
    xh, r2 = S.solve(b, cfg, host=True)
    assert r1.iterations == r2.iterations
    np.testing.assert_array_equal(xd.cpu().numpy(), xh)


@pytest.mark.filterwarnings("ignore:kh =")
@pytest.mark.parametrize("method", ["gmres", "bicgstab", "idrs"])
def test_closed_off_methods_match_oracle(hf, oracle, method):
    """Reference demo_convergence problem (ClosedOff 33^3, k=20, Dirichlet u=1):
    all three Krylov methods, native vs oracle (reference counts 27/44/34)."""
    from paper_2308_06085_b200 import problems
    p = problems.closed_off_problem(33, 20.0)
    x, rep, xo, ro = _solve_pair(hf, oracle, p, np.full(p.grid.shape, 20.0), method=method)
    assert rep.converged and ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert abs(rep.matvec_count - ro["matvec_count"]) <= 2
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-8
    if method == "gmres":
        hist = np.array(rep.residual_history)
        assert np.all(hist[1:] <= hist[:-1] * (1 + 1e-12))     # monotone (krylov.py:349)


def test_gmres_restart(hf, oracle):
    from paper_2308_06085_b200 import problems
    p = problems.point_source_cube(33, 20.0, "sommerfeld")
    x, rep, xo, ro = _solve_pair(hf, oracle, p, np.full(p.grid.shape, 20.0), method="gmres")
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    spec, b = problems.build_problem(p)
    A = StencilOperator(spec, p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
    xr, rr = Solver(A, hier).solve(b, SolverConfig(method="gmres", restart=5, maxit=200))
    assert rr.converged
    assert np.linalg.norm(xr.cpu().numpy() - xo) / np.linalg.norm(xo) < 1e-5


def test_repeat_solves_bit_identical(hf):
    """Deterministic reductions and race-free kernels: repeated solves (with
    different host polling intervals) give bit-identical solutions."""
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    p = problems.point_source_cube(65, 40.0, "sommerfeld")
    spec, b = problems.build_problem(p)
    A = StencilOperator(spec, p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
    S = Solver(A, hier)
    ref = None
    for every in (1, 3, 4):
        x, rep = S.solve(b, SolverConfig(method="bicgstab", check_every=every))
        x = x.cpu().numpy()
        if ref is None:
            ref, ref_it = x, rep.iterations
        assert rep.iterations == ref_it
        assert np.array_equal(x, ref)


@pytest.mark.parametrize("bc", ["sommerfeld", "dirichlet"])
def test_palette_level_matches_oracle(hf, oracle, bc, hfopt):
    """Wide planes (n3 > 256) of a layered medium: k stored as 8-bit palette
    indices, a_p / D^-1 from per-(index, face count) tables -- against the
    oracle's cycle and apply, and against the same level without the palette."""
    from paper_2308_06085_b200.multigrid import mg_precondition
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld, StencilOperator
    n = (33, 17, 289)
    z = np.linspace(0, 1, n[2])[None, None, :]
    x = np.linspace(0, 1, n[0])[:, None, None]
    k = np.broadcast_to(np.where(z > 0.4 + 0.2 * x, 30.0, np.where(z > 0.8 - 0.2 * x, 45.0, 20.0)), n).copy()
    hier, oh = _pair(hf, oracle, n, bc, k)
    r = _rand(n, 31)
    got = mg_precondition(hier, r).cpu().numpy()
    assert _rel(got, oh.precondition(r)) < 1e-9
    spec = OperatorSpec("helmholtz", 1.0, 0.0, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), k)
    grid = hf.make_grid(*n, 1.0 / (n[0] - 1))
    v = StencilOperator(spec, grid).apply(r).cpu().numpy()
    assert _rel(v, oracle.apply(k, r, grid.h, 1.0, bc)) < 1e-12
    hfopt("no_palette", 1)
    hier2, _ = _pair(hf, oracle, n, bc, k)
    assert _rel(mg_precondition(hier2, r).cpu().numpy(), got) < 1e-12
