"""The wide-plane sweep family (csrc/hf_wide.cu: 32 x 8P tiles, P rows per
thread, bulk-copied tile rows) against the C oracle.  The family serves planes
wider than 256 vertices; `force_wide` routes every level through it so the
ragged small grids (partial tiles, mirrored rows / columns inside a tile,
one-plane chunks) are covered, for the strip heights (two rows per thread by
default, `wide_p3` / `wide_p4`), the three wavenumber layouts (constant, float64 field, 8-bit
palette) and both boundary conditions."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _medium(kind, n, seed=3):
    if kind == "const":
        return np.full(n, 9.0)
    if kind == "field":
        return np.random.default_rng(seed).uniform(6.0, 12.0, n)
    # layered: three distinct values -> palette indices
    z = np.linspace(0, 1, n[2])[None, None, :]
    x = np.linspace(0, 1, n[0])[:, None, None]
    y = np.linspace(0, 1, n[1])[None, :, None]
    return np.broadcast_to(np.where(z > 0.4 + 0.2 * x, 11.0, np.where(y > 0.7 - 0.2 * x, 7.0, 9.0)), n).copy()


@pytest.fixture(scope="module")
def hf():
    import paper_2308_06085_b200 as pkg
    from paper_2308_06085_b200 import _native
    _native.load()
    return pkg


GRIDS = [(5, 5, 5), (5, 7, 9), (9, 33, 34), (6, 34, 65), (17, 40, 33), (4, 9, 70)]


# every grid with the default strips; two ragged grids with the optional strip heights
SWEEP_CASES = [(d, "") for d in GRIDS] + [(d, s) for s in ("wide_p1", "wide_p3", "wide_p4", "wide_big")
                                            for d in ((5, 7, 9), (6, 34, 65))]


@pytest.mark.parametrize("dims,strips", SWEEP_CASES)
@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
@pytest.mark.parametrize("medium", ["const", "field", "layered"])
def test_wide_sweeps_match_oracle(hf, oracle, dims, strips, bc, medium, hfopt):
    """A u, the Jacobi sweep and the zero-guess sweep + residual, kernel by kernel."""
    from paper_2308_06085_b200.multigrid import jacobi_smooth
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld, StencilOperator
    hfopt("force_wide", 1)
    if strips:
        hfopt(strips, 1)
    h = 0.125
    k = _medium(medium, dims)
    u0, b = _rand(dims, 2), _rand(dims, 8)
    bcs = Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld()
    grid = hf.make_grid(*dims, h)
    for kind, beta2 in (("helmholtz", 0.0), ("cslp", -0.5)):
        spec = OperatorSpec(kind, 1.0, beta2, bcs, k)
        got = StencilOperator(spec, grid).apply(u0).cpu().numpy()
        assert _rel(got, oracle.apply(k, u0, h, spec.shift, bc)) < 1e-12
    spec = OperatorSpec("cslp", 1.0, -0.5, bcs, k)
    op = StencilOperator(spec, grid)
    oh = oracle.Hierarchy(k, h, beta2=-0.5, bc=bc, threshold=10 ** 9)
    u = torch.as_tensor(u0).cuda()
    jacobi_smooth(op, u, b, 0.8, 2)
    assert _rel(u.cpu().numpy(), oh.jacobi(0, u0, b, 0.8, 2)) < 1e-12


_CYCLE_REF = {}
CYCLE_CASES = [
    ((33, 33, 33), "sommerfeld", "field", {}),
    ((33, 33, 33), "dirichlet", "layered", {}),
    ((33, 33, 65), "sommerfeld", "layered", dict(cycle="F")),
    ((33, 33, 49), "sommerfeld", "const", dict(nu1=2, nu2=1)),
    ((33, 33, 33), "dirichlet", "const", {}),
    ((33, 41, 33), "sommerfeld", "field", dict(nu1=0, nu2=1)),
]


@pytest.mark.parametrize("n,bc,medium,cfg,strips",
                         [c + ("",) for c in CYCLE_CASES] +
                         [c + (s,) for s in ("wide_p1", "wide_p3", "wide_p4", "wide_big") for c in CYCLE_CASES[1:4]])
def test_wide_cycle_matches_oracle(hf, oracle, n, bc, medium, cfg, strips, hfopt):
    """Whole cycles with every level's sweeps on the wide family (split
    down-sweep: the fused flat kernel is switched off), against the oracle and
    against the default kernels."""
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld
    k = _medium(medium, n)
    grid = hf.make_grid(*n, 1.0 / (n[0] - 1))
    spec = OperatorSpec("cslp", 1.0, -0.5, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), k)
    mg = MGConfig(**cfg)
    r = _rand(n, 10)
    key = (n, bc, medium, tuple(sorted(cfg.items())))
    if key not in _CYCLE_REF:        # the oracle cycle and the default kernels, once per case
        oh = oracle.Hierarchy(k, grid.h, beta2=-0.5, bc=bc, nu1=mg.nu1, nu2=mg.nu2, omega=mg.omega,
                              cycle=mg.cycle, threshold=mg.coarsest_threshold,
                              threshold_cmp=mg.threshold_cmp)
        _CYCLE_REF[key] = (oh.precondition(r),
                           mg_precondition(build_hierarchy(grid, None, spec, mg), r).cpu().numpy())
    want, base = _CYCLE_REF[key]
    hfopt("force_wide", 1)
    hfopt("no_dr", 1)
    if strips:
        hfopt(strips, 1)
    hier = build_hierarchy(grid, None, spec, mg)
    got = mg_precondition(hier, r).cpu().numpy()
    assert _rel(got, want) < 1e-9
    assert _rel(got, base) < 1e-12


@pytest.mark.parametrize("medium,strips", [("const", ""), ("layered", ""), ("layered", "wide_p1"),
                                            ("const", "wide_p3"), ("layered", "wide_p4"), ("layered", "wide_big")])
def test_wide_solve_matches_default(hf, oracle, medium, strips, hfopt):
    """Bi-CGSTAB with the matvec's inner products (r~^H v; t^H t, t^H s)
    accumulated by the wide sweeps: iteration count and solution of the default
    kernels, and the oracle's."""
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    p = problems.point_source_cube(33, 20.0, "sommerfeld")
    spec, b = problems.build_problem(p)
    k = np.full(p.grid.shape, 20.0) if medium == "const" else _medium("layered", p.grid.shape) * 2.0
    spec = OperatorSpec("helmholtz", 1.0, 0.0, spec.bc, k)

    def run():
        A = StencilOperator(spec, p.grid)
        M = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, k), MGConfig())
        x, rep = Solver(A, M).solve(b, SolverConfig(method="bicgstab", tol=1e-8, maxit=200))
        return x.cpu().numpy(), rep

    x0, r0 = run()
    hfopt("force_wide", 1)
    hfopt("no_dr", 1)
    if strips:
        hfopt(strips, 1)
    x1, r1 = run()
    assert r0.converged and r1.converged
    assert abs(r0.iterations - r1.iterations) <= 1
    assert np.linalg.norm(x1 - x0) / np.linalg.norm(x0) < 1e-7
    xo, ro = oracle.solve(k, b, p.grid.h, bc="sommerfeld", method="bicgstab", tol=1e-8, maxit=200)
    assert abs(r1.iterations - ro["iterations"]) <= 1
    assert np.linalg.norm(x1 - xo) / np.linalg.norm(xo) < 1e-7
