"""The reference's coarsest solve on the device (coarsest_method="gmres",
k_coarse_gmres; /root/reference/pkg/src/helmfree/multigrid.py:300-323):
unpreconditioned GMRES to coarsest_tol within coarsest_maxit, failures
counted in coarsest_flags, and the automatic fallback of the direct method
when the coarsest grid has no exact factorisation."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _kfield(shape, seed, lo, hi):
    return np.random.default_rng(seed).uniform(lo, hi, shape)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _hier(n, bc, k, **cfg):
    from paper_2308_06085_b200.grid import make_grid
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld
    grid = make_grid(*n, 1.0 / (n[0] - 1))
    spec = OperatorSpec("cslp", 1.0, -0.5, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), k)
    return grid, build_hierarchy(grid, None, spec, MGConfig(**cfg))


@pytest.mark.parametrize("bc", ["sommerfeld", "dirichlet"])
@pytest.mark.parametrize("kind", ["const", "field"])
def test_coarsest_gmres_meets_tolerance(oracle, bc, kind):
    from paper_2308_06085_b200.multigrid import coarsest_solve
    n = (33, 33, 33)
    k = np.full(n, 20.0) if kind == "const" else _kfield(n, 3, 15, 25)
    grid, H = _hier(n, bc, k, coarsest_method="gmres")
    assert H.coarsest_kind == "gmres"
    _, Hd = _hier(n, bc, k)
    nc = H.coarsest.grid.shape
    b = _rand(nc, 4)
    if bc == "dirichlet":      # working vectors carry zeros on the boundary planes
        b[0], b[-1], b[:, 0], b[:, -1], b[:, :, 0], b[:, :, -1] = 0, 0, 0, 0, 0, 0
    x = coarsest_solve(H, b).cpu().numpy()
    kc = k[::2, ::2, ::2]
    from paper_2308_06085_b200.operators import OperatorSpec
    shift = OperatorSpec("cslp", 1.0, -0.5, None, kc).shift
    r = b - oracle.apply(kc, x, H.coarsest.grid.h, shift, bc)
    assert np.linalg.norm(r) / np.linalg.norm(b) <= 1.01e-11
    assert H.coarsest_flags == []
    xd = coarsest_solve(Hd, b).cpu().numpy()
    assert _rel(x, xd) < 1e-8


def test_cycle_with_gmres_coarsest_matches_oracle(oracle):
    """V-cycle with the device GMRES coarsest solve against the oracle's (GMRES
    to 1e-11 as the reference; CGS2 vs MGS orthogonalisation: rounding only)."""
    from paper_2308_06085_b200.multigrid import mg_precondition
    n = (33, 33, 33)
    k = _kfield(n, 9, 15, 25)
    grid, H = _hier(n, "sommerfeld", k, coarsest_method="gmres")
    oh = oracle.Hierarchy(k, grid.h)
    r = _rand(n, 10)
    got = mg_precondition(H, r).cpu().numpy()
    assert _rel(got, oh.precondition(r)) < 1e-9


def test_solve_with_gmres_coarsest_matches_oracle(oracle):
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    p = problems.wedge3_problem(33)
    spec, b = problems.build_problem(p)
    k = np.ascontiguousarray(spec.k_field)
    A = StencilOperator(spec, p.grid)
    H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, k),
                        MGConfig(coarsest_method="gmres"))
    x, rep = Solver(A, H).solve(b, SolverConfig(method="bicgstab", maxit=300))
    xo, ro = oracle.solve(k, b, p.grid.h, maxit=300)
    assert rep.converged and abs(rep.iterations - ro["iterations"]) <= 1
    assert _rel(x.cpu().numpy(), xo) < 1e-8


def test_soft_failure_counted_in_coarsest_flags():
    from paper_2308_06085_b200.multigrid import coarsest_solve
    n = (33, 33, 33)
    k = _kfield(n, 5, 15, 25)
    grid, H = _hier(n, "sommerfeld", k, coarsest_method="gmres", coarsest_maxit=3,
                    coarsest_tol=1e-14)
    b = _rand(H.coarsest.grid.shape, 6)
    coarsest_solve(H, b)
    coarsest_solve(H, b)
    assert sum(f["count"] for f in H.coarsest_flags) == 2


def test_direct_falls_back_to_gmres_on_large_coarsest(oracle):
    """129 x 129 x 33 with a varying medium coarsens to 65 x 65 x 17 = 71825
    vertices: no exact factorisation (dense limit 60000), so the direct method
    falls back to the reference's GMRES instead of failing."""
    from paper_2308_06085_b200.multigrid import mg_precondition
    n = (129, 129, 33)
    k = _kfield(n, 11, 30, 50)
    grid, H = _hier(n, "sommerfeld", k)
    assert H.coarsest.grid.shape == (65, 65, 17)
    assert H.coarsest_kind == "gmres"
    oh = oracle.Hierarchy(k, grid.h)
    r = _rand(n, 12)
    assert _rel(mg_precondition(H, r).cpu().numpy(), oh.precondition(r)) < 1e-8
