"""Properties the reference's own tests assert (pkg/tests/test_operators.py,
test_multigrid.py, test_krylov.py), checked on the native B200 path at sizes
where the flat bulk-copy kernels, the fused down-kernel and the separable
coarsest solve are the code that runs."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _op(n, kind="cslp", bc="sommerfeld", k=None, beta2=-0.5):
    from paper_2308_06085_b200 import make_grid
    from paper_2308_06085_b200.operators import Dirichlet, OperatorSpec, Sommerfeld, StencilOperator
    grid = make_grid(*n, 1.0 / (n[0] - 1))
    kf = np.full(n, 30.0) if k is None else k
    spec = OperatorSpec(kind, 1.0, beta2, Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld(), kf)
    return StencilOperator(spec, grid), spec, grid


def _hier(n, bc="sommerfeld", k=None, **cfg):
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    A, spec, grid = _op(n, "cslp", bc, k)
    return build_hierarchy(grid, None, spec, MGConfig(**cfg)), A, spec, grid


# ---- operators (test_operators.py) -------------------------------------------
@pytest.mark.parametrize("bc", ["dirichlet", "sommerfeld"])
def test_operator_zero_in_zero_out_and_linearity(bc):
    A, _, _ = _op((65, 65, 65), "helmholtz", bc, k=np.random.default_rng(0).uniform(20, 30, (65,) * 3))
    z = torch.zeros((65,) * 3, dtype=torch.complex128, device="cuda")
    assert float(A.apply(z).abs().max()) == 0.0
    u, v = _rand((65,) * 3, 1), _rand((65,) * 3, 2)
    a, b = 0.3 - 1.7j, -2.1 + 0.4j
    lhs = A.apply(a * u + b * v).cpu().numpy()
    rhs = a * A.apply(u).cpu().numpy() + b * A.apply(v).cpu().numpy()
    assert _rel(lhs, rhs) < 1e-13


def test_sommerfeld_operator_row_scaled_symmetric():
    """S A is complex symmetric, S = 2^-faces (reference TestComplexSymmetry):
    <S A u, v> = <u, S A v> with the bilinear (unconjugated) product."""
    n = (33, 33, 33)
    A, _, _ = _op(n, "helmholtz", "sommerfeld")
    i, j, m = np.meshgrid(*[np.arange(s) for s in n], indexing="ij")
    faces = sum((x == 0).astype(int) + (x == s - 1).astype(int) for x, s in zip((i, j, m), n))
    S = 2.0 ** (-faces)
    u, v = _rand(n, 3), _rand(n, 4)
    lhs = np.sum(S * A.apply(u).cpu().numpy() * v)
    rhs = np.sum(u * S * A.apply(v).cpu().numpy())
    assert abs(lhs - rhs) / abs(lhs) < 1e-12


def test_cslp_beta_one_zero_equals_helmholtz():
    n = (65, 65, 65)
    Ah, _, _ = _op(n, "helmholtz")
    Ac, _, _ = _op(n, "cslp", beta2=0.0)
    u = _rand(n, 5)
    assert np.array_equal(Ah.apply(u).cpu().numpy(), Ac.apply(u).cpu().numpy())


def test_zero_diagonal_rejected():
    from paper_2308_06085_b200.operators import ZeroDiagonalError
    h = 1.0 / 16
    k = np.sqrt(6.0) / h          # k^2 h^2 = 6: the interior stencil diagonal vanishes
    with pytest.raises(ZeroDiagonalError):
        _op((17, 17, 17), "helmholtz", "dirichlet", k=np.full((17,) * 3, k))


# ---- multigrid (test_multigrid.py) --------------------------------------------
@pytest.mark.parametrize("n,cmp,levels", [(129, "gt", [129, 65, 33, 17]), (65, "gt", [65, 33, 17]),
                                          (65, "ge", [65, 33, 17, 9]), (33, "ge", [33, 17, 9])])
def test_stop_rule_levels(n, cmp, levels):
    """reference test_65_default / test_65_inclusive / test_33_inclusive_stop_rule"""
    hier, *_ = _hier((n,) * 3, bc="dirichlet", k=np.full((n,) * 3, 10.0), threshold_cmp=cmp)
    assert [lv.grid.n1 for lv in hier.levels] == levels


def test_unknown_cycle_rejected():
    from paper_2308_06085_b200.multigrid import MultigridError
    with pytest.raises(MultigridError):
        _hier((33,) * 3, cycle="W")


def test_restriction_preserves_constants():
    from paper_2308_06085_b200.multigrid import restrict_fw
    hier, *_ = _hier((129,) * 3)
    ones = torch.ones((129,) * 3, dtype=torch.complex128, device="cuda")
    rc = restrict_fw(ones, hier.levels[0], hier.levels[1]).cpu().numpy()
    assert np.abs(rc - 1.0).max() < 1e-14


def test_restriction_is_scaled_transpose_of_prolongation_interior():
    """<R u, e>_interior = 1/8 <u, P e> for u supported in the interior."""
    from paper_2308_06085_b200.multigrid import prolong_tl, restrict_fw
    n = (65, 65, 65)
    hier, *_ = _hier(n)
    u = np.zeros(n, complex)
    u[4:-4, 4:-4, 4:-4] = _rand(n, 6)[4:-4, 4:-4, 4:-4]
    e = _rand(hier.levels[1].extent.shape, 7)
    Ru = restrict_fw(u, hier.levels[0], hier.levels[1]).cpu().numpy()
    Pe = prolong_tl(e, hier.levels[1], hier.levels[0]).cpu().numpy()
    lhs, rhs = np.sum(Ru * e), np.sum(u * Pe) / 8.0
    assert abs(lhs - rhs) / abs(rhs) < 1e-12


def test_prolongation_coincident_impulse():
    from paper_2308_06085_b200.multigrid import prolong_tl
    hier, *_ = _hier((65,) * 3)
    e = np.zeros(hier.levels[1].extent.shape, complex)
    e[10, 12, 14] = 1.0
    Pe = prolong_tl(e, hier.levels[1], hier.levels[0]).cpu().numpy()
    assert Pe[20, 24, 28] == 1.0 and Pe[21, 24, 28] == 0.5 and Pe[21, 25, 29] == 0.125
    assert abs(Pe.sum() - 8.0) < 1e-12          # (0.5, 1, 0.5) per direction


@pytest.mark.parametrize("n", [65, 129])
def test_cycle_zero_in_zero_out_and_linearity(n):
    from paper_2308_06085_b200.multigrid import mg_precondition
    hier, *_ = _hier((n,) * 3)
    z = torch.zeros((n,) * 3, dtype=torch.complex128, device="cuda")
    assert float(mg_precondition(hier, z).abs().max()) == 0.0
    u, v = _rand((n,) * 3, 8), _rand((n,) * 3, 9)
    a, b = 1.5 - 0.5j, -0.25 + 2j
    lhs = mg_precondition(hier, a * u + b * v).cpu().numpy()
    rhs = a * mg_precondition(hier, u).cpu().numpy() + b * mg_precondition(hier, v).cpu().numpy()
    assert _rel(lhs, rhs) < 1e-12


def test_cycle_contracts_on_shifted_operator():
    """One V-cycle reduces the CSLP residual: |r - M z| < |r| (reference
    test_contraction_on_shifted_operator), with M the CSLP operator itself."""
    from paper_2308_06085_b200.multigrid import mg_precondition
    n = (65,) * 3
    hier, _, spec, grid = _hier(n)
    from paper_2308_06085_b200.operators import StencilOperator
    M = StencilOperator(spec, grid)
    r = torch.as_tensor(_rand(n, 10)).cuda()
    z = mg_precondition(hier, r)
    res = (r - M.apply(z)).norm() / r.norm()
    assert float(res) < 0.9


def test_f_cycle_beats_v_cycle():
    from paper_2308_06085_b200.multigrid import mg_precondition
    from paper_2308_06085_b200.operators import StencilOperator
    n = (65,) * 3
    hv, _, spec, grid = _hier(n, cycle="V")
    hf, *_ = _hier(n, cycle="F")
    M = StencilOperator(spec, grid)
    r = torch.as_tensor(_rand(n, 11)).cuda()
    rv = float((r - M.apply(mg_precondition(hv, r))).norm())
    rf = float((r - M.apply(mg_precondition(hf, r))).norm())
    assert rf < rv


# ---- Krylov (test_krylov.py) ---------------------------------------------------
def _solver(n=65, k=40.0):
    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    p = problems.point_source_cube(n, k, "sommerfeld")
    spec, b = problems.build_problem(p)
    A = StencilOperator(spec, p.grid)
    H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
    return Solver(A, H), A, b


@pytest.mark.parametrize("method", ["bicgstab", "gmres", "idrs"])
def test_zero_rhs_converges_immediately(method):
    from paper_2308_06085_b200.krylov import SolverConfig
    S, A, b = _solver()
    x, rep = S.solve(np.zeros_like(b), SolverConfig(method=method))
    assert rep.converged and rep.iterations == 0 and float(x.abs().max()) == 0.0


def test_bicgstab_two_matvecs_per_iteration_and_true_residual():
    from paper_2308_06085_b200.krylov import SolverConfig
    S, A, b = _solver()
    x, rep = S.solve(b, SolverConfig(method="bicgstab", tol=1e-6))
    assert rep.converged
    # a full iteration costs two matvecs; convergence at the half step one
    assert rep.matvec_count in (2 * rep.iterations, 2 * rep.iterations - 1)
    bd = torch.as_tensor(b).cuda()
    true = float((bd - A.apply(x)).norm() / bd.norm())
    assert abs(true - rep.final_relres) < 1e-3 * max(true, 1e-12) + 1e-9
    assert true < 1.05e-6


def test_gmres_matvec_count_and_monotone_history():
    from paper_2308_06085_b200.krylov import SolverConfig
    S, A, b = _solver()
    x, rep = S.solve(b, SolverConfig(method="gmres", tol=1e-6))
    assert rep.converged and rep.matvec_count == rep.iterations
    h = np.array(rep.residual_history)
    assert np.all(np.diff(h) <= 1e-12)


def test_nonconvergence_reported_honestly():
    from paper_2308_06085_b200.krylov import SolverConfig
    S, A, b = _solver()
    x, rep = S.solve(b, SolverConfig(method="bicgstab", tol=1e-12, maxit=3))
    assert not rep.converged and rep.iterations == 3 and rep.breakdown is None


def test_idrs_seed_reproducible_and_seeds_differ():
    from paper_2308_06085_b200.krylov import SolverConfig
    S, A, b = _solver(33, 20.0)
    x1, r1 = S.solve(b, SolverConfig(method="idrs", s=4, rng_seed=7))
    x2, r2 = S.solve(b, SolverConfig(method="idrs", s=4, rng_seed=7))
    x3, r3 = S.solve(b, SolverConfig(method="idrs", s=4, rng_seed=8))
    assert r1.converged and r1.residual_history == r2.residual_history
    assert np.array_equal(x1.cpu().numpy(), x2.cpu().numpy())
    assert r3.residual_history != r1.residual_history


def test_unknown_method_and_invalid_s_rejected():
    from paper_2308_06085_b200.krylov import KrylovError, SolverConfig
    S, A, b = _solver(33, 20.0)
    with pytest.raises((KrylovError, ValueError)):
        S.solve(b, SolverConfig(method="cg"))
    with pytest.raises((KrylovError, ValueError)):
        S.solve(b, SolverConfig(method="idrs", s=0))


@pytest.mark.parametrize("method", ["gmres", "bicgstab", "idrs"])
def test_exact_preconditioner_converges_in_one_step(method):
    """reference test_left_preconditioning_exact_inverse: with the operator
    itself as the CSLP and a one-level hierarchy (the exact separable coarsest
    solve), M^-1 = A^-1 and the Krylov method stops after one application."""
    from paper_2308_06085_b200 import make_grid
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, Sommerfeld, StencilOperator
    n = (17, 17, 17)
    grid = make_grid(*n, 1.0 / 16)
    spec = OperatorSpec("cslp", 1.0, -0.5, Sommerfeld(), np.full(n, 30.0))
    A = StencilOperator(spec, grid)
    H = build_hierarchy(grid, None, spec, MGConfig(coarsest_threshold=64))
    assert len(H.levels) == 1 and H.coarsest_kind == "separable"
    b = _rand(n, 12)
    x, rep = Solver(A, H).solve(b, SolverConfig(method=method, tol=1e-10))
    assert rep.converged and rep.iterations <= 1, rep
    r = torch.as_tensor(b).cuda() - A.apply(x)
    assert float(r.norm() / np.linalg.norm(b)) < 1e-10
