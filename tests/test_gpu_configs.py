"""Parity of the BASELINE workload builders and of the seeded-shadow extension
at sizes the C oracle solves in seconds.

* configs[4] medium (seeded Gaussian random field + ellipsoidal 4500 m/s body,
  kh = 0.625 at the slowest velocity) on a 65 x 65 x 33 grid: native vs oracle
  within +-1 iteration and 1e-8;
* SolverConfig.shadow = "random" (HF_SHADOW_HASH, the B200 addition that
  converges where the reference's r~ = b stops on the rho test): native vs the
  oracle's restatement of the same hash vector: identical early residual
  histories (1e-8), +-1 iteration, solutions within the tolerance band, on the
  wedge and the random medium.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _native(p, k, b, shadow="rhs", maxit=600):
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, Sommerfeld, StencilOperator
    A = StencilOperator(OperatorSpec("helmholtz", 1.0, 0.0, Sommerfeld(), k), p.grid)
    H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, Sommerfeld(), k), MGConfig())
    x, rep = Solver(A, H).solve(b, SolverConfig(method="bicgstab", maxit=maxit, shadow=shadow))
    return x.cpu().numpy(), rep


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _case(name):
    from paper_2308_06085_b200 import problems
    if name == "random":
        p = problems.random_medium_problem((65, 65, 33))
    else:
        p = problems.wedge3_problem(65)
    spec, b = problems.build_problem(p)
    return p, np.ascontiguousarray(spec.k_field, dtype=np.float64), b


def test_random_medium_matches_oracle(oracle):
    p, k, b = _case("random")
    assert k.max() * p.grid.h <= 0.625 * (1 + 1e-12) and np.ptp(k) > 0
    x, rep = _native(p, k, b)
    xo, ro = oracle.solve(k, b, p.grid.h, maxit=600)
    assert rep.converged == ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert _rel(x, xo) < 1e-8


@pytest.mark.parametrize("name", ["wedge", "random"])
def test_random_shadow_matches_oracle(oracle, name):
    p, k, b = _case(name)
    x, rep = _native(p, k, b, shadow="random")
    xo, ro = oracle.solve(k, b, p.grid.h, maxit=600, shadow="random", rng_seed=1234)
    # the same shadow vector drives both: the residual histories coincide until
    # rounding amplification sets in
    np.testing.assert_allclose(rep.residual_history[:10], ro["residual_history"][:10], rtol=1e-8)
    assert rep.converged and ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    # with a dense random shadow the end of the solve is rounding-sensitive
    # (measured: 6.8e-7 relative at 65^3, both at relres <= 1e-6): the solutions
    # agree to the tolerance band, not to 1e-8 as with r~ = b at this size
    assert _rel(x, xo) < 1e-5
