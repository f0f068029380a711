"""Parity at BASELINE sizes, pinned to the REFERENCE itself.

tests/golden/large_*.json hold runs of the reference package (helmfree)
through its own solve path (tests/golden/make_golden_large.py): BASELINE
configs[1] (129^3 k=80 cube) and the configs[2] wedge at 65^3 and 129^3,
solved with the inner product re-associated (np.vdot as shipped, pairwise,
256/1024/4096/65536-chunked, reversed, reversed-chunked; four orders at 65^3).
Those runs ARE the reference's rounding band:

  * wedge 65^3   iterations 40 in every order,  solutions within 7e-13
  * cube 129^3   iterations 90..95 (8 orders),  solutions within 7.1e-6
  * wedge 129^3  iterations 197..216 (8 orders), solutions within 1.1e-5

so the north_star bar (+-1 iteration, 1e-8 relative L2) is what the reference
itself meets at 65^3, and at 129^3 the reference does not meet it against
itself.  The tests assert:
  * at 129^3 the CPU oracle and the native B200 solve inside the reference's
    band widened by half its width (eight samples of a rounding distribution
    understate its tails; the native path also differs from the reference by
    an exact coarsest solve and FMA contraction, perturbations of the same
    rounding size), solutions within twice the band;
  * at 65^3 the bar itself: +-1 iteration and 1e-8 on the solution sample;
  * the iterate after a FIXED number of iterations (15, before rounding
    amplification dominates) against the reference's;
  * full residual histories against the reference's until they leave the band;
  * resolved solutions: native and oracle both to tol 1e-12 agree to 1e-8.
"""

import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(case):
    with open(os.path.join(GOLD, f"large_{case}.json")) as f:
        return json.load(f)


def _band(g):
    """(lo, hi, sol): the reference's iteration range widened by half its width
    (at least the bar's +-1), and its largest solution spread."""
    its = [r["iterations"] for r in g["runs"]]
    sol = max([r.get("x_rel_diff_vs_vdot", 0.0) for r in g["runs"]])
    m = max(1, (max(its) - min(its) + 1) // 2)
    return min(its) - m, max(its) + m, sol


def _sample(x, g, run=None):
    st = (run or g["runs"][0])["sample_stride"]
    return x[::st, ::st, ::st].ravel()


def _ref_sample(run):
    return np.asarray(run["x_sample_re"]) + 1j * np.asarray(run["x_sample_im"])


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _problem(case):
    from paper_2308_06085_b200 import problems
    if case == "cube129":
        p = problems.point_source_cube(129, 80.0, "sommerfeld")
    else:
        p = problems.wedge3_problem(int(case[5:]))
    spec, b = problems.build_problem(p)
    return p, np.ascontiguousarray(spec.k_field, dtype=np.float64), b


def test_fixtures_are_reference_runs():
    for case in ("cube129", "wedge65", "wedge129"):
        g = _gold(case)
        assert "reference helmfree" in g["generated_by"]
        assert {"vdot", "pairwise", "chunk4096", "reversed"} <= {r["variant"] for r in g["runs"]}
        for r in g["runs"]:
            assert r["converged"] and r["final_relres"] <= 1e-6
            assert len(r["residual_history"]) == r["iterations"]


def test_problem_inputs_match_fixture():
    for case in ("cube129", "wedge65"):
        g = _gold(case)
        p, k, b = _problem(case)
        assert list(p.grid.shape) == g["shape"] and abs(p.grid.h - g["h"]) < 1e-15
        assert [int(i) for i in np.unravel_index(np.argmax(np.abs(b)), b.shape)] == g["source"]
        assert np.isclose(k.min(), g["k_min"], rtol=0, atol=0) and k.max() == g["k_max"]


def test_oracle_meets_bar_at_65(oracle):
    """65^3 wedge: the C oracle (GMRES coarsest as the reference) within +-1
    iteration and 1e-8 of every reference run."""
    g = _gold("wedge65")
    p, k, b = _problem("wedge65")
    x, rep = oracle.solve(k, b, p.grid.h, maxit=400)
    for r in g["runs"]:
        assert abs(rep["iterations"] - r["iterations"]) <= 1
    assert _rel(_sample(x, g), _ref_sample(g["runs"][0])) < 1e-8
    np.testing.assert_allclose(rep["residual_history"], g["runs"][0]["residual_history"], rtol=1e-6)


def test_oracle_fixed_iterations_65(oracle):
    g = _gold("wedge65")
    p, k, b = _problem("wedge65")
    x, rep = oracle.solve(k, b, p.grid.h, maxit=g["fixed"]["iterations"])
    assert rep["iterations"] == g["fixed"]["iterations"]
    assert _rel(_sample(x, g, g["fixed"]), _ref_sample(g["fixed"])) < 1e-10


def test_oracle_inside_reference_band_cube129(oracle):
    g = _gold("cube129")
    lo, hi, sol = _band(g)
    p, k, b = _problem("cube129")
    x, rep = oracle.solve(k, b, p.grid.h, maxit=400)
    assert lo <= rep["iterations"] <= hi, (rep["iterations"], lo, hi)
    assert _rel(_sample(x, g), _ref_sample(g["runs"][0])) < 2 * sol


# ----------------------------------------------------------------------------
# native B200 solve
# ----------------------------------------------------------------------------
def _native_solve(p, spec_k, b, tol=1e-6, maxit=400, shadow="rhs"):
    import torch

    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, Sommerfeld, StencilOperator
    A = StencilOperator(OperatorSpec("helmholtz", 1.0, 0.0, Sommerfeld(), spec_k), p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, Sommerfeld(), spec_k),
                           MGConfig())
    x, rep = Solver(A, hier).solve(torch.as_tensor(b).cuda(),
                                   SolverConfig(method="bicgstab", tol=tol, maxit=maxit,
                                                shadow=shadow))
    return x.cpu().numpy(), rep


@pytest.mark.gpu
def test_native_meets_bar_at_65():
    g = _gold("wedge65")
    p, k, b = _problem("wedge65")
    x, rep = _native_solve(p, k, b)
    for r in g["runs"]:
        assert abs(rep.iterations - r["iterations"]) <= 1
    assert _rel(_sample(x, g), _ref_sample(g["runs"][0])) < 1e-8
    n = min(rep.iterations, g["runs"][0]["iterations"])
    np.testing.assert_allclose(rep.residual_history[:n], g["runs"][0]["residual_history"][:n],
                               rtol=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cube129", "wedge129"])
def test_native_inside_reference_band_129(case):
    g = _gold(case)
    lo, hi, sol = _band(g)
    p, k, b = _problem(case)
    x, rep = _native_solve(p, k, b)
    assert rep.converged and rep.final_relres <= 1e-6
    assert lo <= rep.iterations <= hi, (rep.iterations, lo, hi)
    assert _rel(_sample(x, g), _ref_sample(g["runs"][0])) < 2 * sol
    # histories agree with the reference's until rounding amplification (the
    # reference's own variants agree to 1e-9 over the first 15 iterations)
    np.testing.assert_allclose(rep.residual_history[:15], g["runs"][0]["residual_history"][:15],
                               rtol=1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["cube129", "wedge129", "wedge65"])
def test_native_fixed_iterations_match_reference(case):
    """The iterate after 15 Bi-CGSTAB iterations (rounding not yet amplified)
    against the reference's: the B200 coarsest solve is exact where the
    reference iterates GMRES to 1e-11, which bounds the agreement."""
    g = _gold(case)
    p, k, b = _problem(case)
    x, rep = _native_solve(p, k, b, maxit=g["fixed"]["iterations"])
    assert rep.iterations == g["fixed"]["iterations"]
    assert _rel(_sample(x, g, g["fixed"]), _ref_sample(g["fixed"])) < 1e-8


@pytest.mark.gpu
def test_native_resolved_solution_matches_oracle(oracle):
    """Both solved to 1e-12 (past the rounding band): the solutions agree to 1e-8."""
    p, k, b = _problem("cube129")
    x, rep = _native_solve(p, k, b, tol=1e-12, maxit=1000)
    assert rep.converged
    with oracle.exact_coarsest(k, p.grid.h):
        xo, ro = oracle.solve(k, b, p.grid.h, tol=1e-12, maxit=1000)
    assert ro["converged"]
    assert _rel(x, xo) < 1e-8
