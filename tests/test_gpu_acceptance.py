"""Reference acceptance criteria through the B200 path (runner.run_solve):
criterion 1 at desk size (the reference's demo_convergence matvec counts),
criterion 4 (second-order convergence), criterion 6 (partition invariance)."""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.filterwarnings("ignore:kh =")]

torch = pytest.importorskip("torch")


def _run(*over):
    from paper_2308_06085_b200.config import parse_config
    from paper_2308_06085_b200.runner import run_solve
    return run_solve(parse_config("", overrides=list(over)), write_outputs=False)


@pytest.mark.parametrize("method,matvecs", [("gmres", 27), ("bicgstab", 44), ("idrs", 34)])
def test_demo_convergence_counts(method, matvecs):
    """Reference pkg/out/demo_convergence: ClosedOff 33^3, k=20."""
    rep = _run("problem.n=33", "problem.k=20", f"solver.method={method}")
    assert rep.convergence.converged
    assert abs(rep.convergence.matvec_count - matvecs) <= 2
    assert rep.error_max is not None and abs(rep.error_max - 0.01105) < 1e-4


def test_second_order_convergence():
    """Criterion 4: ClosedOff k=10 on 17/33/65, max error ratios in [3, 5]."""
    errs = [_run(f"problem.n={n}", "problem.k=10", "solver.tol=1e-8",
                 "solver.method=bicgstab").error_max for n in (17, 33, 65)]
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.0 <= r1 <= 5.0 and 3.0 <= r2 <= 5.0, (errs, r1, r2)


def test_partition_invariance():
    """Criterion 6: slab-distributed vs single solve, ClosedOff 33^3 k=20, <= 1e-8."""
    a = _run("problem.n=33", "problem.k=20", "solver.method=bicgstab")
    b = _run("problem.n=33", "problem.k=20", "solver.method=bicgstab", "topology.npx0=2")
    assert abs(a.convergence.iterations - b.convergence.iterations) <= 1
    assert np.abs(a.field - b.field).max() < 1e-8
