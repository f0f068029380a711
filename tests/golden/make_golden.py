"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
package (helmfree, imported from /root/reference/pkg/src) on seeded inputs.

Run in the build container (the reference does not travel to the GPU box):
    python tests/golden/make_golden.py
Outputs:
    kernels.npz   -- apply / restrict / prolong / jacobi / V- and F-cycle outputs
    problems.npz  -- closed-off RHS with Dirichlet lifting, wedge k field, Dirac RHS
    solves.json   -- matvec counts, residual histories and solution samples of
                     full reference solves (incl. BASELINE configs[0])
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from helmfree.grid import HaloField, full_extent, make_grid  # noqa: E402
from helmfree.krylov import SolverConfig, run_solver  # noqa: E402
from helmfree.multigrid import (MGConfig, build_hierarchy, jacobi_smooth,  # noqa: E402
                                mg_precondition, prolong_tl, restrict_fw)
from helmfree.operators import (Dirichlet, OperatorSpec, Sommerfeld,  # noqa: E402
                                StencilOperator)
from helmfree.partition import (DistContext, Exchanger, NullFabric,  # noqa: E402
                                PhaseTimers, Topology)
from helmfree.problems import (ConstantK, ProblemSpec, build_problem,  # noqa: E402
                               closed_off_problem, wedge_problem)

OUT = os.path.dirname(os.path.abspath(__file__))


def ctx_for(grid):
    return DistContext(Topology(1, 1, 1), 0, NullFabric(), grid=grid, extent=full_extent(grid),
                       timers=PhaseTimers())


def field(arr):
    g = HaloField(full_extent(make_grid(*arr.shape, 1.0)))
    g.set_owned(arr.copy())
    return g


def rand(shape, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def kernels():
    out = {}
    rng = np.random.default_rng(2308)
    for dims in [(9, 9, 9), (5, 7, 9)]:
        tag = "x".join(map(str, dims))
        k = rng.uniform(2.0, 6.0, dims)
        u = rand(dims, 1)
        out[f"k_{tag}"] = k
        out[f"u_{tag}"] = u
        for bcn, bc in (("dirichlet", Dirichlet(1.0)), ("sommerfeld", Sommerfeld())):
            for kind in ("helmholtz", "cslp"):
                grid = make_grid(*dims, 0.125)
                op = StencilOperator(OperatorSpec(kind, 1.0, -0.5, bc, k), grid, full_extent(grid))
                f = HaloField(full_extent(grid))
                f.set_owned(u.copy())
                out[f"apply_{tag}_{bcn}_{kind}"] = op.apply(f).owned.copy()
    n = (9, 9, 9)
    k = rng.uniform(2.0, 4.0, n)
    r = rand(n, 3)
    out["k_9"], out["r_9"] = k, r
    for bcn, bc in (("dirichlet", Dirichlet(0.0)), ("sommerfeld", Sommerfeld())):
        grid = make_grid(*n, 1.0 / 8)
        for cyc in ("V", "F"):
            spec = OperatorSpec("cslp", 1.0, -0.5, bc, k)
            hier = build_hierarchy(grid, full_extent(grid), spec,
                                   MGConfig(cycle=cyc, coarsest_threshold=4), ctx_for(grid))
            rf = HaloField(full_extent(grid))
            rf.set_owned(r.copy())
            out[f"cycle_{cyc}_{bcn}"] = mg_precondition(hier, rf).owned.copy()
        fine, coarse = hier.levels[0], hier.levels[1]
        rf = HaloField(full_extent(grid))
        rf.set_owned(r.copy())
        out[f"restrict_{bcn}"] = restrict_fw(rf, fine, coarse).owned.copy()
        ec = rand(coarse.grid.shape, 4)
        out["e_5"] = ec
        fc = HaloField(coarse.extent)
        fc.set_owned(ec.copy())
        out[f"prolong_{bcn}"] = prolong_tl(fc, coarse, fine).owned.copy()
        u = HaloField(full_extent(grid))
        u.set_owned(rand(n, 5))
        b = HaloField(full_extent(grid))
        b.set_owned(r.copy())
        jacobi_smooth(fine.op, u, b, 0.8, 2)
        out[f"jacobi2_{bcn}"] = u.owned.copy()
    out["u0_jacobi"] = rand(n, 5)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def problems():
    out = {}
    p = closed_off_problem(9, 10.0)
    spec, rhs = build_problem(p, full_extent(p.grid))
    out["closed_off_9_k10_rhs"] = rhs.owned.copy()
    w = wedge_problem(shape=(13, 13, 21))
    spec, rhs = build_problem(w, full_extent(w.grid))
    out["wedge_13_k"] = spec.k_field.copy()
    out["wedge_13_rhs"] = rhs.owned.copy()
    np.savez_compressed(os.path.join(OUT, "problems.npz"), **out)


def solve_case(name, grid, k, bc, rhs, method, beta2=-0.5, mg=None, tol=1e-6, maxit=400):
    ext = full_extent(grid)
    ctx = ctx_for(grid)
    exch = Exchanger(ctx.topo, 0, ctx.fabric)
    A = StencilOperator(OperatorSpec("helmholtz", 1.0, 0.0, bc, k), grid, ext, exchanger=exch)
    hier = build_hierarchy(grid, ext, OperatorSpec("cslp", 1.0, beta2, bc, k), mg or MGConfig(), ctx)
    xb, rb = HaloField(ext), HaloField(ext)

    def aa(x):
        xb.owned[...] = x
        xb.invalidate_halo()
        return A.apply(xb).owned.copy()

    def mm(x):
        rb.owned[...] = x
        rb.invalidate_halo()
        return mg_precondition(hier, rb).owned.copy()

    x, rep = run_solver(aa, mm, rhs.copy(), ctx, SolverConfig(method=method, tol=tol, maxit=maxit))
    return {
        "name": name, "shape": list(grid.shape), "h": grid.h, "method": method, "beta2": beta2,
        "bc": "dirichlet" if isinstance(bc, Dirichlet) else "sommerfeld",
        "matvec_count": rep.matvec_count, "iterations": rep.iterations,
        "converged": rep.converged, "final_relres": rep.final_relres,
        "residual_history": rep.residual_history,
        "x_norm": float(np.linalg.norm(x)),
        "x_sample_re": np.real(x[::4, ::4, ::4]).ravel().tolist(),
        "x_sample_im": np.imag(x[::4, ::4, ::4]).ravel().tolist(),
    }


def solves():
    cases = []
    # BASELINE configs[0]: 33^3, k=20, zero Dirichlet, centre unit point source
    n = 33
    grid = make_grid(n, n, n, 1.0 / (n - 1))
    ps = ProblemSpec("PointSource", grid, ConstantK(20.0), Dirichlet(0.0),
                     {"type": "dirac", "at": (0.5, 0.5, 0.5)})
    spec, rhs = build_problem(ps, full_extent(grid))
    k = spec.k_field
    cases.append(solve_case("config0_dirichlet_33_k20", grid, k, Dirichlet(0.0), rhs.owned, "bicgstab"))
    ps = ProblemSpec("PointSource", grid, ConstantK(20.0), Sommerfeld(),
                     {"type": "dirac", "at": (0.5, 0.5, 0.5)})
    spec, rhs = build_problem(ps, full_extent(grid))
    cases.append(solve_case("sommerfeld_33_k20", grid, k, Sommerfeld(), rhs.owned, "bicgstab"))
    # closed-off anchor at desk size, all three methods (README demo_convergence)
    p = closed_off_problem(33, 20.0)
    spec, rhs = build_problem(p, full_extent(p.grid))
    for m in ("gmres", "bicgstab", "idrs"):
        cases.append(solve_case(f"closed_off_33_k20_{m}", p.grid, spec.k_field, p.bc, rhs.owned, m))
    with open(os.path.join(OUT, "solves.json"), "w") as f:
        json.dump(cases, f, indent=1)


if __name__ == "__main__":
    kernels()
    problems()
    solves()
    print("golden fixtures written to", OUT)
