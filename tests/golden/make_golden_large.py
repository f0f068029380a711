"""Reference-produced fixtures at BASELINE sizes (test infrastructure only).

Runs the REFERENCE package (helmfree, imported from /root/reference/pkg/src)
through its own solve path -- StencilOperator / build_hierarchy /
mg_precondition / run_solver, exactly as runner.worker_body wires them
(/root/reference/pkg/src/helmfree/runner.py:95-131) -- on:

  * BASELINE configs[1]: the 129^3 k=80 Sommerfeld cube, centre point source;
  * the BASELINE configs[2] three-layer wedge at 65^3 and 129^3;
  * the 257^3 wedge (optional, hours of CPU): where the native solver stops on
    the reference's rho breakdown test (krylov.py:236).

For each case it stores the iteration / matvec counts, the FULL residual
history, the breakdown flag, the solution norm and a strided solution sample,
plus the iterate after a fixed number of iterations (maxit=K, K=15).

The rounding band: the reference's inner product is np.vdot
(partition.py:611-617), whose summation order is the BLAS build's choice.  The
same solve is repeated with ctx.dot re-implemented in seven other summation
orders (pairwise, 256/1024/4096/65536-chunked, reversed, reversed 4096-chunked),
and every variant's iteration count, history and distance from the shipped
order's solution is stored; the parity tests assert native results inside
the band the reference itself spans.

The wedge's k field is the BASELINE configs[2] medium from
paper_2308_06085_b200.problems.PlaneLayeredMedium (the reference has no
tilted-plane-in-unit-depth builder; the medium is an input array to its
operators, operators.py:122-147).

Usage (build container; the reference does not travel to the GPU box):
    python tests/golden/make_golden_large.py cube129 wedge65 wedge129 [wedge257]
Outputs tests/golden/large_<case>.json (one file per case).
"""

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from helmfree.grid import HaloField, full_extent, make_grid  # noqa: E402
from helmfree.krylov import SolverConfig, run_solver  # noqa: E402
from helmfree.multigrid import MGConfig, build_hierarchy, mg_precondition  # noqa: E402
from helmfree.operators import OperatorSpec, Sommerfeld, StencilOperator  # noqa: E402
from helmfree.partition import (DistContext, Exchanger, NullFabric,  # noqa: E402
                                PhaseTimers, Topology)

OUT = os.path.dirname(os.path.abspath(__file__))
FIXED_K = 15


class _Medium:
    def __init__(self, k):
        self.k = k

    def k_field(self, grid, extent):
        return self.k


def _dot_chunked(chunk):
    def dot(self, u, v):
        a, b = np.conj(u.ravel()), v.ravel()
        n = a.size
        parts = [np.dot(a[i:i + chunk], b[i:i + chunk]) for i in range(0, n, chunk)]
        return complex(sum(parts))
    return dot


def _dot_reversed(self, u, v):
    return complex(np.dot(np.conj(u.ravel()[::-1]), v.ravel()[::-1]))


def _dot_pairwise(self, u, v):
    return complex(np.sum(np.conj(u) * v))


def _dot_reversed_chunked(chunk):
    f = _dot_chunked(chunk)

    def dot(self, u, v):
        return f(self, u.ravel()[::-1], v.ravel()[::-1])
    return dot


VARIANTS = {
    "vdot": None,  # the reference as shipped (np.vdot, BLAS order)
    "pairwise": _dot_pairwise,
    "chunk4096": _dot_chunked(4096),
    "reversed": _dot_reversed,
    "chunk256": _dot_chunked(256),
    "chunk1024": _dot_chunked(1024),
    "chunk65536": _dot_chunked(65536),
    "reversed_chunk4096": _dot_reversed_chunked(4096),
}


def problem(case):
    """(grid, k field, rhs) built with the reference's own builders."""
    from helmfree.problems import ConstantK, ProblemSpec, build_problem
    if case == "cube129":
        n = 129
        grid = make_grid(n, n, n, 1.0 / (n - 1))
        ps = ProblemSpec("PointSource", grid, ConstantK(80.0), Sommerfeld(),
                         {"type": "dirac", "at": (0.5, 0.5, 0.5)})
    elif case.startswith("wedge"):
        n = int(case[5:])
        from paper_2308_06085_b200.problems import wedge3_problem
        from paper_2308_06085_b200.grid import full_extent as my_full
        mine = wedge3_problem(n)
        grid = make_grid(n, n, n, 1.0 / (n - 1))
        k = mine.medium.k_field(mine.grid, my_full(mine.grid))
        ps = ProblemSpec("Wedge3", grid, _Medium(np.ascontiguousarray(k)), Sommerfeld(),
                         {"type": "dirac", "at": (0.5, 0.5, 0.1)})
    else:
        raise SystemExit(f"unknown case {case}")
    spec, rhs = build_problem(ps, full_extent(grid))
    return grid, spec.k_field, rhs.owned.copy()


def solve(grid, k, rhs, maxit, variant, tol=1e-6, x_ref=None):
    ext = full_extent(grid)
    ctx = DistContext(Topology(1, 1, 1), 0, NullFabric(), grid=grid, extent=ext,
                      timers=PhaseTimers())
    if VARIANTS[variant] is not None:
        ctx.dot = VARIANTS[variant].__get__(ctx)
    exch = Exchanger(ctx.topo, 0, ctx.fabric)
    A = StencilOperator(OperatorSpec("helmholtz", 1.0, 0.0, Sommerfeld(), k), grid, ext,
                        exchanger=exch)
    hier = build_hierarchy(grid, ext, OperatorSpec("cslp", 1.0, -0.5, Sommerfeld(), k),
                           MGConfig(), ctx)
    xb, rb = HaloField(ext), HaloField(ext)

    def aa(x):
        xb.owned[...] = x
        xb.invalidate_halo()
        return A.apply(xb).owned.copy()

    def mm(x):
        rb.owned[...] = x
        rb.invalidate_halo()
        return mg_precondition(hier, rb).owned.copy()

    t0 = time.perf_counter()
    x, rep = run_solver(aa, mm, rhs.copy(), ctx, SolverConfig(method="bicgstab", tol=tol,
                                                             maxit=maxit))
    st = max(1, (grid.n1 - 1) // 8)
    out = {
        "variant": variant, "maxit": maxit, "tol": tol,
        "iterations": rep.iterations, "matvec_count": rep.matvec_count,
        "converged": bool(rep.converged), "breakdown": rep.breakdown,
        "final_relres": rep.final_relres, "residual_history": rep.residual_history,
        "x_norm": float(np.linalg.norm(x)),
        "sample_stride": st,
        "x_sample_re": np.real(x[::st, ::st, ::st]).ravel().tolist(),
        "x_sample_im": np.imag(x[::st, ::st, ::st]).ravel().tolist(),
        "wall_s": time.perf_counter() - t0,
    }
    if x_ref is not None:   # band: the variant's distance from the shipped-order run
        out["x_rel_diff_vs_vdot"] = float(np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
        del out["x_sample_re"], out["x_sample_im"]
    return out, x


def main(cases):
    for case in cases:
        grid, k, rhs = problem(case)
        big = case == "wedge257"
        maxit = 3000 if case.startswith("wedge") else 400
        out = {"case": case, "shape": list(grid.shape), "h": grid.h,
               "k_min": float(np.min(k)), "k_max": float(np.max(k)),
               "beta": [1.0, -0.5], "mg": "V(1,1) omega=0.8 (MGConfig defaults)",
               "source": [int(i) for i in np.unravel_index(np.argmax(np.abs(rhs)), rhs.shape)],
               "generated_by": "tests/golden/make_golden_large.py (reference helmfree)",
               "runs": []}
        variants = ["vdot"] if big else list(VARIANTS)
        x0 = None
        for v in variants:
            r, x = solve(grid, k, rhs, maxit, v, x_ref=x0)
            if x0 is None:
                x0 = x
            print(case, v, r["iterations"], r["breakdown"], r["final_relres"],
                  f"{r['wall_s']:.0f}s", flush=True)
            out["runs"].append(r)
            _write(case, out)
        if not big:
            r, _ = solve(grid, k, rhs, FIXED_K, "vdot")
            out["fixed"] = r
            print(case, "fixed", FIXED_K, r["final_relres"], flush=True)
        _write(case, out)


def _write(case, out):
    with open(os.path.join(OUT, f"large_{case}.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main(sys.argv[1:] or ["cube129", "wedge65", "wedge129"])
