"""Run the C oracle (the reference algorithm restated, test infrastructure) on the
BASELINE configs[2] wedge at a given size and record where Bi-CGSTAB stops:
iteration count, breakdown flag, full residual history, true residual at the
source vertex (rho = conj(b_s) r_s for the reference's shadow r~ = b,
krylov.py:229-238).

    python tools/oracle_wedge.py 257 [--chunks 256] > profiles/r02_oracle_wedge257.json
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from oracle import oracle as O
    from paper_2308_06085_b200 import problems
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("--maxit", type=int, default=3000)
    ap.add_argument("--chunks", type=int, default=256)
    ap.add_argument("--exact-coarsest", action="store_true")
    ap.add_argument("--shadow", default="rhs", choices=["rhs", "random"])
    a = ap.parse_args()
    p = problems.wedge3_problem(a.n)
    spec, b = problems.build_problem(p)
    k = np.ascontiguousarray(spec.k_field)
    O.lib().or_set_dot_chunks(a.chunks)
    t0 = time.perf_counter()
    if a.exact_coarsest:
        with O.exact_coarsest(k, p.grid.h):
            x, rep = O.solve(k, b, p.grid.h, maxit=a.maxit, shadow=a.shadow)
    else:
        x, rep = O.solve(k, b, p.grid.h, maxit=a.maxit, shadow=a.shadow)
    dt = time.perf_counter() - t0
    src = np.unravel_index(np.argmax(np.abs(b)), b.shape)
    r = b - O.apply(k, x, p.grid.h)
    out = {"problem": "wedge3", "n": a.n, "impl": "C oracle (reference algorithm restated)",
           "threads": O.num_threads(), "dot_chunks": a.chunks, "shadow": a.shadow,
           "coarsest": "exact" if a.exact_coarsest else "GMRES to 1e-11 (reference)",
           "iterations": rep["iterations"], "matvec_count": rep["matvec_count"],
           "converged": rep["converged"], "breakdown": rep["breakdown"],
           "final_relres": rep["final_relres"],
           "true_relres": float(np.linalg.norm(r) / np.linalg.norm(b)),
           "source": [int(v) for v in src], "b_source_abs": float(abs(b[src])),
           "r_source_abs": float(abs(r[src])),
           "coarsest_fail": rep["coarsest_fail"], "wall_s": round(dt, 1),
           "residual_history": rep["residual_history"]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
