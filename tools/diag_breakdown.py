"""Bi-CGSTAB rho breakdown on the wedge: stop just before it and look at the
true residual at the source vertex (rho = conj(b_s) r_s for a point source)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    n = int(sys.argv[1])
    p = problems.wedge3_problem(n)
    spec, b = problems.build_problem(p)
    A = StencilOperator(spec, p.grid)
    H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field), MGConfig())
    S = Solver(A, H)
    bd = torch.as_tensor(b).cuda()
    src = np.unravel_index(np.argmax(np.abs(b)), b.shape)
    x, rep = S.solve(bd, SolverConfig(method="bicgstab", tol=1e-6, maxit=3000))
    it = rep.iterations
    out = {"iterations": it, "breakdown": rep.breakdown, "source": [int(v) for v in src]}
    for m in (it - 3, it - 2, it - 1):
        x, rep2 = S.solve(bd, SolverConfig(method="bicgstab", tol=1e-6, maxit=m))
        r = (bd - A.apply(x)).cpu().numpy()
        out[f"it{m}"] = {"r_source": [float(r[src].real), float(r[src].imag)],
                         "r_norm": float(np.linalg.norm(r)), "b_source": float(abs(b[src])),
                         "max_abs_r": float(np.abs(r).max()),
                         "r_source_neighbours": [float(abs(r[src[0], src[1], src[2] + d])) for d in (-1, 1)]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
