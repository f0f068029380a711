"""Solve one BASELINE.json workload on cuda:0 and print a JSON summary.

    python tools/run_config.py wedge3 --n 257      (configs[2] at reduced size)
    python tools/run_config.py wedge3 --n 513      (configs[2])
    python tools/run_config.py cube --n 129        (configs[1])
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2308_06085_b200 import problems
    from paper_2308_06085_b200.grid import full_extent
    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator

    ap = argparse.ArgumentParser()
    ap.add_argument("which", choices=["cube", "wedge3", "random"])
    ap.add_argument("--n", type=int, default=129)
    ap.add_argument("--maxit", type=int, default=2000)
    ap.add_argument("--method", default="bicgstab", choices=["bicgstab", "gmres", "idrs"])
    ap.add_argument("--restart", type=int, default=0)
    ap.add_argument("--btol", type=float, default=1e-30)
    ap.add_argument("--shadow", default="rhs", choices=["rhs", "random"])
    args = ap.parse_args()
    t0 = time.perf_counter()
    if args.which == "cube":
        p = problems.point_source_cube(args.n, 80.0 * (args.n - 1) / 128, "sommerfeld")
    elif args.which == "wedge3":
        p = problems.wedge3_problem(args.n)
    else:
        p = problems.random_medium_problem((args.n, args.n, (args.n + 1) // 2))
    spec, b = problems.build_problem(p)
    k = np.asarray(spec.k_field)
    t_host = time.perf_counter() - t0
    t0 = time.perf_counter()
    A = StencilOperator(spec, p.grid)
    H = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, k), MGConfig())
    S = Solver(A, H)
    bd = torch.as_tensor(b).cuda()
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    cfg = SolverConfig(method=args.method, tol=1e-6, maxit=args.maxit, restart=args.restart or None,
                       breakdown_tol=args.btol, shadow=args.shadow, check_every=16)
    x, rep = S.solve(bd, cfg)
    n = p.grid.num_vertices
    print(json.dumps({"problem": args.which, "method": args.method, "shadow": args.shadow,
                      "coarsest": H.coarsest_kind, "breakdown_tol": args.btol, "grid": list(p.grid.shape), "unknowns": n,
                      "kh_max": float(np.max(k) * p.grid.h), "levels": [lv.grid.n1 for lv in H.levels],
                      "iterations": rep.iterations, "converged": rep.converged,
                      "final_relres": rep.final_relres, "breakdown": rep.breakdown,
                      "history_tail": [float(v) for v in rep.residual_history[-3:]],
                      "history_every100": [float(v) for v in rep.residual_history[::100]], "solve_s": rep.wall_time,
                      "munknowns_iter_per_s": n * rep.iterations / rep.wall_time / 1e6,
                      "setup_s": t_setup, "host_problem_s": t_host,
                      "gpu_mem_gb": torch.cuda.max_memory_allocated() / 1e9}))


if __name__ == "__main__":
    main()
