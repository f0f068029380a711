"""Virtual-slab solve on one GPU: host-scalar driver (SlabSolver.solve) vs the
device-resident one (solve_device), 129^3, 1/2/4 slabs."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    from paper_2308_06085_b200.dist import SlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import LocalSlabComm, slab_partition
    p, spec, b = bench._problem("c1")
    for ns in (1, 2, 4):
        ext = slab_partition(p.grid, ns)
        S = SlabSolver(p.grid, ext, spec.k_field, p.bc, LocalSlabComm(ns))
        bs = [b[e.lo1 - 1:e.hi1] for e in ext]
        for name, fn in (("host", S.solve), ("device", S.solve_device)):
            fn(bs, SolverConfig(method="bicgstab"))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, rep = fn(bs, SolverConfig(method="bicgstab"))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"slabs {ns} {name:6s}: {dt * 1e3:8.1f} ms  iterations {rep.iterations}  "
                  f"{dt / rep.iterations * 1e6:7.1f} us/iteration", flush=True)


if __name__ == "__main__":
    main()
