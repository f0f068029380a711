"""Diagnostic: native vs oracle for apply / one MG cycle on several grids."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2308_06085_b200.grid import make_grid  # noqa: E402
from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy, mg_precondition  # noqa: E402
from paper_2308_06085_b200.operators import OperatorSpec, Sommerfeld, Dirichlet, StencilOperator  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


rng = np.random.default_rng(0)
for n, kv, bc, th in [(33, 20.0, "sommerfeld", 17), (65, 40.0, "sommerfeld", 17), (65, 40.0, "sommerfeld", 33),
                      (65, 40.0, "dirichlet", 17), (129, 80.0, "sommerfeld", 65)]:
    g = make_grid(n, n, n, 1.0 / (n - 1))
    k = np.full(g.shape, kv)
    r = rng.standard_normal(g.shape) + 1j * rng.standard_normal(g.shape)
    B = Sommerfeld() if bc == "sommerfeld" else Dirichlet(0.0)
    spec = OperatorSpec("cslp", 1.0, -0.5, B, k)
    hier = build_hierarchy(g, None, spec, MGConfig(coarsest_threshold=th))
    oh = O.Hierarchy(k, g.h, bc=bc, threshold=th)
    z = mg_precondition(hier, r).cpu().numpy()
    zo = oh.precondition(r)
    a = StencilOperator(spec, g).apply(r).cpu().numpy()
    ao = O.apply(k, r, g.h, spec.shift, bc)
    print(n, kv, bc, "levels", [l.grid.n1 for l in hier.levels], "apply", rel(a, ao), "cycle", rel(z, zo), flush=True)
