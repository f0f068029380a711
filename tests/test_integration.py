"""The reference-side binding (integration/helmfree_b200.py): the ctypes shim
a maintainer adds to the reference package as helmfree/b200.py.

CPU: every entry point it calls is declared with full argtypes (pointers as
c_void_p -- undeclared ctypes arguments are truncated to a C int), the C
config structs are built from the REFERENCE's own RunConfig (beta1/beta2,
cycle, coarsest settings taken from it, not hard-coded), invalid values are
rejected before any native call.  GPU: a full solve through the shim matches
the C oracle (+-1 iteration, 1e-8)."""

import ctypes
import importlib.util
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def _shim():
    spec = importlib.util.spec_from_file_location("helmfree_b200_shim",
                                                  os.path.join(ROOT, "integration", "helmfree_b200.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _ref_config(overrides=()):
    if not os.path.isdir(REF):
        pytest.skip("reference package not present (build container only)")
    sys.path.insert(0, REF)
    try:
        from helmfree.config import parse_config
    finally:
        sys.path.remove(REF)
    return parse_config("", overrides)


def test_every_called_entry_point_is_declared():
    shim = _shim()
    from paper_2308_06085_b200 import build_native
    build_native.build()
    L = shim.load()
    for name, (args, res) in shim.SIGNATURES.items():
        fn = getattr(L, name)
        assert fn.argtypes == args and fn.restype == res, name
        for a in args:
            assert a not in (ctypes.c_long, ctypes.c_int64) or name == "hf_dot", name
    # a 64-bit host address survives the declared pointer argument
    big = 0x7FCDB7CF8010
    assert ctypes.c_void_p(big).value == big
    assert L.hf_solve_host.argtypes[2] is ctypes.c_void_p


def test_configs_come_from_reference_runconfig():
    shim = _shim()
    cfg = _ref_config(["preconditioner.beta2=0.5", "preconditioner.cycle=F",
                       "solver.method=bicgstab", "preconditioner.coarsest_tol=1e-9",
                       "preconditioner.threshold_cmp=ge", "solver.rng_seed=77"])
    mg, sc, b1, b2 = shim.c_configs(cfg)
    assert (b1, b2) == (1.0, 0.5)                 # not hard-coded
    assert mg.cycle == 1 and mg.threshold_ge == 1 and mg.coarsest_tol == 1e-9
    assert mg.nu1 == cfg.preconditioner["nu1"] and mg.omega == cfg.preconditioner["omega"]
    assert sc.method == 1 and sc.tol == cfg.solver["tol"] and sc.maxit == cfg.solver["maxit"]
    assert sc.shadow_kind == 0 and sc.shadow_seed == 77
    mg, sc, b1, b2 = shim.c_configs(_ref_config())
    assert (b1, b2) == (1.0, -0.5) and sc.method == 0   # reference defaults: gmres, beta2 -0.5


def test_invalid_configs_rejected_before_native_calls():
    shim = _shim()
    good = {"solver": {"method": "bicgstab", "tol": 1e-6, "maxit": 10, "s": 4, "rng_seed": 1,
                       "restart": 0},
            "preconditioner": {"beta1": 1.0, "beta2": -0.5, "omega": 0.8, "nu1": 1, "nu2": 1,
                               "cycle": "V", "coarsest_threshold": 17, "threshold_cmp": "gt",
                               "coarsest_tol": 1e-11, "coarsest_maxit": 2000}}
    shim.c_configs(good)
    for sec, key, val in (("solver", "method", "cg"), ("preconditioner", "cycle", "W"),
                          ("preconditioner", "threshold_cmp", "lt")):
        bad = {s: dict(v) for s, v in good.items()}
        bad[sec][key] = val
        with pytest.raises(shim.B200Error):
            shim.c_configs(bad)

    class G:
        n1 = n2 = n3 = 9
        h = 0.125

    class Spec:
        bc = type("Sommerfeld", (), {})()
        k_field = np.full((9, 9, 9), 4.0)
    with pytest.raises(shim.B200Error, match="rhs shape"):
        shim.solve_on_b200(good, G, Spec, np.zeros((9, 9, 8), complex))


@pytest.mark.gpu
def test_solve_through_shim_matches_oracle(oracle):
    shim = _shim()
    from paper_2308_06085_b200 import problems
    p = problems.point_source_cube(33, 20.0, "sommerfeld")
    spec, b = problems.build_problem(p)
    cfg = {"solver": {"method": "bicgstab", "tol": 1e-6, "maxit": 200, "s": 4, "rng_seed": 1234,
                      "restart": 0},
           "preconditioner": {"beta1": 1.0, "beta2": -0.5, "omega": 0.8, "nu1": 1, "nu2": 1,
                              "cycle": "V", "coarsest_threshold": 17, "threshold_cmp": "gt",
                              "coarsest_tol": 1e-11, "coarsest_maxit": 2000}}
    x, rep = shim.solve_on_b200(cfg, p.grid, spec, b)
    k = np.full(p.grid.shape, 20.0)
    xo, ro = oracle.solve(k, b, p.grid.h, maxit=200)
    its = rep["iterations"] if isinstance(rep, dict) else rep.iterations
    assert abs(its - ro["iterations"]) <= 1
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) < 1e-8
