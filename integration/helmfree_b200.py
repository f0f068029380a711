"""helmfree/b200.py -- the reference-side binding of libhelmfree_b200.so.

This is the file a maintainer adds to the reference package (helmfree,
arxiv 2308.06085) to run its solve path on a B200: a ctypes shim over the C
ABI in include/helmfree_b200.h.  It replaces the solve of
`runner.worker_body` (/root/reference/pkg/src/helmfree/runner.py:95-131) on
one worker that owns the whole grid: StencilOperator + build_hierarchy +
mg_precondition + run_solver become hf_operator_create + hf_hierarchy_create
+ hf_solver_create + hf_solve_host.  It takes the reference's own RunConfig
(solver and preconditioner sections, beta1/beta2 included), Grid3,
OperatorSpec and right-hand side, and returns the reference's
ConvergenceReport.  Only numpy and ctypes are needed (no torch).

Every entry point has full argtypes/restype: a 64-bit pointer passed to an
undeclared ctypes function is truncated to a C int.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["B200Error", "load", "c_configs", "solve_on_b200"]

_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                            "paper_2308_06085_b200", "_lib", "libhelmfree_b200.so")

BC_DIRICHLET, BC_SOMMERFELD = 0, 1
METHODS = {"gmres": 0, "bicgstab": 1, "idrs": 2}
CYCLES = {"V": 0, "F": 1}
COARSEST = {"direct": 0, "gmres": 1}
BREAKDOWNS = {0: None, 1: "arnoldi", 2: "rho", 3: "omega", 4: "projection"}


class B200Error(RuntimeError):
    pass


class MGConfigC(ctypes.Structure):          # hf_mg_config (multigrid.py:42-51 MGConfig)
    _fields_ = [("nu1", ctypes.c_int), ("nu2", ctypes.c_int), ("omega", ctypes.c_double),
                ("cycle", ctypes.c_int), ("coarsest_threshold", ctypes.c_int),
                ("threshold_ge", ctypes.c_int), ("coarsest_tol", ctypes.c_double),
                ("coarsest_maxit", ctypes.c_int), ("coarsest_method", ctypes.c_int)]


class SolverConfigC(ctypes.Structure):      # hf_solver_config (krylov.py:34-43 SolverConfig)
    _fields_ = [("method", ctypes.c_int), ("tol", ctypes.c_double), ("maxit", ctypes.c_int),
                ("s", ctypes.c_int), ("restart", ctypes.c_int),
                ("breakdown_tol", ctypes.c_double), ("shadow_host", ctypes.c_void_p),
                ("check_every", ctypes.c_int), ("shadow_kind", ctypes.c_int),
                ("shadow_seed", ctypes.c_uint64)]


class ReportC(ctypes.Structure):            # hf_report (krylov.py:46-64 ConvergenceReport)
    _fields_ = [("matvec_count", ctypes.c_int), ("iterations", ctypes.c_int),
                ("converged", ctypes.c_int), ("breakdown", ctypes.c_int),
                ("final_relres", ctypes.c_double), ("history_host", ctypes.c_void_p),
                ("history_cap", ctypes.c_int), ("coarsest_flags", ctypes.c_int),
                ("solve_ms", ctypes.c_double), ("kernel_launches", ctypes.c_int)]


_vp, _i, _d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
SIGNATURES = {
    "hf_last_error": ([], ctypes.c_char_p),
    "hf_version": ([], _i),
    "hf_operator_create": ([_i, _i, _i, _i, _i, _d, _d, _d, _i, _vp, _d], _vp),
    "hf_operator_destroy": ([_vp], None),
    "hf_hierarchy_create": ([_i, _i, _i, _i, _i, _d, _d, _d, _i, _vp, _d,
                             ctypes.POINTER(MGConfigC)], _vp),
    "hf_hierarchy_destroy": ([_vp], None),
    "hf_solver_create": ([_vp, _vp], _vp),
    "hf_solver_destroy": ([_vp], None),
    "hf_solve_host": ([_vp, ctypes.POINTER(SolverConfigC), _vp, _vp, ctypes.POINTER(ReportC)], _i),
}
_libs = {}


def load(path: str | None = None):
    """The library with every entry point this shim calls declared."""
    path = path or os.environ.get("HELMFREE_B200_LIB") or _DEFAULT_LIB
    if path not in _libs:
        if not os.path.exists(path):
            raise B200Error(f"{path} not found (build it: python -c 'import __graft_entry__ as g; g.build()')")
        L = ctypes.CDLL(path)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes, fn.restype = args, res
        if L.hf_version() < 2:
            raise B200Error("libhelmfree_b200.so older than ABI version 2")
        _libs[path] = L
    return _libs[path]


def _section(cfg, name):
    sec = getattr(cfg, name, None)
    if sec is None and isinstance(cfg, dict):
        sec = cfg.get(name)
    if sec is None:
        raise B200Error(f"RunConfig has no [{name}] section")
    return sec


def c_configs(cfg, shadow: str = "rhs"):
    """(MGConfigC, SolverConfigC, beta1, beta2) from a reference RunConfig
    (config.py DEFAULTS: [solver] and [preconditioner]).  Raises B200Error for
    values the reference itself would reject (runner.py:77-92)."""
    s, p = _section(cfg, "solver"), _section(cfg, "preconditioner")
    if s["method"] not in METHODS:
        raise B200Error(f"unknown solver.method {s['method']!r}")
    if p["cycle"] not in CYCLES:
        raise B200Error(f"unknown preconditioner.cycle {p['cycle']!r}")
    if p["threshold_cmp"] not in ("gt", "ge"):
        raise B200Error(f"threshold_cmp must be 'gt' or 'ge', got {p['threshold_cmp']!r}")
    if shadow not in ("rhs", "random"):
        raise B200Error(f"unknown shadow {shadow!r}")
    mg = MGConfigC(int(p["nu1"]), int(p["nu2"]), float(p["omega"]), CYCLES[p["cycle"]],
                   int(p["coarsest_threshold"]), 1 if p["threshold_cmp"] == "ge" else 0,
                   float(p["coarsest_tol"]), int(p["coarsest_maxit"]),
                   COARSEST[p.get("coarsest_method", "direct")])
    sc = SolverConfigC(METHODS[s["method"]], float(s["tol"]), int(s["maxit"]), int(s["s"]),
                       int(s["restart"] or 0), 1e-30, None, 4,
                       2 if shadow == "random" else 0, int(s["rng_seed"]) & (2**64 - 1))
    return mg, sc, float(p["beta1"]), float(p["beta2"])


def _bc_code(bc):
    name = type(bc).__name__
    if name == "Sommerfeld":
        return BC_SOMMERFELD
    if name == "Dirichlet":
        return BC_DIRICHLET
    raise B200Error(f"unsupported boundary condition {bc!r}")


def _shadow_space(shape, s, seed):
    """IDR shadow vectors as the reference draws them (krylov.py:279-289)."""
    rng = np.random.default_rng(seed)
    P = []
    for _ in range(s):
        q = (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).astype(np.complex128)
        for pi in P:
            q = q - complex(np.vdot(pi, q)) * pi
        P.append(q / float(np.sqrt(max(np.vdot(q, q).real, 0.0))))
    return np.ascontiguousarray(np.stack(P))


def solve_on_b200(cfg, grid, op_spec, rhs, shadow: str = "rhs", lib_path: str | None = None):
    """Drop-in for the solve of runner.worker_body on one worker owning the
    whole grid.  cfg: reference RunConfig; grid: Grid3 (n1, n2, n3, h); op_spec:
    the Helmholtz OperatorSpec of build_problem (bc, k_field); rhs: complex
    ndarray of grid.shape.  Returns (x, ConvergenceReport)."""
    mg, sc, beta1, beta2 = c_configs(cfg, shadow)
    shape = (int(grid.n1), int(grid.n2), int(grid.n3))
    b = np.ascontiguousarray(rhs, dtype=np.complex128)
    if b.shape != shape:
        raise B200Error(f"rhs shape {b.shape} does not match grid {shape}")
    k = np.ascontiguousarray(np.broadcast_to(np.asarray(op_spec.k_field, dtype=np.float64), shape))
    bc = _bc_code(op_spec.bc)   # Dirichlet lifting lives in the rhs (problems.py:274-300)
    L = load(lib_path)
    n1, n2, n3 = shape
    h = float(grid.h)
    # a constant medium is passed as a scalar (no per-vertex k traffic on the device)
    kconst = float(k.flat[0]) if np.all(k == k.flat[0]) else 0.0
    kp = None if kconst else k.ctypes.data
    A = L.hf_operator_create(n1, n2, n3, 0, n1, h, 1.0, 0.0, bc, kp, kconst)
    if not A:
        raise B200Error(L.hf_last_error().decode())
    M = S = None
    try:
        M = L.hf_hierarchy_create(n1, n2, n3, 0, n1, h, beta1, beta2, bc, kp, kconst,
                                  ctypes.byref(mg))
        if not M:
            raise B200Error(L.hf_last_error().decode())
        S = L.hf_solver_create(A, M)
        if not S:
            raise B200Error(L.hf_last_error().decode())
        P = None
        if sc.method == METHODS["idrs"]:
            P = _shadow_space(shape, sc.s, int(_section(cfg, "solver")["rng_seed"]))
            sc.shadow_host = P.ctypes.data
        x = np.empty_like(b)
        hist = np.zeros(sc.maxit + 2)
        rep = ReportC()
        rep.history_host, rep.history_cap = hist.ctypes.data, len(hist)
        if L.hf_solve_host(S, ctypes.byref(sc), b.ctypes.data, x.ctypes.data, ctypes.byref(rep)):
            raise B200Error(L.hf_last_error().decode())
    finally:
        if S:
            L.hf_solver_destroy(S)
        if M:
            L.hf_hierarchy_destroy(M)
        L.hf_operator_destroy(A)
    fields = dict(method=_section(cfg, "solver")["method"], matvec_count=rep.matvec_count,
                  iterations=rep.iterations, residual_history=hist[:rep.iterations].tolist(),
                  converged=bool(rep.converged), final_relres=float(rep.final_relres),
                  breakdown=BREAKDOWNS[rep.breakdown], wall_time=rep.solve_ms / 1e3)
    try:
        from helmfree.krylov import ConvergenceReport   # inside the reference package
        out = ConvergenceReport(method=fields["method"])
        for key, val in fields.items():
            setattr(out, key, val)
    except ImportError:
        out = fields
    return x, out
