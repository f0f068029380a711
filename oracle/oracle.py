"""ctypes front end of the C oracle (oracle/helmfree_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference leg of bench.py -- never by the product
package.  Arrays follow the reference layout: complex128 / float64 of shape
(n1, n2, n3), C order.

Each wrapper names the reference function it restates
(/root/reference/pkg/src/helmfree/...).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libhelmfree_oracle.so")
_lib = None

BC_CODES = {"dirichlet": 0, "sommerfeld": 1}
METHODS = {"gmres": 0, "bicgstab": 1, "idrs": 2}
BREAKDOWNS = {0: None, 1: "arnoldi", 2: "rho", 3: "omega", 4: "projection"}

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p


def build() -> str:
    """Compile the oracle with its Makefile (gcc + OpenMP)."""
    env = dict(os.environ)
    subprocess.run(["make", "-s", "-C", _HERE], check=True, env=env)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_apply.argtypes = [ctypes.c_int] * 3 + [ctypes.c_double] * 3 + [ctypes.c_int, _dp, _vp, _vp]
        L.or_apply.restype = None
        L.or_hier_create.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_double] * 3 + [ctypes.c_int, _dp]
                                     + [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                        ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int])
        L.or_hier_create.restype = _vp
        L.or_hier_free.argtypes = [_vp]
        L.or_hier_nlev.argtypes = [_vp]
        L.or_hier_nlev.restype = ctypes.c_int
        L.or_hier_level_dims.argtypes = [_vp, ctypes.c_int, _ip]
        L.or_hier_stats.argtypes = [_vp, _ip]
        L.or_hier_apply.argtypes = [_vp, ctypes.c_int, _vp, _vp]
        L.or_hier_diag.argtypes = [_vp, ctypes.c_int, _vp]
        L.or_hier_jacobi.argtypes = [_vp, ctypes.c_int, _vp, _vp, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.or_hier_restrict.argtypes = [_vp, ctypes.c_int, _vp, _vp]
        L.or_hier_prolong.argtypes = [_vp, ctypes.c_int, _vp, _vp]
        L.or_hier_coarsest.argtypes = [_vp, _vp, _vp]
        L.or_mg_precondition.argtypes = [_vp, _vp, _vp]
        L.or_solve.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_double, ctypes.c_int, _dp, _vp, _vp,
                                                   ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                                   ctypes.c_int, _vp, ctypes.c_double, ctypes.c_double,
                                                   ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                                   ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                                   _ip, _ip, _ip, _ip, _dp, _dp, ctypes.c_int, _ip])
        L.or_solve.restype = ctypes.c_int
        L.or_num_threads.restype = ctypes.c_int
        L.or_set_coarse_inverse.argtypes = [_vp, ctypes.c_size_t]
        L.or_set_dot_chunks.argtypes = [ctypes.c_int]
        L.or_set_bicgstab_shadow.argtypes = [ctypes.c_int, ctypes.c_ulonglong]
        L.or_solver_create.argtypes = ([ctypes.c_int] * 3 + [ctypes.c_double, ctypes.c_int, _dp,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_double, ctypes.c_int])
        L.or_solver_create.restype = _vp
        L.or_solver_free.argtypes = [_vp]
        L.or_solver_solve.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                      _ip, _ip, _ip, _dp]
        _lib = L
    return _lib


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return lib().or_num_threads()


def apply(k, u, h, shift=1.0 + 0.0j, bc="sommerfeld"):
    """v = A u (shift 1) or M u (CSLP shift) -- operators.py:200-254."""
    k = _f64(k)
    u = _c128(u)
    v = np.empty_like(u)
    n1, n2, n3 = u.shape
    lib().or_apply(n1, n2, n3, float(h), float(np.real(shift)), float(np.imag(shift)),
                   BC_CODES[bc], k.ctypes.data_as(_dp), _ptr(u), _ptr(v))
    return v


class Hierarchy:
    """multigrid.py:101-128 build_hierarchy on the full grid (one worker)."""

    def __init__(self, k, h, beta1=1.0, beta2=-0.5, bc="sommerfeld", nu1=1, nu2=1, omega=0.8,
                 cycle="V", threshold=17, threshold_cmp="gt", coarsest_tol=1e-11,
                 coarsest_maxit=2000):
        self.k = _f64(k)
        n1, n2, n3 = self.k.shape
        self._h = lib().or_hier_create(n1, n2, n3, float(h), float(beta1), float(beta2),
                                       BC_CODES[bc], self.k.ctypes.data_as(_dp), int(nu1), int(nu2),
                                       float(omega), 1 if cycle.upper() == "F" else 0,
                                       int(threshold), 1 if threshold_cmp == "ge" else 0,
                                       float(coarsest_tol), int(coarsest_maxit))
        self.nlev = lib().or_hier_nlev(self._h)
        self.shapes = []
        for l in range(self.nlev):
            d = (ctypes.c_int * 3)()
            lib().or_hier_level_dims(self._h, l, d)
            self.shapes.append((d[0], d[1], d[2]))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_hier_free(self._h)
            self._h = None

    def stats(self):
        d = (ctypes.c_int * 3)()
        lib().or_hier_stats(self._h, d)
        return {"coarsest_calls": d[0], "coarsest_iters": d[1], "coarsest_fail": d[2]}

    def apply(self, l, u):
        u = _c128(u)
        v = np.empty_like(u)
        lib().or_hier_apply(self._h, l, _ptr(u), _ptr(v))
        return v

    def diag(self, l):
        d = np.empty(self.shapes[l], dtype=np.complex128)
        lib().or_hier_diag(self._h, l, _ptr(d))
        return d

    def jacobi(self, l, u, b, omega=0.8, sweeps=1, assume_zero=False):
        u = _c128(u).copy()
        b = _c128(b)
        lib().or_hier_jacobi(self._h, l, _ptr(u), _ptr(b), float(omega), int(sweeps),
                             1 if assume_zero else 0)
        return u

    def restrict(self, l, r):
        r = _c128(r)
        out = np.empty(self.shapes[l + 1], dtype=np.complex128)
        lib().or_hier_restrict(self._h, l, _ptr(r), _ptr(out))
        return out

    def prolong(self, l, e):
        e = _c128(e)
        out = np.empty(self.shapes[l], dtype=np.complex128)
        lib().or_hier_prolong(self._h, l, _ptr(e), _ptr(out))
        return out

    def coarsest(self, b):
        b = _c128(b)
        x = np.empty_like(b)
        lib().or_hier_coarsest(self._h, _ptr(b), _ptr(x))
        return x

    def precondition(self, r):
        r = _c128(r)
        z = np.empty_like(r)
        lib().or_mg_precondition(self._h, _ptr(r), _ptr(z))
        return z


def shadow_space(shape, s, seed):
    """krylov.py:279-289 + partition.py:623-629: s orthonormal random complex
    vectors drawn from numpy default_rng(seed) over the full grid (MGS with
    the conjugated inner product)."""
    rng = np.random.default_rng(seed)
    P = []
    for _ in range(s):
        q = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        q = q.astype(np.complex128)
        for pi in P:
            q = q - complex(np.vdot(pi, q)) * pi
        nrm = float(np.sqrt(max(np.vdot(q, q).real, 0.0)))
        P.append(q / nrm)
    return np.ascontiguousarray(np.stack(P)) if P else None


def solve(k, b, h, bc="sommerfeld", method="bicgstab", tol=1e-6, maxit=400, restart=0, s=4,
          rng_seed=1234, beta1=1.0, beta2=-0.5, nu1=1, nu2=1, omega=0.8, cycle="V",
          threshold=17, threshold_cmp="gt", coarsest_tol=1e-11, coarsest_maxit=2000,
          shadow="rhs"):
    """runner.py:95-131 worker body on one worker: Helmholtz A, CSLP cycle
    preconditioner, Krylov method.  Returns (x, report dict).  shadow="random":
    Bi-CGSTAB with the seeded hash shadow vector (seed rng_seed) of the B200
    path's SolverConfig.shadow extension instead of the reference's r~ = b."""
    lib().or_set_bicgstab_shadow(2 if shadow == "random" else 0, int(rng_seed) & (2**64 - 1))
    k = _f64(k)
    b = _c128(b)
    x = np.empty_like(b)
    n1, n2, n3 = b.shape
    P = shadow_space(b.shape, s, rng_seed) if method == "idrs" else None
    hist = np.zeros(maxit + 2, dtype=np.float64)
    mv, it, conv, bd = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    fr = ctypes.c_double()
    stats = (ctypes.c_int * 3)()
    lib().or_solve(n1, n2, n3, float(h), BC_CODES[bc], k.ctypes.data_as(_dp), _ptr(b), _ptr(x),
                   METHODS[method], float(tol), int(maxit), int(restart), int(s),
                   _ptr(P) if P is not None else None, float(beta1), float(beta2), int(nu1),
                   int(nu2), float(omega), 1 if cycle.upper() == "F" else 0, int(threshold),
                   1 if threshold_cmp == "ge" else 0, float(coarsest_tol), int(coarsest_maxit),
                   ctypes.byref(mv), ctypes.byref(it), ctypes.byref(conv), ctypes.byref(bd),
                   ctypes.byref(fr), hist.ctypes.data_as(_dp), len(hist), stats)
    report = {
        "method": method, "matvec_count": mv.value, "iterations": it.value,
        "converged": bool(conv.value), "breakdown": BREAKDOWNS[bd.value],
        "final_relres": fr.value, "residual_history": hist[:it.value].tolist(),
        "coarsest_calls": stats[0], "coarsest_iters": stats[1], "coarsest_fail": stats[2],
    }
    return x, report


def coarse_matrix(H: "Hierarchy") -> np.ndarray:
    """Dense matrix of the coarsest-level operator, column by column through the
    oracle's own matrix-free apply (test helper)."""
    l = H.nlev - 1
    shape = H.shapes[l]
    n = int(np.prod(shape))
    A = np.empty((n, n), dtype=np.complex128)
    e = np.zeros(n, dtype=np.complex128)
    for j in range(n):
        e[j] = 1.0
        A[:, j] = H.apply(l, e.reshape(shape)).ravel()
        e[j] = 0.0
    return A


class exact_coarsest:
    """Context manager: make the oracle's coarsest solve an exact dense-inverse
    GEMV (the B200 path's coarsest_method="direct") instead of GMRES."""

    def __init__(self, k, h, bc="sommerfeld", beta2=-0.5, **mg):
        H = Hierarchy(k, h, beta2=beta2, bc=bc, **mg)
        self.inv = np.ascontiguousarray(np.linalg.inv(coarse_matrix(H)))

    def __enter__(self):
        lib().or_set_coarse_inverse(self.inv.ctypes.data, self.inv.shape[0])
        return self

    def __exit__(self, *exc):
        lib().or_set_coarse_inverse(None, 0)
        return False


class PersistentSolver:
    """A and the CSLP hierarchy built once (or_solver_create); solve() runs one
    Krylov solve without the setup -- the CPU legs of bench.py time this, like
    the native arm, which also excludes its setup."""

    def __init__(self, k, h, bc="sommerfeld", beta1=1.0, beta2=-0.5, nu1=1, nu2=1, omega=0.8,
                 cycle="V", threshold=17, threshold_cmp="gt", coarsest_tol=1e-11,
                 coarsest_maxit=2000):
        self.k = _f64(k)
        n1, n2, n3 = self.k.shape
        self._h = lib().or_solver_create(n1, n2, n3, float(h), BC_CODES[bc],
                                         self.k.ctypes.data_as(_dp), float(beta1), float(beta2),
                                         int(nu1), int(nu2), float(omega),
                                         1 if cycle.upper() == "F" else 0, int(threshold),
                                         1 if threshold_cmp == "ge" else 0, float(coarsest_tol),
                                         int(coarsest_maxit))

    def __del__(self):
        if getattr(self, "_h", None):
            lib().or_solver_free(self._h)
            self._h = None

    def solve(self, b, method="bicgstab", tol=1e-6, maxit=400, x=None):
        b = _c128(b)
        x = np.empty_like(b) if x is None else x
        lib().or_set_bicgstab_shadow(0, 0)
        it, conv, bd = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        fr = ctypes.c_double()
        lib().or_solver_solve(self._h, _ptr(b), _ptr(x), METHODS[method], float(tol), int(maxit),
                              ctypes.byref(it), ctypes.byref(conv), ctypes.byref(bd),
                              ctypes.byref(fr))
        return x, {"iterations": it.value, "converged": bool(conv.value),
                   "breakdown": BREAKDOWNS[bd.value], "final_relres": fr.value}
