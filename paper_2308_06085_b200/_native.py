"""ctypes bindings of the C ABI declared in include/helmfree_b200.h.

The product path has no fallback: if libhelmfree_b200.so is missing or
cannot be loaded, importing a compute entry point raises NativeUnavailable.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HF_LIB_PATH") or os.path.join(_HERE, "_lib", "libhelmfree_b200.so")   # override: A/B builds

HF_GHOST = 2
BC = {"dirichlet": 0, "sommerfeld": 1}
CYCLE = {"V": 0, "F": 1}
METHOD = {"gmres": 0, "bicgstab": 1, "idrs": 2}
COARSEST = {"direct": 0, "gmres": 1, "external": 2}
SHADOW = {"rhs": 0, "random": 2}
BREAKDOWN = {0: None, 1: "arnoldi", 2: "rho", 3: "omega", 4: "projection"}
ERR_ARG = -1
ERR_ZERO_DIAGONAL = -3
ERR_UNSUPPORTED = -4
TRANSPORT = {"local": 0, "nccl": 1}

# every symbol include/helmfree_b200.h declares
EXPORTED = (
    "hf_last_error", "hf_version", "hf_set_stream", "hf_device_synchronize",
    "hf_set_option", "hf_get_option",
    "hf_operator_create", "hf_operator_destroy", "hf_operator_apply", "hf_operator_diag",
    "hf_jacobi_smooth", "hf_hierarchy_create", "hf_hierarchy_destroy",
    "hf_hierarchy_num_levels", "hf_hierarchy_level_shape", "hf_restrict_fw", "hf_prolong_tl",
    "hf_coarsest_solve", "hf_coarsest_kind", "hf_coarsest_flags", "hf_mg_precondition", "hf_level_down1", "hf_level_down_restrict", "hf_level_up", "hf_level_correct", "hf_level_correct_ext",
    "hf_level_smooth", "hf_solver_create", "hf_solver_destroy",
    "hf_solve", "hf_solve_host", "hf_dot", "hf_solver_bench_vec",
    "hf_bcg_create", "hf_bcg_destroy", "hf_bcg_step", "hf_bcg_read", "hf_bcg_vec_init", "hf_bcg_vec_p",
    "hf_bcg_vec_s", "hf_bcg_vec_xr", "hf_bcg_vec_xhalf", "hf_operator_apply_dot",
    "hf_nccl_init", "hf_nccl_unique_id", "hf_slab_create", "hf_slab_destroy", "hf_slab_solve",
)


class NativeUnavailable(ImportError):
    pass


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[hf {code}] {msg}")
        self.code = code


class MGConfigC(ctypes.Structure):
    _fields_ = [("nu1", ctypes.c_int), ("nu2", ctypes.c_int), ("omega", ctypes.c_double),
                ("cycle", ctypes.c_int), ("coarsest_threshold", ctypes.c_int),
                ("threshold_ge", ctypes.c_int), ("coarsest_tol", ctypes.c_double),
                ("coarsest_maxit", ctypes.c_int), ("coarsest_method", ctypes.c_int)]


class SolverConfigC(ctypes.Structure):
    _fields_ = [("method", ctypes.c_int), ("tol", ctypes.c_double), ("maxit", ctypes.c_int),
                ("s", ctypes.c_int), ("restart", ctypes.c_int),
                ("breakdown_tol", ctypes.c_double), ("shadow_host", ctypes.c_void_p),
                ("check_every", ctypes.c_int), ("shadow_kind", ctypes.c_int),
                ("shadow_seed", ctypes.c_uint64)]


class ReportC(ctypes.Structure):
    _fields_ = [("matvec_count", ctypes.c_int), ("iterations", ctypes.c_int),
                ("converged", ctypes.c_int), ("breakdown", ctypes.c_int),
                ("final_relres", ctypes.c_double), ("history_host", ctypes.c_void_p),
                ("history_cap", ctypes.c_int), ("coarsest_flags", ctypes.c_int),
                ("solve_ms", ctypes.c_double), ("kernel_launches", ctypes.c_int)]


_lib = None


def load(path: str = LIB_PATH):
    """Load the native library (once).  Raises NativeUnavailable if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeUnavailable(
            f"{path} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    try:
        L = ctypes.CDLL(path)
    except OSError as exc:
        raise NativeUnavailable(f"cannot load {path}: {exc}") from exc
    vp, dp, ip, i, d = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_double
    sig = {
        "hf_last_error": ([], ctypes.c_char_p),
        "hf_version": ([], i),
        "hf_set_stream": ([vp], None),
        "hf_set_option": ([ctypes.c_char_p, i], i),
        "hf_get_option": ([ctypes.c_char_p], i),
        "hf_device_synchronize": ([], i),
        "hf_operator_create": ([i, i, i, i, i, d, d, d, i, vp, d], vp),
        "hf_operator_destroy": ([vp], None),
        "hf_operator_apply": ([vp, vp, vp], i),
        "hf_operator_diag": ([vp, vp], i),
        "hf_jacobi_smooth": ([vp, vp, vp, d, i, i, vp], i),
        "hf_hierarchy_create": ([i, i, i, i, i, d, d, d, i, vp, d, ctypes.POINTER(MGConfigC)], vp),
        "hf_hierarchy_destroy": ([vp], None),
        "hf_hierarchy_num_levels": ([vp], i),
        "hf_hierarchy_level_shape": ([vp, i, ip], i),
        "hf_restrict_fw": ([vp, i, vp, vp], i),
        "hf_prolong_tl": ([vp, i, vp, vp], i),
        "hf_coarsest_solve": ([vp, vp, vp], i),
        "hf_coarsest_kind": ([vp], i),
        "hf_coarsest_flags": ([vp, i], i),
        "hf_mg_precondition": ([vp, vp, vp], i),
        "hf_level_down1": ([vp, i, vp, vp], i),
        "hf_level_down_restrict": ([vp, i, vp, vp], i),
        "hf_level_up": ([vp, i, vp, vp, vp], i),
        "hf_level_correct": ([vp, i, vp, vp, vp], i),
        "hf_level_correct_ext": ([vp, i, vp, vp, vp], i),
        "hf_level_smooth": ([vp, i, vp, vp, vp], i),
        "hf_solver_create": ([vp, vp], vp),
        "hf_solver_destroy": ([vp], None),
        "hf_solver_bench_vec": ([vp, i, i, ctypes.POINTER(ctypes.c_float)], i),
        "hf_bcg_create": ([vp, d, i, d], vp),
        "hf_bcg_destroy": ([vp], None),
        "hf_bcg_step": ([vp, i, vp], i),
        "hf_bcg_read": ([vp, ip, ctypes.POINTER(ctypes.c_double), vp, i], i),
        "hf_bcg_vec_init": ([vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp], i),
        "hf_bcg_vec_p": ([vp, ctypes.c_int64, vp, vp, vp], i),
        "hf_bcg_vec_s": ([vp, ctypes.c_int64, vp, vp, vp, vp], i),
        "hf_bcg_vec_xr": ([vp, ctypes.c_int64, vp, vp, vp, vp, vp, vp, vp, vp], i),
        "hf_bcg_vec_xhalf": ([vp, ctypes.c_int64, vp, vp], i),
        "hf_operator_apply_dot": ([vp, vp, i, vp, vp, vp, vp], i),
        "hf_solve": ([vp, ctypes.POINTER(SolverConfigC), vp, vp, ctypes.POINTER(ReportC)], i),
        "hf_solve_host": ([vp, ctypes.POINTER(SolverConfigC), vp, vp, ctypes.POINTER(ReportC)], i),
        "hf_dot": ([ctypes.c_int64, vp, vp, dp], i),
        "hf_nccl_init": ([ctypes.c_char_p], i),
        "hf_nccl_unique_id": ([vp], i),
        "hf_slab_create": ([i, i, i, d, d, d, i, vp, d, ctypes.POINTER(MGConfigC), i, ip, ip, i, i, i,
                            vp, i], vp),
        "hf_slab_destroy": ([vp], None),
        "hf_slab_solve": ([vp, ctypes.POINTER(SolverConfigC), ctypes.POINTER(vp), ctypes.POINTER(vp),
                           ctypes.POINTER(ReportC)], i),
    }
    for name in EXPORTED:
        fn = getattr(L, name)
        fn.argtypes, fn.restype = sig[name]
    _lib = L
    return L


def last_error() -> str:
    return load().hf_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc != 0:
        raise NativeError(rc, last_error())


def check_handle(h):
    if not h:
        msg = last_error()
        code = ERR_ZERO_DIAGONAL if "diagonal vanishes" in msg else -1
        raise NativeError(code, msg)
    return h


def set_stream_from_torch() -> None:
    import torch
    load().hf_set_stream(ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))


OPTIONS = ("no_pdl", "no_flat", "no_flat_dr", "no_dr", "tiled_dr", "flat_up", "fuse_up", "no_fuse",
           "coarsest_dense", "no_palette")


def set_option(name: str, value) -> None:
    """Kernel-variant selection (hf_set_option): A/B measurements and the parity
    tests that compare variants.  Every variant computes the same arithmetic."""
    check(load().hf_set_option(name.encode(), 1 if value else 0))


class options:
    """Context manager: `with options(no_flat=1, no_dr=1): ...` (restores on exit)."""

    def __init__(self, **kw):
        self.kw = kw
        self.prev = {}

    def __enter__(self):
        L = load()
        for k, v in self.kw.items():
            self.prev[k] = L.hf_get_option(k.encode())
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.prev.items():
            set_option(k, v)
        return False
