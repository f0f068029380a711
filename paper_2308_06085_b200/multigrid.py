"""Geometric multigrid approximation of the CSLP inverse, on the B200.

Mirrors /root/reference/pkg/src/helmfree/multigrid.py: MGConfig (:42-51),
build_hierarchy (:101-128), jacobi_smooth (:138-157), restrict_fw
(:171-202), prolong_tl (:238-297), coarsest_solve (:300-323), V/F cycles
(:326-370), mg_precondition (:395-419).  All levels, transfers and the
coarsest solve live in libhelmfree_b200.so.

Coarsest solve: the reference runs unpreconditioned full GMRES to a relative
residual of coarsest_tol (1e-11), max-iterations being a soft failure recorded
in hier.coarsest_flags.  coarsest_method="gmres" runs exactly that on the
device (one cooperative launch per solve, coarsest_tol / coarsest_maxit
honoured, failures counted).  The default, coarsest_method="direct",
factorises the fixed coarsest operator once at setup (fast diagonalisation for
a constant medium, a packed symmetric or dense inverse otherwise) and meets
the same tolerance exactly up to round-off with one pass instead of ~50-70
latency-bound GMRES iterations; it falls back to GMRES when the coarsest grid
has no exact factorisation (over 60000 vertices with a varying medium or
Dirichlet faces).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .grid import BlockExtent, Grid3, HaloField, coarsen, full_extent
from .operators import (OperatorError, OperatorSpec, StencilOperator, ZeroDiagonalError,
                        as_device, bc_name, k_arguments)

__all__ = ["MGConfig", "MGLevel", "MGHierarchy", "MultigridError", "build_hierarchy",
           "jacobi_smooth", "restrict_fw", "prolong_tl", "mg_precondition", "coarsest_solve",
           "keep_coarsening"]


class MultigridError(RuntimeError):
    pass


@dataclass
class MGConfig:
    nu1: int = 1
    nu2: int = 1
    omega: float = 0.8
    cycle: str = "V"
    coarsest_threshold: int = 17
    threshold_cmp: str = "gt"
    coarsest_tol: float = 1e-11
    coarsest_maxit: int = 2000
    coarsest_method: str = "direct"


def keep_coarsening(grid: Grid3, cfg: MGConfig) -> bool:
    """multigrid.py:90-98 stop rule."""
    th = cfg.coarsest_threshold
    if cfg.threshold_cmp == "ge":
        ok = all(n >= th for n in grid.shape)
    elif cfg.threshold_cmp == "gt":
        ok = all(n > th for n in grid.shape)
    else:
        raise MultigridError(f"threshold_cmp must be 'ge' or 'gt', got {cfg.threshold_cmp!r}")
    return ok and grid.is_coarsenable()


@dataclass
class MGLevel:
    grid: Grid3
    extent: BlockExtent
    index: int
    hier: "MGHierarchy"


class MGHierarchy:
    """Native hierarchy handle plus per-level descriptors."""

    def __init__(self, handle, levels_meta, config: MGConfig, ctx=None, spec=None):
        self._h = handle
        self.config = config
        self.ctx = ctx
        self.spec = spec
        self.levels = [MGLevel(g, e, i, self) for i, (g, e) in enumerate(levels_meta)]
        self.coarsest_flags = []

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.load().hf_hierarchy_destroy(h)
            except Exception:   # interpreter shutdown
                pass
            self._h = None

    @property
    def finest(self) -> MGLevel:
        return self.levels[0]

    @property
    def coarsest(self) -> MGLevel:
        return self.levels[-1]

    @property
    def coarsest_kind(self) -> str:
        """Coarsest solve in use: "separable" (fast diagonalisation, constant
        k), "symmetric" / "dense" (inverse), "gmres", or "external"."""
        kind = _native.load().hf_coarsest_kind(self._h)
        return {0: "external", 1: "dense", 2: "symmetric", 3: "separable", 4: "gmres"}[kind]

    def sync_coarsest_flags(self) -> list:
        """Append the device count of coarsest GMRES solves that stopped at
        coarsest_maxit (multigrid.py:320-322) to coarsest_flags and reset it."""
        n = _native.load().hf_coarsest_flags(self._h, 1)
        if n < 0:
            _native.check(n)
        if n:
            self.coarsest_flags.append({"count": int(n)})
        return self.coarsest_flags


def build_hierarchy(finest_grid: Grid3, finest_extent: BlockExtent | None,
                    finest_spec: OperatorSpec, config: MGConfig | None = None,
                    ctx=None) -> MGHierarchy:
    """Hierarchy under the global-coarsening stop rule (multigrid.py:101-128)."""
    config = config or MGConfig()
    extent = finest_extent or full_extent(finest_grid)
    if config.cycle.upper() not in ("V", "F"):
        raise MultigridError(f"unknown cycle type {config.cycle!r}")
    keep_coarsening(finest_grid, config)     # validates threshold_cmp
    if config.coarsest_method not in _native.COARSEST:
        raise MultigridError(f"unknown coarsest_method {config.coarsest_method!r}")
    kfull, kc, keep = k_arguments(finest_spec, finest_grid, extent)
    c = _native.MGConfigC(int(config.nu1), int(config.nu2), float(config.omega),
                          _native.CYCLE[config.cycle.upper()], int(config.coarsest_threshold),
                          1 if config.threshold_cmp == "ge" else 0, float(config.coarsest_tol),
                          int(config.coarsest_maxit), _native.COARSEST[config.coarsest_method])
    L = _native.load()
    _native.set_stream_from_torch()
    h = L.hf_hierarchy_create(finest_grid.n1, finest_grid.n2, finest_grid.n3, extent.lo1 - 1,
                              extent.nx, finest_grid.h, float(finest_spec.beta1),
                              float(finest_spec.beta2), _native.BC[bc_name(finest_spec.bc)],
                              kfull.ctypes.data if kfull is not None else None, kc,
                              ctypes.byref(c))
    if not h:
        msg = _native.last_error()
        if "diagonal vanishes" in msg:
            raise ZeroDiagonalError(msg)
        if "level-incompatible" in msg:
            from .partition import PartitionError
            raise PartitionError(msg)
        raise MultigridError(msg)
    meta = []
    grid = finest_grid
    for l in range(L.hf_hierarchy_num_levels(h)):
        d = (ctypes.c_int * 5)()
        _native.check(L.hf_hierarchy_level_shape(h, l, d))
        if l > 0:
            grid = coarsen(grid)
        assert grid.shape == (d[0], d[1], d[2])
        meta.append((grid, BlockExtent(d[3] + 1, 1, 1, d[3] + d[4], d[1], d[2])))
    return MGHierarchy(h, meta, config, ctx, finest_spec)


def _out_like(shape, out):
    import torch
    if out is not None:
        return out.owned if isinstance(out, HaloField) else out
    return torch.empty(shape, dtype=torch.complex128, device="cuda")


def restrict_fw(r_fine, fine_level: MGLevel, coarse_level: MGLevel, out=None):
    """Full weighting onto the coarse slab (multigrid.py:171-221)."""
    hier = fine_level.hier
    if coarse_level.index != fine_level.index + 1:
        raise MultigridError("restrict_fw needs adjacent levels")
    src = as_device(r_fine)
    dst = _out_like(coarse_level.extent.shape, out)
    _native.set_stream_from_torch()
    _native.check(_native.load().hf_restrict_fw(hier._h, fine_level.index, src.data_ptr(),
                                                 dst.data_ptr()))
    return out if out is not None else dst


def prolong_tl(e_coarse, coarse_level: MGLevel, fine_level: MGLevel, out=None):
    """Trilinear prolongation onto the fine slab (multigrid.py:238-297)."""
    hier = fine_level.hier
    if coarse_level.index != fine_level.index + 1:
        raise MultigridError("prolong_tl needs adjacent levels")
    src = as_device(e_coarse)
    dst = _out_like(fine_level.extent.shape, out)
    _native.set_stream_from_torch()
    _native.check(_native.load().hf_prolong_tl(hier._h, fine_level.index, src.data_ptr(),
                                                dst.data_ptr()))
    return out if out is not None else dst


def jacobi_smooth(op: StencilOperator, u, b, omega: float, sweeps: int, scratch=None,
                  assume_zero: bool = False):
    """Damped Jacobi in place on u (multigrid.py:138-157)."""
    uu = u.owned if isinstance(u, HaloField) else u
    bb = as_device(b)
    sc = scratch.owned if isinstance(scratch, HaloField) else scratch
    _native.set_stream_from_torch()
    _native.check(_native.load().hf_jacobi_smooth(op._h, uu.data_ptr(), bb.data_ptr(),
                                                   float(omega), int(sweeps),
                                                   1 if assume_zero else 0,
                                                   sc.data_ptr() if sc is not None else None))
    if isinstance(u, HaloField):
        u.invalidate_halo()
    return u


def coarsest_solve(hier: MGHierarchy, b, out=None):
    """Coarsest-level solve (multigrid.py:300-323)."""
    src = as_device(b)
    dst = _out_like(hier.coarsest.extent.shape, out)
    _native.set_stream_from_torch()
    _native.check(_native.load().hf_coarsest_solve(hier._h, src.data_ptr(), dst.data_ptr()))
    if hier.coarsest_kind == "gmres":
        hier.sync_coarsest_flags()
    return out if out is not None else dst


def mg_precondition(hier: MGHierarchy, r, out=None):
    """z ~= M^-1 r: one V- or F-cycle from a zero guess (multigrid.py:395-419)."""
    src = as_device(r)
    if tuple(src.shape) != hier.finest.extent.shape:
        raise MultigridError(f"field shape {tuple(src.shape)} != {hier.finest.extent.shape}")
    dst = _out_like(hier.finest.extent.shape, out)
    _native.set_stream_from_torch()
    _native.check(_native.load().hf_mg_precondition(hier._h, src.data_ptr(), dst.data_ptr()))
    return out if out is not None else dst
