"""Matrix-free Helmholtz / CSLP operators on the B200 (native kernels).

Mirrors /root/reference/pkg/src/helmfree/operators.py: Dirichlet/Sommerfeld
(:58-74), OperatorSpec (:77-99), interior_coeffs (:115-119),
StencilOperator (:122-254), apply_operator (:257-262), reduce_to_spec
(:265-274).  The stencil itself runs in libhelmfree_b200.so (k_apply in
csrc/hf_kernels.cu); there is no CPU implementation here.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Union

import numpy as np

from . import _native
from .grid import BlockExtent, Grid3, HaloField, full_extent

__all__ = ["Dirichlet", "Sommerfeld", "OperatorSpec", "StencilCoeffs", "StencilOperator",
           "OperatorError", "StaleHaloError", "ZeroDiagonalError", "interior_coeffs",
           "apply_operator", "reduce_to_spec", "as_device", "sequential_operator"]


class OperatorError(ValueError):
    pass


class StaleHaloError(OperatorError):
    pass


class ZeroDiagonalError(OperatorError):
    pass


@dataclass(frozen=True)
class Dirichlet:
    value: complex = 1.0


class Sommerfeld:
    def __eq__(self, other):
        return isinstance(other, Sommerfeld)

    def __hash__(self):
        return hash("sommerfeld")

    def __repr__(self):
        return "Sommerfeld()"


BoundaryCondition = Union[Dirichlet, Sommerfeld]


def bc_name(bc) -> str:
    if isinstance(bc, Dirichlet):
        return "dirichlet"
    if isinstance(bc, Sommerfeld):
        return "sommerfeld"
    raise OperatorError(f"unknown boundary condition {bc!r}")


@dataclass(frozen=True)
class OperatorSpec:
    """kind "helmholtz" (shift 1) or "cslp" (shift beta1 - i beta2).

    k_field is the wavenumber on this worker's block (reference semantics)
    or on the whole grid (needed when a slab reads neighbour ghost planes).
    """

    kind: str
    beta1: float
    beta2: float
    bc: BoundaryCondition
    k_field: np.ndarray

    def __post_init__(self):
        if self.kind not in ("helmholtz", "cslp"):
            raise OperatorError(f"unknown operator kind {self.kind!r}")

    @property
    def shift(self) -> complex:
        if self.kind == "helmholtz":
            return 1.0 + 0.0j
        return self.beta1 - 1j * self.beta2


@dataclass(frozen=True)
class StencilCoeffs:
    ap: complex
    aw: complex
    ae: complex
    as_: complex
    an: complex
    ad: complex
    au: complex


def interior_coeffs(spec: OperatorSpec, h: float, k: float) -> StencilCoeffs:
    off = -1.0 / h**2
    ap = (6.0 - spec.shift * k**2 * h**2) / h**2
    return StencilCoeffs(ap, off, off, off, off, off, off)


def as_device(x):
    """numpy / torch -> contiguous complex128 CUDA tensor (no copy if already one)."""
    import torch
    if isinstance(x, HaloField):
        return x.owned
    t = torch.as_tensor(x)
    if t.dtype != torch.complex128:
        t = t.to(torch.complex128)
    if not t.is_cuda:
        t = t.cuda()
    if not t.is_contiguous():
        t = t.contiguous()
    return t


def _ptr(t) -> int:
    return t.data_ptr()


def k_arguments(spec: OperatorSpec, grid: Grid3, extent: BlockExtent):
    """(k_full_or_None, k_const, keepalive) for the native constructors.

    A constant field is passed as a scalar (no per-vertex k traffic).  A
    block-shaped field is accepted when it covers the full grid or when the
    slab has no interior faces to read across.
    """
    k = np.asarray(spec.k_field, dtype=np.float64)
    if k.size and np.all(k == k.flat[0]):
        kc = float(k.flat[0])
        if kc <= 0:
            raise OperatorError(f"wavenumber must be positive, got {kc}")
        return None, kc, None
    if k.shape == grid.shape:
        full = np.ascontiguousarray(k)
    elif k.shape == extent.shape:
        if extent.shape != grid.shape:
            if not extent.is_slab_of(grid):
                raise OperatorError("B200 layout: blocks must be i1 slabs")
            full = np.zeros(grid.shape)
            full[extent.lo1 - 1:extent.hi1] = k
            if extent.lo1 != 1 or extent.hi1 != grid.n1:
                raise OperatorError(
                    "a slab with interior faces needs the global k_field (ghost planes)")
        else:
            full = np.ascontiguousarray(k)
    else:
        raise OperatorError(f"k_field shape {k.shape} != block shape {extent.shape}")
    if np.min(full[extent.lo1 - 1:extent.hi1]) <= 0:
        raise OperatorError("wavenumber must be positive")
    return full, 0.0, full


class StencilOperator:
    """Native matrix-free v = A u (operators.py:122-223)."""

    def __init__(self, spec: OperatorSpec, grid: Grid3, extent: BlockExtent | None = None,
                 exchanger=None, timers=None, phase: str = "matvec"):
        extent = extent or full_extent(grid)
        if not extent.is_slab_of(grid):
            raise OperatorError("B200 layout: blocks must be i1 slabs (full i2/i3 range)")
        k = np.asarray(spec.k_field)
        if k.shape not in (extent.shape, grid.shape):
            raise OperatorError(f"k_field shape {k.shape} != block shape {extent.shape}")
        self.spec, self.grid, self.extent = spec, grid, extent
        self.exchanger, self.timers, self.phase = exchanger, timers, phase
        self.h = grid.h
        self.apply_count = 0
        kfull, kc, self._keep = k_arguments(spec, grid, extent)
        L = _native.load()
        s = spec.shift
        kp = kfull.ctypes.data if kfull is not None else None
        h = L.hf_operator_create(grid.n1, grid.n2, grid.n3, extent.lo1 - 1, extent.nx, grid.h,
                                 float(np.real(s)), float(np.imag(s)), _native.BC[bc_name(spec.bc)],
                                 kp, kc)
        if not h:
            msg = _native.last_error()
            if "diagonal vanishes" in msg:
                raise ZeroDiagonalError(msg)
            raise OperatorError(msg)
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.load().hf_operator_destroy(h)
            except Exception:   # interpreter shutdown
                pass
            self._h = None

    @property
    def has_interior_faces(self) -> bool:
        return self.extent.lo1 != 1 or self.extent.hi1 != self.grid.n1

    def ensure_halo(self, u):
        if not self.has_interior_faces:
            return
        if not isinstance(u, HaloField):
            raise StaleHaloError("slab with interior faces needs a HaloField input")
        if not u.halo_valid:
            if self.exchanger is None:
                raise StaleHaloError("halo faces are stale and no exchanger is attached")
            self.exchanger.exchange(u)

    def apply(self, u, out=None):
        """v = A u on the owned slab; returns a CUDA tensor (or fills `out`)."""
        import torch
        if isinstance(u, HaloField):
            if u.extent.shape != self.extent.shape:
                raise OperatorError(f"field shape {u.extent.shape} != {self.extent.shape}")
            self.ensure_halo(u)
            src = u.owned
        else:
            if self.has_interior_faces:
                raise StaleHaloError("slab with interior faces needs a HaloField input")
            src = as_device(u)
            if tuple(src.shape) != self.extent.shape:
                raise OperatorError(f"field shape {tuple(src.shape)} != {self.extent.shape}")
        dst = out.owned if isinstance(out, HaloField) else out
        if dst is None:
            dst = torch.empty(self.extent.shape, dtype=torch.complex128, device=src.device)
        _native.set_stream_from_torch()
        _native.check(_native.load().hf_operator_apply(self._h, _ptr(src), _ptr(dst)))
        self.apply_count += 1
        if isinstance(out, HaloField):
            out.invalidate_halo()
            return out
        return dst

    def diag(self):
        import torch
        d = torch.empty(self.extent.shape, dtype=torch.complex128, device="cuda")
        _native.check(_native.load().hf_operator_diag(self._h, _ptr(d)))
        return d


def apply_operator(spec: OperatorSpec, u, grid: Grid3, exchanger=None):
    """One-shot v = A u (operators.py:257-262).  numpy in -> numpy out."""
    extent = u.extent if isinstance(u, HaloField) else full_extent(grid)
    op = StencilOperator(spec, grid, extent, exchanger=exchanger)
    v = op.apply(u)
    if isinstance(u, np.ndarray):
        return v.cpu().numpy()
    return v


def reduce_to_spec(spec: OperatorSpec, fine_extent: BlockExtent,
                   coarse_extent: BlockExtent) -> OperatorSpec:
    """Rediscretised coarse spec: k subsampled at the 2i-1 map (operators.py:265-274)."""
    s1 = 2 * coarse_extent.lo1 - 1 - fine_extent.lo1
    s2 = 2 * coarse_extent.lo2 - 1 - fine_extent.lo2
    s3 = 2 * coarse_extent.lo3 - 1 - fine_extent.lo3
    k = np.asarray(spec.k_field)
    kc = k[s1::2, s2::2, s3::2][:coarse_extent.nx, :coarse_extent.ny, :coarse_extent.nz]
    return replace(spec, k_field=np.ascontiguousarray(kc))


def sequential_operator(spec: OperatorSpec, grid: Grid3) -> StencilOperator:
    return StencilOperator(spec, grid, full_extent(grid))
