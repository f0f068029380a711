"""Model problems: media (k = 2*pi*f/c), right-hand sides, error norms.

Host-side setup (numpy), mirroring /root/reference/pkg/src/helmfree/problems.py:
ConstantK (:56-65), LayeredMedium (:68-100), VelocityGridMedium (:103-119),
closed_off_problem (:159-166), wedge_problem (:169-184), salt_problem
(:187-201), build_problem (:220-236), build_rhs (:239-253), Dirac placement
(:256-271), closed-off RHS with Dirichlet lifting (:274-300), error_norms
(:335-357), velocity file I/O (:364-381), gen_salt_surrogate (:383-401).

Plus the BASELINE.json workloads: a centre point source in a constant-k
cube, the three-layer tilted-plane wedge, and a seeded smooth random medium
with an ellipsoidal inclusion.
"""

from __future__ import annotations

import os
import warnings
from dataclasses import dataclass

import numpy as np

from .grid import BlockExtent, Grid3, full_extent, make_grid
from .operators import Dirichlet, OperatorSpec, Sommerfeld

__all__ = ["ProblemError", "ConstantK", "LayeredMedium", "PlaneLayeredMedium",
           "VelocityGridMedium", "ProblemSpec", "closed_off_analytical", "closed_off_problem",
           "wedge_problem", "salt_problem", "point_source_cube", "wedge3_problem",
           "random_medium_problem", "build_problem", "build_rhs", "zero_dirichlet_boundary",
           "fill_dirichlet_boundary", "error_norms", "read_velocity_grid", "write_velocity_grid",
           "gen_salt_surrogate", "KH_LIMIT"]

KH_LIMIT = 0.625
SALT_VMIN = 1500.0
SALT_VMAX = 4482.0


class ProblemError(ValueError):
    pass


def _check_velocity(c):
    cmin = float(np.min(c))
    if cmin <= 0.0:
        raise ProblemError(f"non-positive velocity {cmin} in medium")


@dataclass(frozen=True)
class ConstantK:
    k: float

    def k_field(self, grid: Grid3, extent: BlockExtent) -> np.ndarray:
        if self.k <= 0:
            raise ProblemError(f"wavenumber must be positive, got {self.k}")
        return np.full(extent.shape, float(self.k))


@dataclass(frozen=True)
class LayeredMedium:
    """Layers split by interfaces dipping along x1 (problems.py:68-100)."""

    frequency: float
    velocities: tuple = (2000.0, 1500.0, 3000.0)
    interfaces: tuple = ((-200.0, -400.0), (-500.0, -700.0))
    x1_span: tuple = (0.0, 600.0)

    def velocity(self, x1, x3):
        if len(self.velocities) != len(self.interfaces) + 1:
            raise ProblemError("need one velocity per layer "
                               "(len(velocities) == len(interfaces) + 1)")
        a, b = self.x1_span
        t = (x1 - a) / (b - a) if b != a else np.zeros_like(x1)
        c = np.full(np.broadcast(x1, x3).shape, self.velocities[0])
        for (z0, z1), v_below in zip(self.interfaces, self.velocities[1:]):
            c = np.where(x3 < z0 + t * (z1 - z0), v_below, c)
        return c

    def k_field(self, grid: Grid3, extent: BlockExtent) -> np.ndarray:
        x1 = grid.axis_coords(0, extent.lo1, extent.hi1)[:, None, None]
        x3 = grid.axis_coords(2, extent.lo3, extent.hi3)[None, None, :]
        c = np.broadcast_to(self.velocity(x1, x3), extent.shape)
        _check_velocity(c)
        return 2.0 * np.pi * self.frequency / c


@dataclass(frozen=True)
class PlaneLayeredMedium:
    """BASELINE configs[2] wedge: velocities top/middle/bottom split by the tilted
    planes z = a0 + a1*x (x, z normalised to the unit cube, z = depth)."""

    frequency: float
    velocities: tuple = (2000.0, 1500.0, 3000.0)
    planes: tuple = ((0.4, 0.2), (0.8, -0.2))

    def k_field(self, grid: Grid3, extent: BlockExtent) -> np.ndarray:
        L = (grid.n1 - 1) * grid.h
        D = (grid.n3 - 1) * grid.h
        x = (grid.axis_coords(0, extent.lo1, extent.hi1) - grid.origin[0])[:, None, None] / L
        z = (grid.axis_coords(2, extent.lo3, extent.hi3) - grid.origin[2])[None, None, :] / D
        c = np.full(np.broadcast(x, z).shape, self.velocities[0])
        for (a0, a1), v in zip(self.planes, self.velocities[1:]):
            c = np.where(z > a0 + a1 * x, v, c)
        c = np.broadcast_to(c, extent.shape)
        return 2.0 * np.pi * self.frequency / c


@dataclass(frozen=True)
class VelocityGridMedium:
    frequency: float
    velocities: object = None

    def k_field(self, grid: Grid3, extent: BlockExtent) -> np.ndarray:
        v = self.velocities
        if v.shape != grid.shape:
            raise ProblemError(f"velocity dims {v.shape} do not match grid {grid.shape}")
        e = extent
        block = np.asarray(v[e.lo1 - 1:e.hi1, e.lo2 - 1:e.hi2, e.lo3 - 1:e.hi3], dtype=np.float64)
        _check_velocity(block)
        return 2.0 * np.pi * self.frequency / block


@dataclass
class ProblemSpec:
    name: str
    grid: Grid3
    medium: object
    bc: object
    source: dict
    domain: tuple = None
    analytical = None

    def has_analytical(self) -> bool:
        return self.analytical is not None


def closed_off_analytical(x1, x2, x3):
    return np.sin(np.pi * x1) * np.sin(2.0 * np.pi * x2) * np.sin(4.0 * np.pi * x3) + 1.0


def _closed_off_source(x1, x2, x3, k):
    return ((21.0 * np.pi**2 - k**2) * np.sin(np.pi * x1) * np.sin(2.0 * np.pi * x2)
            * np.sin(4.0 * np.pi * x3) - k**2)


def closed_off_problem(n: int, k: float) -> ProblemSpec:
    grid = make_grid(n, n, n, 1.0 / (n - 1))
    spec = ProblemSpec("ClosedOff", grid, ConstantK(k), Dirichlet(1.0), {"type": "closed_off"},
                       ((0.0, 1.0),) * 3)
    spec.analytical = closed_off_analytical
    return spec


def _grid_for_domain(shape, domain) -> Grid3:
    hs = [(b - a) / (n - 1) for (a, b), n in zip(domain, shape)]
    for h in hs[1:]:
        if abs(h - hs[0]) > 1e-12 * max(abs(hs[0]), abs(h)):
            raise ProblemError(f"domain/grid pairs imply non-uniform spacing {hs}; "
                               "choose extents and vertex counts giving one h")
    return make_grid(*shape, h=hs[0], origin=tuple(a for a, _ in domain))


def wedge_problem(shape=(61, 61, 101), domain=((0.0, 600.0), (0.0, 600.0), (-1000.0, 0.0)),
                  frequency=20.0, velocities=(2000.0, 1500.0, 3000.0),
                  interfaces=((-200.0, -400.0), (-500.0, -700.0)),
                  source_at=(300.0, 300.0, 0.0)) -> ProblemSpec:
    grid = _grid_for_domain(shape, domain)
    medium = LayeredMedium(frequency, tuple(velocities), tuple(tuple(p) for p in interfaces),
                           domain[0])
    return ProblemSpec("Wedge", grid, medium, Sommerfeld(), {"type": "dirac", "at": tuple(source_at)},
                       domain)


def salt_problem(velocities, shape=(641, 641, 193),
                 domain=((0.0, 12800.0), (0.0, 12800.0), (0.0, 3840.0)), frequency=2.0,
                 source_at=(3200.0, 3200.0, 0.0)) -> ProblemSpec:
    grid = _grid_for_domain(shape, domain)
    vmin, vmax = float(np.min(velocities)), float(np.max(velocities))
    if vmin < SALT_VMIN or vmax > SALT_VMAX:
        warnings.warn(f"velocity range [{vmin:g}, {vmax:g}] outside the expected "
                      f"[{SALT_VMIN:g}, {SALT_VMAX:g}] m/s band", stacklevel=2)
    return ProblemSpec("Salt", grid, VelocityGridMedium(frequency, velocities), Sommerfeld(),
                       {"type": "dirac", "at": tuple(source_at)}, domain)


def point_source_cube(n: int, k: float, bc="sommerfeld") -> ProblemSpec:
    """BASELINE configs[0]/[1]/[3]: unit cube, constant k, unit point source at the
    centre node (Dirac 1/h^3), zero-Dirichlet or first-order Sommerfeld faces."""
    grid = make_grid(n, n, n, 1.0 / (n - 1))
    bcv = Dirichlet(0.0) if bc == "dirichlet" else Sommerfeld()
    return ProblemSpec("PointSource", grid, ConstantK(k), bcv,
                       {"type": "dirac", "at": (0.5, 0.5, 0.5)}, ((0.0, 1.0),) * 3)


def wedge3_problem(n: int = 513, frequency: float | None = None) -> ProblemSpec:
    """BASELINE configs[2]: unit-depth three-layer wedge, planes z=0.4+0.2x and
    z=0.8-0.2x, v = 2000/1500/3000 m/s, source at (0.5, 0.5, 0.1), Sommerfeld.
    Frequency defaults to the largest with k h <= 0.625 at the slowest layer."""
    grid = make_grid(n, n, n, 1.0 / (n - 1))
    if frequency is None:
        frequency = KH_LIMIT * 1500.0 / (2.0 * np.pi * grid.h)
    medium = PlaneLayeredMedium(frequency)
    return ProblemSpec("Wedge3", grid, medium, Sommerfeld(), {"type": "dirac", "at": (0.5, 0.5, 0.1)},
                       ((0.0, 1.0),) * 3)


def random_medium_velocity(shape, seed: int = 2308, corr: float = 0.05) -> np.ndarray:
    """BASELINE configs[4]: seeded smooth Gaussian random field (correlation length
    `corr` of the domain) mapped to 1500-4500 m/s plus an ellipsoidal 4500 m/s body."""
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal(shape)
    f = np.fft.rfftn(noise)
    ks = [np.fft.fftfreq(n) * (n - 1) for n in shape[:-1]] + [np.fft.rfftfreq(shape[-1]) * (shape[-1] - 1)]
    kx, ky, kz = np.meshgrid(*ks, indexing="ij", sparse=True)
    f *= np.exp(-0.5 * (2 * np.pi * corr) ** 2 * (kx**2 + ky**2 + kz**2))
    g = np.fft.irfftn(f, s=shape, axes=(0, 1, 2))
    g = (g - g.mean()) / (g.std() + 1e-300)
    c = 3000.0 + 750.0 * g
    c = np.clip(c, 1500.0, 4500.0)
    x = np.linspace(0, 1, shape[0])[:, None, None]
    y = np.linspace(0, 1, shape[1])[None, :, None]
    z = np.linspace(0, 1, shape[2])[None, None, :]
    cx, cy, cz = rng.uniform(0.35, 0.65, 3)
    body = ((x - cx) / 0.2) ** 2 + ((y - cy) / 0.15) ** 2 + ((z - cz) / 0.12) ** 2 <= 1.0
    return np.where(body, 4500.0, c)


def random_medium_problem(shape=(1025, 1025, 513), seed: int = 2308) -> ProblemSpec:
    n1 = shape[0]
    grid = make_grid(*shape, h=1.0 / (n1 - 1))
    vel = random_medium_velocity(shape, seed)
    frequency = KH_LIMIT * 1500.0 / (2.0 * np.pi * grid.h)
    depth = (shape[2] - 1) * grid.h
    return ProblemSpec("RandomMedium", grid, VelocityGridMedium(frequency, vel), Sommerfeld(),
                       {"type": "dirac", "at": (0.5, 0.5 * (shape[1] - 1) * grid.h, 0.05 * depth)},
                       None)


def build_problem(pspec: ProblemSpec, extent: BlockExtent | None = None):
    """(Helmholtz OperatorSpec, rhs ndarray) for this worker's block (problems.py:220-236)."""
    grid = pspec.grid
    extent = extent or full_extent(grid)
    k_field = pspec.medium.k_field(grid, extent)
    kh = float(np.max(k_field)) * grid.h
    if kh > KH_LIMIT * (1.0 + 1e-12):
        warnings.warn(f"kh = {kh:.4g} exceeds {KH_LIMIT} (fewer than ten points per wavelength)",
                      stacklevel=2)
    spec = OperatorSpec("helmholtz", 1.0, 0.0, pspec.bc, k_field)
    return spec, build_rhs(pspec, extent, k_field)


def _nearest_vertex(grid: Grid3, at):
    idx = []
    for dim, x in enumerate(at):
        i = int(round((x - grid.origin[dim]) / grid.h)) + 1
        idx.append(min(max(i, 1), grid.shape[dim]))
    return tuple(idx)


def build_rhs(pspec: ProblemSpec, extent: BlockExtent | None = None, k_field=None) -> np.ndarray:
    grid = pspec.grid
    extent = extent or full_extent(grid)
    b = np.zeros(extent.shape, dtype=np.complex128)
    kind = pspec.source["type"]
    if kind == "dirac":
        g = _nearest_vertex(grid, pspec.source["at"])
        if extent.contains(g):
            b[g[0] - extent.lo1, g[1] - extent.lo2, g[2] - extent.lo3] = 1.0 / grid.h**3
    elif kind == "closed_off":
        if not isinstance(pspec.bc, Dirichlet):
            raise ProblemError("closed-off source assumes Dirichlet boundaries")
        if k_field is None:
            k_field = pspec.medium.k_field(grid, extent)
        x1 = grid.axis_coords(0, extent.lo1, extent.hi1)[:, None, None]
        x2 = grid.axis_coords(1, extent.lo2, extent.hi2)[None, :, None]
        x3 = grid.axis_coords(2, extent.lo3, extent.hi3)[None, None, :]
        b[...] = _closed_off_source(x1, x2, x3, k_field)
        g, ih2 = pspec.bc.value, 1.0 / grid.h**2
        for dim in range(3):
            n, lo, hi = grid.shape[dim], extent.lo[dim], extent.hi[dim]
            for plane in (2, n - 1):
                if lo <= plane <= hi:
                    sl = [slice(None)] * 3
                    sl[dim] = plane - lo
                    b[tuple(sl)] += g * ih2
        zero_dirichlet_boundary(b, grid, extent)
    else:
        raise ProblemError(f"unknown source type {kind!r}")
    return b


def _boundary_planes(grid, extent):
    for dim in range(3):
        if extent.lo[dim] == 1:
            yield dim, 0
        if extent.hi[dim] == grid.shape[dim]:
            yield dim, extent.shape[dim] - 1


def zero_dirichlet_boundary(owned, grid, extent):
    for dim, idx in _boundary_planes(grid, extent):
        sl = [slice(None)] * 3
        sl[dim] = idx
        owned[tuple(sl)] = 0.0


def fill_dirichlet_boundary(owned, grid, extent, value):
    for dim, idx in _boundary_planes(grid, extent):
        sl = [slice(None)] * 3
        sl[dim] = idx
        owned[tuple(sl)] = value


def error_norms(u_num: np.ndarray, pspec: ProblemSpec):
    if not pspec.has_analytical():
        raise ProblemError(f"{pspec.name} has no analytical solution")
    grid = pspec.grid
    if u_num.shape != grid.shape:
        raise ProblemError(f"field shape {u_num.shape} != grid {grid.shape}")
    x1 = grid.axis_coords(0, 1, grid.n1)[:, None, None]
    x2 = grid.axis_coords(1, 1, grid.n2)[None, :, None]
    x3 = grid.axis_coords(2, 1, grid.n3)[None, None, :]
    err = np.abs(u_num - pspec.analytical(x1, x2, x3))
    with np.errstate(divide="ignore"):
        log_err = np.log10(err, out=np.full(err.shape, -16.0), where=err > 1e-16)
    return float(err.max()), float(np.sqrt(np.sum(err**2) * grid.h**3)), log_err


def read_velocity_grid(path, dims, frequency: float = 2.0) -> VelocityGridMedium:
    n1, n2, n3 = dims
    expected = n1 * n2 * n3 * 4
    actual = os.path.getsize(path)
    if actual != expected:
        raise ProblemError(f"velocity file {path}: {actual} bytes, expected {expected} for dims {dims}")
    v = np.memmap(path, dtype="<f4", mode="r", shape=(n1, n2, n3), order="F")
    return VelocityGridMedium(frequency, v)


def write_velocity_grid(path, velocities) -> None:
    with open(path, "wb") as f:
        f.write(np.asarray(velocities, dtype="<f4").tobytes(order="F"))


def gen_salt_surrogate(path, dims) -> np.ndarray:
    n1, n2, n3 = dims
    z = np.linspace(0.0, 1.0, n3)[None, None, :]
    x = np.linspace(0.0, 1.0, n1)[:, None, None]
    y = np.linspace(0.0, 1.0, n2)[None, :, None]
    c = 1500.0 + 2200.0 * z
    body = ((x - 0.5) / 0.28) ** 2 + ((y - 0.5) / 0.22) ** 2 + ((z - 0.45) / 0.30) ** 2 <= 1.0
    c = np.where(body, SALT_VMAX, c)
    c = np.ascontiguousarray(np.clip(np.broadcast_to(c, (n1, n2, n3)), SALT_VMIN, SALT_VMAX),
                             dtype=np.float32)
    write_velocity_grid(path, c)
    return c
