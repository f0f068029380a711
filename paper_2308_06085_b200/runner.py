"""Run orchestration around the native path: build the problem, solve on the
B200, report.

Mirrors /root/reference/pkg/src/helmfree/runner.py (problem_from_config
:39-62, worker_body :95-147, run_solve :170-187) and the HFF1 / residual-CSV
writers of io.py (:127-170) and RunReport of reporting.py (:24-52).
topology.npx0 > 1 splits the grid into slabs: fabric "local" runs them as
virtual slabs on this GPU, fabric "nccl" expects one process per slab
(torch.distributed already initialised, e.g. under torchrun).
"""

from __future__ import annotations

import json
import os
import struct
import time
from dataclasses import asdict, dataclass, field

import numpy as np

from . import problems as P
from .config import ConfigError, RunConfig
from .grid import full_extent
from .krylov import ConvergenceReport, Solver, SolverConfig
from .multigrid import MGConfig, build_hierarchy
from .operators import Dirichlet, OperatorSpec, StencilOperator

__all__ = ["RunReport", "problem_from_config", "run_solve", "write_field", "read_field",
           "write_residual_csv"]

_HFF = struct.Struct("<4sIII")


@dataclass
class RunReport:
    convergence: ConvergenceReport
    config: dict = field(default_factory=dict)
    workers: int = 1
    fabric: str = "none"
    error_max: float | None = None
    error_l2: float | None = None

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=2, sort_keys=True, default=float)


def problem_from_config(cfg: RunConfig):
    p = cfg.problem
    name = p["name"]
    if name == "ClosedOff":
        return P.closed_off_problem(p["n"], p["k"])
    if name == "PointSource":
        return P.point_source_cube(p["n"], p["k"], p["bc"])
    if name == "Wedge3":
        return P.wedge3_problem(p["n"])
    dom = p["domain"]
    if len(dom) != 6:
        raise ConfigError(f"problem.domain needs 6 numbers, got {len(dom)}")
    domain = ((dom[0], dom[1]), (dom[2], dom[3]), (dom[4], dom[5]))
    if name == "Wedge":
        it = p["interfaces"]
        if len(it) % 2:
            raise ConfigError("problem.interfaces needs an even count of numbers")
        return P.wedge_problem(tuple(p["shape"]), domain, p["frequency"], tuple(p["velocities"]),
                               tuple((it[i], it[i + 1]) for i in range(0, len(it), 2)),
                               tuple(p["source"]))
    if name == "Salt":
        if not p["velocity_file"]:
            raise ConfigError("Salt requires problem.velocity_file")
        m = P.read_velocity_grid(p["velocity_file"], tuple(p["shape"]), p["frequency"])
        return P.salt_problem(m.velocities, tuple(p["shape"]), domain, p["frequency"],
                              tuple(p["source"]))
    raise ConfigError(f"unknown problem name {name!r}")


def _mg(cfg):
    q = cfg.preconditioner
    return MGConfig(q["nu1"], q["nu2"], q["omega"], q["cycle"], q["coarsest_threshold"],
                    q["threshold_cmp"], q["coarsest_tol"], q["coarsest_maxit"], q["coarsest_method"])


def _solver_cfg(cfg):
    s = cfg.solver
    return SolverConfig(method=s["method"], tol=s["tol"], maxit=s["maxit"], s=s["s"],
                        rng_seed=s["rng_seed"], restart=s["restart"] or None,
                        check_every=s["check_every"])


def run_solve(cfg: RunConfig, write_outputs: bool = True) -> RunReport:
    """Build and solve per config; returns the report (runner.py:170-187)."""
    pspec = problem_from_config(cfg)
    grid = pspec.grid
    spec, rhs = P.build_problem(pspec)
    k_full = np.asarray(spec.k_field)
    pre = cfg.preconditioner
    nslab = cfg.topology["npx0"]
    t0 = time.perf_counter()
    if nslab == 1:
        A = StencilOperator(spec, grid)
        hier = build_hierarchy(grid, None, OperatorSpec("cslp", pre["beta1"], pre["beta2"],
                                                        spec.bc, k_full), _mg(cfg))
        x, conv = Solver(A, hier).solve(rhs, _solver_cfg(cfg))
        full = x.cpu().numpy()
        fabric = "none"
    else:
        from .dist import NativeSlabSolver, SlabSolver
        from .partition import LocalSlabComm, TorchSlabComm, slab_partition
        if cfg.solver["method"] != "bicgstab":
            raise ConfigError("the slab driver runs Bi-CGSTAB")
        ext = slab_partition(grid, nslab)
        if cfg.topology["fabric"] == "local":
            comm, mine = LocalSlabComm(nslab), ext
        else:
            comm = TorchSlabComm()
            if comm.size != nslab:
                raise ConfigError(f"topology.npx0={nslab} but the process group has {comm.size}")
            mine = [ext[comm.rank]]
        native = cfg.topology["fabric"] == "local" or comm.dist.get_backend(comm.group) == "nccl"
        if native:     # the whole iteration in the native library, one CUDA graph
            S = NativeSlabSolver(grid, mine, k_full, spec.bc, comm, pre["beta1"], pre["beta2"],
                                 _mg(cfg), maxit=cfg.solver["maxit"])
            xs, conv = S.solve([rhs[e.lo1 - 1:e.hi1] for e in mine], _solver_cfg(cfg))
        else:          # gloo process group: device scalars, Python-driven levels
            S = SlabSolver(grid, mine, k_full, spec.bc, comm, pre["beta1"], pre["beta2"], _mg(cfg))
            xs, conv = S.solve_device([rhs[e.lo1 - 1:e.hi1] for e in mine], _solver_cfg(cfg))
        parts = [x.cpu().numpy() for x in xs]
        if cfg.topology["fabric"] == "local":
            full = np.concatenate(parts, 0)
        else:
            import torch
            counts = [e.nx for e in ext]
            full = comm.allgather_planes(torch.as_tensor(parts[0]).cuda(), counts).cpu().numpy()
        fabric = cfg.topology["fabric"]
    conv.wall_time = time.perf_counter() - t0
    if isinstance(pspec.bc, Dirichlet):
        P.fill_dirichlet_boundary(full, grid, full_extent(grid), pspec.bc.value)
    rep = RunReport(convergence=conv, config=cfg.to_dict(), workers=nslab, fabric=fabric)
    if pspec.has_analytical() and conv.converged:
        rep.error_max, rep.error_l2, _ = P.error_norms(full, pspec)
    out = cfg.output["dir"]
    if write_outputs and out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "report.json"), "w") as f:
            f.write(rep.to_json() + "\n")
        write_residual_csv(os.path.join(out, "residual.csv"), conv.residual_history)
        if cfg.output["write_field"]:
            write_field(os.path.join(out, "field.hff"), full)
    rep.field = full
    return rep


def write_field(path, field) -> None:
    """HFF1: magic + n1, n2, n3 (little-endian u32), complex128, i1 fastest (io.py:127-134)."""
    arr = np.asarray(field, dtype=np.complex128)
    with open(path, "wb") as f:
        f.write(_HFF.pack(b"HFF1", *arr.shape))
        f.write(arr.tobytes(order="F"))


def read_field(path):
    with open(path, "rb") as f:
        magic, n1, n2, n3 = _HFF.unpack(f.read(_HFF.size))
        if magic != b"HFF1":
            raise ValueError(f"{path}: bad magic {magic!r}")
        data = np.fromfile(f, dtype=np.complex128, count=n1 * n2 * n3)
    return data.reshape((n1, n2, n3), order="F")


def write_residual_csv(path, history) -> None:
    with open(path, "w") as f:
        f.write("iteration,relres\n")
        for i, r in enumerate(history):
            f.write(f"{i},{r!r}\n")
