"""Benchmark: CSLP-preconditioned Bi-CGSTAB time-to-solution on the B200.

Workload (BASELINE.json configs[1]): unit cube, constant k = 80, h = 1/128
(129^3 vertices, kh = 0.625), first-order Sommerfeld faces, unit point
source at the centre node, complex128; CSLP shift beta1 = 1, |beta2| = 0.5 in
the reference's damping-consistent sign (beta2 = -0.5, shift 1 + 0.5i), one
V(1,1)-cycle with damped Jacobi (omega 0.8), full weighting, trilinear
prolongation, Bi-CGSTAB to relative residual 1e-6.

One step = one full solve from a resident right-hand side.  The metric is
Munknowns*iter/s = (vertices x Bi-CGSTAB iterations) / solve time, summed over
all GPUs.  L2 is flushed (256 MiB write) before every timed step; each step is
timed with CUDA events on the current stream (the library orders its private
stream after it and back).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_GRID = 129
K_WAVE = 80.0
TOL = 1e-6
MAXIT = 400
METRIC = "cslp_bicgstab_munknowns_iter_per_s"
UNIT = "Munknowns*iter/s"


def _env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed ncu --set full summary (profiles/ncu_traffic.json,
    written by tools/ncu_traffic.py); None when it was captured for another kernel."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        return d["traffic_bytes_per_launch"] if d.get("kernel") == kernel else None
    except Exception:
        return None


def _problem():
    from paper_2308_06085_b200 import problems
    p = problems.point_source_cube(N_GRID, K_WAVE, "sommerfeld")
    spec, b = problems.build_problem(p)
    return p, spec, b


def _config_dict(extra=None):
    d = {"workload": "configs[1]: 129^3 unit cube, k=80 (kh=0.625), Sommerfeld, centre point "
                     "source, complex128, CSLP(1, 0.5i-damped) V(1,1) omega=0.8, Bi-CGSTAB tol 1e-6",
         "unknowns": N_GRID ** 3, "grid": [N_GRID] * 3, "k": K_WAVE, "tol": TOL,
         "l2": "flushed (256 MiB write) before every timed step"}
    if extra:
        d.update(extra)
    return d


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during timing."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


def _event_time(fn, reps):
    import torch
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2308_06085_b200.krylov import Solver, SolverConfig
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator

    rank, world, local = _env_rank()
    if world > 1:
        return run_slabs(args)
    torch.cuda.set_device(local)
    p, spec, b_host = _problem()
    n = p.grid.num_vertices
    t_setup = time.perf_counter()
    A = StencilOperator(spec, p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field),
                           MGConfig())
    solver = Solver(A, hier)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    cfg = SolverConfig(method="bicgstab", tol=TOL, maxit=MAXIT, check_every=4)
    b = torch.as_tensor(b_host).cuda()
    x = torch.empty_like(b)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        _, rep = solver.solve(b, cfg, x=x)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times, reps = [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            _, rep = solver.solve(b, cfg, x=x)
            e.record()
            torch.cuda.synchronize()
            times.append(s.elapsed_time(e))
            reps.append(rep)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = float(np.sum(times))
    if world > 1:
        t = torch.tensor([total_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    iters = reps[-1].iterations
    ms_step = total_ms / args.steps
    value = world * n * iters / (ms_step / 1e3) / 1e6

    # ---- e2e: public API from pinned host buffers (H2D + solve + D2H) ----
    bh = torch.as_tensor(b_host).pin_memory().numpy()
    xh = torch.empty(b_host.shape, dtype=torch.complex128).pin_memory().numpy()
    solver.solve(bh, cfg, x=xh, host=True)
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 5))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep_h = solver.solve(bh, cfg, x=xh, host=True)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_step = float(np.mean(e2e_ms))
    e2e_value = world * n * rep_h.iterations / (e2e_step / 1e3) / 1e6

    # ---- kernel roofline: live CUDA-event timing of the hot kernels ----
    hbm, peak_kind = _peaks()
    kern = kernel_table(A, hier, n, ms_step / max(iters, 1), solver=solver)
    dom = max((k_ for k_ in kern if kern[k_]["bound"] == "hbm" and kern[k_]["role"] == "solve"),
              key=lambda k_: kern[k_]["share"])
    kd = kern[dom]
    roofline = {"bound": "hbm", "kernel": dom, "achieved": kd["gbs"], "peak": hbm,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": round(kd["gbs"] / hbm, 4),
                "traffic": _ncu_traffic(dom), "algorithmic_bytes_per_launch": kd["bytes"],
                "launch_ms": kd["ms"],
                "kernels": {k_: {"gbs": v_["gbs"], "frac": round(v_["gbs"] / hbm, 4),
                                 "ms": v_["ms"], "share": v_["share"], "bound": v_["bound"],
                                 "role": v_["role"]}
                            for k_, v_ in kern.items()}}
    roofline["kernels"]["coarsest_solve"]["kind"] = kern["coarsest_solve"]["kind"]

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (BASELINE configs[1] point-source problem, built in-process)",
        "config": _config_dict({"parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                                "iterations": iters, "matvecs": reps[-1].matvec_count,
                                "final_relres": reps[-1].final_relres,
                                "time_to_solution_s": round(ms_step / 1e3, 6),
                                "setup_s": round(t_setup, 3)}),
        "clocks": clk.summary(),
        "gpu_launches": int(sum(r.kernel_launches for r in reps)),
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT,
                "h2d_bytes_per_step": int(b_host.nbytes), "d2h_bytes_per_step": int(b_host.nbytes),
                "ms_per_step": round(e2e_step, 4)},
        "roofline": roofline,
    }
    if rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(MAXIT)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_slabs(args):
    """N > 1: the 129^3 solve split into N slabs along i1, one per GPU
    (strong scaling).  Halos P2P over NCCL, the Bi-CGSTAB scalars on the device
    (partial sums NCCL-all-reduced, no host sync per inner product), coarsest
    level all-gathered and solved on every rank."""
    import torch
    import torch.distributed as dist

    from paper_2308_06085_b200.dist import SlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import TorchSlabComm, slab_partition

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p, spec, b_host = _problem()
    n = p.grid.num_vertices
    e = slab_partition(p.grid, world)[rank]
    comm = TorchSlabComm()
    t_setup = time.perf_counter()
    S = SlabSolver(p.grid, [e], spec.k_field, p.bc, comm)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    cfg = SolverConfig(method="bicgstab", tol=TOL, maxit=MAXIT)
    b = [torch.as_tensor(b_host[e.lo1 - 1:e.hi1]).cuda()]
    for _ in range(args.warmup):
        _, rep = S.solve_device(b, cfg)
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            e0 = torch.cuda.Event(enable_timing=True)
            s0.record()
            _, rep = S.solve_device(b, cfg)
            e0.record()
            torch.cuda.synchronize()
            times.append(s0.elapsed_time(e0))
    t = torch.tensor([float(np.sum(times))], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    iters = rep.iterations
    # e2e: host slab in, host slab out
    bh = torch.as_tensor(b_host[e.lo1 - 1:e.hi1]).pin_memory()
    dist.barrier()
    t0 = time.perf_counter()
    xs, rep_h = S.solve_device([bh.cuda(non_blocking=True)], cfg)
    xh = xs[0].cpu()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3
    te = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    if rank == 0:
        out = {
            "metric": METRIC, "value": round(n * iters / (ms_step / 1e3) / 1e6, 2), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (BASELINE configs[1] point-source problem, built in-process)",
            "config": _config_dict({"parallelism": f"{world} slabs along i1 (halo P2P + NCCL allreduce)",
                                    "iterations": iters, "matvecs": rep.matvec_count,
                                    "final_relres": rep.final_relres,
                                    "time_to_solution_s": round(ms_step / 1e3, 6),
                                    "setup_s": round(t_setup, 3)}),
            "clocks": clk.summary(), "gpu_launches": None,
            "e2e": {"value": round(n * rep_h.iterations / (e2e_ms / 1e3) / 1e6, 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(b_host.nbytes), "d2h_bytes_per_step": int(b_host.nbytes),
                    "ms_per_step": round(e2e_ms, 4)},
            "roofline": None,
        }
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def kernel_table(A, hier, n, t_iter_ms, reps=20, solver=None):
    """Live CUDA-event timing of the path's kernels on the finest level.  The
    129^3 fields are 34 MB (L2 is 126 MB), so consecutive launches rotate over
    NSET independent operand sets (> 2x L2 in total): every launch streams its
    operands from HBM, back to back as in the solve.  The Bi-CGSTAB vector
    kernels run back to back on the solver's own workspace.  Bytes are the
    algorithmic traffic of one launch (constant medium: no k traffic);
    share = launches per Bi-CGSTAB iteration x ms / iteration time."""
    import ctypes

    import torch

    from paper_2308_06085_b200 import _native

    L = _native.load()
    _native.set_stream_from_torch()
    NSET = 4
    shape = hier.levels[0].extent.shape
    cshape = hier.levels[1].extent.shape
    rnd = lambda sh: torch.randn(sh, dtype=torch.complex128, device="cuda")
    sets = [dict(u=rnd(shape), b=rnd(shape), v=rnd(shape), t=rnd(shape), ec=rnd(cshape), bc=rnd(cshape))
            for _ in range(NSET)]
    H = hier._h
    nc_f = cshape[0] * cshape[1] * cshape[2]
    ncs = hier.coarsest.grid.num_vertices
    xc, rc = rnd(hier.coarsest.grid.shape), rnd(hier.coarsest.grid.shape)
    nt = -(-ncs // 64)
    sym_bytes = nt * (nt + 1) // 2 * 64 * 64 * 16 + 2 * nt * (nt + 1) // 2 * 64 * 16 * 2
    p = lambda x: x.data_ptr()
    # on the solve path (each launched twice per Bi-CGSTAB iteration, once per
    # matvec / V-cycle): matvec (+dot), down_restrict (k_flat_dr), prolong_correct
    # (k_corr) + jacobi_postsmooth (k_flat_stencil); "api" = C-ABI level entry
    # points not on the 129^3 solve path (split presmooth+residual / restriction,
    # hf_level_up)
    cases = {
        "device_copy": (lambda s: s["v"].copy_(s["u"]), 32.0 * n, "ceiling"),
        "helmholtz_matvec": (lambda s: L.hf_operator_apply(A._h, p(s["u"]), p(s["v"])), 32.0 * n, "solve"),
        "down_restrict": (lambda s: L.hf_level_down_restrict(H, 0, p(s["b"]), p(s["bc"])),
                          16.0 * n + 16.0 * nc_f, "solve"),
        "prolong_correct": (lambda s: L.hf_level_correct(H, 0, p(s["b"]), p(s["ec"]), p(s["t"])),
                            32.0 * n + 16.0 * nc_f, "solve"),
        "jacobi_postsmooth": (lambda s: L.hf_level_smooth(H, 0, p(s["t"]), p(s["b"]), p(s["u"])), 48.0 * n,
                              "solve"),
        "cslp_presmooth_residual": (lambda s: L.hf_level_down1(H, 0, p(s["b"]), p(s["v"])), 32.0 * n, "api"),
        "restrict_fw": (lambda s: L.hf_restrict_fw(H, 0, p(s["v"]), p(s["bc"])), 16.0 * n + 16.0 * nc_f,
                        "api"),
        "level_up": (lambda s: L.hf_level_up(H, 0, p(s["b"]), p(s["ec"]), p(s["u"])), 32.0 * n + 16.0 * nc_f,
                     "api"),
    }
    kind = hier.coarsest_kind
    # separable (fast diagonalisation): b, two scratch passes, 1/D and x -- a
    # latency-bound 3-launch solve, reported for its share only
    cbytes = {"separable": 112.0 * ncs, "symmetric": float(sym_bytes),
              "dense": 16.0 * ncs * ncs}.get(kind, 0.0)
    cases["coarsest_solve"] = (lambda s: L.hf_coarsest_solve(H, p(rc), p(xc)), cbytes, "solve")
    out = {}

    def put(name, ms, nbytes, role, launches):
        out[name] = {"ms": round(ms, 5), "bytes": nbytes, "gbs": round(nbytes / (ms / 1e3) / 1e9, 1),
                     "share": round(launches * ms / t_iter_ms, 4) if role == "solve" else None,
                     "role": role,
                     "bound": ("latency" if name == "coarsest_solve" and kind == "separable"
                               else "ceiling" if name == "device_copy" else "hbm")}

    reps = max(NSET, reps // NSET * NSET)
    for name, (fn, nbytes, role) in cases.items():
        for s in sets:
            fn(s)
        k = [0]

        def run():
            fn(sets[k[0] % NSET])
            k[0] += 1
        put(name, _event_time(run, reps), nbytes, role, 2)
    if solver is not None:   # Bi-CGSTAB vector kernels, once per iteration (krylov.py:240-269)
        # back to back on the solver's workspace (working sets 137-241 MB: mostly
        # streamed from HBM, partly L2-resident for the p update)
        for nm, which, nb in (("bcg_p_update", 0, 64.0), ("bcg_s_update", 1, 48.0),
                              ("bcg_xr_update", 2, 128.0)):
            ms = ctypes.c_float()
            _native.check(L.hf_solver_bench_vec(solver._h, which, reps, ctypes.byref(ms)))
            put(nm, ms.value, nb * n, "solve", 1)
    out["coarsest_solve"]["kind"] = kind
    return out


def cpu_baseline(iters: int, threads: int | None = None):
    """The C oracle (a port of the reference algorithm) on this host's cores,
    OpenMP over all of them, on the same workload: up to `iters` Bi-CGSTAB
    iterations of the 129^3 solve (the full solve when iters >= its count),
    reported in the same metric."""
    from oracle import oracle as O
    p, spec, b = _problem()
    k = np.asarray(spec.k_field, dtype=np.float64)
    t0 = time.perf_counter()
    _, rep = O.solve(k, b, p.grid.h, bc="sommerfeld", method="bicgstab", tol=TOL, maxit=iters)
    dt = time.perf_counter() - t0
    n = p.grid.num_vertices
    return {"value": round(n * rep["iterations"] / dt / 1e6, 3), "unit": UNIT,
            "cores": O.num_threads(), "kind": "port",
            "sample": f"first {rep['iterations']} Bi-CGSTAB iterations of the 129^3 solve "
                      f"(incl. hierarchy setup), {dt:.2f} s"}


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    vals, samples, secs = [], [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(args.cpu_iters)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            vals.append(cb["value"])
            samples.append(cb)
            secs.append(dt)
    value = float(np.mean(vals))
    out = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "impl": "reference",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           # one step = one bounded sample (the oracle's solve, setup included)
           "ms_per_step": round(float(np.mean(secs)) * 1e3, 2),
           "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "c128", "data": "synthetic",
           "config": _config_dict({"parallelism": "host cores (OpenMP)"}),
           "cpu_baseline": {**samples[-1], "value": round(value, 3)},
           "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    # reference arm: each step is the full 129^3 solve (~3 s on the box's 16 cores)
    ap.add_argument("--cpu-iters", type=int, default=MAXIT)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
