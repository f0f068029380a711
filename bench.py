"""Benchmark: CSLP-preconditioned Bi-CGSTAB on the B200 (BASELINE.json metric
"CSLP-Bi-CGSTAB time-to-solution, Munknowns*iter/s and stencil HBM GB/s").

Default workload (--config c2) = BASELINE configs[2], the configuration the
metric is quoted on that fits one B200: the 513^3 three-layer wedge
(2000/1500/3000 m/s split by z = 0.4 + 0.2x and z = 0.8 - 0.2x, kh = 0.625 at
the slowest layer), first-order Sommerfeld faces, point source at
(0.5, 0.5, 0.1), complex128, CSLP shift beta1 = 1, |beta2| = 0.5 (the
reference's damping-consistent sign, beta2 = -0.5), one V(1,1) cycle with
damped Jacobi omega = 0.8, full weighting, trilinear prolongation, Bi-CGSTAB
tol 1e-6 with the reference's shadow vector r~ = b.  One step = a FIXED
budget of 100 Bi-CGSTAB iterations from a resident right-hand side (the
reference algorithm stops on its rho breakdown test after 389-978 iterations
on this grid, so a full solve is not the unit).  The
metric is Munknowns*iter/s = (vertices x iterations) / device time, summed
over all GPUs.  The 2.2 GB fields are ~17x L2, so every launch streams from
HBM; L2 is also flushed (256 MiB write) before every timed step.

Besides the headline line the run reports, in `config`:
  * time_to_solution of configs[2] with the seeded shadow vector
    (SolverConfig.shadow = "random", converges where r~ = b breaks down);
  * configs[1] (129^3, k = 80 cube) time to solution at tol 1e-6.

`roofline.kernels` is the live CUDA-event table of the finest-level kernels on
the DEFAULT path of this workload (wide sweep family: pre-smoothing + residual
sweep, restriction, fused up-sweep, matvec, matvec with t^H t / t^H s, the three
vector updates), `share` = launches per iteration x ms / ms per iteration; the
kernels of other variants appear with share null.  `--opt name=0|1` sets a
kernel-variant option of the library for an A/B run,
`--no-tts` / `--no-cpu` skip the secondary measurements.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1] [--impl reference]
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cslp_bicgstab_munknowns_iter_per_s"
UNIT = "Munknowns*iter/s"
TOL = 1e-6
L2_BYTES = 126 * 1024 * 1024

CONFIGS = {
    "c2": {
        "workload": ("configs[2]: 513^3 three-layer wedge (2000/1500/3000 m/s, tilted planes "
                     "z=0.4+0.2x, z=0.8-0.2x), kh<=0.625, Sommerfeld, source (0.5,0.5,0.1), "
                     "complex128, CSLP(1, 0.5i-damped) V(1,1) omega=0.8, Bi-CGSTAB tol 1e-6 "
                     "(r~=b), fixed budget of 100 iterations per step"),
        "iters": 100, "fixed": True, "cpu_iters": 1,
    },
    "c1": {
        "workload": ("configs[1]: 129^3 unit cube, k=80 (kh=0.625), Sommerfeld, centre point "
                     "source, complex128, CSLP(1, 0.5i-damped) V(1,1) omega=0.8, Bi-CGSTAB tol 1e-6"),
        "iters": 400, "fixed": False, "cpu_iters": 400,
    },
}


def _problem(name):
    from paper_2308_06085_b200 import problems
    p = problems.wedge3_problem(513) if name == "c2" else problems.point_source_cube(129, 80.0)
    spec, b = problems.build_problem(p)
    return p, spec, b


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


def _ncu_traffic(kernel, config):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant
    kernel, from the committed ncu --set full summary (profiles/ncu_traffic.json,
    tools/ncu_traffic.py); None when it was captured for another kernel/config."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            d = json.load(f)
        e = d.get(config, {})
        if "kernel" in e:             # single-kernel entry
            e = {e["kernel"]: e}
        return e[kernel]["traffic_bytes_per_launch"] if kernel in e else None
    except Exception:
        return None


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


def _solver_for(p, spec):
    from paper_2308_06085_b200.krylov import Solver
    from paper_2308_06085_b200.multigrid import MGConfig, build_hierarchy
    from paper_2308_06085_b200.operators import OperatorSpec, StencilOperator
    A = StencilOperator(spec, p.grid)
    hier = build_hierarchy(p.grid, None, OperatorSpec("cslp", 1.0, -0.5, spec.bc, spec.k_field),
                           MGConfig())
    return A, hier, Solver(A, hier)


def run_gpu(args):
    import torch

    from paper_2308_06085_b200.krylov import SolverConfig

    rank, world, local = _env_rank()
    if world > 1:
        return run_slabs(args)
    torch.cuda.set_device(local)
    C = CONFIGS[args.config]
    p, spec, b_host = _problem(args.config)
    n = p.grid.num_vertices
    t_setup = time.perf_counter()
    A, hier, solver = _solver_for(p, spec)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    cfg = SolverConfig(method="bicgstab", tol=TOL, maxit=C["iters"], check_every=4)
    b = torch.as_tensor(b_host).cuda()
    x = torch.empty_like(b)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    for _ in range(args.warmup):
        _, rep = solver.solve(b, cfg, x=x)
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
    total_ms = float(np.sum(times))
    iters = reps[-1].iterations
    ms_step = total_ms / args.steps
    value = n * iters / (ms_step / 1e3) / 1e6

    # ---- e2e: public API from pinned host buffers (H2D + solve + D2H) ----
    bh = torch.as_tensor(b_host).pin_memory().numpy()
    xh = torch.empty(b_host.shape, dtype=torch.complex128).pin_memory().numpy()
    solver.solve(bh, cfg, x=xh, host=True)
    e2e_ms, e2e_it = [], []
    for _ in range(max(1, min(args.steps, 3))):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _, rep_h = solver.solve(bh, cfg, x=xh, host=True)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_it.append(rep_h.iterations)
    e2e_step = float(np.mean(e2e_ms))
    e2e_value = n * float(np.mean(e2e_it)) / (e2e_step / 1e3) / 1e6

    # ---- kernel roofline: live CUDA-event timing of the path's kernels ----
    hbm, peak_kind = _peaks()
    t_iter = ms_step / max(iters, 1)
    kern = kernel_table(A, hier, solver, n, t_iter, sparse_shadow=np.count_nonzero(b_host) <= 16)
    dom = max((k_ for k_ in kern if kern[k_]["bound"] == "hbm" and kern[k_]["share"]),
              key=lambda k_: kern[k_]["share"])
    kd = kern[dom]
    roofline = {"bound": "hbm", "kernel": dom, "kernel_symbol": kd["symbol"],
                "achieved": kd["gbs"], "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
                "frac": round(kd["gbs"] / hbm, 4), "traffic": _ncu_traffic(dom, args.config),
                "algorithmic_bytes_per_launch": kd["bytes"], "bytes_per_vertex": kd["bpv"],
                "launch_ms": kd["ms"],
                "kernels": {k_: {"gbs": v_["gbs"], "frac": round(v_["gbs"] / hbm, 4),
                                 "ms": v_["ms"], "share": v_["share"], "bound": v_["bound"],
                                 "bytes_per_vertex": v_["bpv"], "symbol": v_["symbol"]}
                            for k_, v_ in kern.items()}}

    extra = {"unknowns": n, "grid": list(p.grid.shape),
             "k_range": [float(np.min(spec.k_field)), float(np.max(spec.k_field))],
             "tol": TOL, "maxit_per_step": C["iters"], "parallelism": "single GPU",
             "l2": "fields 2.2 GB (17x L2) and a 256 MiB L2 flush before every timed step"
             if args.config == "c2" else "flushed (256 MiB write) before every timed step",
             "iterations": iters, "matvecs": reps[-1].matvec_count,
             "converged": reps[-1].converged, "breakdown": reps[-1].breakdown,
             "final_relres": reps[-1].final_relres, "ms_per_iteration": round(t_iter, 4),
             "setup_s": round(t_setup, 3)}
    if not C["fixed"]:
        extra["time_to_solution_s"] = round(ms_step / 1e3, 6)
    if args.config == "c2" and not args.no_tts:
        extra["time_to_solution_random_shadow"] = tts_random_shadow(solver, b, x, n)
        del A, hier, solver
        torch.cuda.empty_cache()
        extra["configs1"] = configs1_tts()

    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": f"synthetic (BASELINE {C['workload'][:10]} problem, built in-process)",
        "config": {"workload": C["workload"], **extra},
        "clocks": clk.summary(),
        "gpu_launches": int(sum(r.kernel_launches for r in reps)),
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT,
                "h2d_bytes_per_step": int(b_host.nbytes), "d2h_bytes_per_step": int(b_host.nbytes),
                "ms_per_step": round(e2e_step, 4)},
        "roofline": roofline,
    }
    if rank == 0 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args.config, min(args.cpu_iters or C["cpu_iters"],
                                                            C["cpu_iters"]))
    print(json.dumps(out), flush=True)


def tts_random_shadow(solver, b, x, n):
    """One full configs[2] solve to tol 1e-6 with the seeded shadow vector
    (SolverConfig.shadow = "random"): the time to solution where the
    reference's r~ = b stops on the rho breakdown test."""
    import torch

    from paper_2308_06085_b200.krylov import SolverConfig
    cfg = SolverConfig(method="bicgstab", tol=TOL, maxit=4000, shadow="random", check_every=8)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    _, rep = solver.solve(b, cfg, x=x)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    return {"shadow": "random (HF_SHADOW_HASH, seed 1234)", "iterations": rep.iterations,
            "converged": rep.converged, "breakdown": rep.breakdown,
            "final_relres": rep.final_relres, "time_to_solution_s": round(ms / 1e3, 4),
            "munknowns_iter_per_s": round(n * rep.iterations / (ms / 1e3) / 1e6, 2)}


def configs1_tts(steps=5):
    """configs[1] (129^3, k = 80) time to solution at tol 1e-6, device-timed."""
    import torch

    from paper_2308_06085_b200.krylov import SolverConfig
    p, spec, b_host = _problem("c1")
    A, hier, solver = _solver_for(p, spec)
    cfg = SolverConfig(method="bicgstab", tol=TOL, maxit=400, check_every=4)
    b = torch.as_tensor(b_host).cuda()
    x = torch.empty_like(b)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(2):
        solver.solve(b, cfg, x=x)
    ts = []
    for _ in range(steps):
        flush.fill_(1.0)
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        _, rep = solver.solve(b, cfg, x=x)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ms = float(np.mean(ts))
    n = p.grid.num_vertices
    return {"workload": CONFIGS["c1"]["workload"], "iterations": rep.iterations,
            "converged": rep.converged, "time_to_solution_s": round(ms / 1e3, 6),
            "munknowns_iter_per_s": round(n * rep.iterations / (ms / 1e3) / 1e6, 2)}


def run_slabs(args):
    """N > 1: the grid split into N slabs along i1, one per GPU, run by the
    native slab driver (dist.NativeSlabSolver): each iteration one CUDA graph
    with the halo exchanges as ncclSend/ncclRecv between neighbours, the inner
    products as one ncclAllReduce each and the coarsest slabs ncclAllGather-ed
    and solved on every rank."""
    import torch
    import torch.distributed as dist

    from paper_2308_06085_b200.dist import NativeSlabSolver
    from paper_2308_06085_b200.krylov import SolverConfig
    from paper_2308_06085_b200.partition import TorchSlabComm, slab_partition

    rank, world, local = _env_rank()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    C = CONFIGS[args.config]
    p, spec, b_host = _problem(args.config)
    n = p.grid.num_vertices
    e = slab_partition(p.grid, world)[rank]
    comm = TorchSlabComm()
    t_setup = time.perf_counter()
    S = NativeSlabSolver(p.grid, [e], spec.k_field, p.bc, comm, maxit=C["iters"])
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    cfg = SolverConfig(method="bicgstab", tol=TOL, maxit=C["iters"])
    b = [torch.as_tensor(b_host[e.lo1 - 1:e.hi1]).cuda()]
    for _ in range(args.warmup):
        _, rep = S.solve(b, cfg)
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            dist.barrier()
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            e0 = torch.cuda.Event(enable_timing=True)
            s0.record()
            _, rep = S.solve(b, cfg)
            e0.record()
            torch.cuda.synchronize()
            times.append(s0.elapsed_time(e0))
    t = torch.tensor([float(np.sum(times))], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    iters = rep.iterations
    bh = torch.as_tensor(b_host[e.lo1 - 1:e.hi1]).pin_memory()
    dist.barrier()
    t0 = time.perf_counter()
    xs, rep_h = S.solve([bh.cuda(non_blocking=True)], cfg)
    xs[0].cpu()
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
            "data": f"synthetic (BASELINE {C['workload'][:10]} problem, built in-process)",
            "config": {"workload": C["workload"], "unknowns": n, "grid": list(p.grid.shape),
                       "parallelism": f"{world} slabs along i1 (native slab graph: NCCL P2P halos, "
                                      "NCCL allreduce for the inner products)",
                       "iterations": iters, "matvecs": rep.matvec_count,
                       "converged": rep.converged, "breakdown": rep.breakdown,
                       "final_relres": rep.final_relres, "setup_s": round(t_setup, 3)},
            "clocks": clk.summary(), "gpu_launches": None,
            "e2e": {"value": round(n * rep_h.iterations / (e2e_ms / 1e3) / 1e6, 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(bh.numel() * 16),
                    "d2h_bytes_per_step": int(bh.numel() * 16), "ms_per_step": round(e2e_ms, 4)},
            "roofline": None,
        }
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


def kernel_table(A, hier, solver, n, t_iter_ms, reps=12, sparse_shadow=True):
    """Live CUDA-event timing of the kernels the finest level of THIS workload's
    solve launches (the fused flat down-kernel where the plane is <= 255 wide,
    the split presmooth+residual / restriction pair otherwise; correction +
    Jacobi sweep; matvec; Bi-CGSTAB vector updates), each on operands that
    stream from HBM: fields larger than L2 are used directly, smaller ones
    rotate over sets whose total is > 2x L2.

    bytes_per_vertex = algorithmic HBM bytes per fine vertex of one launch:
    16 per complex field read or written, + 8 for k when the medium varies
    (constant media pass k as a scalar) and + 16 where a kernel streams the
    stored D^-1 field (k_corr, k_flat_dr; the stencil sweeps form D^-1 from k),
    + 16 / 8 per fine vertex for coarse fields.  share = launches per
    Bi-CGSTAB iteration x ms / (ms per iteration)."""
    import torch

    from paper_2308_06085_b200 import _native

    L = _native.load()
    _native.set_stream_from_torch()
    lv0, lv1 = hier.levels[0], hier.levels[1]
    shape, cshape = lv0.extent.shape, lv1.extent.shape
    nf = int(np.prod(shape))
    nc = int(np.prod(cshape))
    cr = nc / nf
    kvar = A._keep is not None     # k passed per vertex (operators.k_arguments)
    kb, db = (8.0, 16.0) if kvar else (0.0, 0.0)
    # palette levels (wide planes, <= 256 distinct k): 1-byte indices, no D^-1
    # field; the pre-smoothing sweep still streams the 8-byte k
    pal = kvar and shape[2] > 256 and len(np.unique(np.asarray(A.spec.k_field)[::7, ::7, ::7])) <= 256 \
        and not _native.load().hf_get_option(b"no_palette")
    kp, dp = (1.0, 0.0) if pal else (kb, db)
    nset = 1 if nf * 16 > 2 * L2_BYTES else 4
    rnd = lambda sh: torch.randn(sh, dtype=torch.complex128, device="cuda")
    sets = [dict(u=rnd(shape), b=rnd(shape), v=rnd(shape), t=rnd(shape), ec=rnd(cshape),
                 bc=rnd(cshape)) for _ in range(nset)]
    H = hier._h
    ncs = hier.coarsest.grid.num_vertices
    xc, rc = rnd(hier.coarsest.grid.shape), rnd(hier.coarsest.grid.shape)
    p = lambda x: x.data_ptr()
    fused_down = shape[2] <= 255
    wide = not fused_down and not L.hf_get_option(b"no_wide")
    wide_all = wide and bool(L.hf_get_option(b"wide_all"))
    wide_up = wide and not L.hf_get_option(b"no_wide_up") and not L.hf_get_option(b"no_fuse")
    sweep = "k_flat_stencil" if fused_down else ("k_wide" if wide_all else "k_stencil")
    cases = {
        "device_copy": (lambda s: s["v"].copy_(s["u"]), 32.0, "ceiling", 0, "torch copy_"),
        # the first matvec of an iteration (sparse shadow: r~^H v is gathered, no inner-product
        # pass); the second one carries t^H t and t^H s (matvec_dot2 below)
        "helmholtz_matvec": (lambda s: L.hf_operator_apply(A._h, p(s["u"]), p(s["v"])),
                             32.0 + kp, "hbm", 1 if sparse_shadow else 0, "k_wide<LOAD,APPLY0>" if wide else f"{sweep}<LOAD,EpiApply>"),
        # split up-sweep: on the default path only where the fused up-sweep does not apply
        "prolong_correct": (lambda s: L.hf_level_correct(H, 0, p(s["b"]), p(s["ec"]), p(s["t"])),
                            32.0 + (1.0 if pal else db) + 16.0 * cr, "hbm", 0 if wide_up else 2,
                            "k_corr_flat<1>"),
        "jacobi_postsmooth": (lambda s: L.hf_level_smooth(H, 0, p(s["t"]), p(s["b"]), p(s["u"])),
                              48.0 + kp, "hbm", 0 if wide_up else 2, f"{sweep}<LOAD,EpiJacobi>"),
    }
    if fused_down:
        cases["down_restrict"] = (lambda s: L.hf_level_down_restrict(H, 0, p(s["b"]), p(s["bc"])),
                                  16.0 + kb + db + 16.0 * cr, "hbm", 2, "k_flat_dr")
    else:
        # the wide family's pre-smoothing sweep reads the palette index (1 B), the tiled one k (8 B)
        cases["presmooth_residual"] = (lambda s: L.hf_level_down1(H, 0, p(s["b"]), p(s["v"])),
                                       32.0 + (kp if wide else kb), "hbm", 2,
                                       "k_wide<PRE,RESID>" if wide else "k_stencil<PRE,EpiResid>")
        cases["restrict_fw"] = (lambda s: L.hf_restrict_fw(H, 0, p(s["v"]), p(s["bc"])),
                                16.0 + 16.0 * cr, "hbm", 2, "k_restrict_flat")
        if wide_up:
            # fused up-sweep: b, palette index / k, coarse e in; u out (t never written)
            cases["up_fused"] = (lambda s: L.hf_level_up(H, 0, p(s["b"]), p(s["ec"]), p(s["u"])),
                                 32.0 + kp + 16.0 * cr, "hbm", 2, "k_wide<UP,JACOBI>")
        # the tiled fused alternatives on wide planes (not on the default path: share None)
        cases["down_restrict_tiled"] = (lambda s: L.hf_level_down_restrict(H, 0, p(s["b"]), p(s["bc"])),
                                        16.0 + kb + 16.0 * cr, "hbm", 0, "k_down_restrict")
        kp_up = kb       # the tiled fused up-sweep stages the 8-byte k (D^-1 of every staged entry)

        def up_fused(s):
            with _native.options(fuse_up=1):
                L.hf_level_up(H, 0, p(s["b"]), p(s["ec"]), p(s["u"]))
        cases["up_fused_tiled"] = (up_fused, 32.0 + kp_up + 16.0 * cr, "hbm", 0, "k_stencil<UP,EpiJacobi>")
    kind = hier.coarsest_kind
    nt = -(-ncs // 64)
    cbytes = {"separable": 112.0 * ncs,
              "symmetric": float(nt * (nt + 1) // 2 * 64 * 64 * 16 + 2 * nt * (nt + 1) // 2 * 64 * 32),
              "dense": 16.0 * ncs * ncs}.get(kind, 0.0)
    out = {}

    def put(name, ms, bpv, bound, launches, symbol, total_bytes=None):
        nbytes = total_bytes if total_bytes is not None else bpv * nf
        out[name] = {"ms": round(ms, 5), "bytes": nbytes, "bpv": round(bpv, 3),
                     "gbs": round(nbytes / (ms / 1e3) / 1e9, 1),
                     "share": round(launches * ms / t_iter_ms, 4) if launches else None,
                     "bound": bound, "symbol": symbol}

    r = max(nset, reps // nset * nset)
    for name, (fn, bpv, bound, launches, sym) in cases.items():
        for s in sets:
            fn(s)
        k = [0]

        def run():
            fn(sets[k[0] % nset])
            k[0] += 1
        put(name, _event_time(run, r), bpv, bound, launches, sym)
    ms = _event_time(lambda: L.hf_coarsest_solve(H, p(rc), p(xc)), r)
    put("coarsest_solve", ms, 0.0, "latency" if kind == "separable" else "hbm", 2,
        f"coarsest ({kind})", total_bytes=cbytes)
    # Bi-CGSTAB vector kernels, once per iteration (krylov.py:240-269), back to
    # back on the solver's workspace
    # the x/r update reads r~ only when the shadow vector is dense; a point
    # source with the reference's r~ = b is sparse (gathered)
    sparse = bool(sparse_shadow)
    for nm, which, bpv in (("bcg_p_update", 0, 64.0), ("bcg_s_update", 1, 48.0),
                           ("bcg_xr_update", 3 if sparse else 2, 112.0 if sparse else 128.0),
                           ("matvec_dot2", 4, 48.0 + kp)):
        m = ctypes.c_float()
        _native.check(L.hf_solver_bench_vec(solver._h, which, r, ctypes.byref(m)))
        # (the solver's own vectors: HBM-streaming when a vector is larger than L2, else the
        # launches re-read L2-resident data and the figure is not an HBM fraction)
        put(nm, m.value, bpv, "hbm" if nf * 16 > L2_BYTES else "l2-resident", 1 if which != 4 or sparse else 2,
            ("k_bcg_p", "k_bcg_s", "k_bcg_xr", "k_bcg_xr (sparse r~)", f"{sweep}<LOAD,EpiApply<2>>")[which])
    return out


def cpu_baseline(config: str, iters: int, steps: int = 1):
    """The C oracle (a port of the reference algorithm: same operators, cycle,
    GMRES coarsest solve and Bi-CGSTAB) on this host's cores (OpenMP over all of
    them), on the same workload: `iters` Bi-CGSTAB iterations per sample, the
    hierarchy built once outside the timed region (as in the native arm)."""
    from oracle import oracle as O
    p, spec, b = _problem(config)
    k = np.asarray(spec.k_field, dtype=np.float64)
    S = O.PersistentSolver(k, p.grid.h)
    x = np.empty_like(b)
    n = p.grid.num_vertices
    vals, secs = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        _, rep = S.solve(b, "bicgstab", TOL, iters, x=x)
        dt = time.perf_counter() - t0
        vals.append(n * rep["iterations"] / dt / 1e6)
        secs.append(dt)
    return {"value": round(float(np.mean(vals)), 3), "unit": UNIT, "cores": O.num_threads(),
            "kind": "port",
            "sample": f"first {rep['iterations']} Bi-CGSTAB iterations of the {CONFIGS[config]['workload'][:10]} "
                      f"{'x'.join(map(str, p.grid.shape))} solve (hierarchy built once, untimed), "
                      f"{float(np.mean(secs)):.2f} s",
            "ms_per_sample": round(float(np.mean(secs)) * 1e3, 2)}


def run_reference(args):
    rank, world, _ = _env_rank()
    if rank != 0:
        return
    C = CONFIGS[args.config]
    iters = args.cpu_iters or C["cpu_iters"]
    cb = cpu_baseline(args.config, iters, steps=args.warmup + args.steps)
    out = {"metric": METRIC, "value": cb["value"], "unit": UNIT, "impl": "reference",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": cb["ms_per_sample"],
           "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "c128", "data": "synthetic",
           "config": {"workload": C["workload"], "parallelism": "host cores (OpenMP)"},
           "cpu_baseline": {k: v for k, v in cb.items() if k != "ms_per_sample"},
           "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="GPUs of this node; >1 runs under torchrun (one rank per GPU)")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    # CPU legs: Bi-CGSTAB iterations per sample (default: 1 at 513^3, ~5 s on 16 cores;
    # the full solve at 129^3)
    ap.add_argument("--cpu-iters", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tts", action="store_true", help="skip the secondary solves in config")
    ap.add_argument("--opt", action="append", default=[], metavar="NAME=0|1",
                    help="kernel-variant option of the library (hf_set_option), for A/B runs")
    args = ap.parse_args()
    if args.opt and args.impl == "native":
        from paper_2308_06085_b200 import _native
        for kv in args.opt:
            name, _, val = kv.partition("=")
            _native.set_option(name, int(val or 1))
    _, world, _ = _env_rank()
    if args.gpus != world and args.impl == "native":
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torchrun")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
