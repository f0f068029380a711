"""Multi-slab CSLP-preconditioned Bi-CGSTAB (one slab per GPU, or several
virtual slabs on one GPU).

The SPMD structure of the reference's worker_body (runner.py:95-131) with
its distributed V-cycle (multigrid.py:326-343) and global inner products
(partition.py:611-621), re-laid for slabs along i1:

  level l < L-1 :  halo(b) -> r = b - M(w D^-1 b) -> halo(r) -> R r
  coarsest      :  all-gather the coarse slabs, exact solve (replicated)
  level l       :  halo(e) -> t = w D^-1 b + P e -> halo(t) -> Jacobi sweep

Every stencil / transfer / smoother step is a native kernel on the slab
(hf_level_down1, hf_restrict_fw, hf_level_correct, hf_level_smooth,
hf_operator_apply, hf_coarsest_solve); halos and inner products go through
the slab fabric (partition.TorchSlabComm or LocalSlabComm).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .grid import HF_GHOST, BlockExtent, Grid3, HaloField, full_extent, make_grid
from .krylov import ConvergenceReport, SolverConfig
from .multigrid import MGConfig
from .operators import OperatorSpec, StencilOperator, bc_name, k_arguments

__all__ = ["SlabSolver", "NativeSlabSolver"]


def _ptr(t):
    return t.data_ptr()


class SlabSolver:
    """Bi-CGSTAB over the slabs owned by this process (krylov.py:207-276)."""

    def __init__(self, grid: Grid3, extents, k_field, bc, comm, beta1=1.0, beta2=-0.5,
                 mg: MGConfig | None = None):
        import torch
        self.torch = torch
        self.grid, self.comm = grid, comm
        self.extents = list(extents)
        self.mg = mg or MGConfig()
        if self.mg.cycle.upper() != "V" or self.mg.nu1 != 1 or self.mg.nu2 != 1:
            raise NotImplementedError("slab driver implements the V(1,1) cycle")
        L = _native.load()
        self.L = L
        kfull, kc, self._keep = k_arguments(
            OperatorSpec("helmholtz", 1.0, 0.0, bc, np.asarray(k_field)), grid, full_extent(grid))
        kp = kfull.ctypes.data if kfull is not None else None
        bcc = _native.BC[bc_name(bc)]
        c = _native.MGConfigC(1, 1, float(self.mg.omega), 0, int(self.mg.coarsest_threshold),
                              1 if self.mg.threshold_cmp == "ge" else 0, float(self.mg.coarsest_tol),
                              int(self.mg.coarsest_maxit), _native.COARSEST["external"])
        _native.set_stream_from_torch()
        self.A, self.H, self.levels = [], [], []
        for e in self.extents:
            A = L.hf_operator_create(grid.n1, grid.n2, grid.n3, e.lo1 - 1, e.nx, grid.h, 1.0, 0.0,
                                     bcc, kp, kc)
            H = L.hf_hierarchy_create(grid.n1, grid.n2, grid.n3, e.lo1 - 1, e.nx, grid.h,
                                      float(beta1), float(beta2), bcc, kp, kc, ctypes.byref(c))
            if not A or not H:
                raise RuntimeError(_native.last_error())
            self.A.append(A)
            self.H.append(H)
            lv = []
            for l in range(L.hf_hierarchy_num_levels(H)):
                d = (ctypes.c_int * 5)()
                _native.check(L.hf_hierarchy_level_shape(H, l, d))
                lv.append(BlockExtent(d[3] + 1, 1, 1, d[3] + d[4], d[1], d[2]))
            self.levels.append(lv)
        self.nlev = len(self.levels[0])
        # fused down + restriction per level: needs an HF_GHOST-deep halo of b, so
        # every slab of that level must own at least HF_GHOST planes
        nsl = len(self.extents) if len(self.extents) > 1 else getattr(comm, "size", 1)
        self._fuse_down = [all(e.nx >= HF_GHOST for e in _level_extents(grid, nsl, l + 1))
                           for l in range(self.nlev)]
        d = (ctypes.c_int * 5)()
        _native.check(L.hf_hierarchy_level_shape(self.H[0], self.nlev - 1, d))
        cgrid = make_grid(d[0], d[1], d[2], grid.h * 2 ** (self.nlev - 1))
        self.cgrid = cgrid
        # coarsest level: the whole coarse grid on every process (exact solve, replicated)
        kc_full = None
        if kfull is not None:
            s = 2 ** (self.nlev - 1)
            kc_full = np.ascontiguousarray(kfull[::s, ::s, ::s])
            self._keep_c = kc_full
        cc = _native.MGConfigC(1, 1, float(self.mg.omega), 0, max(cgrid.shape) + 1, 0,
                               float(self.mg.coarsest_tol), int(self.mg.coarsest_maxit),
                               _native.COARSEST["direct"])
        self.Hc = L.hf_hierarchy_create(cgrid.n1, cgrid.n2, cgrid.n3, 0, cgrid.n1, cgrid.h,
                                        float(beta1), float(beta2), bcc,
                                        kc_full.ctypes.data if kc_full is not None else None,
                                        kc if kfull is None else 0.0, ctypes.byref(cc))
        if not self.Hc:
            raise RuntimeError(_native.last_error())
        self.ccounts = [lv[-1].nx for lv in self.levels] if len(self.extents) > 1 else None
        # level fields per local slab: b, r, u, t (with ghost planes)
        f = lambda e: HaloField(e)
        self.fb = [[f(lv[l]) for l in range(self.nlev)] for lv in self.levels]
        self.fr = [[f(lv[l]) for l in range(self.nlev)] for lv in self.levels]
        self.fu = [[f(lv[l]) for l in range(self.nlev)] for lv in self.levels]
        self.ft = [[f(lv[l]) for l in range(self.nlev)] for lv in self.levels]
        self.xc = torch.empty(cgrid.shape, dtype=torch.complex128, device="cuda")

    def __del__(self):
        try:
            for h in getattr(self, "A", []):
                self.L.hf_operator_destroy(h)
            for h in getattr(self, "H", []):
                self.L.hf_hierarchy_destroy(h)
            if getattr(self, "Hc", None):
                self.L.hf_hierarchy_destroy(self.Hc)
        except Exception:   # interpreter shutdown
            pass

    # ---- building blocks -------------------------------------------------
    def _halo(self, fields):
        self.comm.exchange([h.data for h in fields], planes=1)

    def _dot(self, a, b):
        out = (ctypes.c_double * 2)()
        vals = []
        for x, y in zip(a, b):
            _native.check(self.L.hf_dot(x.numel(), _ptr(x), _ptr(y), out))
            vals.append(complex(out[0], out[1]))
        return self.comm.allreduce(vals)

    def precondition(self, src, dst):
        """dst = one V(1,1) cycle applied to src (lists of per-slab HaloFields)."""
        L, n = self.L, self.nlev
        S = range(len(self.extents))
        for r in S:
            self.fb[r][0].owned.copy_(src[r].owned)
        for l in range(n - 1):
            if self._fuse_down[l]:
                # one HF_GHOST-deep halo of b, then the fused down + restriction
                self.comm.exchange([self.fb[r][l].data for r in S], planes=HF_GHOST)
                for r in S:
                    _native.check(L.hf_level_down_restrict(self.H[r], l, _ptr(self.fb[r][l].owned),
                                                           _ptr(self.fb[r][l + 1].owned)))
                continue
            self._halo([self.fb[r][l] for r in S])
            for r in S:
                _native.check(L.hf_level_down1(self.H[r], l, _ptr(self.fb[r][l].owned),
                                               _ptr(self.fr[r][l].owned)))
            self._halo([self.fr[r][l] for r in S])
            for r in S:
                _native.check(L.hf_restrict_fw(self.H[r], l, _ptr(self.fr[r][l].owned),
                                               _ptr(self.fb[r][l + 1].owned)))
        # coarsest: gather the coarse slabs, exact solve, keep this slab's planes
        parts = [self.fb[r][n - 1].owned for r in S]
        if len(self.extents) > 1 or getattr(self.comm, "size", 1) > 1:
            if len(self.extents) > 1:
                bc = self.comm.allgather_planes(parts, self.ccounts)
            else:
                counts = [e.nx for e in _coarse_extents(self.grid, self.comm.size, n)]
                bc = self.comm.allgather_planes(parts[0], counts)
        else:
            bc = parts[0]
        bc = bc.contiguous()
        _native.check(L.hf_coarsest_solve(self.Hc, _ptr(bc), _ptr(self.xc)))
        for r in S:
            e = self.levels[r][n - 1]
            self.fu[r][n - 1].owned.copy_(self.xc[e.lo1 - 1:e.hi1])
        for l in range(n - 2, -1, -1):
            self._halo([self.fu[r][l + 1] for r in S])
            # t on the owned planes and the interior-face ghost planes (b's halo from the
            # down-sweep is still valid): no halo exchange of t before the sweep
            for r in S:
                _native.check(L.hf_level_correct_ext(self.H[r], l, _ptr(self.fb[r][l].owned),
                                                     _ptr(self.fu[r][l + 1].owned),
                                                     _ptr(self.ft[r][l].owned)))
            for r in S:
                out = dst[r] if l == 0 else self.fu[r][l]
                _native.check(L.hf_level_smooth(self.H[r], l, _ptr(self.ft[r][l].owned),
                                                _ptr(self.fb[r][l].owned), _ptr(out.owned)))

    def apply_A(self, src, dst):
        self._halo(src)
        for r in range(len(self.extents)):
            _native.check(self.L.hf_operator_apply(self.A[r], _ptr(src[r].owned), _ptr(dst[r])))

    # ---- Bi-CGSTAB (krylov.py:207-276) ------------------------------------
    def solve(self, b_slabs, cfg: SolverConfig | None = None):
        """b_slabs: per local slab, the right-hand side (owned shape).  Returns
        (x per slab, ConvergenceReport)."""
        torch = self.torch
        cfg = cfg or SolverConfig(method="bicgstab")
        _native.set_stream_from_torch()
        S = range(len(self.extents))
        own = lambda: [torch.zeros(e.shape, dtype=torch.complex128, device="cuda") for e in self.extents]
        halo = lambda: [HaloField(e) for e in self.extents]
        b = [torch.as_tensor(x).to("cuda", torch.complex128) for x in b_slabs]
        x, v, t = own(), own(), own()
        p, s, ph, sh = halo(), halo(), halo(), halo()
        rep = ConvergenceReport(method="bicgstab")
        bnorm = abs(self._dot(b, b)) ** 0.5
        if bnorm == 0.0:
            rep.converged, rep.final_relres = True, 0.0
            return x, rep
        r = [bi.clone() for bi in b]
        rs = [bi.clone() for bi in b]
        rho = alpha = omega = 1.0 + 0j
        while rep.iterations < cfg.maxit:
            rho_new = self._dot(rs, r)
            if abs(rho_new) < cfg.breakdown_tol:
                rep.breakdown = "rho"
                break
            beta = (rho_new / rho) * (alpha / omega)
            for i in S:
                p[i].owned.copy_(r[i] + beta * (p[i].owned - omega * v[i]))
            self.precondition(p, ph)
            self.apply_A(ph, v)
            rep.matvec_count += 1
            den = self._dot(rs, v)
            if abs(den) < cfg.breakdown_tol:
                rep.breakdown = "rho"
                break
            alpha = rho_new / den
            for i in S:
                s[i].owned.copy_(r[i] - alpha * v[i])
            snorm = abs(self._dot([si.owned for si in s], [si.owned for si in s])) ** 0.5
            if snorm / bnorm <= cfg.tol:
                for i in S:
                    x[i] += alpha * ph[i].owned
                rep.record(snorm / bnorm)
                rep.converged = True
                return x, rep
            self.precondition(s, sh)
            self.apply_A(sh, t)
            rep.matvec_count += 1
            tt = self._dot(t, t)
            if abs(tt) < cfg.breakdown_tol:
                rep.breakdown = "omega"
                break
            omega = self._dot(t, [si.owned for si in s]) / tt
            if abs(omega) < cfg.breakdown_tol:
                rep.breakdown = "omega"
                break
            for i in S:
                x[i] += alpha * ph[i].owned + omega * sh[i].owned
                r[i] = s[i].owned - omega * t[i]
            rho = rho_new
            relres = abs(self._dot(r, r)) ** 0.5 / bnorm
            rep.record(relres)
            if relres <= cfg.tol:
                rep.converged = True
                return x, rep
        rep.converged = False
        return x, rep

    # ---- device-resident Bi-CGSTAB (same recurrences, scalars on the device) ----
    def solve_device(self, b_slabs, cfg: SolverConfig | None = None, poll_every: int = 4):
        """Bi-CGSTAB with the scalars advanced on the device (hf_bcg_*): each
        reduction leaves this slab's partial sums on the device, the comm adds
        them over slabs / ranks (an NCCL all-reduce across processes), and a
        one-thread kernel updates the state.  The host only polls the state
        every `poll_every` iterations; kernels launched past convergence are
        no-ops on the state and on x.  Returns (x per slab, ConvergenceReport)."""
        torch, L = self.torch, self.L
        cfg = cfg or SolverConfig(method="bicgstab")
        _native.set_stream_from_torch()
        S = range(len(self.extents))
        own = lambda: [torch.zeros(e.shape, dtype=torch.complex128, device="cuda") for e in self.extents]
        halo = lambda: [HaloField(e) for e in self.extents]
        b = [torch.as_tensor(x).to("cuda", torch.complex128).contiguous() for x in b_slabs]
        x, v, t, r, rs = own(), own(), own(), own(), own()
        p, s, ph, sh = halo(), halo(), halo(), halo()
        n = [e.nx * e.ny * e.nz for e in self.extents]
        big = max(S, key=lambda i: n[i])
        B = L.hf_bcg_create(self.A[big], float(cfg.tol), int(cfg.maxit), float(cfg.breakdown_tol))
        if not B:
            raise RuntimeError(_native.last_error())
        sums = [torch.zeros(2, dtype=torch.complex128, device="cuda") for _ in S]
        chk = _native.check
        keep = []

        def reduce_step(op):
            tot = self.comm.allreduce_device(sums)
            keep.append(tot)            # alive until the kernel reading it has run
            chk(L.hf_bcg_step(B, op, _ptr(tot)))

        try:
            for i in S:
                chk(L.hf_bcg_vec_init(B, n[i], _ptr(b[i]), _ptr(r[i]), _ptr(rs[i]), _ptr(x[i]),
                                      _ptr(p[i].owned), _ptr(v[i]), _ptr(sums[i])))
            reduce_step(1)
            st = (ctypes.c_int * 6)()
            relres = ctypes.c_double()
            while True:
                chk(L.hf_bcg_read(B, st, ctypes.byref(relres), None, 0))
                keep.clear()
                if st[1] or st[0] >= cfg.maxit:
                    break
                for _ in range(poll_every):
                    for i in S:
                        chk(L.hf_bcg_vec_p(B, n[i], _ptr(r[i]), _ptr(p[i].owned), _ptr(v[i])))
                    self.precondition(p, ph)
                    self._halo(ph)
                    for i in S:
                        chk(L.hf_operator_apply_dot(self.A[i], B, 1, _ptr(ph[i].owned), _ptr(v[i]),
                                                    _ptr(rs[i]), _ptr(sums[i])))
                    reduce_step(2)
                    for i in S:
                        chk(L.hf_bcg_vec_s(B, n[i], _ptr(r[i]), _ptr(v[i]), _ptr(s[i].owned),
                                           _ptr(sums[i])))
                    reduce_step(3)
                    self.precondition(s, sh)
                    self._halo(sh)
                    for i in S:
                        chk(L.hf_operator_apply_dot(self.A[i], B, 2, _ptr(sh[i].owned), _ptr(t[i]),
                                                    _ptr(s[i].owned), _ptr(sums[i])))
                    reduce_step(4)
                    for i in S:
                        chk(L.hf_bcg_vec_xr(B, n[i], _ptr(x[i]), _ptr(ph[i].owned), _ptr(sh[i].owned),
                                            _ptr(s[i].owned), _ptr(t[i]), _ptr(r[i]), _ptr(rs[i]),
                                            _ptr(sums[i])))
                    reduce_step(5)
            if st[5]:                    # converged at the half step: x += alpha ph
                for i in S:
                    chk(L.hf_bcg_vec_xhalf(B, n[i], _ptr(x[i]), _ptr(ph[i].owned)))
            hist = np.zeros(cfg.maxit + 2)
            chk(L.hf_bcg_read(B, st, ctypes.byref(relres), hist.ctypes.data, len(hist)))
        finally:
            torch.cuda.synchronize()
            L.hf_bcg_destroy(B)
        rep = ConvergenceReport(method="bicgstab")
        rep.iterations, rep.matvec_count = int(st[0]), int(st[4])
        rep.converged = bool(st[2])
        rep.breakdown = _native.BREAKDOWN[int(st[3])]
        rep.final_relres = float(relres.value)
        rep.residual_history = hist[:rep.iterations].tolist()
        return x, rep


def _coarse_extents(grid, nslabs, nlev):
    return _level_extents(grid, nslabs, nlev)


def _level_extents(grid, nslabs, nlev):
    """Every slab's extent on level nlev - 1 (level 0 = the fine partition)."""
    from .partition import derive_coarse_extent, slab_partition
    out = []
    for e in slab_partition(grid, nslabs):
        for _ in range(nlev - 1):
            e = derive_coarse_extent(e)
        out.append(e)
    return out


def _nccl_library_path() -> str:
    """The libnccl torch.distributed uses (the torch wheel's nvidia-nccl), so the
    native slab driver and torch share one NCCL build."""
    try:
        import nvidia.nccl
        import os
        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        path = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(path):
            return path
    except Exception:
        pass
    return "libnccl.so.2"


class NativeSlabSolver:
    """Multi-slab CSLP-preconditioned Bi-CGSTAB run entirely by the native
    library (hf_slab_*): one stream-ordered iteration -- vector updates, slab
    V(1,1) cycle, halo exchanges, coarsest gather, inner-product all-reduces,
    scalar update -- captured once as a CUDA graph and replayed.

    comm = LocalSlabComm(n): all n slabs of the decomposition in this process
    (virtual ranks on one GPU, halos as device copies).  comm = TorchSlabComm()
    over an NCCL process group: one slab per rank, halos ncclSend/ncclRecv with
    the neighbours and sums one ncclAllReduce inside the graph (the NCCL unique
    id is broadcast through torch.distributed once at setup).  Same recurrences
    and arithmetic as SlabSolver / the single-slab solve (runner.py:95-131)."""

    def __init__(self, grid: Grid3, extents, k_field, bc, comm, beta1=1.0, beta2=-0.5,
                 mg: MGConfig | None = None, maxit: int = 4000):
        from .partition import LocalSlabComm
        self.grid, self.comm = grid, comm
        self.extents = list(extents)
        self.mg = mg or MGConfig()
        self.maxit = int(maxit)
        L = _native.load()
        self.L = L
        kfull, kc, self._keep = k_arguments(
            OperatorSpec("helmholtz", 1.0, 0.0, bc, np.asarray(k_field)), grid, full_extent(grid))
        kp = kfull.ctypes.data if kfull is not None else None
        c = _native.MGConfigC(int(self.mg.nu1), int(self.mg.nu2), float(self.mg.omega),
                              _native.CYCLE[self.mg.cycle.upper()], int(self.mg.coarsest_threshold),
                              1 if self.mg.threshold_cmp == "ge" else 0, float(self.mg.coarsest_tol),
                              int(self.mg.coarsest_maxit), _native.COARSEST["direct"])
        nloc = len(self.extents)
        lo = (ctypes.c_int * nloc)(*[e.lo1 - 1 for e in self.extents])
        nx = (ctypes.c_int * nloc)(*[e.nx for e in self.extents])
        nid = None
        if isinstance(comm, LocalSlabComm):
            transport, world, rank = _native.TRANSPORT["local"], nloc, 0
        else:
            if comm.dist.get_backend(comm.group) != "nccl":
                raise NotImplementedError("the native slab driver runs over NCCL (or LocalSlabComm)")
            transport, world, rank = _native.TRANSPORT["nccl"], comm.size, comm.rank
            _native.check(L.hf_nccl_init(_nccl_library_path().encode()))
            buf = (ctypes.c_char * 128)()
            if rank == 0:
                _native.check(L.hf_nccl_unique_id(buf))
            obj = [bytes(buf)]
            comm.dist.broadcast_object_list(obj, src=0, group=comm.group)
            nid = (ctypes.c_char * 128).from_buffer_copy(obj[0])
        _native.set_stream_from_torch()
        h = L.hf_slab_create(grid.n1, grid.n2, grid.n3, grid.h, float(beta1), float(beta2),
                             _native.BC[bc_name(bc)], kp, kc, ctypes.byref(c), nloc, lo, nx, world,
                             rank, transport, ctypes.addressof(nid) if nid is not None else None,
                             self.maxit)
        if not h:
            raise RuntimeError(_native.last_error())
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                self.L.hf_slab_destroy(h)
            except Exception:
                pass
            self._h = None

    def solve(self, b_slabs, cfg: SolverConfig | None = None, x_slabs=None):
        """b_slabs: per local slab, the right-hand side (owned planes, device or
        host).  Returns (x per slab, ConvergenceReport)."""
        import torch
        cfg = cfg or SolverConfig(method="bicgstab")
        if cfg.method != "bicgstab":
            raise NotImplementedError("the native slab driver runs Bi-CGSTAB")
        if cfg.maxit > self.maxit:
            raise ValueError(f"maxit {cfg.maxit} above this solver's capacity {self.maxit}")
        b = [torch.as_tensor(x).to("cuda", torch.complex128).contiguous() for x in b_slabs]
        x = x_slabs or [torch.empty_like(bi) for bi in b]
        nloc = len(b)
        bp = (ctypes.c_void_p * nloc)(*[t.data_ptr() for t in b])
        xp = (ctypes.c_void_p * nloc)(*[t.data_ptr() for t in x])
        kind = _native.SHADOW[cfg.shadow]
        c = _native.SolverConfigC(_native.METHOD["bicgstab"], float(cfg.tol), int(cfg.maxit), 0, 0,
                                  float(cfg.breakdown_tol), None, int(cfg.check_every), kind,
                                  int(cfg.rng_seed) & (2**64 - 1))
        hist = np.zeros(cfg.maxit + 2)
        rep = _native.ReportC()
        rep.history_host, rep.history_cap = hist.ctypes.data, len(hist)
        _native.set_stream_from_torch()
        _native.check(self.L.hf_slab_solve(self._h, ctypes.byref(c), bp, xp, ctypes.byref(rep)))
        out = ConvergenceReport(method="bicgstab", matvec_count=rep.matvec_count,
                                iterations=rep.iterations,
                                residual_history=hist[:rep.iterations].tolist(),
                                converged=bool(rep.converged),
                                final_relres=float(rep.final_relres),
                                breakdown=_native.BREAKDOWN[rep.breakdown],
                                kernel_launches=rep.kernel_launches)
        return x, out
