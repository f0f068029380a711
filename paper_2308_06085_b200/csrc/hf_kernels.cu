// hf_kernels.cu -- sm_100a kernels of the CSLP / multigrid / Bi-CGSTAB path.
//
// Stencil kernels march along i1 (one thread per (i2, i3) column, a chunk of
// planes per block).  Multigrid kernels are fused where the reference's
// sequence allows it without changing results:
//   k_down1 : pre-smooth from zero + residual   r = b - M (w D^-1 b)
//             (multigrid.py:373-386, nu1 == 1)
//   k_up1   : prolong + correct + post-smooth   u = u1 + w D^-1 (b - M u1),
//             u1 = w D^-1 b + P e                 (multigrid.py:389-392, 138-157)
// Krylov vector updates carry their inner products in the same pass, with a
// deterministic last-block reduction that also advances the Bi-CGSTAB scalars
// on the device (krylov.py:207-276).
#include "hf_kernels.cuh"

namespace hf {

// ---------------------------------------------------------------------------
// Bi-CGSTAB scalar state machine (krylov.py:234-273), run by one thread.
// ---------------------------------------------------------------------------
__device__ static void bcg_record(BcgState *st, double relres) {
    if (st->hist && st->iter < st->hist_cap) st->hist[st->iter] = relres;
    st->iter += 1;
    st->relres = relres;
}

__device__ void bcg_finalize(BcgState *st, int op, const cd *sums) {
    switch (op) {
    case FIN_BCG_INIT: {            // krylov.py:217-232
        double bb = sums[0].x;
        st->bnorm = sqrt(bb > 0.0 ? bb : 0.0);
        st->rho = st->alpha = st->omega = mk(1.0, 0.0);
        st->iter = 0; st->matvecs = 0; st->breakdown = 0; st->s_conv = 0;
        st->converged = 0; st->done = 0;
        if (st->bnorm == 0.0) { st->converged = 1; st->done = 1; st->relres = 0.0; return; }
        st->relres = st->bnorm / st->bnorm;
        if (st->relres <= st->tol) { st->converged = 1; st->done = 1; return; }
        if (st->iter >= st->maxit) { st->done = 1; return; }
        st->rho_new = sums[1];
        if (cabsd(st->rho_new) < st->btol) { st->breakdown = HF_BREAKDOWN_RHO; st->done = 1; return; }
        st->beta = cmul(cdiv(st->rho_new, st->rho), cdiv(st->alpha, st->omega));
        return;
    }
    case FIN_BCG_ALPHA: {           // krylov.py:242-247
        st->matvecs += 1;
        cd den = sums[0];
        if (cabsd(den) < st->btol) { st->breakdown = HF_BREAKDOWN_RHO; st->done = 1; return; }
        st->alpha = cdiv(st->rho_new, den);
        return;
    }
    case FIN_BCG_S: {               // krylov.py:248-255
        double ss = sums[0].x;
        double snorm = sqrt(ss > 0.0 ? ss : 0.0);
        if (snorm / st->bnorm <= st->tol) {
            bcg_record(st, snorm / st->bnorm);
            st->s_conv = 1; st->converged = 1; st->done = 1;
        }
        return;
    }
    case FIN_BCG_OMEGA: {           // krylov.py:257-265
        st->matvecs += 1;
        cd tt = sums[0], ts = sums[1];
        if (cabsd(tt) < st->btol) { st->breakdown = HF_BREAKDOWN_OMEGA; st->done = 1; return; }
        st->omega = cdiv(ts, tt);
        if (cabsd(st->omega) < st->btol) { st->breakdown = HF_BREAKDOWN_OMEGA; st->done = 1; return; }
        return;
    }
    case FIN_BCG_RHO: {             // krylov.py:266-273, then the loop head 234-239
        st->rho = st->rho_new;
        double rr = sums[0].x;
        double relres = sqrt(rr > 0.0 ? rr : 0.0) / st->bnorm;
        bcg_record(st, relres);
        if (relres <= st->tol) { st->converged = 1; st->done = 1; return; }
        if (st->iter >= st->maxit) { st->done = 1; return; }
        st->rho_new = sums[1];
        if (cabsd(st->rho_new) < st->btol) { st->breakdown = HF_BREAKDOWN_RHO; st->done = 1; return; }
        st->beta = cmul(cdiv(st->rho_new, st->rho), cdiv(st->alpha, st->omega));
        return;
    }
    default:
        return;
    }
}

__device__ __forceinline__ bool is_done(const int *done) { return done && *(volatile const int *)done; }

// ---------------------------------------------------------------------------
// marching stencil kernels
// ---------------------------------------------------------------------------
#define MARCH_BX 32
#define MARCH_BY 8

struct ColCtx {
    int j, m, i0, i1;
    bool act;
};
__device__ __forceinline__ ColCtx col_ctx(const Lvl &L, int chunk) {
    ColCtx c;
    c.m = blockIdx.x * MARCH_BX + threadIdx.x;
    c.j = blockIdx.y * MARCH_BY + threadIdx.y;
    c.i0 = blockIdx.z * chunk;
    c.i1 = min(c.i0 + chunk, L.nx);
    c.act = c.m < L.n3 && c.j < L.n2;
    return c;
}

// v = M u  (+ optional fused inner products)
//   DOT == 0: none
//   DOT == 1: sum conj(w) v                 (Bi-CGSTAB v = A p_hat, den)
//   DOT == 2: sum conj(v) v, sum conj(v) w   (Bi-CGSTAB t = A s_hat, tt & ts)
template <int DOT>
__global__ void __launch_bounds__(256) k_apply(Lvl L, const cd *__restrict__ u, cd *__restrict__ v,
                                               const cd *__restrict__ w, int chunk, RedSlot rs,
                                               const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(L, chunk);
    LoadField U{u, L.plane, L.n3};
    constexpr int ND = DOT == 0 ? 1 : DOT;
    cd acc[ND];
#pragma unroll
    for (int d = 0; d < ND; d++) acc[d] = mk(0, 0);
    if (c.act) {
        for (int i = c.i0; i < c.i1; i++) {
            long long q = (long long)i * L.plane + (long long)c.j * L.n3 + c.m;
            cd uc = __ldg(u + q);
            cd val = stencil_row(L, i, c.j, c.m, uc, kat(L, q), U);
            v[q] = val;
            if (DOT == 1) acc[0] = cadd(acc[0], cjmul(__ldg(w + q), val));
            if (DOT == 2) {
                acc[0] = cadd(acc[0], cjmul(val, val));
                acc[ND - 1] = cadd(acc[ND - 1], cjmul(val, __ldg(w + q)));
            }
        }
    }
    if (DOT) reduce_finish<ND>(acc, rs);
}

// r = b - M u   (multigrid.py:383-386)
__global__ void __launch_bounds__(256) k_residual(Lvl L, const cd *__restrict__ u,
                                                  const cd *__restrict__ b, cd *__restrict__ r,
                                                  int chunk, const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(L, chunk);
    if (!c.act) return;
    LoadField U{u, L.plane, L.n3};
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * L.plane + (long long)c.j * L.n3 + c.m;
        cd mu = stencil_row(L, i, c.j, c.m, __ldg(u + q), kat(L, q), U);
        r[q] = csub(__ldg(b + q), mu);
    }
}

// uo = u + w D^-1 (b - M u)   (multigrid.py:153-156), out of place
__global__ void __launch_bounds__(256) k_jacobi(Lvl L, const cd *__restrict__ u,
                                                const cd *__restrict__ b, cd *__restrict__ uo,
                                                double omega, int chunk, const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(L, chunk);
    if (!c.act) return;
    LoadField U{u, L.plane, L.n3};
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * L.plane + (long long)c.j * L.n3 + c.m;
        double kk = kat(L, q);
        cd uc = __ldg(u + q);
        cd mu = stencil_row(L, i, c.j, c.m, uc, kk, U);
        cd res = csub(__ldg(b + q), mu);
        cd d = diag_of(L, kk, nbnd(L, L.lo1 + i, c.j, c.m));
        cd upd = cdiv(res, d);
        uo[q] = mk(uc.x + omega * upd.x, uc.y + omega * upd.y);
    }
}

// u = w D^-1 b   (multigrid.py:148-151, assume_zero first sweep)
__global__ void __launch_bounds__(256) k_jacobi0(Lvl L, const cd *__restrict__ b,
                                                 cd *__restrict__ u, double omega, int chunk,
                                                 const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(L, chunk);
    if (!c.act) return;
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * L.plane + (long long)c.j * L.n3 + c.m;
        cd d = diag_of(L, kat(L, q), nbnd(L, L.lo1 + i, c.j, c.m));
        u[q] = cscal(cdiv(__ldg(b + q), d), omega);
    }
}

// value of the zero-guess pre-smoothed iterate w D^-1 b at a (possibly ghost) point
struct PreSmooth {
    Lvl L;
    const cd *b;
    double omega;
    __device__ __forceinline__ cd operator()(int i, int j, int m) const {
        long long q = (long long)i * L.plane + (long long)j * L.n3 + m;
        cd d = diag_of(L, kat(L, q), nbnd(L, L.lo1 + i, j, m));
        return cscal(cdiv(__ldg(b + q), d), omega);
    }
};

// r = b - M (w D^-1 b)  -- fused pre-smooth (nu1 = 1, zero guess) + residual
__global__ void __launch_bounds__(256) k_down1(Lvl L, const cd *__restrict__ b,
                                               cd *__restrict__ r, double omega, int chunk,
                                               const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(L, chunk);
    if (!c.act) return;
    PreSmooth P{L, b, omega};
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * L.plane + (long long)c.j * L.n3 + c.m;
        cd mu = stencil_row(L, i, c.j, c.m, P(i, c.j, c.m), kat(L, q), P);
        r[q] = csub(__ldg(b + q), mu);
    }
}

// trilinear prolongation value at fine local (i, j, m) (multigrid.py:238-297)
struct Prolong {
    Lvl F, C;
    const cd *e;   // coarse field, owned plane 0
    __device__ __forceinline__ cd operator()(int i, int j, int m) const {
        int gi = F.lo1 + i;
        int c1 = (gi >> 1) - C.lo1, e1 = (gi & 1) ? 2 : 1;
        int c2 = j >> 1, e2 = (j & 1) ? 2 : 1;
        int c3 = m >> 1, e3 = (m & 1) ? 2 : 1;
        cd acc = mk(0, 0);
        for (int d1 = 0; d1 < e1; d1++)
            for (int d2 = 0; d2 < e2; d2++)
                for (int d3 = 0; d3 < e3; d3++) {
                    long long q = (long long)(c1 + d1) * C.plane + (long long)(c2 + d2) * C.n3 + (c3 + d3);
                    acc = cadd(acc, __ldg(e + q));
                }
        int ns = e1 * e2 * e3;
        if (ns > 1) acc = mk(acc.x / ns, acc.y / ns);
        return acc;
    }
};

// out = P e (ADD=0) or out += P e (ADD=1)
template <int ADD>
__global__ void __launch_bounds__(256) k_prolong(Lvl F, Lvl C, const cd *__restrict__ e,
                                                 cd *__restrict__ out, int chunk, const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(F, chunk);
    if (!c.act) return;
    Prolong P{F, C, e};
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * F.plane + (long long)c.j * F.n3 + c.m;
        cd pe = P(i, c.j, c.m);
        out[q] = ADD ? cadd(out[q], pe) : pe;
    }
}

// u1 = [w D^-1 b] + P e  (pre-smoothed from zero + coarse correction)
template <int PRE>
struct Corrected {
    PreSmooth S;
    Prolong P;
    __device__ __forceinline__ cd operator()(int i, int j, int m) const {
        cd pe = P(i, j, m);
        if (PRE) {
            cd s = S(i, j, m);
            return cadd(s, pe);
        }
        return pe;
    }
};

// u = u1 + w D^-1 (b - M u1)  -- fused prolong + correct + one post-smoothing sweep
template <int PRE>
__global__ void __launch_bounds__(256) k_up1(Lvl L, Lvl C, const cd *__restrict__ b,
                                             const cd *__restrict__ e, cd *__restrict__ u,
                                             double omega, int chunk, const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(L, chunk);
    if (!c.act) return;
    Corrected<PRE> V{PreSmooth{L, b, omega}, Prolong{L, C, e}};
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * L.plane + (long long)c.j * L.n3 + c.m;
        double kk = kat(L, q);
        cd u1 = V(i, c.j, c.m);
        cd mu = stencil_row(L, i, c.j, c.m, u1, kk, V);
        cd res = csub(__ldg(b + q), mu);
        cd d = diag_of(L, kk, nbnd(L, L.lo1 + i, c.j, c.m));
        cd upd = cdiv(res, d);
        u[q] = mk(u1.x + omega * upd.x, u1.y + omega * upd.y);
    }
}

// full-weighting restriction, one thread per coarse vertex (multigrid.py:171-221)
__global__ void __launch_bounds__(256) k_restrict(Lvl F, Lvl C, const cd *__restrict__ r,
                                                  cd *__restrict__ out, int chunk,
                                                  const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(C, chunk);
    if (!c.act) return;
    const double w1[3] = {1.0, 2.0, 1.0};
    for (int ci = c.i0; ci < c.i1; ci++) {
        int gci = C.lo1 + ci;
        int fi0 = 2 * gci - F.lo1;      // fine local plane of the coarse vertex image
        int fj0 = 2 * c.j, fm0 = 2 * c.m;
        cd acc = mk(0, 0);
#pragma unroll
        for (int o1 = -1; o1 <= 1; o1++) {
            int gfi = 2 * gci + o1;
            bool in1 = gfi >= 0 && gfi < F.n1;
#pragma unroll
            for (int o2 = -1; o2 <= 1; o2++) {
                int fj = fj0 + o2;
                bool in2 = in1 && fj >= 0 && fj < F.n2;
#pragma unroll
                for (int o3 = -1; o3 <= 1; o3++) {
                    int fm = fm0 + o3;
                    double w = w1[o1 + 1] * w1[o2 + 1] * w1[o3 + 1];
                    if (in2 && fm >= 0 && fm < F.n3) {
                        cd val = __ldg(r + (long long)(fi0 + o1) * F.plane + (long long)fj * F.n3 + fm);
                        acc.x += w * val.x;
                        acc.y += w * val.y;
                    }
                }
            }
        }
        acc = mk(acc.x / 64.0, acc.y / 64.0);
        int onb = (gci == 0 || gci == C.n1 - 1) + (c.j == 0 || c.j == C.n2 - 1) +
                  (c.m == 0 || c.m == C.n3 - 1);
        if (onb) {
            if (C.bc == HF_BC_DIRICHLET) acc = mk(0, 0);
            else
                for (int d = 0; d < onb; d++) acc = cscal(acc, 64.0 / 48.0);
        }
        out[(long long)ci * C.plane + (long long)c.j * C.n3 + c.m] = acc;
    }
}

// ---------------------------------------------------------------------------
// 1-D vector kernels (owned region, contiguous)
// ---------------------------------------------------------------------------
#define VEC_BLOCKS 592   // 4 x 148 SMs, fixed => deterministic reductions

// Bi-CGSTAB start (krylov.py:217-232): r = b, rs = b, x = p = v = 0; |b|^2, rs^H r
__global__ void __launch_bounds__(256) k_bcg_init(long long n, const cd *__restrict__ b,
                                                  cd *__restrict__ r, cd *__restrict__ rs,
                                                  cd *__restrict__ x, cd *__restrict__ p,
                                                  cd *__restrict__ v, RedSlot red) {
    cd acc[2] = {mk(0, 0), mk(0, 0)};
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd bv = __ldg(b + q);
        r[q] = bv; rs[q] = bv;
        x[q] = mk(0, 0); p[q] = mk(0, 0); v[q] = mk(0, 0);
        acc[0] = cadd(acc[0], cjmul(bv, bv));
    }
    acc[1] = acc[0];
    reduce_finish<2>(acc, red);
}

// p = r + beta (p - omega v)   (krylov.py:240)
__global__ void __launch_bounds__(256) k_bcg_p(long long n, const BcgState *st,
                                               const cd *__restrict__ r, cd *__restrict__ p,
                                               const cd *__restrict__ v, const int *done) {
    if (is_done(done)) return;
    cd beta = st->beta, om = st->omega;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd t = csub(p[q], cmul(om, __ldg(v + q)));
        p[q] = cadd(__ldg(r + q), cmul(beta, t));
    }
}

// s = r - alpha v ; |s|^2   (krylov.py:248-249)
__global__ void __launch_bounds__(256) k_bcg_s(long long n, const BcgState *st,
                                               const cd *__restrict__ r, const cd *__restrict__ v,
                                               cd *__restrict__ s, RedSlot red, const int *done) {
    if (is_done(done)) return;
    cd al = st->alpha;
    cd acc[1] = {mk(0, 0)};
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd sv = csub(__ldg(r + q), cmul(al, __ldg(v + q)));
        s[q] = sv;
        acc[0] = cadd(acc[0], cjmul(sv, sv));
    }
    reduce_finish<1>(acc, red);
}

// x += alpha ph + omega sh ; r = s - omega t ; |r|^2, rs^H r   (krylov.py:266-269)
__global__ void __launch_bounds__(256) k_bcg_xr(long long n, const BcgState *st,
                                                cd *__restrict__ x, const cd *__restrict__ ph,
                                                const cd *__restrict__ sh, const cd *__restrict__ s,
                                                const cd *__restrict__ t, cd *__restrict__ r,
                                                const cd *__restrict__ rs, RedSlot red,
                                                const int *done) {
    if (is_done(done)) return;
    cd al = st->alpha, om = st->omega;
    cd acc[2] = {mk(0, 0), mk(0, 0)};
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd xv = cadd(cadd(x[q], cmul(al, __ldg(ph + q))), cmul(om, __ldg(sh + q)));
        x[q] = xv;
        cd rv = csub(__ldg(s + q), cmul(om, __ldg(t + q)));
        r[q] = rv;
        acc[0] = cadd(acc[0], cjmul(rv, rv));
        acc[1] = cadd(acc[1], cjmul(__ldg(rs + q), rv));
    }
    reduce_finish<2>(acc, red);
}

// x += alpha ph  (convergence at the half step, krylov.py:250-255)
__global__ void k_bcg_xhalf(long long n, const BcgState *st, cd *__restrict__ x,
                            const cd *__restrict__ ph) {
    cd al = st->alpha;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256)
        x[q] = cadd(x[q], cmul(al, __ldg(ph + q)));
}

// generic y = a x + b y with host scalars (GMRES / IDR helpers)
__global__ void k_axpby(long long n, cd a, const cd *__restrict__ x, cd b, cd *__restrict__ y) {
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd yv = (b.x == 0.0 && b.y == 0.0) ? mk(0, 0) : cmul(b, y[q]);
        y[q] = cadd(cmul(a, __ldg(x + q)), yv);
    }
}

// y = x - sum_i c_i V_i  with c on the device (dense coefficient vector)
__global__ void k_dot_store(long long n, const cd *__restrict__ a, const cd *__restrict__ b,
                            RedSlot red) {
    cd acc[1] = {mk(0, 0)};
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256)
        acc[0] = cadd(acc[0], cjmul(__ldg(a + q), __ldg(b + q)));
    reduce_finish<1>(acc, red);
}

// ---------------------------------------------------------------------------
// coarsest level: dense inverse applied as one GEMV (HBM-bound)
// ---------------------------------------------------------------------------
// x = Minv b, Minv row-major N x N.  One warp per row.
__global__ void __launch_bounds__(256) k_gemv(int N, const cd *__restrict__ Minv,
                                              const cd *__restrict__ b, cd *__restrict__ x,
                                              const int *done) {
    if (is_done(done)) return;
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= N) return;
    const cd *row = Minv + (long long)warp * N;
    cd a0 = mk(0, 0), a1 = mk(0, 0);
    int j = lane;
    for (; j + 32 < N; j += 64) {
        cd m0 = __ldcs(row + j), m1 = __ldcs(row + j + 32);
        cd b0 = __ldg(b + j), b1 = __ldg(b + j + 32);
        a0 = cadd(a0, cmul(m0, b0));
        a1 = cadd(a1, cmul(m1, b1));
    }
    if (j < N) a0 = cadd(a0, cmul(__ldcs(row + j), __ldg(b + j)));
    a0 = warp_sum(cadd(a0, a1));
    if (lane == 0) x[warp] = a0;
}

// Row-major dense CSLP matrix of a full (single-slab) level: A[r * N + c].
__global__ void k_assemble(Lvl L, cd *__restrict__ A) {
    long long N = (long long)L.n1 * L.plane;
    long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (r >= N) return;
    int i = (int)(r / L.plane);
    int rem = (int)(r - (long long)i * L.plane);
    int j = rem / L.n3, m = rem - j * L.n3;
    int nb = nbnd(L, i, j, m);
    cd *row = A + r * N;
    if (L.bc == HF_BC_DIRICHLET && nb) { row[r] = mk(1.0, 0.0); return; }
    double kk = L.k ? L.k[r] : L.kc;
    row[r] = ap_of(L, kk, nb);
    const double off = -L.ih2;
    int ii[6] = {i - 1, i + 1, i, i, i, i};
    int jj[6] = {j, j, j - 1, j + 1, j, j};
    int mm[6] = {m, m, m, m, m - 1, m + 1};
    int ri[6] = {i + 1, i - 1, i, i, i, i};
    int rj[6] = {j, j, j + 1, j - 1, j, j};
    int rm[6] = {m, m, m, m, m + 1, m - 1};
    for (int d = 0; d < 6; d++) {
        int a = ii[d], bq = jj[d], cq = mm[d];
        if (a < 0 || a >= L.n1 || bq < 0 || bq >= L.n2 || cq < 0 || cq >= L.n3) {
            a = ri[d]; bq = rj[d]; cq = rm[d];   // Sommerfeld: doubled inward neighbour
        }
        long long col = (long long)a * L.plane + (long long)bq * L.n3 + cq;
        row[col] = cadd(row[col], mk(off, 0.0));
    }
}

__global__ void k_set_identity(long long N, cd *__restrict__ B) {
    long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q < N) B[q * N + q] = mk(1.0, 0.0);
}

__global__ void k_zero(long long n, cd *__restrict__ y) {
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256)
        y[q] = mk(0, 0);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
static dim3 march_grid(const Lvl &L, int &chunk) {
    int gx = (L.n3 + MARCH_BX - 1) / MARCH_BX;
    int gy = (L.n2 + MARCH_BY - 1) / MARCH_BY;
    long long cols = (long long)gx * gy;
    long long target = 148 * 6;     // resident blocks on B200 at 256 threads
    int gz = (int)((target + cols - 1) / cols);
    if (gz < 1) gz = 1;
    if (gz > L.nx) gz = L.nx;
    chunk = (L.nx + gz - 1) / gz;
    gz = (L.nx + chunk - 1) / chunk;
    return dim3(gx, gy, gz);
}
static const dim3 kMarchBlock(MARCH_BX, MARCH_BY, 1);

int march_blocks(const Lvl &L) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    return g.x * g.y * g.z;
}

void launch_apply(const Lvl &L, const cd *u, cd *v, cudaStream_t s, const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    RedSlot rs{};
    k_apply<0><<<g, kMarchBlock, 0, s>>>(L, u, v, nullptr, chunk, rs, done);
}
void launch_apply_dot1(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    k_apply<1><<<g, kMarchBlock, 0, s>>>(L, u, v, w, chunk, rs, done);
}
void launch_apply_dot2(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    k_apply<2><<<g, kMarchBlock, 0, s>>>(L, u, v, w, chunk, rs, done);
}
void launch_residual(const Lvl &L, const cd *u, const cd *b, cd *r, cudaStream_t s,
                     const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    k_residual<<<g, kMarchBlock, 0, s>>>(L, u, b, r, chunk, done);
}
void launch_jacobi(const Lvl &L, const cd *u, const cd *b, cd *uo, double omega,
                   cudaStream_t s, const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    k_jacobi<<<g, kMarchBlock, 0, s>>>(L, u, b, uo, omega, chunk, done);
}
void launch_jacobi0(const Lvl &L, const cd *b, cd *u, double omega, cudaStream_t s,
                    const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    k_jacobi0<<<g, kMarchBlock, 0, s>>>(L, b, u, omega, chunk, done);
}
void launch_down1(const Lvl &L, const cd *b, cd *r, double omega, cudaStream_t s,
                  const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    k_down1<<<g, kMarchBlock, 0, s>>>(L, b, r, omega, chunk, done);
}
void launch_restrict(const Lvl &F, const Lvl &C, const cd *r, cd *out, cudaStream_t s,
                     const int *done) {
    int chunk;
    dim3 g = march_grid(C, chunk);
    k_restrict<<<g, kMarchBlock, 0, s>>>(F, C, r, out, chunk, done);
}
void launch_prolong(const Lvl &F, const Lvl &C, const cd *e, cd *out, bool add, cudaStream_t s,
                    const int *done) {
    int chunk;
    dim3 g = march_grid(F, chunk);
    if (add) k_prolong<1><<<g, kMarchBlock, 0, s>>>(F, C, e, out, chunk, done);
    else k_prolong<0><<<g, kMarchBlock, 0, s>>>(F, C, e, out, chunk, done);
}
void launch_up1(const Lvl &L, const Lvl &C, const cd *b, const cd *e, cd *u, double omega,
                bool pre, cudaStream_t s, const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    if (pre) k_up1<1><<<g, kMarchBlock, 0, s>>>(L, C, b, e, u, omega, chunk, done);
    else k_up1<0><<<g, kMarchBlock, 0, s>>>(L, C, b, e, u, omega, chunk, done);
}
void launch_gemv(int N, const cd *Minv, const cd *b, cd *x, cudaStream_t s, const int *done) {
    int blocks = (N + 7) / 8;
    k_gemv<<<blocks, 256, 0, s>>>(N, Minv, b, x, done);
}
void launch_assemble(const Lvl &L, cd *A, cudaStream_t s) {
    long long N = (long long)L.n1 * L.plane;
    k_assemble<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(L, A);
}
void launch_set_identity(long long N, cd *B, cudaStream_t s) {
    k_set_identity<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, B);
}
void launch_zero(long long n, cd *y, cudaStream_t s) {
    k_zero<<<VEC_BLOCKS, 256, 0, s>>>(n, y);
}
void launch_axpby(long long n, cd a, const cd *x, cd b, cd *y, cudaStream_t s) {
    k_axpby<<<VEC_BLOCKS, 256, 0, s>>>(n, a, x, b, y);
}
void launch_dot(long long n, const cd *a, const cd *b, const RedSlot &rs, cudaStream_t s) {
    k_dot_store<<<VEC_BLOCKS, 256, 0, s>>>(n, a, b, rs);
}
void launch_bcg_init(long long n, const cd *b, cd *r, cd *rs, cd *x, cd *p, cd *v,
                     const RedSlot &red, cudaStream_t s) {
    k_bcg_init<<<VEC_BLOCKS, 256, 0, s>>>(n, b, r, rs, x, p, v, red);
}
void launch_bcg_p(long long n, const BcgState *st, const cd *r, cd *p, const cd *v,
                  cudaStream_t s, const int *done) {
    k_bcg_p<<<VEC_BLOCKS, 256, 0, s>>>(n, st, r, p, v, done);
}
void launch_bcg_s(long long n, const BcgState *st, const cd *r, const cd *v, cd *sv,
                  const RedSlot &red, cudaStream_t s, const int *done) {
    k_bcg_s<<<VEC_BLOCKS, 256, 0, s>>>(n, st, r, v, sv, red, done);
}
void launch_bcg_xr(long long n, const BcgState *st, cd *x, const cd *ph, const cd *sh,
                   const cd *sv, const cd *t, cd *r, const cd *rs, const RedSlot &red,
                   cudaStream_t s, const int *done) {
    k_bcg_xr<<<VEC_BLOCKS, 256, 0, s>>>(n, st, x, ph, sh, sv, t, r, rs, red, done);
}
void launch_bcg_xhalf(long long n, const BcgState *st, cd *x, const cd *ph, cudaStream_t s) {
    k_bcg_xhalf<<<VEC_BLOCKS, 256, 0, s>>>(n, st, x, ph);
}

}  // namespace hf
