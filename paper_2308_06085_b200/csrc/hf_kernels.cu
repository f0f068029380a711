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
#include <algorithm>

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

// ---------------------------------------------------------------------------
// shared-memory 2.5D tiled stencil kernels
//
// A block owns a TX x TY tile of (i3, i2) columns and marches along i1 over a
// chunk of planes.  For each plane the block evaluates the stencil input f
// ONCE per point (tile + 1-point halo) into a 3-plane rolling shared-memory
// window; each thread then forms M f from shared memory.  f is a functor:
// a plain load (matvec / residual / Jacobi), the zero-guess pre-smoothed
// iterate w D^-1 b (fused pre-smooth + residual), or w D^-1 b + P e (fused
// prolongation + correction + post-smooth).  The epilogue consumes (f, M f).
// ---------------------------------------------------------------------------
#define TILE_X 32
#define TILE_Y 8
#define HALO_X (TILE_X + 2)
#define HALO_Y (TILE_Y + 2)

// v = a f - h^-2 sum(neighbours), neighbours already mirrored for Sommerfeld
__device__ __forceinline__ cd stencil_nb(const Lvl &L, int gi, int j, int m, cd fc, double kk,
                                         cd xm, cd xp, cd ym, cd yp, cd zm, cd zp, int &nb) {
    const bool bxl = gi == 0, bxh = gi == L.n1 - 1;
    const bool byl = j == 0, byh = j == L.n2 - 1;
    const bool bzl = m == 0, bzh = m == L.n3 - 1;
    nb = (int)bxl + bxh + byl + byh + bzl + bzh;
    if (L.bc == HF_BC_DIRICHLET && nb) return fc;
    if (bxl) xm = xp;
    if (bxh) xp = xm;
    if (byl) ym = yp;
    if (byh) yp = ym;
    if (bzl) zm = zp;
    if (bzh) zp = zm;
    cd s = cadd(cadd(cadd(xm, xp), cadd(ym, yp)), cadd(zm, zp));
    cd a = ap_of(L, kk, nb);
    cd v = cmul(a, fc);
    v.x -= L.ih2 * s.x;
    v.y -= L.ih2 * s.y;
    return v;
}

// stencil inputs --------------------------------------------------------------
struct ProdLoad {
    const cd *u;
    long long plane;
    int n3;
    __device__ __forceinline__ cd operator()(const Lvl &, int i, int j, int m) const {
        return __ldg(u + (long long)i * plane + (long long)j * n3 + m);
    }
};

// zero-guess pre-smoothed iterate w D^-1 b (multigrid.py:148-151)
struct ProdPre {
    const cd *b;
    double omega;
    __device__ __forceinline__ cd operator()(const Lvl &L, int i, int j, int m) const {
        long long q = (long long)i * L.plane + (long long)j * L.n3 + m;
        cd d = diag_of(L, kat(L, q), nbnd(L, L.lo1 + i, j, m));
        return cscal(cdiv(__ldg(b + q), d), omega);
    }
};

// trilinear prolongation value at fine local (i, j, m) (multigrid.py:238-297);
// the reference divides the 2/4/8-point sums, exact here as a power-of-two scale
struct Prolong {
    Lvl C;
    const cd *e;   // coarse field, owned plane 0
    __device__ __forceinline__ cd operator()(const Lvl &F, int i, int j, int m) const {
        int gi = F.lo1 + i;
        int c1 = (gi >> 1) - C.lo1, e1 = (gi & 1) ? 2 : 1;
        int c2 = j >> 1, e2 = (j & 1) ? 2 : 1;
        int c3 = m >> 1, e3 = (m & 1) ? 2 : 1;
        const cd *p = e + (long long)c1 * C.plane + (long long)c2 * C.n3 + c3;
        cd acc = __ldg(p);
        if (e3 == 2) acc = cadd(acc, __ldg(p + 1));
        if (e2 == 2) {
            acc = cadd(acc, __ldg(p + C.n3));
            if (e3 == 2) acc = cadd(acc, __ldg(p + C.n3 + 1));
        }
        if (e1 == 2) {
            const cd *p1 = p + C.plane;
            acc = cadd(acc, __ldg(p1));
            if (e3 == 2) acc = cadd(acc, __ldg(p1 + 1));
            if (e2 == 2) {
                acc = cadd(acc, __ldg(p1 + C.n3));
                if (e3 == 2) acc = cadd(acc, __ldg(p1 + C.n3 + 1));
            }
        }
        int ns = e1 * e2 * e3;
        if (ns > 1) acc = cscal(acc, 1.0 / ns);
        return acc;
    }
};

// w D^-1 b + P e (PRE=1) or P e (PRE=0): iterate after pre-smoothing from zero
// and the coarse-grid correction (multigrid.py:337-341)
template <int PRE>
struct ProdCorr {
    ProdPre S;
    Prolong P;
    __device__ __forceinline__ cd operator()(const Lvl &L, int i, int j, int m) const {
        cd pe = P(L, i, j, m);
        if (PRE) return cadd(S(L, i, j, m), pe);
        return pe;
    }
};

// epilogues --------------------------------------------------------------------
// called as epi(q, f_centre, (M f)_centre, w D^-1_centre, staged operand, acc)
// v = M f (+ inner products), DOT: 0 none, 1 conj(w) v, 2 conj(v) v & conj(v) w
template <int DOT>
struct EpiApply {
    cd *v;
    static constexpr bool kAux = DOT > 0;   // w is staged as the aux field
    static constexpr bool kDinv = false;
    __device__ __forceinline__ void operator()(long long q, cd, cd mf, cd, cd aux,
                                               cd (&acc)[2]) const {
        v[q] = mf;
        if (DOT == 1) acc[0] = cadd(acc[0], cjmul(aux, mf));
        if (DOT == 2) {
            acc[0] = cadd(acc[0], cjmul(mf, mf));
            acc[1] = cadd(acc[1], cjmul(mf, aux));
        }
    }
};

// r = b - M f (residual; with MODE_PRE the fused pre-smooth + residual)
struct EpiResid {
    cd *r;
    static constexpr bool kAux = true;      // b
    static constexpr bool kDinv = false;
    __device__ __forceinline__ void operator()(long long q, cd, cd mf, cd, cd b, cd (&)[2]) const {
        r[q] = csub(b, mf);
    }
};

// u = f + w D^-1 (b - M f) (one damped Jacobi sweep on f, multigrid.py:153-156)
struct EpiJacobi {
    cd *u;
    static constexpr bool kAux = true;      // b
    static constexpr bool kDinv = true;
    __device__ __forceinline__ void operator()(long long q, cd fc, cd mf, cd wd, cd b,
                                               cd (&)[2]) const {
        cd upd = cmul(wd, csub(b, mf));
        u[q] = cadd(fc, upd);
    }
};

// ---------------------------------------------------------------------------
// cp.async-pipelined tiled stencil kernel (instruction-lean)
//
// Raw inputs of plane i+2 and i+3 (the stencil field or right-hand side, the
// wavenumber when it varies, the epilogue operand, and the two coarse planes
// the prolongation reads) are in flight global->shared (cp.async) while plane
// i is computed.  For each plane the block evaluates the stencil input f ONCE
// per point of the tile + 1-point halo into a 3-plane window; every thread
// then forms the 7-point row M f from shared memory.  Per-thread fill
// metadata (shared-memory slots, 32-bit in-plane offsets, boundary counts,
// prolongation taps) is computed once per block, and for a constant medium
// the stencil centre a_p and w D^-1 come from a 4-entry table indexed by the
// number of physical faces (no FP64 division in the loop).
// ---------------------------------------------------------------------------
#define PIPE_S 4
#define PIPE_MASK 3
#define CT_Y (TILE_Y / 2 + 2)
#define CT_X (TILE_X / 2 + 2)
#define NFILL (HALO_Y * HALO_X)
#define NCOARSE (2 * CT_Y * CT_X)

enum { MODE_LOAD = 0, MODE_PRE = 1, MODE_CORR1 = 2, MODE_CORR0 = 3 };

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int MODE, bool KVAR, bool AUX>
struct StencilSmem {
    static constexpr bool kCoarse = MODE == MODE_CORR1 || MODE == MODE_CORR0;
    static constexpr bool kAuxArr = AUX && MODE == MODE_LOAD;
    cd f[3][NFILL];                              // stencil input window
    cd raw[PIPE_S][NFILL];                       // field / rhs planes (tile + halo)
    double kr[KVAR ? PIPE_S : 1][NFILL];         // wavenumber planes
    cd cr[kCoarse ? PIPE_S : 1][NCOARSE];        // coarse planes for the prolongation
    cd ax[kAuxArr ? PIPE_S : 1][TILE_Y * TILE_X];   // epilogue operand, centre only
};

// per-thread fill entry: halo point e of the tile
struct FillEnt {
    int go;        // in-plane global offset j*n3 + m
    int nbjm;      // physical faces touched in i2 / i3
    int co;        // prolongation: coarse tap offset in the staged coarse plane
    int e23;       // prolongation: bit0 = i3 odd, bit1 = i2 odd
    bool ok;       // inside the grid in i2 / i3
};

// 4-entry register table indexed by the boundary-face count (no local memory)
struct Tab4 {
    cd t0, t1, t2, t3;
    __device__ __forceinline__ cd operator[](int nb) const {
        return nb == 0 ? t0 : (nb == 1 ? t1 : (nb == 2 ? t2 : t3));
    }
};

template <int MODE, class Epi, int ND, bool KVAR>
__global__ void __launch_bounds__(TILE_X *TILE_Y) k_stencil(Lvl L, Lvl C, const cd *__restrict__ src,
                                                           const cd *__restrict__ ec,
                                                           const cd *__restrict__ aux, double omega,
                                                           Epi epi, int chunk, RedSlot rs,
                                                           const int *done) {
    using SM = StencilSmem<MODE, KVAR, Epi::kAux>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SM &sm = *reinterpret_cast<SM *>(smem_raw);
    if (is_done(done)) return;
    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * TILE_X + tx;
    const int m0 = blockIdx.x * TILE_X, j0 = blockIdx.y * TILE_Y;
    const int i0 = blockIdx.z * chunk, i1 = min(i0 + chunk, L.nx);
    const int m = m0 + tx, j = j0 + ty;
    const bool act = m < L.n3 && j < L.n2;
    const int cj0 = (j0 - 1) >> 1, cm0 = (m0 - 1) >> 1;   // coarse tile origin (floor)

    // ---- per-thread metadata (once per block) ----
    FillEnt fe[2];
    const bool has1 = tid + TILE_X * TILE_Y < NFILL;
#pragma unroll
    for (int k = 0; k < 2; k++) {
        int e = tid + k * TILE_X * TILE_Y;
        int hy = e / HALO_X, hx = e - hy * HALO_X;
        int jj = j0 - 1 + hy, mm = m0 - 1 + hx;
        fe[k].ok = jj >= 0 && jj < L.n2 && mm >= 0 && mm < L.n3;
        fe[k].go = jj * L.n3 + mm;
        fe[k].nbjm = (jj == 0) + (jj == L.n2 - 1) + (mm == 0) + (mm == L.n3 - 1);
        fe[k].co = ((jj >> 1) - cj0) * CT_X + ((mm >> 1) - cm0);
        fe[k].e23 = (mm & 1) | ((jj & 1) << 1);
    }
    // coarse staging entry of this thread
    const bool hasc = SM::kCoarse && tid < NCOARSE;
    int cgo = 0, cplane = 0;
    bool cok = false;
    if (hasc) {
        cplane = tid / (CT_Y * CT_X);
        int r = tid - cplane * (CT_Y * CT_X);
        int cy = r / CT_X, cx = r - cy * CT_X;
        int cj = cj0 + cy, cm = cm0 + cx;
        cok = cj >= 0 && cj < C.n2 && cm >= 0 && cm < C.n3;
        cgo = cj * C.n3 + cm;
    }
    // centre of this thread
    const int cfill = (ty + 1) * HALO_X + (tx + 1);
    const int nbjm_c = (j == 0) + (j == L.n2 - 1) + (m == 0) + (m == L.n3 - 1);
    const bool byl = j == 0, byh = j == L.n2 - 1, bzl = m == 0, bzh = m == L.n3 - 1;
    // constant medium: a_p and w D^-1 by boundary-face count
    Tab4 apt{}, wdt{};
    if (!KVAR) {
        auto wdinv = [&](int nb) { return cscal(cdiv(mk(1.0, 0.0), diag_of(L, L.kc, nb)), omega); };
        apt = Tab4{ap_of(L, L.kc, 0), ap_of(L, L.kc, 1), ap_of(L, L.kc, 2), ap_of(L, L.kc, 3)};
        wdt = Tab4{wdinv(0), wdinv(1), wdinv(2), wdinv(3)};
    }
    cd acc[2] = {mk(0, 0), mk(0, 0)};

    int stage_slot = 0, prod_slot = 0;
    // issue the raw copies of plane i (one commit group per call)
    auto stage = [&](int i) {
        const int slot = stage_slot;
        stage_slot = (stage_slot + 1) & PIPE_MASK;
        const int gi = L.lo1 + i;
        const bool pok = i <= i1 && gi >= 0 && gi < L.n1;
        const long long pbase = (long long)i * L.plane;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            if (k == 1 && !has1) break;
            const int e = tid + k * TILE_X * TILE_Y;
            const bool ok = pok && fe[k].ok;
            cp_async16(&sm.raw[slot][e], ok ? src + pbase + fe[k].go : src, ok);
            if (KVAR) cp_async8(&sm.kr[slot & (KVAR ? PIPE_MASK : 0)][e], ok ? L.k + pbase + fe[k].go : L.k, ok);
        }
        if (SM::kAuxArr) {
            const bool ok = pok && act && i < i1;
            cp_async16(&sm.ax[slot & (SM::kAuxArr ? PIPE_MASK : 0)][tid],
                       ok ? aux + pbase + j * L.n3 + m : aux, ok);
        }
        if (hasc) {
            const int c1 = (gi >> 1) - C.lo1 + cplane;     // local coarse plane
            const int cg = C.lo1 + c1;
            const bool ok = pok && cok && cg >= 0 && cg < C.n1;
            cp_async16(&sm.cr[slot & (SM::kCoarse ? PIPE_MASK : 0)][tid],
                       ok ? ec + (long long)c1 * C.plane + cgo : ec, ok);
        }
        cp_commit();
    };

    // stencil input f at plane i from its staged raw data, into window w
    auto produce = [&](int i, int w) {
        const int slot = prod_slot;
        prod_slot = (prod_slot + 1) & PIPE_MASK;
        const int gi = L.lo1 + i;
        const bool pok = gi >= 0 && gi < L.n1;
        const int nbi = (gi == 0) + (gi == L.n1 - 1);
        const bool xodd = gi & 1;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            if (k == 1 && !has1) break;
            const int e = tid + k * TILE_X * TILE_Y;
            cd v = mk(0, 0);
            if (pok && fe[k].ok) {
                const cd rv = sm.raw[slot][e];
                if (MODE == MODE_LOAD) {
                    v = rv;
                } else {
                    if (MODE == MODE_PRE || MODE == MODE_CORR1) {
                        const int nb = nbi + fe[k].nbjm;
                        cd wd;
                        if (KVAR) wd = cscal(cdiv(mk(1.0, 0.0), diag_of(L, sm.kr[slot & (KVAR ? PIPE_MASK : 0)][e], nb)), omega);
                        else wd = wdt[nb];
                        v = cmul(rv, wd);
                    }
                    if (SM::kCoarse) {
                        const cd *cp = sm.cr[slot & (SM::kCoarse ? PIPE_MASK : 0)];
                        const int co = fe[k].co;
                        const bool e3 = fe[k].e23 & 1, e2 = fe[k].e23 & 2;
                        cd a = cp[co];
                        if (e3) a = cadd(a, cp[co + 1]);
                        if (e2) {
                            a = cadd(a, cp[co + CT_X]);
                            if (e3) a = cadd(a, cp[co + CT_X + 1]);
                        }
                        if (xodd) {
                            const cd *cq = cp + CT_Y * CT_X;
                            a = cadd(a, cq[co]);
                            if (e3) a = cadd(a, cq[co + 1]);
                            if (e2) {
                                a = cadd(a, cq[co + CT_X]);
                                if (e3) a = cadd(a, cq[co + CT_X + 1]);
                            }
                        }
                        const int ns = (1 + (int)xodd) * (1 + (int)e2) * (1 + (int)e3);
                        if (ns > 1) a = cscal(a, ns == 2 ? 0.5 : (ns == 4 ? 0.25 : 0.125));
                        v = (MODE == MODE_CORR1) ? cadd(v, a) : a;
                    }
                }
            }
            sm.f[w][e] = v;
        }
    };

    // prologue: raw planes i0-1 .. i0+2 in flight; f(i0-1), f(i0) produced
    for (int s = 0; s < PIPE_S; s++) stage(i0 - 1 + s);
    cp_wait<PIPE_S - 1>();
    __syncthreads();
    produce(i0 - 1, 0);
    cp_wait<PIPE_S - 2>();
    __syncthreads();
    produce(i0, 1);
    int wp = 0, wc = 1, wn = 2;
    int cslot = 1;   // stage slot of the plane being computed
    for (int i = i0; i < i1; i++) {
        cp_wait<PIPE_S - 3>();          // raw(i+1) landed
        __syncthreads();
        produce(i + 1, wn);
        stage(i + PIPE_S - 1);          // reuses the slot of raw(i-1)
        __syncthreads();
        if (act) {
            const long long q = (long long)i * L.plane + j * L.n3 + m;
            const int gi = L.lo1 + i;
            const bool bxl = gi == 0, bxh = gi == L.n1 - 1;
            const int nb = (int)bxl + (int)bxh + nbjm_c;
            const cd fc = sm.f[wc][cfill];
            cd mf;
            cd ap;
            double kk = 0.0;
            if (KVAR) {
                kk = sm.kr[cslot & (KVAR ? PIPE_MASK : 0)][cfill];
                ap = ap_of(L, kk, nb);
            } else {
                ap = apt[nb];
            }
            if (L.bc == HF_BC_DIRICHLET && nb) {
                mf = fc;
            } else {
                cd xm = sm.f[wp][cfill], xp = sm.f[wn][cfill];
                cd ym = sm.f[wc][cfill - HALO_X], yp = sm.f[wc][cfill + HALO_X];
                cd zm = sm.f[wc][cfill - 1], zp = sm.f[wc][cfill + 1];
                if (bxl) xm = xp;
                if (bxh) xp = xm;
                if (byl) ym = yp;
                if (byh) yp = ym;
                if (bzl) zm = zp;
                if (bzh) zp = zm;
                cd sum = cadd(cadd(cadd(xm, xp), cadd(ym, yp)), cadd(zm, zp));
                mf = cmul(ap, fc);
                mf.x -= L.ih2 * sum.x;
                mf.y -= L.ih2 * sum.y;
            }
            cd av = mk(0, 0);
            if (Epi::kAux) av = SM::kAuxArr ? sm.ax[cslot & (SM::kAuxArr ? PIPE_MASK : 0)][tid]
                                            : sm.raw[cslot][cfill];
            cd wd = mk(0, 0);
            if (Epi::kDinv) {
                if (KVAR) wd = cscal(cdiv(mk(1.0, 0.0), diag_of(L, kk, nb)), omega);
                else wd = wdt[nb];
            }
            epi(q, fc, mf, wd, av, acc);
        }
        int t = wp; wp = wc; wc = wn; wn = t;
        cslot = (cslot + 1) & PIPE_MASK;
    }
    cp_wait<0>();
    constexpr int NR = (ND > 0) ? ND : 1;
    if (ND > 0) {
        cd a2[NR];
#pragma unroll
        for (int d = 0; d < NR; d++) a2[d] = acc[d];
        reduce_finish<NR>(a2, rs);
    }
}

// u = w D^-1 b   (multigrid.py:148-151, assume_zero first sweep)
__global__ void __launch_bounds__(256) k_jacobi0(Lvl L, const cd *__restrict__ b,
                                                 cd *__restrict__ u, double omega, int chunk,
                                                 const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(L, chunk);
    if (!c.act) return;
    ProdPre P{b, omega};
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * L.plane + (long long)c.j * L.n3 + c.m;
        u[q] = P(L, i, c.j, c.m);
    }
}

// out = P e (ADD=0) or out += P e (ADD=1)
template <int ADD>
__global__ void __launch_bounds__(256) k_prolong(Lvl F, Lvl C, const cd *__restrict__ e,
                                                 cd *__restrict__ out, int chunk, const int *done) {
    if (is_done(done)) return;
    ColCtx c = col_ctx(F, chunk);
    if (!c.act) return;
    Prolong P{C, e};
    for (int i = c.i0; i < c.i1; i++) {
        long long q = (long long)i * F.plane + (long long)c.j * F.n3 + c.m;
        cd pe = P(F, i, c.j, c.m);
        out[q] = ADD ? cadd(out[q], pe) : pe;
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

// Modified Gram-Schmidt step (krylov.py:151-154): w -= c[0] * vprev (if c),
// then the conjugated dot of vcur with the updated w (or |w|^2 when vcur is
// null) into red.out -- one pass over w per MGS step.
__global__ void __launch_bounds__(256) k_mgs(long long n, cd *__restrict__ w, const cd *c,
                                             const cd *__restrict__ vprev,
                                             const cd *__restrict__ vcur, RedSlot red) {
    cd cc = c ? *c : mk(0, 0);
    cd acc[1] = {mk(0, 0)};
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd wv = w[q];
        if (c) {
            wv = csub(wv, cmul(cc, __ldg(vprev + q)));
            w[q] = wv;
        }
        acc[0] = cadd(acc[0], vcur ? cjmul(__ldg(vcur + q), wv) : cjmul(wv, wv));
    }
    reduce_finish<1>(acc, red);
}

// x += sum_i y_i V_i (GMRES solution update, krylov.py:178-180), V given as a
// device array of pointers; each V_i is streamed once.
__global__ void __launch_bounds__(256) k_multi_axpy(long long n, int m, const cd *const *V,
                                                    const cd *y, cd *__restrict__ x) {
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd xv = x[q];
        for (int i = 0; i < m; i++) xv = cadd(xv, cmul(y[i], __ldg(V[i] + q)));
        x[q] = xv;
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
// x = Minv b, Minv row-major N x N.  One warp per row, 64-thread blocks (fine
// grained so rows spread evenly over the 148 SMs), eight 512 B row segments in
// flight per warp.
__global__ void __launch_bounds__(64) k_gemv(int N, const cd *__restrict__ Minv,
                                             const cd *__restrict__ b, cd *__restrict__ x,
                                             const int *done) {
    if (is_done(done)) return;
    int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (warp >= N) return;
    const cd *row = Minv + (long long)warp * N;
    cd a[8];
#pragma unroll
    for (int u = 0; u < 8; u++) a[u] = mk(0, 0);
    int j = lane;
    for (; j + 224 < N; j += 256) {
        cd mv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) mv[u] = __ldcs(row + j + 32 * u);
#pragma unroll
        for (int u = 0; u < 8; u++) a[u] = cadd(a[u], cmul(mv[u], __ldg(b + j + 32 * u)));
    }
    for (; j < N; j += 32) a[0] = cadd(a[0], cmul(__ldcs(row + j), __ldg(b + j)));
#pragma unroll
    for (int u = 1; u < 8; u++) a[0] = cadd(a[0], a[u]);
    a[0] = warp_sum(a[0]);
    if (lane == 0) x[warp] = a[0];
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

static dim3 tile_grid(const Lvl &L, int &chunk) {
    int gx = (L.n3 + TILE_X - 1) / TILE_X;
    int gy = (L.n2 + TILE_Y - 1) / TILE_Y;
    long long cols = (long long)gx * gy;
    long long target = 148 * 8;     // resident 256-thread blocks on B200
    int gz = (int)((target + cols - 1) / cols);
    gz = std::max(1, std::min(gz, L.nx));
    chunk = std::max((L.nx + gz - 1) / gz, 4);
    chunk = std::min(chunk, L.nx);
    gz = (L.nx + chunk - 1) / chunk;
    return dim3(gx, gy, gz);
}
static const dim3 kTileBlock(TILE_X, TILE_Y, 1);

template <int MODE, class Epi, int ND, bool KVAR>
static void stencil_launch(const Lvl &L, const Lvl &C, const cd *src, const cd *ec, const cd *aux,
                           double omega, const Epi &e, const RedSlot &rs, cudaStream_t s,
                           const int *done) {
    int chunk;
    dim3 g = tile_grid(L, chunk);
    size_t smem = sizeof(StencilSmem<MODE, KVAR, Epi::kAux>);
    k_stencil<MODE, Epi, ND, KVAR><<<g, kTileBlock, smem, s>>>(L, C, src, ec, aux ? aux : src, omega,
                                                               e, chunk, rs, done);
}
template <int MODE, class Epi, int ND>
static void stencil(const Lvl &L, const Lvl &C, const cd *src, const cd *ec, const cd *aux,
                    double omega, const Epi &e, const RedSlot &rs, cudaStream_t s, const int *done) {
    if (L.k) stencil_launch<MODE, Epi, ND, true>(L, C, src, ec, aux, omega, e, rs, s, done);
    else stencil_launch<MODE, Epi, ND, false>(L, C, src, ec, aux, omega, e, rs, s, done);
}

template <int MODE, class Epi, int ND>
static void set_attr() {
    cudaFuncSetAttribute(k_stencil<MODE, Epi, ND, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(StencilSmem<MODE, true, Epi::kAux>));
    cudaFuncSetAttribute(k_stencil<MODE, Epi, ND, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(StencilSmem<MODE, false, Epi::kAux>));
}

// opt the pipelined stencil kernels into > 48 KB dynamic shared memory (once, outside capture)
void init_kernel_attributes() {
    static bool done = false;
    if (done) return;
    set_attr<MODE_LOAD, EpiApply<0>, 0>();
    set_attr<MODE_LOAD, EpiApply<1>, 1>();
    set_attr<MODE_LOAD, EpiApply<2>, 2>();
    set_attr<MODE_LOAD, EpiResid, 0>();
    set_attr<MODE_LOAD, EpiJacobi, 0>();
    set_attr<MODE_PRE, EpiResid, 0>();
    set_attr<MODE_CORR1, EpiJacobi, 0>();
    set_attr<MODE_CORR0, EpiJacobi, 0>();
    done = true;
}

int tile_blocks(const Lvl &L) {
    int chunk;
    dim3 g = tile_grid(L, chunk);
    return g.x * g.y * g.z;
}

void launch_apply(const Lvl &L, const cd *u, cd *v, cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiApply<0>, 0>(L, L, u, nullptr, nullptr, 0.0, EpiApply<0>{v},
                                       RedSlot{}, s, done);
}
void launch_apply_dot1(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiApply<1>, 1>(L, L, u, nullptr, w, 0.0, EpiApply<1>{v}, rs, s, done);
}
void launch_apply_dot2(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiApply<2>, 2>(L, L, u, nullptr, w, 0.0, EpiApply<2>{v}, rs, s, done);
}
void launch_residual(const Lvl &L, const cd *u, const cd *b, cd *r, cudaStream_t s,
                     const int *done) {
    stencil<MODE_LOAD, EpiResid, 0>(L, L, u, nullptr, b, 0.0, EpiResid{r}, RedSlot{}, s, done);
}
void launch_jacobi(const Lvl &L, const cd *u, const cd *b, cd *uo, double omega,
                   cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiJacobi, 0>(L, L, u, nullptr, b, omega, EpiJacobi{uo}, RedSlot{}, s,
                                     done);
}
void launch_jacobi0(const Lvl &L, const cd *b, cd *u, double omega, cudaStream_t s,
                    const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    k_jacobi0<<<g, kMarchBlock, 0, s>>>(L, b, u, omega, chunk, done);
}
void launch_down1(const Lvl &L, const cd *b, cd *r, double omega, cudaStream_t s,
                  const int *done) {
    stencil<MODE_PRE, EpiResid, 0>(L, L, b, nullptr, b, omega, EpiResid{r}, RedSlot{}, s, done);
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
    if (pre)
        stencil<MODE_CORR1, EpiJacobi, 0>(L, C, b, e, b, omega, EpiJacobi{u}, RedSlot{}, s, done);
    else
        stencil<MODE_CORR0, EpiJacobi, 0>(L, C, b, e, b, omega, EpiJacobi{u}, RedSlot{}, s, done);
}
void launch_gemv(int N, const cd *Minv, const cd *b, cd *x, cudaStream_t s, const int *done) {
    int blocks = (N + 1) / 2;
    k_gemv<<<blocks, 64, 0, s>>>(N, Minv, b, x, done);
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
void launch_mgs(long long n, cd *w, const cd *c, const cd *vprev, const cd *vcur,
                const RedSlot &rs, cudaStream_t s) {
    k_mgs<<<VEC_BLOCKS, 256, 0, s>>>(n, w, c, vprev, vcur, rs);
}
void launch_multi_axpy(long long n, int m, const cd *const *V, const cd *y, cd *x, cudaStream_t s) {
    k_multi_axpy<<<VEC_BLOCKS, 256, 0, s>>>(n, m, V, y, x);
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
