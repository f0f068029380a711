// hf_device.cuh -- device-side building blocks of the B200 CSLP path.
//
// Layout: complex128 fields as double2, shape (nx, n2, n3) C order (i3
// fastest), slab along i1 with HF_GHOST ghost planes before/after the owned
// planes.  Helpers for complex arithmetic, the per-level stencil description,
// the boundary-row coefficients and deterministic block reductions.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/helmfree_b200.h"

namespace hf {

typedef double2 cd;

__device__ __forceinline__ cd mk(double x, double y) { return make_double2(x, y); }
__device__ __forceinline__ cd cadd(cd a, cd b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cd csub(cd a, cd b) { return mk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ cd cscal(cd a, double s) { return mk(a.x * s, a.y * s); }
__device__ __forceinline__ cd cmul(cd a, cd b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * b + c
__device__ __forceinline__ cd cfma(cd a, cd b, cd c) {
    return mk(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// conj(a) * b
__device__ __forceinline__ cd cjmul(cd a, cd b) {
    return mk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ cd cdiv(cd a, cd b) {
    double inv = 1.0 / (b.x * b.x + b.y * b.y);
    return mk((a.x * b.x + a.y * b.y) * inv, (a.y * b.x - a.x * b.y) * inv);
}
__device__ __forceinline__ double cabs2(cd a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double cabsd(cd a) { return hypot(a.x, a.y); }

// One grid level on one slab (operators.py:122-183 StencilOperator state).
struct Lvl {
    int n1, n2, n3;      // global vertex counts
    int lo1, nx;         // owned global planes [lo1, lo1 + nx)
    long long plane;     // n2 * n3
    double h, h2, ih2, twoh;  // h, h^2, 1/h^2, 2/h
    double sre, sim;     // shift = beta1 - i beta2
    int bc;              // HF_BC_*
    const double *k;     // wavenumber at owned plane 0 (ghost planes valid), or null
    double kc;           // constant wavenumber when k == null
    const double2 *dinv; // D^-1 at owned plane 0 (ghost planes valid) when k varies, else null
    const double2 *tab;  // constant k, nb physical faces: tab[nb] = a_p, tab[4 + nb] = D^-1,
                         // tab[8 + nb] = D^-1(nb) / D^-1(0)
    // palette (wide levels of a medium with <= 256 distinct wavenumbers): k as an
    // 8-bit index into kpal, a_p and D^-1 per (index, face count) in apal / dpal
    // (4 entries per index) -- 1 byte of k traffic per vertex instead of 8, no
    // D^-1 field and no reciprocal
    const unsigned char *kidx;   // at owned plane 0 (ghost planes valid), or null
    int npal;                    // palette entries in use
    const double *kpal;
    const double2 *apal, *dpal;
};


__device__ __forceinline__ double kat(const Lvl &L, long long q) {
    return L.k ? __ldg(L.k + q) : L.kc;
}

// Number of physical faces the vertex touches (edges/corners count each face).
__device__ __forceinline__ int nbnd(const Lvl &L, int gi, int j, int m) {
    return (gi == 0) + (gi == L.n1 - 1) + (j == 0) + (j == L.n2 - 1) + (m == 0) + (m == L.n3 - 1);
}

// Stencil centre ap (operators.py:163-172): (6 - s k^2 h^2)/h^2, minus 2ik/h per
// physical face for Sommerfeld.
__device__ __forceinline__ cd ap_of(const Lvl &L, double kk, int nb) {
    double k2h2 = kk * kk * L.h2;
    cd a = mk((6.0 - L.sre * k2h2) * L.ih2, (-L.sim * k2h2) * L.ih2);
    if (L.bc == HF_BC_SOMMERFELD) a.y -= (double)nb * (kk * L.twoh);
    return a;
}

// Jacobi diagonal (operators.py:173-178): Dirichlet boundary rows are identities.
__device__ __forceinline__ cd diag_of(const Lvl &L, double kk, int nb) {
    if (L.bc == HF_BC_DIRICHLET && nb) return mk(1.0, 0.0);
    return ap_of(L, kk, nb);
}

// D^-1 from the wavenumber: one complex reciprocal (same formula as the stored
// D^-1 field of k_dinv, so both give identical bits).  Cheaper than streaming
// the 16-byte field: a varying medium reads k (8 B) anyway.
__device__ __forceinline__ cd dinv_of(const Lvl &L, double kk, int nb) {
    const cd d = diag_of(L, kk, nb);
    // 1 / |d|^2 without the IEEE division's special-case branch: the MUFU
    // approximation refined by two Newton steps (|d|^2 is a normal number here,
    // the diagonal is bounded away from 0 and overflow; result within 1 ulp)
    const double m = d.x * d.x + d.y * d.y;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(m));
    r = fma(r, fma(-m, r, 1.0), r);
    r = fma(r, fma(-m, r, 1.0), r);
    return mk(d.x * r, -d.y * r);
}

// D^-1 at local linear index q of a vertex touching nb physical faces: the
// stored field where the level keeps one (a pointwise kernel without ALU slack
// -- k_corr -- is faster streaming 16 B than dividing), else from k
__device__ __forceinline__ double2 dinv_at(const Lvl &L, long long q, int nb) {
    if (L.kidx) return __ldg(L.dpal + 4 * __ldg(L.kidx + q) + nb);
    if (L.dinv) return __ldg(L.dinv + q);
    return L.k ? dinv_of(L, __ldg(L.k + q), nb) : __ldg(L.tab + 4 + nb);
}

// ---------------------------------------------------------------------------
// deterministic reductions: per-block partials + last-block finalize
// ---------------------------------------------------------------------------
#define HF_RED_THREADS 256
#define HF_MAX_DOTS 2

struct BcgState;   // fwd

// finalize op codes
enum {
    FIN_STORE = 0,       // write the sums to out[]
    FIN_BCG_INIT = 1,    // sums: |b|^2
    FIN_BCG_ALPHA = 2,   // sums: rs^H v
    FIN_BCG_S = 3,       // sums: |s|^2
    FIN_BCG_OMEGA = 4,   // sums: t^H t, t^H s
    FIN_BCG_RHO = 5,     // sums: |r|^2, rs^H r
};

struct RedSlot {
    cd *partials;        // >= nblocks * HF_MAX_DOTS
    unsigned *counter;   // zero-initialised, reset by the last block
    cd *out;             // FIN_STORE destination (HF_MAX_DOTS)
    int op;
    BcgState *st;
    // sparse shadow (st->nz > 0): sums[gd] = r~^H gvec over the nonzeros of r~,
    // gathered by the last block (the dense pass then skips reading r~)
    const cd *gvec = nullptr;
    int gd = 0;
};

#define HF_NZ_MAX 16   // shadow vectors with at most this many nonzeros are gathered

// Seeded shadow vector entry (SolverConfig.shadow = "random"): splitmix64 of
// (seed, global vertex index) -> two doubles uniform in [-1/2, 1/2) (53-bit
// mantissas, exact).  The C oracle draws the same values (or_shadow_hash).
__host__ __device__ inline unsigned long long splitmix64(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ inline cd shadow_hash(unsigned long long seed, unsigned long long q) {
    const unsigned long long a = splitmix64(seed * 0x632be59bd9b4e019ull + 2 * q);
    const unsigned long long b = splitmix64(seed * 0x632be59bd9b4e019ull + 2 * q + 1);
    const double s = 1.0 / 9007199254740992.0;   // 2^-53
    cd w;
    w.x = (double)(a >> 11) * s - 0.5;
    w.y = (double)(b >> 11) * s - 0.5;
    return w;
}

// Bi-CGSTAB scalars, device resident (krylov.py:207-276).
struct BcgState {
    cd rho, rho_new, alpha, omega, beta;
    double bnorm, tol, btol, relres;
    int iter, maxit, done, converged, breakdown, s_conv, matvecs, pad1;
    double *hist;
    int hist_cap, pad2;
    // nonzeros of the shadow vector r~ (ascending index) when there are at most
    // HF_NZ_MAX of them -- a point source with the reference's r~ = b has one:
    // r~^H v is then conj(r~_s) v_s exactly, without streaming r~
    int nz, nz_count;
    long long nzq[HF_NZ_MAX];
    cd nzw[HF_NZ_MAX];
};

__device__ __forceinline__ cd warp_sum(cd v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_down_sync(0xffffffffu, v.x, o);
        v.y += __shfl_down_sync(0xffffffffu, v.y, o);
    }
    return v;
}

// Block-wide deterministic sum of ND complex accumulators; result valid in
// thread 0.  The first HF_RED_THREADS threads of the block contribute (a block
// may carry extra warps, e.g. a producer warp, whose values are ignored).
template <int ND>
__device__ __forceinline__ void block_sum(cd (&acc)[ND], cd (&out)[ND]) {
    __shared__ cd sm[ND][HF_RED_THREADS / 32];
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int lane = tid & 31, w = tid >> 5;
#pragma unroll
    for (int d = 0; d < ND; d++) {
        cd v = warp_sum(acc[d]);
        if (lane == 0 && w < HF_RED_THREADS / 32) sm[d][w] = v;
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int d = 0; d < ND; d++) {
            cd s = mk(0, 0);
            for (int k = 0; k < HF_RED_THREADS / 32; k++) s = cadd(s, sm[d][k]);
            out[d] = s;
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// Bi-CGSTAB scalar state machine (krylov.py:234-273), run by one thread.
// ---------------------------------------------------------------------------
__device__ inline void bcg_record(BcgState *st, double relres) {
    if (st->hist && st->iter < st->hist_cap) st->hist[st->iter] = relres;
    st->iter += 1;
    st->relres = relres;
}

__device__ inline void bcg_finalize(BcgState *st, int op, const cd *sums) {
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


// Write this block's partials; the last block to arrive reduces all partials in
// fixed block order and runs the finalize step.
template <int ND>
__device__ __forceinline__ void reduce_finish(cd (&acc)[ND], const RedSlot &rs) {
    cd bs[ND];
    block_sum<ND>(acc, bs);
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const unsigned nblk = gridDim.x * gridDim.y * gridDim.z;
    const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    __shared__ bool last;
    if (tid == 0) {
#pragma unroll
        for (int d = 0; d < ND; d++) rs.partials[(size_t)bid * ND + d] = bs[d];
        __threadfence();
        unsigned prev = atomicAdd(rs.counter, 1u);
        last = (prev == nblk - 1);
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    cd a2[ND];
#pragma unroll
    for (int d = 0; d < ND; d++) a2[d] = mk(0, 0);
    // four independent loads in flight per thread (fixed order => deterministic)
    unsigned b = tid < HF_RED_THREADS ? tid : nblk;
    for (; b + 3 * HF_RED_THREADS < nblk; b += 4 * HF_RED_THREADS) {
        cd p[4][ND];
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int d = 0; d < ND; d++)
                p[k][d] = __ldcg(rs.partials + (size_t)(b + k * HF_RED_THREADS) * ND + d);
#pragma unroll
        for (int k = 0; k < 4; k++)
#pragma unroll
            for (int d = 0; d < ND; d++) a2[d] = cadd(a2[d], p[k][d]);
    }
    for (; b < nblk; b += HF_RED_THREADS) {
#pragma unroll
        for (int d = 0; d < ND; d++) a2[d] = cadd(a2[d], __ldcg(rs.partials + (size_t)b * ND + d));
    }
    cd tot[ND];
    block_sum<ND>(a2, tot);
    if (tid == 0) {
        *rs.counter = 0u;
        cd sums[HF_MAX_DOTS];
#pragma unroll
        for (int d = 0; d < HF_MAX_DOTS; d++) sums[d] = d < ND ? tot[d < ND ? d : 0] : mk(0, 0);
        if (rs.op == FIN_STORE) {
#pragma unroll
            for (int d = 0; d < ND; d++) rs.out[d] = tot[d];
        } else {
            if (rs.gvec && rs.st->nz > 0) {   // sparse shadow: fixed ascending order
                cd g = mk(0, 0);
                for (int k = 0; k < rs.st->nz; k++)
                    g = cadd(g, cjmul(rs.st->nzw[k], __ldcg(rs.gvec + rs.st->nzq[k])));
                sums[rs.gd] = g;
            }
            bcg_finalize(rs.st, rs.op, sums);
        }
    }
}

}  // namespace hf
