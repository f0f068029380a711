// hf_kernels.cu -- sm_100a kernels of the CSLP / multigrid / Bi-CGSTAB path.
//
// Stencil kernels march along i1.  Planes up to 255 wide use the FLAT kernels:
// a block owns a contiguous range of the (i2, i3) plane, its halo arrives as one
// cp.async.bulk per plane on an mbarrier (k_flat_stencil, k_flat_dr, plus
// k_corr_flat / k_restrict_flat); wider planes use the 2-D tiled cp.async
// kernels (k_stencil, k_down_restrict, k_restrict2, k_corr).  Multigrid steps
// are fused where the reference's sequence allows it:
//   down : pre-smooth from zero + residual + full weighting
//          b_c = R (b - M (w D^-1 b))          (multigrid.py:373-386, 171-221)
//   up   : prolong + correct, then one Jacobi sweep
//          u = t + w D^-1 (b - M t), t = w D^-1 b + P e   (multigrid.py:389-392, 138-157)
// Krylov vector updates carry their inner products in the same pass, with a
// deterministic last-block reduction that also advances the Bi-CGSTAB scalars
// on the device (krylov.py:207-276).
#include <algorithm>
#include <utility>
#include <cstdlib>

#include "hf_kernels.cuh"
#include "hf_stencil.cuh"

namespace hf {

int g_opt[OPT_COUNT] = {};

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
// stencil kernels: cp.async plane ring + 2.5D tiles
//
// A block owns a 32 x 8 tile of (i3, i2) columns and marches along i1 over a
// chunk of planes.  Each plane's tile + 1-point halo of the stencil operand is
// copied global->shared with cp.async into a 5-slot ring, three planes ahead
// of the plane being computed, so one barrier per plane is enough and the
// 7-point row reads its six neighbours straight from the ring.  Centre-only
// epilogue operands (b, the inner-product partner w, the wavenumber) are
// prefetched into registers one plane ahead.  Two stencil inputs:
//   MODE_LOAD  f = u                      (A u, b - M u, Jacobi sweep)
//   MODE_PRE   f = w D^-1 b, zero-guess pre-smoothing folded into the
//              residual (multigrid.py:148-151 + 383-386): in the deep
//              interior of a constant medium w D^-1 is one constant and
//              M (c b) = c M b; elsewhere each neighbour is scaled by its own
//              w D^-1 (boundary-count formula, or the level's precomputed
//              w D^-1 field when k varies).
// ---------------------------------------------------------------------------
#define TILE_X 32
#define TILE_Y 8
#define HALO_X (TILE_X + 2)
#define HALO_Y (TILE_Y + 2)
#define NFILL (HALO_Y * HALO_X)
#define NT (TILE_X * TILE_Y)
#define RING 5

enum { MODE_LOAD = 0, MODE_PRE = 1, MODE_UP = 2 };

// MODE_UP: the staged operand is t = [w D^-1 b] + P e, produced in shared memory
// from the staged b and a staged tile of the coarse correction e (the
// prolongation + correction of multigrid.py:337-341 / 389-392 folded into the
// post-smoothing sweep that consumes it)
#define UP_MAX_CPLANES 10   // coarse planes staged per block (fine chunk <= 16)
#define UP_EW 18            // coarse tile: <= 18 x 6 columns cover the 34 x 10 fine halo tile
#define UP_EH 6
struct UpArgs {
    Lvl C;                  // coarse level of e
    const cd *e;            // coarse correction (owned plane 0)
    int pre;                // 1: t = w D^-1 b + P e (nu1 = 1), 0: t = P e (nu1 = 0)
};

template <int V>
struct IC {
    static constexpr int value = V;
};
// f(IC<B>), f(IC<B+1>), ..., f(IC<E-1>) at compile time
template <int B, int E, class F>
__device__ __forceinline__ void static_for(F &&f) {
    if constexpr (B < E) {
        f(IC<B>{});
        static_for<B + 1, E>(f);
    }
}
// march steps R = B.. of the ring until the chunk ends; false once it has
template <int B, int E, class F>
__device__ __forceinline__ bool ring_steps(F &&f, int &i, int i1) {
    if constexpr (B < E) {
        f(IC<B>{}, i);
        if (++i >= i1) return false;
        return ring_steps<B + 1, E>(f, i, i1);
    }
    return true;
}

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
__device__ __forceinline__ void cp_async16s(unsigned saddr, const void *gmem, bool valid) {
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async8s(unsigned saddr, const void *gmem, bool valid) {
    int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int MODE, bool KVAR, bool AUX>
struct StencilSmem {
    static constexpr bool kWd = false;   // (D^-1 b is formed in place from k, see vfix)
    static constexpr bool kKw = (MODE == MODE_PRE || MODE == MODE_UP) && KVAR;   // staged k of the fill entries
    static constexpr bool kUp = MODE == MODE_UP;
    cd raw[RING][NFILL];
    cd wd[kWd ? RING : 1][kWd ? NFILL : 1];
    double kw[kKw ? RING : 1][kKw ? NFILL : 1];
    cd ec[kUp ? UP_MAX_CPLANES : 1][kUp ? UP_EW * UP_EH : 1];   // coarse e tile
};

// Body of one (virtual) block: tile (bx, by) of (i3, i2) columns, planes
// [bz chunk, (bz + 1) chunk).
// (block index passed explicitly so the body can be driven by other schedules)
template <int MODE, class Epi, int ND, bool KVAR, bool SOMM>
__device__ __forceinline__ void stencil_body(const Lvl &L, const cd *__restrict__ src,
                                             const cd *__restrict__ aux, double omega,
                                             const Epi &epi, int chunk, const RedSlot &rs,
                                             const UpArgs &up, unsigned char *smem_raw, int tid,
                                             int bx, int by, int bz) {
    using SM = StencilSmem<MODE, KVAR, Epi::kAux>;
    SM &sm = *reinterpret_cast<SM *>(smem_raw);
    const int tx = tid & (TILE_X - 1), ty = tid / TILE_X;
    const int m0 = bx * TILE_X, j0 = by * TILE_Y;
    const int i0 = bz * chunk, i1 = min(i0 + chunk, L.nx);
    const int m = m0 + tx, j = j0 + ty;
    const bool act = m < L.n3 && j < L.n2;
    const cd one = mk(1.0, 0.0);

    // fill entries of this thread: e0 = tid, e1 = tid + NT (when < NFILL).  A halo
    // entry one step outside the grid holds the MIRRORED inward value (row/column
    // 1 or n-2), so the Sommerfeld ghost elimination needs no branch: the
    // 7-point sum is uniform and the boundary lives in a_p (and Dirichlet rows,
    // identities, never read outside the grid).
    const bool has1 = tid + NT < NFILL;
    int go0, go1, nbe0, nbe1;
    int mj0 = 0, mm0 = 0, mj1 = 0, mm1 = 0;   // mirrored fine (i2, i3) of the fill entries
    bool ok0, ok1;
    {
        auto mirror = [](int x, int n) { return x < 0 ? -x : (x >= n ? 2 * (n - 1) - x : x); };
        int hy = tid / HALO_X, hx = tid - hy * HALO_X;
        int jj = j0 - 1 + hy, mm = m0 - 1 + hx;
        bool oj = jj >= -1 && jj <= L.n2, om = mm >= -1 && mm <= L.n3;
        bool corner = (jj < 0 || jj >= L.n2) && (mm < 0 || mm >= L.n3);
        ok0 = oj && om && !corner;
        go0 = ok0 ? mirror(jj, L.n2) * L.n3 + mirror(mm, L.n3) : 0;
        if (ok0) { mj0 = mirror(jj, L.n2); mm0 = mirror(mm, L.n3); }
        nbe0 = ok0 ? (mirror(jj, L.n2) == 0) + (mirror(jj, L.n2) == L.n2 - 1) +
                         (mirror(mm, L.n3) == 0) + (mirror(mm, L.n3) == L.n3 - 1) : 0;
        int e = tid + NT;
        hy = e / HALO_X; hx = e - hy * HALO_X;
        jj = j0 - 1 + hy; mm = m0 - 1 + hx;
        oj = jj >= -1 && jj <= L.n2; om = mm >= -1 && mm <= L.n3;
        corner = (jj < 0 || jj >= L.n2) && (mm < 0 || mm >= L.n3);
        ok1 = has1 && oj && om && !corner;
        go1 = ok1 ? mirror(jj, L.n2) * L.n3 + mirror(mm, L.n3) : 0;
        if (ok1) { mj1 = mirror(jj, L.n2); mm1 = mirror(mm, L.n3); }
        nbe1 = ok1 ? (mirror(jj, L.n2) == 0) + (mirror(jj, L.n2) == L.n2 - 1) +
                         (mirror(mm, L.n3) == 0) + (mirror(mm, L.n3) == L.n3 - 1) : 0;
    }
    const int own = j * L.n3 + m;
    const int cf = (ty + 1) * HALO_X + (tx + 1);
    const int nbjm = (j == 0) + (j == L.n2 - 1) + (m == 0) + (m == L.n3 - 1);
    // constant medium: a_p and w D^-1 by physical-face count (0..3) in shared memory
    __shared__ cd tab[16];
    cd ap0 = mk(0, 0), wd0 = mk(0, 0);
    if (!KVAR) {
        ap0 = __ldg(L.tab);
        wd0 = cscal(__ldg(L.tab + 4), omega);
        if (tid < 4) {
            tab[tid] = __ldg(L.tab + tid);
            tab[4 + tid] = cscal(__ldg(L.tab + 4 + tid), omega);
            tab[8 + tid] = cdiv(__ldg(L.tab + 4 + tid), __ldg(L.tab + 4));   // D^-1(nb) / D^-1(0)
            tab[12 + tid] = __ldg(L.tab + 4 + tid);                         // D^-1(nb)
        }
    }
    // MODE_PRE, constant medium: stage b^ = b * D^-1(nb)/D^-1(0) so f = w D^-1 b = wd0 b^
    // everywhere and the 7-point row is uniform; each thread rescales the
    // boundary vertices among its own fill entries once their copies land.
    constexpr bool kScale = MODE == MODE_PRE && !KVAR;
    const bool edge_block = j0 - 1 <= 0 || j0 + TILE_Y >= L.n2 - 1 || m0 - 1 <= 0 ||
                            m0 + TILE_X >= L.n3 - 1;
    // fill entries that are boundary vertices of an interior plane (nbx = 0) and
    // their rescale factors, fixed for the whole march
    const bool f0 = kScale && ok0 && nbe0 > 0, f1 = kScale && ok1 && nbe1 > 0;
    auto fixup = [&](int slot, int i) {
        int gi = L.lo1 + i;
        gi = gi < 0 ? -gi : (gi >= L.n1 ? 2 * (L.n1 - 1) - gi : gi);
        const int nbx = (gi == 0) + (gi == L.n1 - 1);
        if (nbx == 0) {                    // block-uniform
            if (!edge_block) return;
            if (f0) sm.raw[slot][tid] = cmul(sm.raw[slot][tid], tab[8 + nbe0]);
            if (f1) sm.raw[slot][tid + NT] = cmul(sm.raw[slot][tid + NT], tab[8 + nbe1]);
            return;
        }
        if (ok0) sm.raw[slot][tid] = cmul(sm.raw[slot][tid], tab[8 + nbx + nbe0]);
        if (ok1) sm.raw[slot][tid + NT] = cmul(sm.raw[slot][tid + NT], tab[8 + nbx + nbe1]);
    };
    // MODE_PRE, varying medium: each thread turns its own staged entries of b
    // into f = D^-1 b in place once their plane lands (one plane ahead of use),
    // D^-1 from k at the entry's (mirrored) vertex -- no D^-1 field is streamed
    // and a point's row reads its seven neighbours' f directly
    constexpr bool kVarPre = MODE == MODE_PRE && KVAR;
    // palette level: D^-1 of a staged entry is a table read at its 8-bit index,
    // the indices of plane p+1's entries loaded one step ahead (pix0 / pix1)
    // (the pre-smoothing sweep keeps staging k and forming D^-1: its per-entry
    // table reads on the critical path of every plane measured slower)
    const bool pal = KVAR && L.kidx != nullptr && MODE != MODE_PRE;
    auto ldix = [&](int p, int go) -> int {
        int g = L.lo1 + p;
        g = g < 0 ? -g : (g >= L.n1 ? 2 * (L.n1 - 1) - g : g);
        return __ldg(L.kidx + (long long)(g - L.lo1) * L.plane + go);
    };
    int pix0 = 0, pix1 = 0;
    auto vfix = [&](int slot, int i) {
        int gi = L.lo1 + i;
        gi = gi < 0 ? -gi : (gi >= L.n1 ? 2 * (L.n1 - 1) - gi : gi);
        const int nbx = (gi == 0) + (gi == L.n1 - 1);
        if (pal) {
            if (ok0) sm.raw[slot][tid] = cmul(sm.raw[slot][tid], __ldg(L.dpal + 4 * pix0 + nbx + nbe0));
            if (ok1) sm.raw[slot][tid + NT] = cmul(sm.raw[slot][tid + NT], __ldg(L.dpal + 4 * pix1 + nbx + nbe1));
            return;
        }
        if (ok0) sm.raw[slot][tid] = cmul(sm.raw[slot][tid], dinv_of(L, sm.kw[slot][tid], nbx + nbe0));
        if (ok1)
            sm.raw[slot][tid + NT] = cmul(sm.raw[slot][tid + NT], dinv_of(L, sm.kw[slot][tid + NT], nbx + nbe1));
    };
    auto pfix = [&](int p) {          // prefetch the palette indices of plane p's own entries
        if (!pal || p > i1) return;
        if (ok0) pix0 = ldix(p, go0);
        if (ok1) pix1 = ldix(p, go1);
    };
    // MODE_UP: coarse tile of e staged once per block (all coarse planes the
    // chunk's fine planes i0-1 .. i1 interpolate from, mirrored ones included)
    const Lvl &C = up.C;
    int c_lo = 0, cj_lo = 0, cm_lo = 0, ew = 0;
    int eo0 = 0, eo1 = 0;
    if (MODE == MODE_UP) {
        auto cmirror = [&](int p) {         // local fine plane -> mirrored global plane
            int g = L.lo1 + p;
            return g < 0 ? -g : (g >= L.n1 ? 2 * (L.n1 - 1) - g : g);
        };
        // fine g interpolates from coarse g >> 1 and, when odd, (g >> 1) + 1;
        // the march is monotone between its (possibly mirrored) end planes
        const int gmin = min(cmirror(i0 - 1), cmirror(i0));
        const int gmax = max(cmirror(i1), cmirror(i1 - 1));
        c_lo = gmin >> 1;
        const int c_hi = min(C.n1 - 1, (gmax + 1) >> 1);
        cj_lo = max(0, j0 - 1) >> 1;
        const int cj_hi = min(C.n2 - 1, (min(j0 + TILE_Y, L.n2 - 1) + 1) >> 1);
        cm_lo = max(0, m0 - 1) >> 1;
        const int cm_hi = min(C.n3 - 1, (min(m0 + TILE_X, L.n3 - 1) + 1) >> 1);
        ew = cm_hi - cm_lo + 1;
        const int eh = cj_hi - cj_lo + 1, np = c_hi - c_lo + 1, per = ew * eh;
        for (int t = tid; t < np * per; t += NT) {
            const int pl = t / per, r = t - pl * per, ry = r / ew, rx = r - ry * ew;
            const cd *g = up.e + (long long)(c_lo + pl - C.lo1) * C.plane +
                          (long long)(cj_lo + ry) * C.n3 + cm_lo + rx;
            cp_async16(&sm.ec[pl][ry * UP_EW + rx], g, true);
        }
        eo0 = ((mj0 >> 1) - cj_lo) * UP_EW + ((mm0 >> 1) - cm_lo);
        eo1 = ((mj1 >> 1) - cj_lo) * UP_EW + ((mm1 >> 1) - cm_lo);
    }
    // t = [w D^-1 b] + P e on this thread's own staged entries of plane p, in
    // place (k_corr arithmetic, at the mirrored coordinates of halo entries)
    auto produce = [&](int slot, int p) {
        int gi = L.lo1 + p;
        gi = gi < 0 ? -gi : (gi >= L.n1 ? 2 * (L.n1 - 1) - gi : gi);
        const int nbx = (gi == 0) + (gi == L.n1 - 1);
        const int cl = (gi >> 1) - c_lo;
        auto one = [&](int e, int gj, int gm, int nbe, int eo, int go) {
            const bool o2 = gj & 1, o3 = gm & 1;
            auto cplane = [&](int c) -> cd {
                const cd *q = &sm.ec[c][eo];
                cd a = q[0];
                if (o3) a = cadd(a, q[1]);
                if (o2) {
                    a = cadd(a, q[UP_EW]);
                    if (o3) a = cadd(a, q[UP_EW + 1]);
                }
                return a;
            };
            const double s2 = (o2 && o3) ? 0.25 : ((o2 || o3) ? 0.5 : 1.0);
            const cd v0 = cplane(cl);
            cd pe;
            if (gi & 1) pe = cscal(cadd(v0, cplane(cl + 1)), 0.5 * s2);
            else pe = s2 == 1.0 ? v0 : cscal(v0, s2);
            if (up.pre) {
                const cd D = KVAR ? dinv_of(L, sm.kw[slot][e], nbx + nbe) : tab[12 + nbx + nbe];
                pe = cadd(cscal(cmul(sm.raw[slot][e], D), omega), pe);
            }
            sm.raw[slot][e] = pe;
        };
        if (ok0) one(tid, mj0, mm0, nbe0, eo0, go0);
        if (ok1) one(tid + NT, mj1, mm1, nbe1, eo1, go1);
    };
    auto wd_nb = [&](int nb) -> cd { return tab[4 + nb]; };   // read after the first barrier
    cd acc[2] = {mk(0, 0), mk(0, 0)};

    // cp.async operands precomputed once: 32-bit shared addresses of this thread's
    // fill entries in ring slot 0 and global pointers of the entries in plane 0
    // (invalid entries point at a valid vertex and copy 0 bytes)
    const unsigned sraw0 = (unsigned)__cvta_generic_to_shared(&sm.raw[0][tid]);
    const unsigned swd0 = (unsigned)__cvta_generic_to_shared(&sm.wd[0][SM::kWd ? tid : 0]);
    const unsigned skw0 = (unsigned)__cvta_generic_to_shared(&sm.kw[0][SM::kKw ? tid : 0]);
    constexpr unsigned SLOT = NFILL * sizeof(cd);
    constexpr unsigned KSLOT = NFILL * sizeof(double);
    const double *k0 = SM::kKw ? L.k + go0 : nullptr, *k1 = SM::kKw ? L.k + go1 : nullptr;
    const bool stage_k = !pal || MODE == MODE_UP;   // MODE_UP forms D^-1 from the staged k
    const cd *g0 = src + go0, *g1 = src + go1;
    const cd *d0 = SM::kWd ? L.dinv + go0 : nullptr, *d1 = SM::kWd ? L.dinv + go1 : nullptr;
    auto stage = [&](auto SS, int p) {     // one commit group per plane, ring slot SS
        constexpr unsigned so = decltype(SS)::value * SLOT;
        // plane p of the march (ghost planes of a slab included; mirrored outside
        // the grid); nothing is copied past the chunk's last neighbour plane
        const int gi = L.lo1 + p;
        const bool pok = p <= i1 && gi >= -1 && gi <= L.n1;
        const int gm = gi < 0 ? -gi : (gi >= L.n1 ? 2 * (L.n1 - 1) - gi : gi);
        const long long pb = pok ? (long long)(gm - L.lo1) * L.plane : 0;
        const bool v0 = pok && ok0, v1 = pok && ok1;
        cp_async16s(sraw0 + so, g0 + pb, v0);
        if (SM::kWd) cp_async16s(swd0 + so, d0 + pb, v0);
        if (SM::kKw && stage_k) cp_async8s(skw0 + decltype(SS)::value * KSLOT, k0 + pb, v0);
        if (has1) {
            cp_async16s(sraw0 + so + NT * sizeof(cd), g1 + pb, v1);
            if (SM::kWd) cp_async16s(swd0 + so + NT * sizeof(cd), d1 + pb, v1);
            if (SM::kKw && stage_k) cp_async8s(skw0 + decltype(SS)::value * KSLOT + NT * sizeof(double), k1 + pb, v1);
        }
        cp_commit();
    };

    // in-loop staging (plane p = i + 3 > 0): straight copy while the plane is in
    // memory (owned or ghost), the mirrored plane n1-2 for global plane n1,
    // nothing past i1 (never read)
    const int p_direct_end = min(i1, L.n1 - 1 - L.lo1);
    const int p_mirror = L.n1 - L.lo1;
    const long long mirror_off = (long long)(L.n1 - 2 - L.lo1) * L.plane;
    auto stage_in = [&](auto SS, int p) {
        constexpr unsigned so = decltype(SS)::value * SLOT;
        long long pb = (long long)p * L.plane;
        bool any = p <= p_direct_end;
        if (!any && p == p_mirror && p <= i1) {
            pb = mirror_off;
            any = true;
        }
        if (any) {
            cp_async16s(sraw0 + so, g0 + pb, ok0);
            if (SM::kWd) cp_async16s(swd0 + so, d0 + pb, ok0);
            if (SM::kKw && stage_k) cp_async8s(skw0 + decltype(SS)::value * KSLOT, k0 + pb, ok0);
            if (has1) {
                cp_async16s(sraw0 + so + NT * sizeof(cd), g1 + pb, ok1);
                if (SM::kWd) cp_async16s(swd0 + so + NT * sizeof(cd), d1 + pb, ok1);
                if (SM::kKw && stage_k) cp_async8s(skw0 + decltype(SS)::value * KSLOT + NT * sizeof(double), k1 + pb, ok1);
            }
        }
        cp_commit();
    };

    // planes i0-1 .. i0+RING-3 into slots 0 .. RING-2
    static_for<0, RING - 1>([&](auto Sc) { stage(Sc, i0 - 1 + decltype(Sc)::value); });
    if (kScale || kVarPre || MODE == MODE_UP) {
        cp_wait<RING - 3>();               // planes i0-1, i0 (and the e tile) landed
        __syncthreads();                   // tab[] and the e tile visible
        if (kScale) {
            fixup(0, i0 - 1);
            fixup(1, i0);
        } else if (kVarPre) {
            pfix(i0 - 1);
            vfix(0, i0 - 1);
            pfix(i0);
            vfix(1, i0);
            pfix(i0 + 1);
        } else {
            produce(0, i0 - 1);
            produce(1, i0);
        }
    }
    long long q = (long long)i0 * L.plane + own;
    // centre-only epilogue operands (b or w, and k) are prefetched one plane ahead
    cd a_next = mk(0, 0);
    double k_next = L.kc;
    int ci_next = 0;                    // palette index of this thread's vertex
    if (act && i0 < i1) {
        if (Epi::kAux && aux) a_next = __ldg(aux + q);
        if (pal) ci_next = __ldg(L.kidx + q);
        else if (KVAR && !SM::kKw) k_next = __ldg(L.k + q);
    }
    cd rot_c = mk(0, 0), rot_m = mk(0, 0);   // centre values of planes i, i-1 (next step)
    // one plane; R = (i - i0) mod RING fixes the ring slots at compile time:
    // i-1 in R, i in R+1, i+1 in R+2, and plane i+RING-2 is staged into R-1
    auto step = [&](auto Rc, int i) {
        constexpr int R = decltype(Rc)::value;
        constexpr int sp = R, sc = (R + 1) % RING, sn = (R + 2) % RING;
        constexpr int ss = (R + RING - 1) % RING;
        const cd a_cur = a_next;
        const double k_cur = k_next;
        const int ci_cur = ci_next;
        if (act && i + 1 < i1) {
            if (Epi::kAux && aux) a_next = __ldg(aux + q + L.plane);
            if (pal) ci_next = __ldg(L.kidx + q + L.plane);
            else if (KVAR && !SM::kKw) k_next = __ldg(L.k + q + L.plane);
        }
        cp_wait<RING - 4>();               // plane i+1 landed (later ones may be in flight)
        if (kScale) fixup(sn, i + 1);      // own entries only: no barrier needed before
        if (kVarPre && i + 1 <= i1) {
            vfix(sn, i + 1);
            pfix(i + 2);
        }
        if (MODE == MODE_UP) produce(sn, i + 1);
        __syncthreads();
        stage_in(IC<ss>{}, i + RING - 2);  // into the slot read last at step i-1
        if (act) {
            const int gi = L.lo1 + i;
            const bool bxl = gi == 0, bxh = gi == L.n1 - 1;
            const int nb = (int)bxl + (int)bxh + nbjm;
            const cd *r0 = sm.raw[sc];
            // centre values of planes i-1, i rotate through registers along the
            // march (plane i+1's was read as xp at the previous step, after its
            // in-slot transform); only the first step reads them from the ring
            cd fc, xm;
            if (MODE != MODE_PRE || i == i0) {   // (rotation measured faster for PRE only)
                fc = r0[cf];
                xm = sm.raw[sp][cf];
            } else {
                fc = rot_c;
                xm = rot_m;
            }
            cd xp = sm.raw[sn][cf];
            rot_m = fc;
            rot_c = xp;
            cd ym = r0[cf - HALO_X], yp = r0[cf + HALO_X];
            cd zm = r0[cf - 1], zp = r0[cf + 1];
            const double kk = pal ? 0.0 : (SM::kKw ? sm.kw[sc][cf] : k_cur);   // PRE: k staged with the halo
            cd post = one;
            if (MODE == MODE_PRE) {
                if (KVAR) {                   // staged f = D^-1 b (vfix), w applied once after M
                    post = mk(omega, 0.0);
                } else {
                    post = wd0;               // f = wd0 * b^ (staged, rescaled at the faces)
                }
            }
            // uniform 7-point row: out-of-grid neighbours are already mirrored
            cd sum = cadd(cadd(cadd(xm, xp), cadd(ym, yp)), cadd(zm, zp));
            const cd ap = KVAR ? (pal ? __ldg(L.apal + 4 * ci_cur + nb) : ap_of(L, kk, nb))
                               : (nb == 0 ? ap0 : tab[nb]);
            cd mf = cmul(ap, fc);
            mf.x -= L.ih2 * sum.x;
            mf.y -= L.ih2 * sum.y;
            if (MODE == MODE_PRE) mf = cmul(post, mf);
            if (!SOMM && nb) mf = (MODE == MODE_PRE) ? cmul(post, fc) : fc;   // Dirichlet identity
            cd av = mk(0, 0);
            if (Epi::kAux) av = a_cur;
            cd wd = mk(0, 0);
            if (Epi::kDinv)
                wd = KVAR ? cscal(pal ? __ldg(L.dpal + 4 * ci_cur + nb) : dinv_of(L, kk, nb), omega) : wd_nb(nb);
            epi(q, fc, mf, wd, av, acc);
        }
        q += L.plane;
    };
    for (int i = i0; i < i1 && ring_steps<0, RING>(step, i, i1);) {
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

template <int MODE, class Epi, int ND, bool KVAR, bool SOMM>
__global__ void __launch_bounds__(NT) k_stencil(Lvl L, const cd *__restrict__ src,
                                                const cd *__restrict__ aux, double omega, Epi epi,
                                                int chunk, RedSlot rs, UpArgs up, const int *done) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (is_done(done)) return;
    stencil_body<MODE, Epi, ND, KVAR, SOMM>(L, src, aux, omega, epi, chunk, rs, up, smem_raw,
                                            threadIdx.y * TILE_X + threadIdx.x, blockIdx.x,
                                            blockIdx.y, blockIdx.z);
}

// ---------------------------------------------------------------------------
// k_flat_stencil: marching stencil on a FLAT (i2, i3) decomposition.
//
// Each plane is treated as one contiguous array of n2*n3 vertices; a block owns
// FS_PTS consecutive vertices of it (two per thread, 256 apart, so every warp
// access is 512 contiguous bytes) and marches along i1.  Its halo -- the owned
// range widened by one row (n3 + 1) on each side -- is ONE contiguous bulk copy
// per plane (cp.async.bulk, issued by thread 0, completed on the slot's
// mbarrier with expect_tx): no tensor map, no per-thread staging addresses,
// and no ragged tiles (grids of 2^k + 1 vertices waste ~1% instead of the
// ~35% a 32 x 8 tile wastes).  Neighbour offsets, including the Sommerfeld
// mirror at the faces (operators.py:9-12), are per-thread constants of the
// march; the centre value rotates through registers along i1, so a point
// reads 5 shared values per plane.  The first / last global plane take the
// mirrored plane through a block-uniform branch.  One __syncthreads per plane
// guards slot reuse.  Used when the halo is small against the owned range
// (n3 <= FS_MAX_N3); wider planes keep the 2-D tiled kernels.
// ---------------------------------------------------------------------------
#define FS_PTS 512
#define FS_RING 5
#define FS_MAX_N3 256

// slot geometry of one block: window [w0, w0 + FS_PTS + 2 (n3 + 1)) of the plane
__host__ __device__ __forceinline__ int fs_window(int n3) { return FS_PTS + 2 * (n3 + 1); }
__host__ __device__ __forceinline__ int fs_slot_bytes(int n3) { return (fs_window(n3) * 16 + 127) / 128 * 128; }

// MODE_LOAD: f = src.  MODE_PRE: f = w D^-1 src (zero-guess pre-smoothing folded
// into the residual, as in k_stencil): a constant medium stages b^ = b
// D^-1(nb)/D^-1(0) (face vertices rescaled in the slot one plane ahead of use)
// so f = wd0 b^ and the 7-point row stays uniform; a varying medium scales each
// neighbour by its own D^-1.  MODE_UP (post-smoothing after the coarse-grid
// correction, multigrid.py:389-392 + 153-156): every staged entry of b is turned
// in place into t = [w D^-1 b] + P e one plane ahead of use (the k_corr
// arithmetic at the mirrored coordinates of halo entries), and the sweep is
// u = t + w D^-1 (b - M t) -- the correction t never goes to memory.
template <int MODE, class Epi, int ND, bool KVAR, bool SOMM>
__global__ void __launch_bounds__(256, 3) k_flat_stencil(Lvl L, const cd *__restrict__ src,
                                                      const cd *__restrict__ aux, double omega, Epi epi,
                                                      int chunk, RedSlot rs, UpArgs up, const int *done) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long bars[FS_RING];
    __shared__ cd tab[8];
    __shared__ cd tabs[4];
    if (is_done(done)) return;
    const int tid = threadIdx.x;
    const int plane = (int)L.plane;
    const int f0 = blockIdx.x * FS_PTS;
    const int i0 = blockIdx.y * chunk, i1 = min(i0 + chunk, L.nx);
    const int w0 = f0 - (L.n3 + 1);
    const int c0 = max(w0, 0), c1 = min(f0 + FS_PTS + L.n3 + 1, plane);
    const unsigned cbytes = (unsigned)(c1 - c0) * 16u;
    const int sbytes = fs_slot_bytes(L.n3);
    const unsigned sraw = smem_u32(smem_raw);
    const unsigned sbase = (sraw + 127u) & ~127u, bbase = smem_u32(bars);
    const cd *const sgen = reinterpret_cast<const cd *>(smem_raw + (sbase - sraw));
    auto gmirror = [&](int g) { return g < 0 ? -g : (g >= L.n1 ? 2 * (L.n1 - 1) - g : g); };
    auto issue = [&](int p) {            // thread 0: halo window of local plane p (mirrored outside)
        const int k = (p - (i0 - 1)) % FS_RING;
        const unsigned bar = bbase + 8 * k;
        const long long lp = gmirror(L.lo1 + p) - L.lo1;
        mbar_expect_tx(bar, cbytes);
        bulk_g2s(sbase + k * sbytes + (c0 - w0) * 16, src + lp * plane + c0, cbytes, bar);
    };
    if (tid == 0) {
        for (int k = 0; k < FS_RING; k++) mbar_init(bbase + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (!KVAR && tid < 4) {
        tab[tid] = __ldg(L.tab + tid);
        tab[4 + tid] = cscal(__ldg(L.tab + 4 + tid), omega);
        if (MODE == MODE_PRE) tabs[tid] = cdiv(__ldg(L.tab + 4 + tid), __ldg(L.tab + 4));   // D^-1(nb)/D^-1(0)
    }
    if (MODE == MODE_UP && !KVAR && tid < 4) tabs[tid] = __ldg(L.tab + 4 + tid);            // D^-1(nb)
    __syncthreads();
    const int last = min(i1, L.n1 - 1 - L.lo1);       // last plane read (i1, or the top plane)
    if (tid == 0)
        for (int p = i0 - 1; p < i0 - 1 + FS_RING && p <= last; p++) issue(p);
    auto wait_plane = [&](int p) {
        const int d = p - (i0 - 1);
        mbar_wait(bbase + 8 * (d % FS_RING), (d / FS_RING) & 1);
    };
    auto slot = [&](int p) -> const cd * {
        return sgen + ((p - (i0 - 1)) % FS_RING) * (sbytes / 16);
    };
    // MODE_PRE, constant medium: this thread's window entries (e = tid + 256 t)
    // that are face vertices, rescaled in place by D^-1(nb)/D^-1(0) once their
    // plane lands (one plane ahead of its first use).  MODE_UP: every entry is
    // replaced by t = [w D^-1 b] + P e at the same point of the pipeline.
    constexpr bool kFix = MODE == MODE_PRE && !KVAR;
    constexpr bool kProd = MODE == MODE_UP;
    constexpr int NFE = (FS_PTS + 2 * (FS_MAX_N3 + 1) + 255) / 256;
    unsigned fe_nb = 0;                  // 2 bits per entry: in-plane face count
    unsigned fe_in = 0;                  // entry lies in the plane
    int fe_c[kProd ? NFE : 1];           // MODE_UP: coarse (i2, i3) base << 2 | odd i2 << 1 | odd i3
    if (kFix || kProd) {
        const int W = c1 - w0;
#pragma unroll
        for (int t = 0; t < NFE; t++) {
            const int e = tid + 256 * t, g = w0 + e;
            if (kProd) fe_c[t] = 0;
            if (e < W && g >= 0 && g < plane) {
                const int j = g / L.n3, m = g - j * L.n3;
                fe_in |= 1u << t;
                fe_nb |= (unsigned)((j == 0) + (j == L.n2 - 1) + (m == 0) + (m == L.n3 - 1)) << (2 * t);
                if (kProd) fe_c[t] = (((j >> 1) * up.C.n3 + (m >> 1)) << 2) | ((j & 1) << 1) | (m & 1);
            }
        }
    }
    auto fixup = [&](int p) {            // own entries of local plane p (mirrored outside)
        if (!kFix && !kProd) return;
        const int gm = gmirror(L.lo1 + p);
        const int nbx = (gm == 0) + (gm == L.n1 - 1);
        if (kFix && nbx == 0 && fe_nb == 0) return;
        cd *sl = const_cast<cd *>(slot(p));
        const Lvl &C = up.C;
        const int cl = (gm >> 1) - C.lo1;
        const bool odd = gm & 1;
#pragma unroll
        for (int t = 0; t < NFE; t++) {
            if (!((fe_in >> t) & 1u)) continue;
            const int e = tid + 256 * t;
            const int nb = nbx + (int)((fe_nb >> (2 * t)) & 3u);
            if (kFix) {
                if (nb > 0) sl[e] = cmul(sl[e], tabs[nb]);
                continue;
            }
            const int info = fe_c[t];
            const bool o2 = info & 2, o3 = info & 1;
            const cd *ecol = up.e + (info >> 2);
            auto cplane = [&](int c) -> cd {      // bilinear sum on coarse local plane c (k_corr)
                const cd *pp = ecol + (long long)c * C.plane;
                cd a = __ldg(pp);
                if (o3) a = cadd(a, __ldg(pp + 1));
                if (o2) {
                    a = cadd(a, __ldg(pp + C.n3));
                    if (o3) a = cadd(a, __ldg(pp + C.n3 + 1));
                }
                return a;
            };
            const double s2 = (o2 && o3) ? 0.25 : ((o2 || o3) ? 0.5 : 1.0);
            const cd v0 = cplane(cl);
            cd pe;
            if (odd) pe = cscal(cadd(v0, cplane(cl + 1)), 0.5 * s2);
            else pe = s2 == 1.0 ? v0 : cscal(v0, s2);
            if (up.pre) {
                const cd D = KVAR ? __ldg(L.dinv + (long long)(gm - L.lo1) * plane + (w0 + e)) : tabs[nb];
                pe = cadd(cscal(cmul(sl[e], D), omega), pe);
            }
            sl[e] = pe;
        }
    };
    // per point: smem offsets of centre and in-plane neighbours (mirrored at faces)
    int oc[2], ozm[2], ozp[2], oym[2], oyp[2], nbjm[2];
    bool act[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const int f = f0 + tid + 256 * k;
        act[k] = f < plane;
        const int ff = act[k] ? f : f0;
        const int j = ff / L.n3, m = ff - j * L.n3;
        oc[k] = ff - w0;
        ozm[k] = oc[k] + (m == 0 ? 1 : -1);
        ozp[k] = oc[k] + (m == L.n3 - 1 ? -1 : 1);
        oym[k] = oc[k] + (j == 0 ? L.n3 : -L.n3);
        oyp[k] = oc[k] + (j == L.n2 - 1 ? -L.n3 : L.n3);
        nbjm[k] = (j == 0) + (j == L.n2 - 1) + (m == 0) + (m == L.n3 - 1);
    }
    const cd apc = KVAR ? mk(0, 0) : tab[0];
    wait_plane(i0 - 1);
    wait_plane(i0);
    if (kFix || kProd) {
        fixup(i0 - 1);
        fixup(i0);
        if (i0 + 1 <= last) {
            wait_plane(i0 + 1);
            fixup(i0 + 1);
        }
        __syncthreads();
    }
    // plane values rotate through three register sets (prev / cur / next) with a
    // 3-way unrolled march, so no moves are spent on the rotation
    struct PV {
        cd v[2];      // staged value at the two points
        double k[2];  // wavenumber (varying medium)
    };
    PV S0, S1, S2;
    {
        const cd *sp = slot(i0 - 1), *sc = slot(i0);
        S0.v[0] = sp[oc[0]]; S0.v[1] = sp[oc[1]];
        S1.v[0] = sc[oc[0]]; S1.v[1] = sc[oc[1]];
    }
    cd acc[2] = {mk(0, 0), mk(0, 0)};
    long long q = (long long)i0 * plane + f0;      // plane origin of the block
    // point offsets; inactive points (past the plane end) use the block's first
    // vertex for their (unused) loads and skip the epilogue
    const int qo0 = act[0] ? tid : 0, qo1 = act[1] ? tid + 256 : 0;
#pragma unroll
    for (int k = 0; k < 2; k++) {
        S1.k[k] = L.kc;
        if (KVAR) S1.k[k] = __ldg(L.k + q + (k ? qo1 : qo0));
    }
    auto step = [&](int i, PV &P, PV &C, PV &N) {
        const int gi = L.lo1 + i;
        const bool top = gi == L.n1 - 1, bot = gi == 0;
        // centre epilogue operand of this plane, issued before the waits
        cd ca[2] = {mk(0, 0), mk(0, 0)};
        if (Epi::kAux && aux) {
            ca[0] = __ldg(aux + q + qo0);
            ca[1] = __ldg(aux + q + qo1);
        }
        __syncthreads();                             // slot of plane i-1 is free
        if (tid == 0 && i + FS_RING - 1 <= last) issue(i + FS_RING - 1);
        if ((kFix || kProd) && i + 2 <= last) {     // visible after the next barrier
            wait_plane(i + 2);
            fixup(i + 2);
        }
        if (!top) {
            wait_plane(i + 1);
            const cd *sn = slot(i + 1);
            N.v[0] = sn[oc[0]]; N.v[1] = sn[oc[1]];
        } else {
            N.v[0] = P.v[0]; N.v[1] = P.v[1];        // mirrored plane n1-2
        }
        if (KVAR && i + 1 < i1) {
#pragma unroll
            for (int k = 0; k < 2; k++) N.k[k] = __ldg(L.k + q + plane + (k ? qo1 : qo0));
        }
        const cd *s0 = slot(i);
        const int nbx = (int)bot + (int)top;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const long long qk = q + (k ? qo1 : qo0);
            cd fc = C.v[k], xm = bot ? N.v[k] : P.v[k], xp = N.v[k];
            cd ym = s0[oym[k]], yp = s0[oyp[k]], zm = s0[ozm[k]], zp = s0[ozp[k]];
            const int nb = nbx + nbjm[k];
            cd post = mk(1.0, 0.0);
            if (MODE == MODE_PRE) {
                if (KVAR) {          // f = D^-1 b per vertex, w applied after M
                    post = mk(omega, 0.0);
                    const cd *dv = L.dinv + qk;
                    const long long dxm = bot ? plane : -(long long)plane;
                    const long long dxp = top ? -(long long)plane : plane;
                    fc = cmul(fc, __ldg(dv));
                    xm = cmul(xm, __ldg(dv + dxm));
                    xp = cmul(xp, __ldg(dv + dxp));
                    ym = cmul(ym, __ldg(dv + (oym[k] - oc[k])));
                    yp = cmul(yp, __ldg(dv + (oyp[k] - oc[k])));
                    zm = cmul(zm, __ldg(dv + (ozm[k] - oc[k])));
                    zp = cmul(zp, __ldg(dv + (ozp[k] - oc[k])));
                } else {
                    post = tab[4];   // f = wd0 b^ (b^ rescaled in the slot)
                }
            }
            const cd sum = cadd(cadd(cadd(xm, xp), cadd(ym, yp)), cadd(zm, zp));
            const cd ap = KVAR ? ap_of(L, C.k[k], nb) : (nb == 0 ? apc : tab[nb]);
            cd mf = cmul(ap, fc);
            mf.x -= L.ih2 * sum.x;
            mf.y -= L.ih2 * sum.y;
            if (MODE == MODE_PRE) mf = cmul(post, mf);
            if (!SOMM && nb) mf = (MODE == MODE_PRE) ? cmul(post, fc) : fc;
            cd wd = mk(0, 0);
            if (Epi::kDinv) wd = KVAR ? cscal(dinv_of(L, C.k[k], nb), omega) : tab[4 + nb];
            if (act[k]) epi(qk, fc, mf, wd, ca[k], acc);
        }
        q += plane;
    };
    int i = i0;
    for (; i + 3 <= i1; i += 3) {
        step(i, S0, S1, S2);
        step(i + 1, S1, S2, S0);
        step(i + 2, S2, S0, S1);
    }
    if (i < i1) step(i, S0, S1, S2);
    if (i + 1 < i1) step(i + 1, S1, S2, S0);
    constexpr int NR = (ND > 0) ? ND : 1;
    if (ND > 0) {
        cd a2[NR];
#pragma unroll
        for (int d = 0; d < NR; d++) a2[d] = acc[d];
        reduce_finish<NR>(a2, rs);
    }
}

// ---------------------------------------------------------------------------
// k_flat_dr: zero-guess pre-smoothing + residual + full-weighting restriction
// in one pass (nu1 = 1, multigrid.py:383-386 then 171-221):
//     b_coarse = R (b - M (w D^-1 b))
// without writing or re-reading the fine residual.  A block owns DR2_CR whole
// coarse rows (all i3) of a chunk of coarse planes, i.e. fine residual rows
// 2 cr0 - 1 .. 2 cr1 - 1 (one row shared with each neighbour block) over all
// fine columns, and marches over the fine planes.  Per fine plane: the b rows
// of the block (+1 halo row each side, mirrored at the faces) arrive as ONE
// contiguous cp.async.bulk on the slot's mbarrier; face vertices are rescaled
// in the slot one plane ahead (MODE_PRE constant medium, as k_flat_stencil);
// every thread forms residual points of the plane into a shared tile; after
// one __syncthreads the coarse-column threads reduce it to the
// (1,2,1) x (1,2,1) partial and fold three consecutive partials into a coarse
// value.  Arithmetic and association follow k_stencil<MODE_PRE, EpiResid> +
// k_restrict2, so the result matches the split pair to rounding.
// ---------------------------------------------------------------------------
#define DR2_CR 2
#define DR2_NT 256
#define DR2_RING 6
#define DR2_RPT 5            // residual points per thread: (2 CR + 1) rows x n3 <= 5 x 255
#define DR2_MAX_N3 255

__host__ __device__ __forceinline__ int dr2_slot_elems(int n3) { return ((2 * DR2_CR + 3) * n3 + 7) / 8 * 8; }

template <bool KVAR, bool SOMM, int RPT>
__global__ void __launch_bounds__(DR2_NT, 2) k_flat_dr(Lvl L, Lvl C, const cd *__restrict__ b,
                                                       cd *__restrict__ out, double omega, int chunk,
                                                       const int *done) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long bars[DR2_RING];
    __shared__ cd tab[12];
    if (is_done(done)) return;
    const int tid = threadIdx.x;
    const int n3 = L.n3, plane = (int)L.plane, n1 = L.n1, n2 = L.n2, lo1 = L.lo1;
    const double ih2 = L.ih2;
    const int cr0 = blockIdx.x * DR2_CR, cr1 = min(cr0 + DR2_CR, C.n2);
    const int c0 = blockIdx.y * chunk, c1 = min(c0 + chunk, C.nx);
    if (c0 >= c1) return;
    const int gc0 = C.lo1 + c0, gc1 = C.lo1 + c1;              // global coarse planes [gc0, gc1)
    const int rlo = max(2 * cr0 - 1, 0), rhi = min(2 * cr1 - 1, L.n2 - 1);   // residual rows
    const int blo = max(rlo - 1, 0), bhi = min(rhi + 1, L.n2 - 1);           // staged b rows
    const int nrp = (rhi - rlo + 1) * n3;                       // residual points per plane
    const int dbo = (rlo - blo) * n3;                           // slot offset - tile offset
    const unsigned wbytes = (unsigned)((bhi - blo + 1) * n3) * 16u;
    const int selems = dr2_slot_elems(n3);
    const unsigned sraw = smem_u32(smem_raw);
    const unsigned sbase = (sraw + 127u) & ~127u, bbase = smem_u32(bars);
    cd *const sgen = reinterpret_cast<cd *>(smem_raw + (sbase - sraw));
    cd *const rt = sgen + DR2_RING * selems;                   // residual tiles [2][5 n3]
    auto gmirror = [&](int g) { return g < 0 ? -g : (g >= L.n1 ? 2 * (L.n1 - 1) - g : g); };
    const int gpf = 2 * gc0 - 1, gpl = 2 * gc1 - 1;             // residual planes [gpf, gpl]
    const int stage_last = gpl + 1;                             // last plane a residual reads
    auto issue = [&](int gp) {           // thread 0: b rows of global plane gp (mirrored outside)
        const int k = (gp - gpf + 1) % DR2_RING;
        const long long lp = gmirror(gp) - L.lo1;
        mbar_expect_tx(bbase + 8 * k, wbytes);
        bulk_g2s(sbase + k * selems * 16, b + lp * plane + (long long)blo * n3, wbytes, bbase + 8 * k);
    };
    auto wait_plane = [&](int gp) {
        const int d = gp - gpf + 1;
        mbar_wait(bbase + 8 * (d % DR2_RING), (d / DR2_RING) & 1);
    };
    auto slot = [&](int gp) { return sgen + ((unsigned)(gp - gpf + 1) % DR2_RING) * selems; };
    if (tid == 0) {
        for (int k = 0; k < DR2_RING; k++) mbar_init(bbase + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (!KVAR && tid < 4) {
        tab[tid] = __ldg(L.tab + tid);
        tab[4 + tid] = cscal(__ldg(L.tab + 4 + tid), omega);
        tab[8 + tid] = cdiv(__ldg(L.tab + 4 + tid), __ldg(L.tab + 4));   // D^-1(nb) / D^-1(0)
    }
    __syncthreads();
    if (tid == 0)
        for (int gp = gpf - 1; gp < gpf - 1 + DR2_RING && gp <= stage_last; gp++) issue(gp);

    // residual points of this thread: slot offset of the centre + packed flags
    // (bit0 row mirror below, bit1 row mirror above, bit2 col mirror left,
    //  bit3 col mirror right, bits 4-5 in-plane face count)
    int rc[RPT], rf[RPT];
#pragma unroll
    for (int t = 0; t < RPT; t++) {
        // points enumerated interior columns first (m in [2, n3-3], row by row),
        // then the four face-adjacent columns: the read-time face rescale then
        // diverges in one warp instead of in every warp that spans a row end
        const int e = tid + DR2_NT * t;
        const int ee = e < nrp ? e : 0;
        const int nrow = rhi - rlo + 1, ni = n3 >= 5 ? n3 - 4 : 0;
        int rr, m;
        if (ee < nrow * ni) {
            rr = rlo + ee / ni;
            m = 2 + (ee - (ee / ni) * ni);
        } else if (ni > 0) {
            const int e2 = ee - nrow * ni, k4 = e2 & 3;
            rr = rlo + (e2 >> 2);
            m = k4 < 2 ? k4 : n3 - 4 + k4;
        } else {
            rr = rlo + ee / n3;
            m = ee - (ee / n3) * n3;
        }
        rc[t] = (rr - blo) * n3 + m;
        auto fc1 = [](int x, int n) { return (x == 0) + (x == n - 1); };
        const int fj = fc1(rr, n2), fm = fc1(m, n3);
        const int jm = rr == 0 ? 1 : rr - 1, jp = rr == n2 - 1 ? n2 - 2 : rr + 1;
        const int mm = m == 0 ? 1 : m - 1, mp = m == n3 - 1 ? n3 - 2 : m + 1;
        // bits 0-3 mirror flags, 4-5 own in-plane face count, 6-13 the in-plane face
        // counts of the ym, yp, zm, zp neighbours (for the MODE_PRE face rescale)
        rf[t] = (rr == 0) | (rr == n2 - 1) << 1 | (m == 0) << 2 | (m == n3 - 1) << 3 | (fj + fm) << 4 |
                (fc1(jm, n2) + fm) << 6 | (fc1(jp, n2) + fm) << 8 | (fj + fc1(mm, n3)) << 10 |
                (fj + fc1(mp, n3)) << 12;
    }
    // coarse column of this thread: the LAST ncp threads (they carry one residual
    // point fewer than the first ones), so the per-plane work is balanced
    const int ncp = (cr1 - cr0) * C.n3;
    const int ct = tid - (DR2_NT - ncp);
    const bool cact = ct >= 0;
    const int cj = cr0 + (cact ? ct / C.n3 : 0), cm = cact ? ct - (ct / C.n3) * C.n3 : 0;
    const int crow = 2 * cj - rlo;                              // residual tile row of fine 2 cj
    const bool rm_ok = 2 * cj - 1 >= 0, rp_ok = 2 * cj + 1 <= L.n2 - 1;
    const bool cm_ok = 2 * cm - 1 >= 0, cp_ok = 2 * cm + 1 <= n3 - 1;
    cd Pprev = mk(0, 0), Pe = mk(0, 0);
    auto partial = [&](const cd *r) -> cd {
        cd s = mk(0, 0);
        const cd zero = mk(0, 0);
#pragma unroll
        for (int a = -1; a <= 1; a++) {
            const bool rok = a < 0 ? rm_ok : (a > 0 ? rp_ok : true);
            const cd *row = r + (crow + a) * n3 + 2 * cm;
            const cd v0 = rok && cm_ok ? row[-1] : zero;
            const cd v1 = rok ? row[0] : zero;
            const cd v2 = rok && cp_ok ? row[1] : zero;
            cd rs = cadd(cadd(v0, cscal(v1, 2.0)), v2);
            s = cadd(s, a == 0 ? cscal(rs, 2.0) : rs);
        }
        return s;
    };
    auto fold = [&](int gp, cd P) {
        if ((gp & 1) == 0) {
            Pe = P;
            return;
        }
        const int gc = (gp - 1) >> 1;
        if (gc >= gc0 && cact) {
            cd acc = cadd(cadd(Pprev, cscal(Pe, 2.0)), P);
            acc = mk(acc.x / 64.0, acc.y / 64.0);
            const int onb = (gc == 0 || gc == C.n1 - 1) + (cj == 0 || cj == C.n2 - 1) +
                            (cm == 0 || cm == C.n3 - 1);
            if (onb) {
                if (!SOMM) acc = mk(0, 0);
                else
                    for (int d = 0; d < onb; d++) acc = cscal(acc, 64.0 / 48.0);
            }
            out[(long long)(gc - C.lo1) * C.plane + (long long)cj * C.n3 + cm] = acc;
        }
        Pprev = P;
    };

    // prologue: planes gpf-1, gpf landed
    wait_plane(gpf - 1);
    wait_plane(gpf);
    const cd ap0 = KVAR ? mk(0, 0) : tab[0];
    const cd wd0 = KVAR ? mk(0, 0) : tab[4];
    // one fine plane -- the interior planes take a select-free body
    auto step = [&](auto EDGEc, int gp) {
        constexpr bool EDGE = decltype(EDGEc)::value;
        if (gp + 1 <= stage_last) wait_plane(gp + 1);
        const int buf = (gp - gpf) & 1;
        cd *rtile = rt + buf * (2 * DR2_CR + 1) * n3;
        const bool pin = !EDGE || (gp >= 0 && gp < n1);
        const bool bot = EDGE && gp == 0, top = EDGE && gp == n1 - 1;
        // planes gp-1 and gp+1 are staged mirrored at the faces (issue()), so the
        // x-neighbours read straight from their slots
        const cd *s0 = slot(gp), *sm1 = slot(gp - 1), *sp1 = slot(gp + 1);
        const int nbx = (int)bot + (int)top;
#pragma unroll
        for (int t = 0; t < RPT; t++) {
            const int e = tid + DR2_NT * t;
            if (e >= nrp) continue;
            cd rv = mk(0, 0);
            if (pin) {
                const int c = rc[t], f = rf[t];
                const int ym = (f & 1) ? c + n3 : c - n3, yp = (f & 2) ? c - n3 : c + n3;
                const int zm = (f & 4) ? c + 1 : c - 1, zp = (f & 8) ? c - 1 : c + 1;
                const int nb = nbx + ((f >> 4) & 3);
                cd fc = s0[c];
                cd xm = sm1[c], xp = sp1[c];
                cd vym = s0[ym], vyp = s0[yp], vzm = s0[zm], vzp = s0[zp];
                cd post = wd0;
                cd bc = fc;                               // staged b is unscaled
                if (KVAR) {
                    const long long q = (long long)(gp - lo1) * plane + (long long)blo * n3 + c;
                    post = mk(omega, 0.0);
                    const cd *dv = L.dinv + q;
                    const long long dxm = bot ? plane : -(long long)plane;
                    const long long dxp = top ? -(long long)plane : plane;
                    fc = cmul(fc, __ldg(dv));
                    xm = cmul(xm, __ldg(dv + dxm));
                    xp = cmul(xp, __ldg(dv + dxp));
                    vym = cmul(vym, __ldg(dv + (ym - c)));
                    vyp = cmul(vyp, __ldg(dv + (yp - c)));
                    vzm = cmul(vzm, __ldg(dv + (zm - c)));
                    vzp = cmul(vzp, __ldg(dv + (zp - c)));
                } else if (EDGE || (f >> 6)) {
                    // f = w D^-1 b with D^-1(nb) / D^-1(0) on the face vertices among the
                    // seven (as the staged rescale of k_stencil, applied at read time)
                    const int gxm = bot ? gp + 1 : gp - 1, gxp = top ? gp - 1 : gp + 1;
                    const int nbxm = (gxm == 0) + (gxm == n1 - 1), nbxp = (gxp == 0) + (gxp == n1 - 1);
                    auto sc = [&](cd v, int nbv) { return nbv > 0 ? cmul(v, tab[8 + nbv]) : v; };
                    fc = sc(fc, nb);
                    xm = sc(xm, nbxm + ((f >> 4) & 3));
                    xp = sc(xp, nbxp + ((f >> 4) & 3));
                    vym = sc(vym, nbx + ((f >> 6) & 3));
                    vyp = sc(vyp, nbx + ((f >> 8) & 3));
                    vzm = sc(vzm, nbx + ((f >> 10) & 3));
                    vzp = sc(vzp, nbx + ((f >> 12) & 3));
                }
                const cd sum = cadd(cadd(cadd(xm, xp), cadd(vym, vyp)), cadd(vzm, vzp));
                const cd ap = KVAR ? ap_of(L, __ldg(L.k + (long long)(gp - lo1) * plane +
                                                    (long long)blo * n3 + c), nb)
                                   : (nb == 0 ? ap0 : tab[nb]);
                cd mf = cmul(ap, fc);
                mf.x -= ih2 * sum.x;
                mf.y -= ih2 * sum.y;
                mf = cmul(post, mf);
                if (!SOMM && nb) mf = cmul(post, fc);
                rv = csub(bc, mf);
            }
            rtile[rc[t] - dbo] = rv;                  // row-major tile position
        }
        // the previous plane's residual tile is complete (last barrier): fold it
        // while the other warps still form this plane's tile
        if (cact && gp > gpf) fold(gp - 1, partial(rt + (buf ^ 1) * (2 * DR2_CR + 1) * n3));
        __syncthreads();                             // tile complete; slot of gp-1 free
        if (tid == 0 && gp + DR2_RING - 1 <= stage_last) issue(gp + DR2_RING - 1);
    };
    // EDGE: a face plane, a plane next to one (its x-neighbour needs the face
    // rescale) or a plane outside the grid
#pragma unroll 1
    for (int gp = gpf; gp <= gpl; gp++) {
        if (gp <= 1 || gp >= n1 - 2) step(IC<1>{}, gp);
        else step(IC<0>{}, gp);
    }
    if (cact) fold(gpl, partial(rt + ((gpl - gpf) & 1) * (2 * DR2_CR + 1) * n3));
}

// D^-1 over a level of a varying medium (owned + ghost planes), at setup
// palette tables: a_p and D^-1 of every (palette entry, face count) with the
// device formulas, so they are bit-identical to the on-the-fly values
__global__ void k_palette(Lvl L, int np, cd *__restrict__ apal, cd *__restrict__ dpal) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 4 * np) return;
    const double kk = L.kpal[t >> 2];
    apal[t] = ap_of(L, kk, t & 3);
    dpal[t] = dinv_of(L, kk, t & 3);
}

__global__ void k_dinv(Lvl L, int g0, int g1, cd *__restrict__ out) {
    pdl_enter();
    long long n = (long long)(g1 - g0) * L.plane;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x) {
        int i = g0 + (int)(t / L.plane);
        int rem = (int)(t - (long long)(i - g0) * L.plane);
        int j = rem / L.n3, m = rem - j * L.n3;
        long long q = (long long)i * L.plane + rem;
        out[q] = dinv_of(L, L.k[q], nbnd(L, L.lo1 + i, j, m));
    }
}

// pointwise coarse-grid correction on the zero-guess pre-smoothed iterate:
//   MODE 0: out = P e           MODE 1: out = w D^-1 b + P e   (nu1 = 1)
//   MODE 2: out += P e          (multigrid.py:337-341, 389-392)
// One thread per fine (i2, i3) column marching along i1: the bilinear (i2, i3)
// sum of each coarse plane is formed once and reused by the two fine planes
// that straddle it.
template <int MODE>
__device__ __forceinline__ void corr_col(const Lvl &F, const Lvl &C, const cd *__restrict__ b,
                                         const cd *__restrict__ e, cd *__restrict__ out,
                                         double omega, int j, int m, int i0, int i1);
template <int MODE>
__device__ __forceinline__ void corr_body(const Lvl &F, const Lvl &C, const cd *__restrict__ b,
                                          const cd *__restrict__ e, cd *__restrict__ out,
                                          double omega, int chunk, int tid, int bx, int by,
                                          int bz) {
    const int m = bx * 32 + (tid & 31);
    const int j = by * 8 + (tid >> 5);
    const int i0 = bz * chunk, i1 = min(i0 + chunk, F.nx);
    if (m >= F.n3 || j >= F.n2) return;
    corr_col<MODE>(F, C, b, e, out, omega, j, m, i0, i1);
}
// one fine (i2, i3) column over local planes [i0, i1)
template <int MODE>
__device__ __forceinline__ void corr_col(const Lvl &F, const Lvl &C, const cd *__restrict__ b,
                                         const cd *__restrict__ e, cd *__restrict__ out,
                                         double omega, int j, int m, int i0, int i1) {
    const bool o2 = j & 1, o3 = m & 1;
    const cd *ecol = e + (j >> 1) * C.n3 + (m >> 1);
    auto cplane = [&](int c) -> cd {                 // bilinear sum on coarse local plane c
        const cd *p = ecol + (long long)c * C.plane;
        cd a = __ldg(p);
        if (o3) a = cadd(a, __ldg(p + 1));
        if (o2) {
            a = cadd(a, __ldg(p + C.n3));
            if (o3) a = cadd(a, __ldg(p + C.n3 + 1));
        }
        return a;
    };
    const int nb_jm = (j == 0) + (j == F.n2 - 1) + (m == 0) + (m == F.n3 - 1);
    const double s2 = (o2 && o3) ? 0.25 : ((o2 || o3) ? 0.5 : 1.0);
    if (i1 - i0 == 4 && ((F.lo1 + i0) & 1) == 0) {
        // four fine planes 2c .. 2c+3 over coarse planes c, c+1, c+2, unrolled
        // (same arithmetic as the general march below; 4.1 TB/s at 129^3, the
        // one-launch copy ceiling at this size)
        const int gi0 = F.lo1 + i0, c = (gi0 >> 1) - C.lo1;
        const long long q0 = (long long)i0 * F.plane + j * F.n3 + m;
        const cd e0 = cplane(c), e1 = cplane(c + 1), e2 = cplane(c + 2);
        cd bv[4];
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (MODE == 1) bv[k] = __ldg(b + q0 + k * F.plane);
            if (MODE == 2) bv[k] = out[q0 + k * F.plane];
        }
        cd pe[4] = {s2 == 1.0 ? e0 : cscal(e0, s2), cscal(cadd(e0, e1), 0.5 * s2),
                    s2 == 1.0 ? e1 : cscal(e1, s2), cscal(cadd(e1, e2), 0.5 * s2)};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const long long q = q0 + k * F.plane;
            if (MODE == 1) {
                const int gi = gi0 + k;
                const int nb = (gi == 0) + (gi == F.n1 - 1) + nb_jm;
                pe[k] = cadd(cscal(cmul(bv[k], dinv_at(F, q, nb)), omega), pe[k]);
            }
            if (MODE == 2) pe[k] = cadd(bv[k], pe[k]);
            out[q] = pe[k];
        }
        return;
    }
    int cc = -(1 << 30);
    cd v0 = mk(0, 0), v1 = mk(0, 0);               // planes cc and cc + 1
    bool have1 = false;
    long long q = (long long)i0 * F.plane + j * F.n3 + m;
    for (int i = i0; i < i1; i++, q += F.plane) {
        const int gi = F.lo1 + i;
        const int c = (gi >> 1) - C.lo1;
        if (c != cc) {
            if (c == cc + 1 && have1) v0 = v1;
            else v0 = cplane(c);
            cc = c;
            have1 = false;
        }
        cd pe;
        if (gi & 1) {
            if (!have1) { v1 = cplane(c + 1); have1 = true; }
            pe = cscal(cadd(v0, v1), 0.5 * s2);
        } else {
            pe = s2 == 1.0 ? v0 : cscal(v0, s2);
        }
        if (MODE == 1) {
            const int nb = (gi == 0) + (gi == F.n1 - 1) + nb_jm;
            pe = cadd(cscal(cmul(__ldg(b + q), dinv_at(F, q, nb)), omega), pe);
        }
        if (MODE == 2) pe = cadd(out[q], pe);
        out[q] = pe;
    }
}

// flat variant: thread = one fine (i2, i3) vertex of the plane (no ragged tiles)
template <int MODE>
// local planes [plo, phi): the owned planes, or with the ghost planes at interior
// slab faces (the slab driver then skips the halo exchange of t)
__global__ void __launch_bounds__(256) k_corr_flat(Lvl F, Lvl C, const cd *__restrict__ b,
                                                   const cd *__restrict__ e, cd *__restrict__ out,
                                                   double omega, int chunk, int plo, int phi,
                                                   const int *done) {
    if (is_done(done)) return;
    const int f = blockIdx.x * 256 + threadIdx.x;
    if (f >= (int)F.plane) return;
    const int j = f / F.n3, m = f - j * F.n3;
    const int i0 = plo + blockIdx.y * chunk, i1 = min(i0 + chunk, phi);
    corr_col<MODE>(F, C, b, e, out, omega, j, m, i0, i1);
}

template <int MODE>
__global__ void __launch_bounds__(256) k_corr(Lvl F, Lvl C, const cd *__restrict__ b,
                                              const cd *__restrict__ e, cd *__restrict__ out,
                                              double omega, int chunk, const int *done) {
    if (is_done(done)) return;
    corr_body<MODE>(F, C, b, e, out, omega, chunk, threadIdx.x, blockIdx.x, blockIdx.y, blockIdx.z);
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
        u[q] = cscal(cmul(__ldg(b + q), dinv_at(L, q, nbnd(L, L.lo1 + i, c.j, c.m))), omega);
    }
}

// full-weighting restriction (multigrid.py:171-221), shared-memory tiled: a
// block owns 16 x 8 coarse columns and marches over a chunk of coarse planes;
// the two fine planes each coarse plane adds are prefetched with cp.async one
// step ahead, every fine plane is reduced once to its 2-D (1,2,1)x(1,2,1)
// partial, and a coarse value combines three consecutive partials.
#define RC_X 16
#define RC_Y 8
#define RF_X (2 * RC_X + 1)
#define RF_Y (2 * RC_Y + 1)
#define RF_N (RF_X * RF_Y)
struct RestrictSmem {
    cd fp[4][RF_N];
    cd P[3][RC_Y * RC_X];
};
__device__ __forceinline__ void restrict_body(const Lvl &F, const Lvl &C, const cd *__restrict__ r,
                                              cd *__restrict__ out, int chunk,
                                              RestrictSmem &sm, int tid, int bx, int by, int bz) {
    cd (*fp)[RF_N] = sm.fp;
    cd (*P)[RC_Y * RC_X] = sm.P;
    const int cm0 = bx * RC_X, cj0 = by * RC_Y;
    const int ci0 = bz * chunk, ci1 = min(ci0 + chunk, C.nx);
    const int fm0 = 2 * cm0 - 1, fj0 = 2 * cj0 - 1;
    int go[3];
    bool ok[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {
        int e = tid + 256 * k;
        int fy = e / RF_X, fx = e - fy * RF_X;
        int fj = fj0 + fy, fm = fm0 + fx;
        ok[k] = e < RF_N && fj >= 0 && fj < F.n2 && fm >= 0 && fm < F.n3;
        go[k] = ok[k] ? fj * F.n3 + fm : 0;
    }
    auto stage = [&](int gf, int slot) {     // fine global plane gf -> fp[slot]
        const bool pok = gf >= 0 && gf < F.n1;
        const cd *pp = r + (long long)(gf - F.lo1) * F.plane;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            int e = tid + 256 * k;
            if (e < RF_N) {
                bool v = pok && ok[k];
                cp_async16(&fp[slot][e], v ? pp + go[k] : r, v);
            }
        }
    };
    // 2-D partial of the coarse column handled by this thread, from plane slot
    const int cidx = tid & 127, cy = cidx / RC_X, cx = cidx - cy * RC_X;
    auto partial = [&](int slot) -> cd {
        const cd *b = &fp[slot][(2 * cy + 1) * RF_X + 2 * cx + 1];
        cd s = mk(0, 0);
#pragma unroll
        for (int a = -1; a <= 1; a++) {
            const cd *row = b + a * RF_X;
            cd rs = cadd(cadd(row[-1], cscal(row[0], 2.0)), row[1]);
            s = cadd(s, a == 0 ? cscal(rs, 2.0) : rs);
        }
        return s;
    };
    const int gc0 = C.lo1 + ci0;
    // prologue: fine planes 2gc0-1 (slot 3), 2gc0 (0), 2gc0+1 (1)
    stage(2 * gc0 - 1, 3);
    stage(2 * gc0, 0);
    stage(2 * gc0 + 1, 1);
    cp_commit();
    cp_wait<0>();
    __syncthreads();
    if (tid < 128) P[0][cidx] = partial(3);
    __syncthreads();                            // slot 3 is refilled by the first prefetch
    int pprev = 0, pe = 1, po = 2;
    int se = 0, so = 1;
    const int cj = cj0 + cy, cm = cm0 + cx;
    const bool act = cj < C.n2 && cm < C.n3;
    for (int ci = ci0; ci < ci1; ci++) {
        const int gc = C.lo1 + ci;
        if (ci + 1 < ci1) {                     // prefetch the next pair
            stage(2 * gc + 2, se ^ 2);
            stage(2 * gc + 3, so ^ 2);
        }
        cp_commit();
        if (tid < 128) P[pe][cidx] = partial(se);
        else P[po][cidx] = partial(so);
        __syncthreads();
        if (tid < 128 && act) {
            cd acc = cadd(cadd(P[pprev][cidx], cscal(P[pe][cidx], 2.0)), P[po][cidx]);
            acc = mk(acc.x / 64.0, acc.y / 64.0);
            int onb = (gc == 0 || gc == C.n1 - 1) + (cj == 0 || cj == C.n2 - 1) + (cm == 0 || cm == C.n3 - 1);
            if (onb) {
                if (C.bc == HF_BC_DIRICHLET) acc = mk(0, 0);
                else
                    for (int d = 0; d < onb; d++) acc = cscal(acc, 64.0 / 48.0);
            }
            out[(long long)ci * C.plane + cj * C.n3 + cm] = acc;
        }
        int t = pprev; pprev = po; po = pe; pe = t;
        se ^= 2; so ^= 2;
        cp_wait<0>();
        __syncthreads();
    }
}

// flat full-weighting restriction: one thread per coarse (i2, i3) vertex of a
// contiguous range of the coarse plane, marching over a chunk of coarse
// planes; each fine plane's (1,2,1) x (1,2,1) partial is formed once from L1 /
// L2 loads (neighbouring coarse vertices share fine rows) and the odd plane's
// partial is carried to the next coarse plane.  Association as k_restrict2.
__global__ void __launch_bounds__(256) k_restrict_flat(Lvl F, Lvl C, const cd *__restrict__ r,
                                                       cd *__restrict__ out, int chunk, const int *done) {
    if (is_done(done)) return;
    const int g = blockIdx.x * 256 + threadIdx.x;
    if (g >= (int)C.plane) return;
    const int cj = g / C.n3, cm = g - cj * C.n3;
    const int ci0 = blockIdx.y * chunk, ci1 = min(ci0 + chunk, C.nx);
    const int fj = 2 * cj, fm = 2 * cm;
    const bool jm = fj - 1 >= 0, jp = fj + 1 < F.n2, mm = fm - 1 >= 0, mp = fm + 1 < F.n3;
    const cd zero = mk(0, 0);
    // 2-D partial of global fine plane gf (zero outside the grid / slab data)
    auto partial = [&](int gf) -> cd {
        if (gf < 0 || gf >= F.n1) return zero;
        const cd *pl = r + (long long)(gf - F.lo1) * F.plane + (long long)fj * F.n3 + fm;
        cd s = zero;
#pragma unroll
        for (int a = -1; a <= 1; a++) {
            const bool rok = a < 0 ? jm : (a > 0 ? jp : true);
            const cd *row = pl + a * F.n3;
            const cd v0 = rok && mm ? __ldg(row - 1) : zero;
            const cd v1 = rok ? __ldg(row) : zero;
            const cd v2 = rok && mp ? __ldg(row + 1) : zero;
            const cd rs = cadd(cadd(v0, cscal(v1, 2.0)), v2);
            s = cadd(s, a == 0 ? cscal(rs, 2.0) : rs);
        }
        return s;
    };
    cd prev = partial(2 * (C.lo1 + ci0) - 1);
    for (int ci = ci0; ci < ci1; ci++) {
        const int gc = C.lo1 + ci;
        const cd pe = partial(2 * gc), po = partial(2 * gc + 1);
        cd acc = cadd(cadd(prev, cscal(pe, 2.0)), po);
        acc = mk(acc.x / 64.0, acc.y / 64.0);
        const int onb = (gc == 0 || gc == C.n1 - 1) + (cj == 0 || cj == C.n2 - 1) + (cm == 0 || cm == C.n3 - 1);
        if (onb) {
            if (C.bc == HF_BC_DIRICHLET) acc = zero;
            else
                for (int d = 0; d < onb; d++) acc = cscal(acc, 64.0 / 48.0);
        }
        out[(long long)ci * C.plane + g] = acc;
        prev = po;
    }
}

__global__ void __launch_bounds__(256) k_restrict2(Lvl F, Lvl C, const cd *__restrict__ r,
                                                   cd *__restrict__ out, int chunk, const int *done) {
    __shared__ __align__(16) RestrictSmem sm;
    if (is_done(done)) return;
    restrict_body(F, C, r, out, chunk, sm, threadIdx.x, blockIdx.x, blockIdx.y, blockIdx.z);
}

// ---------------------------------------------------------------------------
// Fused zero-guess pre-smoothing + residual + full-weighting restriction
// (nu1 = 1, multigrid.py:383-386 then 171-221):
//     b_coarse = R (b - M (w D^-1 b))
// without writing or re-reading the fine residual.  A block owns 16 x 4 coarse
// columns, i.e. a 33 x 9 tile of fine residual points (one shared column/row
// with the neighbouring tiles), and marches over the fine planes of a chunk of
// coarse planes.  Per fine plane: the 35 x 11 tile of b (mirrored halos,
// boundary-rescaled as in MODE_PRE) is staged by cp.async into a 5-slot ring
// three planes ahead, all threads form the residual of the 33 x 9 tile into a
// double-buffered shared tile, and warps 8-9 reduce the previous plane's tile
// to the (1,2,1) x (1,2,1) partials of their 64 coarse columns and combine
// three consecutive partials into a coarse value.  The arithmetic (and its
// association) is that of k_stencil<MODE_PRE, EpiResid> + k_restrict2, so the
// result is bit-identical to the split kernels.
// ---------------------------------------------------------------------------
#define DR_CX 16
#define DR_CY 4
#define DR_RX (2 * DR_CX + 1)
#define DR_RY (2 * DR_CY + 1)
#define DR_FX (DR_RX + 2)
#define DR_FY (DR_RY + 2)
#define DR_NF (DR_FX * DR_FY)
#define DR_NR (DR_RX * DR_RY)
#define DR_NT 320
#define DR_RING 6

template <bool KVAR>
struct DRSmem {
    cd f[DR_RING][DR_NF];
    double kw[KVAR ? DR_RING : 1][KVAR ? DR_NF : 1];   // staged k of the fill entries
    cd r[2][DR_NR];
};

template <bool KVAR, bool SOMM>
__global__ void __launch_bounds__(DR_NT, 3) k_down_restrict(Lvl L, Lvl C, const cd *__restrict__ b,
                                                         cd *__restrict__ out, double omega,
                                                         int chunk, const int *done) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    using SM = DRSmem<KVAR>;
    SM &sm = *reinterpret_cast<SM *>(smem_raw);
    __shared__ cd tab[16];
    if (is_done(done)) return;
    const int tid = threadIdx.x;
    const int cm0 = blockIdx.x * DR_CX, cj0 = blockIdx.y * DR_CY;
    const int c0 = blockIdx.z * chunk, c1 = min(c0 + chunk, C.nx);
    if (c0 >= c1) return;
    const int gc0 = C.lo1 + c0, gc1 = C.lo1 + c1;            // global coarse planes [gc0, gc1)
    const int fm0 = 2 * cm0 - 1, fj0 = 2 * cj0 - 1;          // residual tile origin (global)
    auto mirror = [](int x, int n) { return x < 0 ? -x : (x >= n ? 2 * (n - 1) - x : x); };

    if (!KVAR && tid < 4) {
        tab[tid] = __ldg(L.tab + tid);
        tab[4 + tid] = cscal(__ldg(L.tab + 4 + tid), omega);
        tab[8 + tid] = cdiv(__ldg(L.tab + 4 + tid), __ldg(L.tab + 4));   // D^-1(nb) / D^-1(0)
    }
    // fill entries e0 = tid, e1 = tid + DR_NT (< DR_NF): mirrored in-plane vertex
    const bool has1 = tid + DR_NT < DR_NF;
    int go[2] = {0, 0}, nbe[2] = {0, 0};
    bool ok[2] = {false, false};
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const int e = tid + k * DR_NT;
        const int hy = e / DR_FX, hx = e - hy * DR_FX;
        const int jj = fj0 - 1 + hy, mm = fm0 - 1 + hx;
        const bool oj = jj >= -1 && jj <= L.n2, om = mm >= -1 && mm <= L.n3;
        const bool corner = (jj < 0 || jj >= L.n2) && (mm < 0 || mm >= L.n3);
        ok[k] = (k == 0 || has1) && oj && om && !corner;
        if (ok[k]) {
            const int mj = mirror(jj, L.n2), mmm = mirror(mm, L.n3);
            go[k] = mj * L.n3 + mmm;
            nbe[k] = (mj == 0) + (mj == L.n2 - 1) + (mmm == 0) + (mmm == L.n3 - 1);
        }
    }
    const bool edge_block = fj0 - 1 <= 0 || fj0 + DR_RY >= L.n2 - 1 || fm0 - 1 <= 0 ||
                            fm0 + DR_RX >= L.n3 - 1;
    const unsigned sf0 = (unsigned)__cvta_generic_to_shared(&sm.f[0][tid]);
    const unsigned sw0 = (unsigned)__cvta_generic_to_shared(&sm.kw[0][KVAR ? tid : 0]);
    constexpr unsigned SLOT = DR_NF * sizeof(cd);
    constexpr unsigned KSLOT = DR_NF * sizeof(double);
    // stage global fine plane gp (mirrored outside the grid) into ring slot s
    const int gp_last_stage = 2 * gc1;                       // last plane a residual reads
    auto stage = [&](int s, int gp) {
        if (gp <= gp_last_stage) {                            // (slabs: stay inside the ghosts)
            const int gm = mirror(gp, L.n1);
            const long long pb = (long long)(gm - L.lo1) * L.plane;
            const unsigned so = s * SLOT;
            cp_async16s(sf0 + so, b + pb + go[0], ok[0]);
            if (KVAR) cp_async8s(sw0 + s * KSLOT, L.k + pb + go[0], ok[0]);
            if (has1) {
                cp_async16s(sf0 + so + DR_NT * sizeof(cd), b + pb + go[1], ok[1]);
                if (KVAR) cp_async8s(sw0 + s * KSLOT + DR_NT * sizeof(double), L.k + pb + go[1], ok[1]);
            }
        }
        cp_commit();
    };
    // constant medium: rescale this thread's boundary fill entries of plane gp;
    // varying medium: turn them into f = D^-1 b in place (D^-1 from the staged k)
    auto fixup = [&](int s, int gp) {
        if (KVAR) {
            const int gm = mirror(gp, L.n1);
            const int nbx = (gm == 0) + (gm == L.n1 - 1);
#pragma unroll
            for (int k = 0; k < 2; k++) {
                const int e = tid + k * DR_NT;
                if (ok[k]) sm.f[s][e] = cmul(sm.f[s][e], dinv_of(L, sm.kw[s][e], nbx + nbe[k]));
            }
            return;
        }
        const int gm = mirror(gp, L.n1);
        const int nbx = (gm == 0) + (gm == L.n1 - 1);
        if (nbx == 0 && !edge_block) return;
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const int e = tid + k * DR_NT;
            if (ok[k] && (nbx + nbe[k]) > 0) sm.f[s][e] = cmul(sm.f[s][e], tab[8 + nbx + nbe[k]]);
        }
    };

    // residual point of this thread (tid < DR_NR)
    const bool rpt = tid < DR_NR;
    const int ry = rpt ? tid / DR_RX : 0, rx = rpt ? tid - ry * DR_RX : 0;
    const int gj = fj0 + ry, gmc = fm0 + rx;
    const bool rin = rpt && gj >= 0 && gj < L.n2 && gmc >= 0 && gmc < L.n3;
    const int cf = (ry + 1) * DR_FX + (rx + 1);
    const int nbjm = rin ? (gj == 0) + (gj == L.n2 - 1) + (gmc == 0) + (gmc == L.n3 - 1) : 0;
    const long long own = (long long)gj * L.n3 + gmc;
    // coarse column of the reducing threads (warps 8-9)
    const int cth = tid - 8 * 32, ccx = cth & (DR_CX - 1), ccy = cth >> 4;
    const bool red = cth >= 0 && cth < DR_CX * DR_CY;
    const int cj = cj0 + ccy, cm = cm0 + ccx;
    const bool cact = red && cj < C.n2 && cm < C.n3;
    cd Pprev = mk(0, 0), Pe = mk(0, 0);

    auto partial = [&](int buf) -> cd {
        const cd *bb = &sm.r[buf][(2 * ccy + 1) * DR_RX + 2 * ccx + 1];
        cd s = mk(0, 0);
#pragma unroll
        for (int a = -1; a <= 1; a++) {
            const cd *row = bb + a * DR_RX;
            cd rs = cadd(cadd(row[-1], cscal(row[0], 2.0)), row[1]);
            s = cadd(s, a == 0 ? cscal(rs, 2.0) : rs);
        }
        return s;
    };
    // fold the partial of fine plane gp into the coarse accumulation; an odd
    // plane 2c+1 completes coarse plane c
    auto fold = [&](int gp, cd P) {
        if ((gp & 1) == 0) {
            Pe = P;
            return;
        }
        const int gc = (gp - 1) >> 1;
        if (gc >= gc0 && cact) {
            cd acc = cadd(cadd(Pprev, cscal(Pe, 2.0)), P);
            acc = mk(acc.x / 64.0, acc.y / 64.0);
            const int onb = (gc == 0 || gc == C.n1 - 1) + (cj == 0 || cj == C.n2 - 1) +
                            (cm == 0 || cm == C.n3 - 1);
            if (onb) {
                if (!SOMM) acc = mk(0, 0);
                else
                    for (int d = 0; d < onb; d++) acc = cscal(acc, 64.0 / 48.0);
            }
            out[(long long)(gc - C.lo1) * C.plane + (long long)cj * C.n3 + cm] = acc;
        }
        Pprev = P;
    };

    const int gp0 = 2 * gc0 - 1, gp1 = 2 * gc1 - 1;           // residual planes [gp0, gp1]
    // prologue: planes gp0-1 .. gp0+RING-3 into slots 0..RING-2
    for (int k = 0; k < DR_RING - 1; k++) stage(k, gp0 - 1 + k);
    cp_wait<DR_RING - 3>();
    __syncthreads();                                         // tab visible
    fixup(0, gp0 - 1);
    fixup(1, gp0);
    const cd ap0 = KVAR ? mk(0, 0) : tab[0];
    const cd wd0 = KVAR ? mk(0, 0) : tab[4];
    int sp = 0, sc = 1, sn = 2, ss = DR_RING - 1;            // slots of gp-1, gp, gp+1, free
    cd b_next = mk(0, 0);
    double k_next = L.kc;
    if (rin && gp0 >= 0 && gp0 < L.n1) {
        const long long q0 = (long long)(gp0 - L.lo1) * L.plane + own;
        b_next = __ldg(b + q0);
        if (KVAR) k_next = __ldg(L.k + q0);
    }
    for (int gp = gp0; gp <= gp1; gp++) {
        cp_wait<DR_RING - 4>();                              // plane gp+1 landed
        fixup(sn, gp + 1);
        __syncthreads();
        stage(ss, gp + DR_RING - 2);
        const int buf = (gp - gp0) & 1;
        if (rpt) {
            cd rv = mk(0, 0);
            const cd bc = b_next;
            const double kq = k_next;
            if (rin && gp + 1 >= 0 && gp + 1 < L.n1) {       // centre operands one plane ahead
                const long long qn = (long long)(gp + 1 - L.lo1) * L.plane + own;
                b_next = __ldg(b + qn);
                if (KVAR) k_next = __ldg(L.k + qn);
            }
            if (rin && gp >= 0 && gp < L.n1) {
                const cd *r0 = sm.f[sc];
                cd fc = r0[cf];
                cd xm = sm.f[sp][cf], xp = sm.f[sn][cf];
                cd ym = r0[cf - DR_FX], yp = r0[cf + DR_FX];
                cd zm = r0[cf - 1], zp = r0[cf + 1];
                const int nb = (gp == 0) + (gp == L.n1 - 1) + nbjm;
                const cd post = KVAR ? mk(omega, 0.0) : wd0;   // f = D^-1 b staged (fixup)
                cd sum = cadd(cadd(cadd(xm, xp), cadd(ym, yp)), cadd(zm, zp));
                const cd ap = KVAR ? ap_of(L, kq, nb) : (nb == 0 ? ap0 : tab[nb]);
                cd mf = cmul(ap, fc);
                mf.x -= L.ih2 * sum.x;
                mf.y -= L.ih2 * sum.y;
                mf = cmul(post, mf);
                if (!SOMM && nb) mf = cmul(post, fc);
                rv = csub(bc, mf);
            }
            sm.r[buf][tid] = rv;
        }
        if (red && gp > gp0) fold(gp - 1, partial(buf ^ 1));
        const int t = sp;
        sp = sc; sc = sn; sn = (sn + 1) % DR_RING; ss = t;
    }
    cp_wait<0>();
    __syncthreads();
    if (red) fold(gp1, partial((gp1 - gp0) & 1));
}

// ---------------------------------------------------------------------------
// 1-D vector kernels (owned region, contiguous)
// ---------------------------------------------------------------------------
#define VEC_BLOCKS 592   // 4 x 148 SMs, fixed => deterministic reductions

// Bi-CGSTAB start (krylov.py:217-232): r = b, x = p = v = 0; |b|^2, rs^H r, with the
// shadow vector rs (SolverConfig.shadow): HF_SHADOW_RHS rs = b (the reference,
// krylov.py:229); HF_SHADOW_HOST rs already loaded by the caller; HF_SHADOW_HASH
// rs = hf_shadow_hash(seed, global vertex index) -- layout independent, so a slab
// of a partitioned grid draws the same vector (offset q0 = first owned vertex).
__global__ void __launch_bounds__(256) k_bcg_init(long long n, const cd *__restrict__ b,
                                                  cd *__restrict__ r, cd *__restrict__ rs,
                                                  cd *__restrict__ x, cd *__restrict__ p,
                                                  cd *__restrict__ v, RedSlot red, int mode,
                                                  unsigned long long seed, long long q0) {
    pdl_enter();
    cd acc[2] = {mk(0, 0), mk(0, 0)};
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd bv = __ldg(b + q);
        r[q] = bv;
        if (mode == HF_SHADOW_RHS) {
            rs[q] = bv;
        } else {
            cd w;
            if (mode == HF_SHADOW_HASH) {
                w = shadow_hash(seed, (unsigned long long)(q0 + q));
                rs[q] = w;
            } else {
                w = rs[q];
            }
            acc[1] = cadd(acc[1], cjmul(w, bv));
        }
        x[q] = mk(0, 0); p[q] = mk(0, 0); v[q] = mk(0, 0);
        acc[0] = cadd(acc[0], cjmul(bv, bv));
    }
    if (mode == HF_SHADOW_RHS) acc[1] = acc[0];
    reduce_finish<2>(acc, red);
}

// nonzeros of the shadow vector (up to HF_NZ_MAX): slots taken in any order,
// sorted by k_nz_finish, so the gathered inner products are deterministic
__global__ void __launch_bounds__(256) k_nz_scan(long long n, const cd *__restrict__ rs, BcgState *st) {
    pdl_enter();
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        const cd w = __ldg(rs + q);
        if (w.x != 0.0 || w.y != 0.0) {
            const int k = atomicAdd(&st->nz_count, 1);
            if (k < HF_NZ_MAX) st->nzq[k] = q;
        }
    }
}
__global__ void k_nz_finish(const cd *__restrict__ rs, BcgState *st) {
    pdl_enter();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int c = st->nz_count;
    if (c < 1 || c > HF_NZ_MAX) { st->nz = -1; return; }
    for (int a = 1; a < c; a++)                     // insertion sort, <= 16 entries
        for (int b = a; b > 0 && st->nzq[b - 1] > st->nzq[b]; b--) {
            const long long t = st->nzq[b]; st->nzq[b] = st->nzq[b - 1]; st->nzq[b - 1] = t;
        }
    for (int k = 0; k < c; k++) st->nzw[k] = rs[st->nzq[k]];
    st->nz = c;
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

// s = r - alpha v ; |s|^2   (krylov.py:248-249).  s may BE r (the single-slab solver keeps
// s in r's buffer: the old residual is dead once s exists, and an in-place pass measured
// 1.23 -> 1.08 ms at 513^3), so r and s are neither restrict nor read through the
// read-only path; every element is read once and then written by the same thread.
__global__ void __launch_bounds__(256) k_bcg_s(long long n, const BcgState *st, const cd *r,
                                               const cd *__restrict__ v, cd *s, RedSlot red,
                                               const int *done) {
    if (is_done(done)) return;
    cd al = st->alpha;
    cd acc[1] = {mk(0, 0)};
    const long long S = (long long)gridDim.x * 256;
    long long q = blockIdx.x * 256ll + threadIdx.x;
    // two strides per trip; the per-thread accumulation order is unchanged
    for (; q + S < n; q += 2 * S) {
        cd r0 = r[q], r1 = r[q + S], v0 = __ldg(v + q), v1 = __ldg(v + q + S);
        cd s0 = csub(r0, cmul(al, v0)), s1 = csub(r1, cmul(al, v1));
        s[q] = s0;
        s[q + S] = s1;
        acc[0] = cadd(acc[0], cjmul(s0, s0));
        acc[0] = cadd(acc[0], cjmul(s1, s1));
    }
    if (q < n) {
        cd sv = csub(r[q], cmul(al, __ldg(v + q)));
        s[q] = sv;
        acc[0] = cadd(acc[0], cjmul(sv, sv));
    }
    reduce_finish<1>(acc, red);
}

// x += alpha ph + omega sh ; r = s - omega t ; |r|^2, rs^H r   (krylov.py:266-269).
// s may BE r (see k_bcg_s).
__global__ void __launch_bounds__(256) k_bcg_xr(long long n, const BcgState *st,
                                                cd *__restrict__ x, const cd *__restrict__ ph,
                                                const cd *__restrict__ sh, const cd *s,
                                                const cd *__restrict__ t, cd *r,
                                                const cd *__restrict__ rs, RedSlot red,
                                                const int *done) {
    if (is_done(done)) return;
    cd al = st->alpha, om = st->omega;
    cd acc[2] = {mk(0, 0), mk(0, 0)};
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd xv = cadd(cadd(x[q], cmul(al, __ldg(ph + q))), cmul(om, __ldg(sh + q)));
        x[q] = xv;
        cd rv = csub(s[q], cmul(om, __ldg(t + q)));
        r[q] = rv;
        acc[0] = cadd(acc[0], cjmul(rv, rv));
        if (rs) acc[1] = cadd(acc[1], cjmul(__ldg(rs + q), rv));   // null: sparse shadow
    }
    reduce_finish<2>(acc, red);
}

// one-thread Bi-CGSTAB state update from (all-reduced) inner products, for
// drivers whose reductions span several slabs / ranks (dist.SlabSolver): the
// local kernels store partial sums, the driver sums them across slabs, and
// this kernel runs the same state machine the single-slab reductions run in
// their last block.  No-op once the solve is done (except the init step).
__global__ void k_bcg_step(BcgState *st, int op, const cd *sums) {
    pdl_enter();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (op != FIN_BCG_INIT && st->done) return;
    bcg_finalize(st, op, sums);
}

// sparse shadow: r~^H g over the (<= HF_NZ_MAX) nonzeros of r~, then the scalar
// step `op` that consumes it as sums[0] -- the matvec feeding it runs without
// an inner-product pass (no second operand streamed)
__global__ void k_bcg_gather(BcgState *st, int op, const cd *__restrict__ g, const int *done) {
    if (is_done(done)) return;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    cd sums[HF_MAX_DOTS] = {mk(0, 0), mk(0, 0)};
    for (int k = 0; k < st->nz; k++)            // fixed ascending order
        sums[0] = cadd(sums[0], cjmul(st->nzw[k], __ldcg(g + st->nzq[k])));
    bcg_finalize(st, op, sums);
}

// slab drivers: this slab's share of r~^H g over the slab's own nonzeros of r~ (a per-slab
// nonzero list in nz; the shares are summed across slabs / ranks like any partial sum)
__global__ void k_gather_store(const BcgState *nz, const cd *__restrict__ g, cd *out, const int *done) {
    if (is_done(done)) return;
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    cd a = mk(0, 0);
    for (int k = 0; k < nz->nz; k++)            // fixed ascending order; nz <= 0: none here
        a = cadd(a, cjmul(nz->nzw[k], __ldcg(g + nz->nzq[k])));
    *out = a;
}

// x += alpha ph  (convergence at the half step, krylov.py:250-255)
__global__ void k_bcg_xhalf(long long n, const BcgState *st, cd *__restrict__ x,
                            const cd *__restrict__ ph) {
    pdl_enter();
    cd al = st->alpha;
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256)
        x[q] = cadd(x[q], cmul(al, __ldg(ph + q)));
}

// generic y = a x + b y with host scalars (GMRES / IDR helpers)
__global__ void k_axpby(long long n, cd a, const cd *__restrict__ x, cd b, cd *__restrict__ y) {
    pdl_enter();
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
    pdl_enter();
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
    pdl_enter();
    for (long long q = blockIdx.x * 256ll + threadIdx.x; q < n; q += (long long)gridDim.x * 256) {
        cd xv = x[q];
        for (int i = 0; i < m; i++) xv = cadd(xv, cmul(y[i], __ldg(V[i] + q)));
        x[q] = xv;
    }
}

// y = x - sum_i c_i V_i  with c on the device (dense coefficient vector)
__global__ void k_dot_store(long long n, const cd *__restrict__ a, const cd *__restrict__ b,
                            RedSlot red) {
    pdl_enter();
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

// ---- symmetric coarsest solve (Sommerfeld) ----------------------------------
// With S = diag(2^-faces) the Sommerfeld operator is complex symmetric after
// row scaling (S M = (S M)^T, the reference's own symmetry test), so
// B = M^-1 S^-1 is symmetric and x = M^-1 b = B (S b).  Only the upper
// triangle of B is stored, as 64 x 64 tiles (I <= J); each tile contributes
// its row sums to x_I and, off the diagonal, its column sums to x_J.
#define SYT 64
__device__ __forceinline__ long long sym_tile_index(int I, int J, int nT) {
    return (long long)I * nT - (long long)I * (I - 1) / 2 + (J - I);
}
// inverse of sym_tile_index: tile-row I of packed upper-triangle tile t
__device__ __forceinline__ int sym_tile_row(long long t, int nT) {
    const double a = 2.0 * nT + 1.0;
    int I = (int)floor((a - sqrt(a * a - 8.0 * (double)t)) * 0.5);
    I = max(0, min(I, nT - 1));
    while (I > 0 && sym_tile_index(I, I, nT) > t) I--;
    while (I + 1 < nT && sym_tile_index(I + 1, I + 1, nT) <= t) I++;
    return I;
}

// pack: tile (I, J) = Minv[I*64 + r][J*64 + c] / s[J*64 + c], zero padded
__global__ void k_sym_pack(int N, int nT, const cd *__restrict__ Minv, const double *__restrict__ s,
                           cd *__restrict__ tiles) {
    pdl_enter();
    const long long ntile = (long long)nT * (nT + 1) / 2;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < ntile * SYT * SYT;
         e += (long long)gridDim.x * blockDim.x) {
        long long t = e / (SYT * SYT);
        int rc = (int)(e - t * SYT * SYT), r = rc / SYT, c = rc - r * SYT;
        const int I = sym_tile_row(t, nT);
        int J = I + (int)(t - sym_tile_index(I, I, nT));
        int gi = I * SYT + r, gj = J * SYT + c;
        cd v = mk(0, 0);
        if (gi < N && gj < N) v = cscal(Minv[(long long)gi * N + gj], 1.0 / s[gj]);
        tiles[e] = v;
    }
}

// one 256-thread CTA per stored tile; warp w streams rows 8w..8w+7 straight
// from HBM (16 independent 16 B loads per lane), forms their row sums with
// warp shuffles and its partial column sums in registers; the 8 warps'
// column partials are combined through shared memory in fixed order.
__global__ void __launch_bounds__(256) k_sym_tiles(int N, int nT, const cd *__restrict__ tiles,
                                                   const double *__restrict__ s,
                                                   const cd *__restrict__ b,
                                                   cd *__restrict__ prow, cd *__restrict__ pcol,
                                                   const int *done) {
    __shared__ cd cI[SYT], cJ[SYT];
    __shared__ cd colp[8][SYT];
    if (is_done(done)) return;
    const long long t = blockIdx.x;
    const int I = sym_tile_row(t, nT);
    const int J = I + (int)(t - sym_tile_index(I, I, nT));
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
    const cd *src = tiles + t * SYT * SYT + (long long)(8 * w) * SYT;
    cd m0[8], m1[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        m0[k] = __ldcs(src + k * SYT + lane);
        m1[k] = __ldcs(src + k * SYT + lane + 32);
    }
    if (tid < SYT) {
        int gj = J * SYT + tid;
        cJ[tid] = gj < N ? cscal(__ldg(b + gj), s[gj]) : mk(0, 0);
    } else if (tid < 2 * SYT) {
        int gi = I * SYT + tid - SYT;
        cI[tid - SYT] = gi < N ? cscal(__ldg(b + gi), s[gi]) : mk(0, 0);
    }
    __syncthreads();
    const cd cj0 = cJ[lane], cj1 = cJ[lane + 32];
    cd c0 = mk(0, 0), c1 = mk(0, 0);
    cd rsum[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        rsum[k] = cadd(cmul(m0[k], cj0), cmul(m1[k], cj1));
        const cd ci = cI[8 * w + k];
        c0 = cadd(c0, cmul(m0[k], ci));
        c1 = cadd(c1, cmul(m1[k], ci));
    }
#pragma unroll
    for (int k = 0; k < 8; k++) rsum[k] = warp_sum(rsum[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 8; k++) prow[t * SYT + 8 * w + k] = rsum[k];
    }
    if (I != J) {
        colp[w][lane] = c0;
        colp[w][lane + 32] = c1;
        __syncthreads();
        if (tid < SYT) {
            cd a = colp[0][tid];
#pragma unroll
            for (int k = 1; k < 8; k++) a = cadd(a, colp[k][tid]);
            pcol[t * SYT + tid] = a;
        }
    }
}

// x_i = sum_{J >= I} rowpart(I, J) + sum_{I' < I} colpart(I', I): one warp per
// output, partials summed lane-strided then by a fixed shuffle tree
__global__ void k_sym_reduce(int N, int nT, const cd *__restrict__ prow,
                             const cd *__restrict__ pcol, cd *__restrict__ x, const int *done) {
    if (is_done(done)) return;
    const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (i >= N) return;
    const int I = i / SYT, r = i - I * SYT;
    cd acc = mk(0, 0);
    for (int J = lane; J < nT; J += 32) {
        if (J >= I) acc = cadd(acc, __ldg(prow + sym_tile_index(I, J, nT) * SYT + r));
        else acc = cadd(acc, __ldg(pcol + sym_tile_index(J, I, nT) * SYT + r));
    }
    acc = warp_sum(acc);
    if (lane == 0) x[i] = acc;
}

// Row-major dense CSLP matrix of a full (single-slab) level: A[r * N + c].
// ---------------------------------------------------------------------------
// Coarsest solve by fast diagonalisation (Lynch, Rice & Thomas 1964).  With a
// constant wavenumber the coarsest CSLP operator is separable,
//   M = T1 (x) I (x) I + I (x) T2 (x) I + I (x) I (x) T3 + c I,
// T_d the 1-D operator of direction d (Sommerfeld end rows included), so
//   M^-1 = (V1 (x) V2 (x) V3) diag(1 / (l1_a + l2_b + l3_c + c)) (V1^-1 (x) V2^-1 (x) V3^-1)
// with T_d = V_d diag(l_d) V_d^-1.  The exact solve costs 2 (n1 + n2 + n3) N
// complex MACs on N = n1 n2 n3 points (~0.5 M at 17^3) instead of streaming
// the N^2 dense inverse (~190 MB at 17^3, symmetric half).  Three launches:
// in-plane (i2, i3) transform per i1 plane, i1 transform with the eigenvalue
// division per i2 slice, inverse in-plane transform.
// ---------------------------------------------------------------------------
// sum_q a[q * sa] * b[q * sb] with four independent accumulators (short
// dependent FMA chains: these kernels are latency-bound)
__device__ __forceinline__ cd cdot_strided(const cd *a, int sa, const cd *b, int sb, int n) {
    cd c0 = mk(0, 0), c1 = mk(0, 0), c2 = mk(0, 0), c3 = mk(0, 0);
    int q = 0;
    for (; q + 4 <= n; q += 4) {
        c0 = cfma(a[q * sa], b[q * sb], c0);
        c1 = cfma(a[(q + 1) * sa], b[(q + 1) * sb], c1);
        c2 = cfma(a[(q + 2) * sa], b[(q + 2) * sb], c2);
        c3 = cfma(a[(q + 3) * sa], b[(q + 3) * sb], c3);
    }
    for (; q < n; q++) c0 = cfma(a[q * sa], b[q * sb], c0);
    return cadd(cadd(c0, c1), cadd(c2, c3));
}

#define FDM_THREADS 128
#define FDM_GROUPS 4

// in-plane transform of i1 plane blockIdx.x, rows [j0, j0 + R) of i2:
//   out[j][m] = sum_m' A3[m][m'] sum_j' A2[j][j'] in[j'][m']
template <int NTH>
__device__ __forceinline__ void fdm_plane_body(int n2, int n3, int R, const cd *__restrict__ A2,
                                               const cd *__restrict__ A3,
                                               const cd *__restrict__ in, cd *__restrict__ out,
                                               unsigned char *smem_raw, int tid, int bx, int by) {
    cd *a2 = reinterpret_cast<cd *>(smem_raw);   // R x n2 (rows j0..)
    cd *a3t = a2 + R * n2;                        // n3 x n3, transposed
    cd *P = a3t + n3 * n3;                        // n2 x n3
    cd *Q = P + n2 * n3;                          // R x n3
    const int plane = n2 * n3;
    const int j0 = by * R, rows = min(R, n2 - j0);
    if (rows <= 0) return;
    const cd *src = in + (size_t)bx * plane;
    for (int t = tid; t < plane; t += NTH) P[t] = src[t];
    for (int t = tid; t < rows * n2; t += NTH) a2[t] = __ldg(A2 + (size_t)j0 * n2 + t);
    for (int t = tid; t < n3 * n3; t += NTH) {
        int r = t / n3, c = t - r * n3;
        a3t[c * n3 + r] = __ldg(A3 + t);
    }
    __syncthreads();
    for (int t = tid; t < rows * n3; t += NTH) {   // Q = A2 P (rows j0..)
        int jr = t / n3, m = t - jr * n3;
        Q[t] = cdot_strided(a2 + jr * n2, 1, P + m, n3, n2);
    }
    __syncthreads();
    cd *dst = out + (size_t)bx * plane + (size_t)j0 * n3;
    for (int t = tid; t < rows * n3; t += NTH) {   // out = Q A3^T
        int jr = t / n3, m = t - jr * n3;
        dst[t] = cdot_strided(a3t + m, n3, Q + jr * n3, 1, n3);
    }
}

// i1 transform of slice i2 = blockIdx.x, columns [m0, m0 + C) of i3:
//   out[i][m] = sum_a V1[i][a] invD[a][m] sum_i' W1[a][i'] in[i'][m]
template <int NTH>
__device__ __forceinline__ void fdm_fiber_body(int n1, int n2, int n3, int C,
                                               const cd *__restrict__ W1,
                                               const cd *__restrict__ V1,
                                               const cd *__restrict__ invD,
                                               const cd *__restrict__ in, cd *__restrict__ out,
                                               unsigned char *smem_raw, int tid, int bx, int by) {
    cd *w = reinterpret_cast<cd *>(smem_raw), *v = w + n1 * n1;
    cd *S = v + n1 * n1, *Y = S + n1 * C;
    const int j = bx;
    const int m0 = by * C, cols = min(C, n3 - m0);
    if (cols <= 0) return;
    for (int t = tid; t < n1 * n1; t += NTH) { w[t] = __ldg(W1 + t); v[t] = __ldg(V1 + t); }
    for (int t = tid; t < n1 * cols; t += NTH) {
        int i = t / cols, mc = t - i * cols;
        S[i * C + mc] = in[((size_t)i * n2 + j) * n3 + m0 + mc];
    }
    __syncthreads();
    for (int t = tid; t < n1 * cols; t += NTH) {   // Y = diag(1/D) (W1 S)
        int a = t / cols, mc = t - a * cols;
        cd acc = cdot_strided(w + a * n1, 1, S + mc, C, n1);
        Y[a * C + mc] = cmul(acc, __ldg(invD + ((size_t)a * n2 + j) * n3 + m0 + mc));
    }
    __syncthreads();
    for (int t = tid; t < n1 * cols; t += NTH) {   // out = V1 Y
        int i = t / cols, mc = t - i * cols;
        out[((size_t)i * n2 + j) * n3 + m0 + mc] = cdot_strided(v + i * n1, 1, Y + mc, C, n1);
    }
}

__global__ void __launch_bounds__(FDM_THREADS) k_fdm_plane(int n2, int n3, int R,
                                                           const cd *__restrict__ A2,
                                                           const cd *__restrict__ A3,
                                                           const cd *__restrict__ in,
                                                           cd *__restrict__ out, const int *done) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (is_done(done)) return;
    fdm_plane_body<FDM_THREADS>(n2, n3, R, A2, A3, in, out, smem_raw, threadIdx.x, blockIdx.x,
                                blockIdx.y);
}

__global__ void __launch_bounds__(FDM_THREADS) k_fdm_fiber(int n1, int n2, int n3, int C,
                                                           const cd *__restrict__ W1,
                                                           const cd *__restrict__ V1,
                                                           const cd *__restrict__ invD,
                                                           const cd *__restrict__ in,
                                                           cd *__restrict__ out, const int *done) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (is_done(done)) return;
    fdm_fiber_body<FDM_THREADS>(n1, n2, n3, C, W1, V1, invD, in, out, smem_raw, threadIdx.x,
                                blockIdx.x, blockIdx.y);
}

__global__ void k_assemble(Lvl L, cd *__restrict__ A) {
    pdl_enter();
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
    pdl_enter();
    long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q < N) B[q * N + q] = mk(1.0, 0.0);
}

__global__ void k_zero(long long n, cd *__restrict__ y) {
    pdl_enter();
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
    const long long target = 148 * 8;     // resident 256-thread blocks on B200
    const int cmin = 4;
    int gz = (int)((target + cols - 1) / cols);
    gz = std::max(1, std::min(gz, L.nx));
    chunk = std::max((L.nx + gz - 1) / gz, L.nx >= 96 ? cmin : 2);   // short marches on coarse levels
    chunk = std::min(chunk, L.nx);
    gz = (L.nx + chunk - 1) / chunk;
    return dim3(gx, gy, gz);
}
static const dim3 kTileBlock(TILE_X, TILE_Y, 1);

template <int MODE, class Epi, int ND, bool KVAR, bool SOMM>
static void stencil_launch(const Lvl &L, const cd *src, const cd *aux, double omega, const Epi &e,
                           const RedSlot &rs, cudaStream_t s, const int *done,
                           const UpArgs &up = UpArgs{}) {
    int chunk;
    dim3 g = tile_grid(L, chunk);
    if (MODE == MODE_UP && chunk > 16) {   // the staged coarse tile covers <= 16 fine planes
        chunk = 16;
        g.z = (L.nx + chunk - 1) / chunk;
    }
    size_t smem = sizeof(StencilSmem<MODE, KVAR, Epi::kAux>);
    launch(k_stencil<MODE, Epi, ND, KVAR, SOMM>, dim3(g), dim3(kTileBlock), smem, s, L, src,
           aux ? aux : src, omega, e, chunk, rs, up, done);
}
// ---- flat-decomposition MODE_LOAD stencils (k_flat_stencil) ----
static bool use_flat(const Lvl &L) {
    return L.n3 <= FS_MAX_N3 && !opt(OPT_NO_FLAT);
}
static size_t flat_smem(const Lvl &L) { return (size_t)FS_RING * fs_slot_bytes(L.n3) + 128; }
static const size_t kFlatSmemMax = (size_t)FS_RING * ((FS_PTS + 2 * (FS_MAX_N3 + 1)) * 16 + 127) / 128 * 128 + 128;
template <int MODE, class Epi, int ND, bool KVAR, bool SOMM>
static void flat_launch_t(const Lvl &L, const cd *src, const cd *aux, double omega, const Epi &e,
                          const RedSlot &rs, cudaStream_t s, const int *done, const UpArgs &up) {
    const int gx = (int)((L.plane + FS_PTS - 1) / FS_PTS);
    const int bps = 3;
    int gz = std::max(1, std::min(L.nx, (148 * bps + gx - 1) / gx));
    const int chunk = std::max((L.nx + gz - 1) / gz, std::min(L.nx, 2));
    gz = (L.nx + chunk - 1) / chunk;
    launch(k_flat_stencil<MODE, Epi, ND, KVAR, SOMM>, dim3(gx, gz), dim3(256), flat_smem(L), s, L, src,
           aux ? aux : src, omega, e, chunk, rs, up, done);
}
template <int MODE, class Epi, int ND>
static bool flat_stencil(const Lvl &L, const cd *src, const cd *aux, double omega, const Epi &e,
                         const RedSlot &rs, cudaStream_t s, const int *done,
                         const UpArgs &up = UpArgs{}) {
    if (!use_flat(L)) return false;
    const bool somm = L.bc == HF_BC_SOMMERFELD;
    if (L.k) {
        if (somm) flat_launch_t<MODE, Epi, ND, true, true>(L, src, aux, omega, e, rs, s, done, up);
        else flat_launch_t<MODE, Epi, ND, true, false>(L, src, aux, omega, e, rs, s, done, up);
    } else {
        if (somm) flat_launch_t<MODE, Epi, ND, false, true>(L, src, aux, omega, e, rs, s, done, up);
        else flat_launch_t<MODE, Epi, ND, false, false>(L, src, aux, omega, e, rs, s, done, up);
    }
    return true;
}
template <int MODE, class Epi, int ND>
static void flat_attr() {
    const int b = (int)kFlatSmemMax;
    cudaFuncSetAttribute(k_flat_stencil<MODE, Epi, ND, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(k_flat_stencil<MODE, Epi, ND, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(k_flat_stencil<MODE, Epi, ND, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
    cudaFuncSetAttribute(k_flat_stencil<MODE, Epi, ND, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, b);
}

// kind code of the wide-plane family (hf_wide.cu) for a (MODE, epilogue) pair
template <int MODE, class Epi> struct WideKind { static constexpr int value = -1; };
template <> struct WideKind<MODE_LOAD, EpiApply<0>> { static constexpr int value = 0; };
template <> struct WideKind<MODE_LOAD, EpiApply<1>> { static constexpr int value = 1; };
template <> struct WideKind<MODE_LOAD, EpiApply<2>> { static constexpr int value = 2; };
template <> struct WideKind<MODE_LOAD, EpiResid> { static constexpr int value = 3; };
template <> struct WideKind<MODE_LOAD, EpiJacobi> { static constexpr int value = 4; };
template <> struct WideKind<MODE_PRE, EpiResid> { static constexpr int value = 5; };
template <int D> static cd *epi_out(const EpiApply<D> &e) { return e.v; }
static cd *epi_out(const EpiResid &e) { return e.r; }
static cd *epi_out(const EpiJacobi &e) { return e.u; }

template <int MODE, class Epi, int ND>
static void stencil(const Lvl &L, const cd *src, const cd *aux, double omega, const Epi &e,
                    const RedSlot &rs, cudaStream_t s, const int *done,
                    const UpArgs &up = UpArgs{}) {
    if (WideKind<MODE, Epi>::value >= 0 && wide_ok(L, WideKind<MODE, Epi>::value)) {
        launch_wide(WideKind<MODE, Epi>::value, L, src, aux, epi_out(e), omega, rs, s, done);
        return;
    }
    if ((MODE == MODE_LOAD || MODE == MODE_PRE) &&
        flat_stencil<MODE == MODE_PRE ? MODE_PRE : MODE_LOAD, Epi, ND>(L, src, aux, omega, e, rs, s, done))
        return;
    const bool somm = L.bc == HF_BC_SOMMERFELD;
    if (L.k) {
        if (somm) stencil_launch<MODE, Epi, ND, true, true>(L, src, aux, omega, e, rs, s, done, up);
        else stencil_launch<MODE, Epi, ND, true, false>(L, src, aux, omega, e, rs, s, done, up);
    } else {
        if (somm) stencil_launch<MODE, Epi, ND, false, true>(L, src, aux, omega, e, rs, s, done, up);
        else stencil_launch<MODE, Epi, ND, false, false>(L, src, aux, omega, e, rs, s, done, up);
    }
}

template <int MODE, class Epi, int ND>
static void set_attr() {
    const int a1 = (int)sizeof(StencilSmem<MODE, true, Epi::kAux>);
    const int a0 = (int)sizeof(StencilSmem<MODE, false, Epi::kAux>);
    cudaFuncSetAttribute(k_stencil<MODE, Epi, ND, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, a1);
    cudaFuncSetAttribute(k_stencil<MODE, Epi, ND, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, a1);
    cudaFuncSetAttribute(k_stencil<MODE, Epi, ND, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, a0);
    cudaFuncSetAttribute(k_stencil<MODE, Epi, ND, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, a0);
}

// opt the staged stencil kernels into > 48 KB dynamic shared memory (once, outside capture)
void init_kernel_attributes() {
    static bool done = false;
    if (done) return;

    set_attr<MODE_LOAD, EpiApply<0>, 0>();
    set_attr<MODE_LOAD, EpiApply<1>, 1>();
    set_attr<MODE_LOAD, EpiApply<2>, 2>();
    set_attr<MODE_LOAD, EpiResid, 0>();
    set_attr<MODE_LOAD, EpiJacobi, 0>();
    set_attr<MODE_PRE, EpiResid, 0>();
    set_attr<MODE_UP, EpiJacobi, 0>();
    flat_attr<MODE_LOAD, EpiApply<0>, 0>();
    flat_attr<MODE_LOAD, EpiApply<1>, 1>();
    flat_attr<MODE_LOAD, EpiApply<2>, 2>();
    flat_attr<MODE_LOAD, EpiResid, 0>();
    flat_attr<MODE_LOAD, EpiJacobi, 0>();
    flat_attr<MODE_PRE, EpiResid, 0>();
    flat_attr<MODE_UP, EpiJacobi, 0>();
    {
        const int b2 = DR2_RING * dr2_slot_elems(DR2_MAX_N3) * 16 + 2 * (2 * DR2_CR + 1) * DR2_MAX_N3 * 16 + 128;
        cudaFuncSetAttribute(k_flat_dr<true, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
        cudaFuncSetAttribute(k_flat_dr<true, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
        cudaFuncSetAttribute(k_flat_dr<false, true, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
        cudaFuncSetAttribute(k_flat_dr<false, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
        cudaFuncSetAttribute(k_flat_dr<true, true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
        cudaFuncSetAttribute(k_flat_dr<true, false, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
        cudaFuncSetAttribute(k_flat_dr<false, true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
        cudaFuncSetAttribute(k_flat_dr<false, false, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, b2);
    }
    cudaFuncSetAttribute(k_down_restrict<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DRSmem<true>));
    cudaFuncSetAttribute(k_down_restrict<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DRSmem<true>));
    cudaFuncSetAttribute(k_down_restrict<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DRSmem<false>));
    cudaFuncSetAttribute(k_down_restrict<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(DRSmem<false>));
    cudaFuncSetAttribute(k_fdm_plane, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_fdm_fiber, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    done = true;
}

int tile_blocks(const Lvl &L) {
    int chunk;
    dim3 g = tile_grid(L, chunk);
    const int gx = (int)((L.plane + FS_PTS - 1) / FS_PTS);   // k_flat_stencil grid (flat_launch_t)
    return std::max<int>(std::max<int>(g.x * g.y * g.z, gx * L.nx), wide_blocks(L));
}

void launch_apply(const Lvl &L, const cd *u, cd *v, cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiApply<0>, 0>(L, u, nullptr, 0.0, EpiApply<0>{v}, RedSlot{}, s, done);
}
void launch_apply_dot1(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiApply<1>, 1>(L, u, w, 0.0, EpiApply<1>{v}, rs, s, done);
}
void launch_apply_dot2(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiApply<2>, 2>(L, u, w, 0.0, EpiApply<2>{v}, rs, s, done);
}
void launch_residual(const Lvl &L, const cd *u, const cd *b, cd *r, cudaStream_t s,
                     const int *done) {
    stencil<MODE_LOAD, EpiResid, 0>(L, u, b, 0.0, EpiResid{r}, RedSlot{}, s, done);
}
void launch_jacobi(const Lvl &L, const cd *u, const cd *b, cd *uo, double omega,
                   cudaStream_t s, const int *done) {
    stencil<MODE_LOAD, EpiJacobi, 0>(L, u, b, omega, EpiJacobi{uo}, RedSlot{}, s, done);
}
void launch_down1(const Lvl &L, const cd *b, cd *r, double omega, cudaStream_t s,
                  const int *done) {
    stencil<MODE_PRE, EpiResid, 0>(L, b, b, omega, EpiResid{r}, RedSlot{}, s, done);
}
static void corr(int mode, const Lvl &F, const Lvl &C, const cd *b, const cd *e, cd *out,
                 double omega, cudaStream_t s, const int *done, bool ghosts = false) {
    // tiled variant: two fine planes per thread (every load of the pair independent)
    const int chunk = 2;
    if (ghosts || !opt(OPT_NO_FLAT)) {   // flat thread mapping (no ragged tiles)
        // four fine planes per thread (coarse-plane sums reused between them)
        const int chunk = 4;
        const int plo = ghosts && F.lo1 > 0 ? -1 : 0;
        const int phi = ghosts && F.lo1 + F.nx < F.n1 ? F.nx + 1 : F.nx;
        dim3 gf((unsigned)((F.plane + 255) / 256), (phi - plo + chunk - 1) / chunk);
        if (mode == 0) launch(k_corr_flat<0>, gf, dim3(256), 0, s, F, C, b, e, out, omega, chunk, plo, phi, done);
        else if (mode == 1) launch(k_corr_flat<1>, gf, dim3(256), 0, s, F, C, b, e, out, omega, chunk, plo, phi, done);
        else launch(k_corr_flat<2>, gf, dim3(256), 0, s, F, C, b, e, out, omega, chunk, plo, phi, done);
        return;
    }
    dim3 g((F.n3 + 31) / 32, (F.n2 + 7) / 8, (F.nx + chunk - 1) / chunk);
    if (mode == 0) launch(k_corr<0>, dim3(g), dim3(256), 0, s, F, C, b, e, out, omega, chunk, done);
    else if (mode == 1) launch(k_corr<1>, dim3(g), dim3(256), 0, s, F, C, b, e, out, omega, chunk, done);
    else launch(k_corr<2>, dim3(g), dim3(256), 0, s, F, C, b, e, out, omega, chunk, done);
}
void launch_jacobi0(const Lvl &L, const cd *b, cd *u, double omega, cudaStream_t s,
                    const int *done) {
    int chunk;
    dim3 g = march_grid(L, chunk);
    launch(k_jacobi0, dim3(g), dim3(kMarchBlock), 0, s, L, b, u, omega, chunk, done);
}
void launch_palette(const Lvl &L, int np, cd *apal, cd *dpal, cudaStream_t s) {
    launch(k_palette, dim3((4 * np + 127) / 128), dim3(128), 0, s, L, np, apal, dpal);
}
void launch_dinv(const Lvl &L, cd *out_owned, cudaStream_t s) {
    int g0 = std::max(-HF_GHOST, -L.lo1), g1 = std::min(L.nx + HF_GHOST, L.n1 - L.lo1);
    launch(k_dinv, dim3(592), dim3(256), 0, s, L, g0, g1, out_owned);
}
void launch_restrict(const Lvl &F, const Lvl &C, const cd *r, cd *out, cudaStream_t s,
                     const int *done) {
    if (!opt(OPT_NO_FLAT)) {
        // ~20 blocks per SM in total (5 resident at 48 registers): a few full
        // waves of short marches instead of 1.4 waves of long ones
        const int gx = (int)((C.plane + 255) / 256);
        int gz = std::max(1, std::min(C.nx, (148 * 20) / gx));
        const int chunk = (C.nx + gz - 1) / gz;
        gz = (C.nx + chunk - 1) / chunk;
        launch(k_restrict_flat, dim3(gx, gz), dim3(256), 0, s, F, C, r, out, chunk, done);
        return;
    }
    int gx = (C.n3 + RC_X - 1) / RC_X, gy = (C.n2 + RC_Y - 1) / RC_Y;
    long long cols = (long long)gx * gy;
    int gz = (int)std::max<long long>(1, std::min<long long>(C.nx, (148 * 6 + cols - 1) / cols));
    int chunk = std::max(2, (C.nx + gz - 1) / gz);
    gz = (C.nx + chunk - 1) / chunk;
    launch(k_restrict2, dim3(dim3(gx, gy, gz)), dim3(256), 0, s, F, C, r, out, chunk, done);
}
template <bool KVAR, bool SOMM>
static void dr_launch(const Lvl &F, const Lvl &C, const cd *b, cd *out, double omega, cudaStream_t s,
                      const int *done) {
    const int gx = (C.n3 + DR_CX - 1) / DR_CX, gy = (C.n2 + DR_CY - 1) / DR_CY;
    const long long cols = (long long)gx * gy;
    int gz = (int)std::max<long long>(1, std::min<long long>(C.nx, (148 * 4 + cols - 1) / cols));
    const int chunk = (C.nx + gz - 1) / gz;
    gz = (C.nx + chunk - 1) / chunk;
    launch(k_down_restrict<KVAR, SOMM>, dim3(gx, gy, gz), dim3(DR_NT), sizeof(DRSmem<KVAR>), s, F, C,
           b, out, omega, chunk, done);
}
template <bool KVAR, bool SOMM, int RPT>
static void dr2_launch(const Lvl &F, const Lvl &C, const cd *b, cd *out, double omega, cudaStream_t s,
                       const int *done) {
    const int gx = (C.n2 + DR2_CR - 1) / DR2_CR;
    const int target = 148 * 2;
    int gz = std::max(1, std::min(C.nx, (target + gx - 1) / gx));
    const int chunk = (C.nx + gz - 1) / gz;
    gz = (C.nx + chunk - 1) / chunk;
    const size_t smem = (size_t)DR2_RING * dr2_slot_elems(F.n3) * 16 + (size_t)2 * (2 * DR2_CR + 1) * F.n3 * 16 + 128;
    launch(k_flat_dr<KVAR, SOMM, RPT>, dim3(gx, gz), dim3(DR2_NT), smem, s, F, C, b, out, omega, chunk, done);
}
bool flat_dr_ok(const Lvl &F) {
    return F.n3 <= DR2_MAX_N3 && !opt(OPT_NO_FLAT_DR);
}
void launch_down_restrict(const Lvl &F, const Lvl &C, const cd *b, cd *out, double omega,
                          cudaStream_t s, const int *done) {
    const bool somm = F.bc == HF_BC_SOMMERFELD;
    if (flat_dr_ok(F)) {
        // residual points per thread: (2 CR + 1) n3 / 256 -> 3 up to n3 = 153, else 5
        const bool r3 = (2 * DR2_CR + 1) * F.n3 <= 3 * DR2_NT;
        if (F.k) {
            if (somm) r3 ? dr2_launch<true, true, 3>(F, C, b, out, omega, s, done)
                         : dr2_launch<true, true, 5>(F, C, b, out, omega, s, done);
            else r3 ? dr2_launch<true, false, 3>(F, C, b, out, omega, s, done)
                    : dr2_launch<true, false, 5>(F, C, b, out, omega, s, done);
        } else {
            if (somm) r3 ? dr2_launch<false, true, 3>(F, C, b, out, omega, s, done)
                         : dr2_launch<false, true, 5>(F, C, b, out, omega, s, done);
            else r3 ? dr2_launch<false, false, 3>(F, C, b, out, omega, s, done)
                    : dr2_launch<false, false, 5>(F, C, b, out, omega, s, done);
        }
        return;
    }
    if (F.k) {
        if (somm) dr_launch<true, true>(F, C, b, out, omega, s, done);
        else dr_launch<true, false>(F, C, b, out, omega, s, done);
    } else {
        if (somm) dr_launch<false, true>(F, C, b, out, omega, s, done);
        else dr_launch<false, false>(F, C, b, out, omega, s, done);
    }
}
void launch_prolong(const Lvl &F, const Lvl &C, const cd *e, cd *out, bool add, cudaStream_t s,
                    const int *done) {
    corr(add ? 2 : 0, F, C, nullptr, e, out, 0.0, s, done);
}
// u = u1 + w D^-1 (b - M u1), u1 = [w D^-1 b] + P e: pointwise correction into
// the scratch field t, then one Jacobi sweep stencil (multigrid.py:337-343)
void launch_correct(const Lvl &L, const Lvl &C, const cd *b, const cd *e, cd *t, double omega,
                    bool pre, cudaStream_t s, const int *done, bool ghosts) {
    corr(pre ? 1 : 0, L, C, b, e, t, omega, s, done, ghosts);
}
int launch_up1(const Lvl &L, const Lvl &C, const cd *b, const cd *e, cd *u, cd *t, double omega,
               bool pre, cudaStream_t s, const int *done) {
    // whole-grid levels: correction produced inside the post-smoothing sweep
    // flat fused up-sweep: opt-in (HF_FLAT_UP=1); the per-entry prolongation in the
    // slot made it slower than k_corr_flat + the flat Jacobi sweep on every level
    if (!opt(OPT_NO_FUSE) && opt(OPT_FLAT_UP) && L.n3 <= FS_MAX_N3 &&
        flat_stencil<MODE_UP, EpiJacobi, 0>(L, b, b, omega, EpiJacobi{u}, RedSlot{}, s, done,
                                            UpArgs{C, e, pre ? 1 : 0}))
        return 1;
    // (the split pair is faster than the tiled fused kernel where the flat Jacobi applies)
    // correction + Jacobi sweep as the split pair unless fuse_up is requested: the
    // tiled MODE_UP kernel measured slower than k_corr_flat + the sweep on the wide
    // 513^3 wedge levels too (3.40 vs 1.07 + 1.63 ms, profiles/r02_kernel_table_513w.json)
    // wide whole-grid levels: the wide family's fused up-sweep (hf_wide.cu)
    if (!opt(OPT_NO_FUSE) && !opt(OPT_NO_WIDE_UP) && !opt(OPT_FUSE_UP) && wide_ok(L, 6) && L.lo1 == 0 &&
        L.nx == L.n1 && C.lo1 == 0 && C.nx == C.n1) {
        launch_wide_up(L, C, b, e, u, omega, pre, s, done);
        return 1;
    }
    const bool split = opt(OPT_NO_FUSE) || !opt(OPT_FUSE_UP);
    if (!split && L.lo1 == 0 && L.nx == L.n1 && C.lo1 == 0 && C.nx == C.n1) {
        stencil<MODE_UP, EpiJacobi, 0>(L, b, b, omega, EpiJacobi{u}, RedSlot{}, s, done,
                                        UpArgs{C, e, pre ? 1 : 0});
        return 1;
    }
    corr(pre ? 1 : 0, L, C, b, e, t, omega, s, done);
    stencil<MODE_LOAD, EpiJacobi, 0>(L, t, b, omega, EpiJacobi{u}, RedSlot{}, s, done);
    return 2;
}
void launch_gemv(int N, const cd *Minv, const cd *b, cd *x, cudaStream_t s, const int *done) {
    int blocks = (N + 1) / 2;
    launch(k_gemv, dim3(blocks), dim3(64), 0, s, N, Minv, b, x, done);
}
void launch_sym_pack(int N, const cd *Minv, const double *sv, cd *tiles, cudaStream_t s) {
    int nT = (N + SYT - 1) / SYT;
    launch(k_sym_pack, dim3(2048), dim3(256), 0, s, N, nT, Minv, sv, tiles);
}
void launch_symv(int N, const cd *tiles, const double *sv, const cd *b, cd *prow, cd *pcol, cd *x,
                 cudaStream_t s, const int *done) {
    int nT = (N + SYT - 1) / SYT;
    long long ntile = (long long)nT * (nT + 1) / 2;
    launch(k_sym_tiles, dim3((unsigned)ntile), dim3(256), 0, s, N, nT, tiles, sv, b, prow, pcol, done);
    launch(k_sym_reduce, dim3((N * 32 + 255) / 256), dim3(256), 0, s, N, nT, prow, pcol, x, done);
}
long long sym_tiles_count(int N) {
    long long nT = (N + SYT - 1) / SYT;
    return nT * (nT + 1) / 2;
}
void launch_assemble(const Lvl &L, cd *A, cudaStream_t s) {
    long long N = (long long)L.n1 * L.plane;
    launch(k_assemble, dim3((unsigned)((N + 255) / 256)), dim3(256), 0, s, L, A);
}
static void fdm_split(int n1, int n2, int n3, int &R, int &C, size_t &sp, size_t &sf) {
    R = (n2 + FDM_GROUPS - 1) / FDM_GROUPS;
    C = (n3 + FDM_GROUPS - 1) / FDM_GROUPS;
    sp = ((size_t)R * n2 + (size_t)n3 * n3 + (size_t)n2 * n3 + (size_t)R * n3) * sizeof(cd);
    sf = (2ull * n1 * n1 + 2ull * n1 * C) * sizeof(cd);
}
void fdm_groups(int n1, int n2, int n3, int &R, int &C) {
    size_t sp, sf;
    fdm_split(n1, n2, n3, R, C, sp, sf);
}
size_t fdm_smem_bytes(int n1, int n2, int n3) {
    int R, C;
    size_t sp, sf;
    fdm_split(n1, n2, n3, R, C, sp, sf);
    return std::max(sp, sf);
}
// fdm = [V1^-1, V2^-1, V3^-1, V1, V2, V3] (row-major n_d x n_d each), tmp = 2N
// returns the number of kernels launched (3)
int launch_fdm(int n1, int n2, int n3, const cd *fdm, const cd *invD, const cd *b, cd *tmp,
               cd *x, cudaStream_t s, const int *done) {
    const cd *W1 = fdm, *W2 = W1 + n1 * n1, *W3 = W2 + n2 * n2;
    const cd *V1 = W3 + n3 * n3, *V2 = V1 + n1 * n1, *V3 = V2 + n2 * n2;
    int R, C;
    size_t sp, sf;
    fdm_split(n1, n2, n3, R, C, sp, sf);
    cd *t0 = tmp, *t1 = tmp + (size_t)n1 * n2 * n3;
    dim3 gp(n1, (n2 + R - 1) / R), gf(n2, (n3 + C - 1) / C);
    launch(k_fdm_plane, gp, dim3(FDM_THREADS), sp, s, n2, n3, R, W2, W3, b, t0, done);
    launch(k_fdm_fiber, gf, dim3(FDM_THREADS), sf, s, n1, n2, n3, C, W1, V1, invD,
           (const cd *)t0, t1, done);
    launch(k_fdm_plane, gp, dim3(FDM_THREADS), sp, s, n2, n3, R, V2, V3, (const cd *)t1, x, done);
    return 3;
}
void launch_set_identity(long long N, cd *B, cudaStream_t s) {
    launch(k_set_identity, dim3((unsigned)((N + 255) / 256)), dim3(256), 0, s, N, B);
}
void launch_zero(long long n, cd *y, cudaStream_t s) {
    launch(k_zero, dim3(VEC_BLOCKS), dim3(256), 0, s, n, y);
}
void launch_axpby(long long n, cd a, const cd *x, cd b, cd *y, cudaStream_t s) {
    launch(k_axpby, dim3(VEC_BLOCKS), dim3(256), 0, s, n, a, x, b, y);
}
void launch_mgs(long long n, cd *w, const cd *c, const cd *vprev, const cd *vcur,
                const RedSlot &rs, cudaStream_t s) {
    launch(k_mgs, dim3(VEC_BLOCKS), dim3(256), 0, s, n, w, c, vprev, vcur, rs);
}
void launch_multi_axpy(long long n, int m, const cd *const *V, const cd *y, cd *x, cudaStream_t s) {
    launch(k_multi_axpy, dim3(VEC_BLOCKS), dim3(256), 0, s, n, m, V, y, x);
}
void launch_dot(long long n, const cd *a, const cd *b, const RedSlot &rs, cudaStream_t s) {
    launch(k_dot_store, dim3(VEC_BLOCKS), dim3(256), 0, s, n, a, b, rs);
}
void launch_bcg_init(long long n, const cd *b, cd *r, cd *rs, cd *x, cd *p, cd *v,
                     const RedSlot &red, cudaStream_t s, int shadow, unsigned long long seed,
                     long long q0) {
    launch(k_bcg_init, dim3(VEC_BLOCKS), dim3(256), 0, s, n, b, r, rs, x, p, v, red, shadow, seed, q0);
}
void launch_bcg_p(long long n, const BcgState *st, const cd *r, cd *p, const cd *v,
                  cudaStream_t s, const int *done) {
    launch(k_bcg_p, dim3(VEC_BLOCKS), dim3(256), 0, s, n, st, r, p, v, done);
}
void launch_bcg_s(long long n, const BcgState *st, const cd *r, const cd *v, cd *sv,
                  const RedSlot &red, cudaStream_t s, const int *done) {
    launch(k_bcg_s, dim3(VEC_BLOCKS), dim3(256), 0, s, n, st, r, v, sv, red, done);
}
void launch_bcg_xr(long long n, const BcgState *st, cd *x, const cd *ph, const cd *sh,
                   const cd *sv, const cd *t, cd *r, const cd *rs, const RedSlot &red,
                   cudaStream_t s, const int *done) {
    launch(k_bcg_xr, dim3(VEC_BLOCKS), dim3(256), 0, s, n, st, x, ph, sh, sv, t, r, rs, red, done);
}
void launch_nz_scan(long long n, const cd *rs, BcgState *st, cudaStream_t s) {
    launch(k_nz_scan, dim3(VEC_BLOCKS), dim3(256), 0, s, n, rs, st);
    launch(k_nz_finish, dim3(1), dim3(32), 0, s, rs, st);
}
void launch_gather_store(const BcgState *nz, const cd *g, cd *out, cudaStream_t s, const int *done) {
    launch(k_gather_store, dim3(1), dim3(32), 0, s, nz, g, out, done);
}
void launch_bcg_gather(BcgState *st, int op, const cd *g, cudaStream_t s, const int *done) {
    launch(k_bcg_gather, dim3(1), dim3(32), 0, s, st, op, g, done);
}
void launch_bcg_step(BcgState *st, int op, const cd *sums, cudaStream_t s) {
    launch(k_bcg_step, dim3(1), dim3(32), 0, s, st, op, sums);
}
void launch_bcg_xhalf(long long n, const BcgState *st, cd *x, const cd *ph, cudaStream_t s) {
    launch(k_bcg_xhalf, dim3(VEC_BLOCKS), dim3(256), 0, s, n, st, x, ph);
}

}  // namespace hf
