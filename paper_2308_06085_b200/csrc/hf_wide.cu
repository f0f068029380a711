// hf_wide.cu -- stencil sweeps on WIDE planes (n3 > 256: the 513^3 / 1025^2
// finest levels), sm_100a.
//
// A block owns a 32 x (NCW P) tile of (i3, i2) columns and marches along i1.  It
// is warp-specialised: NCW CONSUMER warps compute (8 for the plain sweeps, 7 for
// the in-slot transform modes: two 8-warp blocks put 4 warps on every SM
// sub-partition, 128 registers without spills), one PRODUCER warp feeds a ring
// of 4 plane slots with cp.async.bulk copies, and the warps are synchronised
// only through mbarriers -- there is no block-wide barrier on the march, so the
// consumer warps drift apart by up to the ring depth and hide each other's
// latencies:
//   full[k]   the producer's copies of a plane have landed (expect_tx)
//   empty[k]  all consumer warps are done reading the slot
//   xf[k]     (transform modes) all consumer warps have transformed their
//             entries of the plane in the slot
// P = 2 rows per thread by default; 1 / 3 / 4 rows and a 15-consumer-warp block
// are kept as options (all measured slower).
// A consumer thread owns P consecutive i2 rows of one i3 column:
//   * the x neighbours rotate through registers along the march (three named
//     register sets, the march unrolled by three: no moves),
//   * the y neighbours inside the thread's own rows are registers too,
//   * per plane a thread reads P (next plane's centres) + 2 (rows above and
//     below its strip) + 2P (z neighbours) shared values for P points --
//     (3P + 2) / P instead of 7 per point.
// A slot holds the tile + one-vertex halo of the stencil operand (one bulk
// copy per tile row, 34 contiguous entries) and, for epilogues with a
// centre-only operand (b, or the inner-product partner w), the tile of that
// operand (one copy per row), so the consumers issue no global loads except
// the wavenumber / palette index of their own points, one plane ahead.  A halo
// row or column one step outside the grid holds the MIRRORED inward row /
// column (operators.py:9-12: Sommerfeld ghost elimination; Dirichlet rows are
// identities and never use them), copied from the mirrored address, so the
// 7-point row is uniform.
//
// Three stencil inputs (same arithmetic as k_stencil / k_flat_stencil):
//   WIDE_LOAD  f = src            (A u with inner products, b - M u, Jacobi sweep)
//   WIDE_PRE   f = D^-1 b: zero-guess pre-smoothing folded into the residual,
//              r = b - M (w D^-1 b) (multigrid.py:148-151 + 383-386).  A thread
//              turns its own centre entries of plane i+1 into D^-1 b in place,
//              keeping b and D^-1 b in registers (its epilogue operand and x+
//              neighbour); threads 0..NHE-1 also one entry each of the ring
//              around the tile's active region.
//   WIDE_UP    f = t = [w D^-1 b] + P e: the coarse-grid correction
//              (prolong_tl + _correct, multigrid.py:238-297, 389-392) produced in
//              the slot like WIDE_PRE's D^-1 b, the k_corr arithmetic at the
//              (mirrored) coordinates of every entry; the coarse tile of e the
//              block's fine planes interpolate from is staged plane by plane, each
//              on its own barrier, and the in-plane sums of a coarse plane are
//              carried in registers over the three fine planes they serve.
//              Epilogue: the post-smoothing Jacobi sweep u = t + w D^-1 (b - M t).
//              The correction t never goes to memory (-32 B per vertex against
//              the split k_corr_flat + Jacobi pair).
// Wavenumber: constant (tables by face count), a float64 field, or the 8-bit
// palette indices of a layered medium (a_p / D^-1 tables per index).
#include <algorithm>

#include "hf_stencil.cuh"

namespace hf {

enum { WIDE_LOAD = 0, WIDE_PRE = 1, WIDE_UP = 2 };
enum { WE_APPLY0 = 0, WE_APPLY1, WE_APPLY2, WE_RESID, WE_JACOBI };
enum { KV_CONST = 0, KV_FIELD = 1, KV_PAL = 2 };

constexpr int WX = 32;            // tile width (i3): one warp row
constexpr int WRS = WX + 2;       // staged entries per tile row
// consumer warps of a block: 8 for the plain sweeps (9 warps, 3 blocks per SM at 72
// registers); 7 for the in-slot transform modes -- registers are allocated per SM
// sub-partition (16 K each), two 8-warp blocks put 4 warps on each (128 registers, no
// spills), two 9-warp blocks up to 5 (96)
// (strips of 3 / 4 rows, options wide_p3 / wide_p4: 5 / 4 consumer warps for the transform
// modes -- fewer, fatter warps, the per-plane barrier traffic paid once per 3 / 4 points)
// P >= 10 encodes the BIG block of the transform modes: P - 10 rows per thread, 15 consumer
// warps + the producer in one 512-thread block per SM (16 warps: 4 per sub-partition, 128
// registers; a 32 x 30 tile: 1.13 instead of 1.21 staged entries per point)
__host__ __device__ constexpr int wide_rows(int P) { return P >= 10 ? P - 10 : P; }
__host__ __device__ constexpr int wide_ncw(int mode, int P = 2) {
    return P >= 10 ? 15 : (mode == 0 || P == 1 ? 8 : (P == 2 ? 7 : (P == 3 ? 5 : 4)));
}
constexpr int WRING = 4;
constexpr int WPAL = 16;          // palette entries held in shared memory (else the k field is used)
// fine planes per block of the fused up-sweep / coarse planes staged per block
__host__ __device__ constexpr int wup_chunk(int P) { return P == 2 || P >= 10 ? 48 : 40; }
__host__ __device__ constexpr int wup_cpl(int P) { return wup_chunk(P) / 2 + 2; }
constexpr int WCW = WX / 2 + 2;   // coarse tile row length
static_assert((WRING & (WRING - 1)) == 0, "ring size is a power of two");

struct WideUp {          // WIDE_UP: the coarse level and its correction
    Lvl C;
    const cd *e;         // coarse correction (owned plane 0)
    int pre;             // 1: t = w D^-1 b + P e (nu1 = 1), 0: t = P e (nu1 = 0)
};

template <int P, bool AUX, bool UP = false, int NCW = 8>
struct WideTile {
    static constexpr int WY = NCW * wide_rows(P); // tile height (i2)
    static constexpr int ROWS = WY + 2;
    static constexpr int ENT = ROWS * WRS;        // stencil operand entries of a slot
    static constexpr int AENT = AUX ? WY * WX : 0;   // centre-only operand entries
    static constexpr int SLOT = ENT + AENT;
    static constexpr int NHE = 2 * WRS + 2 * WY;  // entries of the ring around the tile
    static constexpr int CH = (WY + 1) / 2 + 2;   // coarse tile rows (tiles may start on odd rows)
    static constexpr int CENT = UP ? wup_cpl(P) * CH * WCW : 0;   // staged coarse tile
    static constexpr size_t smem = (size_t)(WRING * SLOT + CENT) * sizeof(cd) + 128;
};

__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}

template <int P>
struct WidePlane {       // register set of one plane of a thread's strip
    cd f[P];             // staged operand at the thread's P points
};

template <int MODE, int EPI, int KV, bool SOMM, int PP>
// registers are allocated per SM sub-partition (16 K each): 3 blocks of 9 warps put up to
// 7 warps on one (72 registers), 2 blocks up to 5 (96) -- the in-slot transform modes and
// the 4-row strips take 2 blocks
__global__ void __launch_bounds__(32 * (wide_ncw(MODE, PP) + 1),
                                  (PP >= 10 ? 1 : (PP >= 4 || (MODE != WIDE_LOAD && PP > 1) || (MODE == WIDE_UP) ? 2 : 3)))
k_wide(Lvl L, const cd *__restrict__ src, const cd *__restrict__ aux, cd *__restrict__ out,
       double omega, int chunk, RedSlot rs, WideUp up, const int *done) {
    constexpr bool kAux = EPI != WE_APPLY0 && MODE == WIDE_LOAD;   // staged centre-only operand
    constexpr bool kXf = MODE != WIDE_LOAD;                        // entries transformed in the slot
    constexpr int P = wide_rows(PP);
    constexpr int NCW = wide_ncw(MODE, PP), WNC = 32 * NCW, WUP_CPL = wup_cpl(PP);
    using T = WideTile<PP, kAux, MODE == WIDE_UP, NCW>;
    constexpr int ND = EPI == WE_APPLY1 ? 1 : (EPI == WE_APPLY2 ? 2 : 0);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ __align__(8) unsigned long long bars[3 * WRING + (MODE == WIDE_UP ? WUP_CPL : 0)];
    __shared__ cd tab[12];
    // palette: a_p and w D^-1 per (index, face count)
    __shared__ cd pal_a[KV == KV_PAL ? 4 * WPAL : 1], pal_d[KV == KV_PAL ? 4 * WPAL : 1];
    if (is_done(done)) return;
    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * WX, j0 = blockIdx.y * T::WY;
    const int i0 = blockIdx.z * chunk, i1 = min(i0 + chunk, L.nx);
    const int n1 = L.n1, n2 = L.n2, n3 = L.n3;
    const long long plane = L.plane;
    const unsigned sraw = smem_u32(smem_raw);
    const unsigned sbase = (sraw + 127u) & ~127u;
    const unsigned b_full = smem_u32(bars), b_empty = b_full + 8 * WRING, b_xf = b_full + 16 * WRING;
    const unsigned b_coarse = b_full + 24 * WRING;     // WIDE_UP: one barrier per staged coarse plane
    cd *const sgen = reinterpret_cast<cd *>(smem_raw + (sbase - sraw));
    auto gmirror = [&](int g) { return g < 0 ? -g : (g >= n1 ? 2 * (n1 - 1) - g : g); };

    if (tid == 0) {
        for (int k = 0; k < WRING; k++) {
            mbar_init(b_full + 8 * k, 1);
            mbar_init(b_empty + 8 * k, WNC / 32);
            mbar_init(b_xf + 8 * k, WNC / 32);
        }
        if (MODE == WIDE_UP)
            for (int k = 0; k < WUP_CPL; k++) mbar_init(b_coarse + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (KV == KV_CONST && tid < 4) {
        tab[tid] = __ldg(L.tab + tid);                                   // a_p(nb)
        tab[4 + tid] = cscal(__ldg(L.tab + 4 + tid), omega);             // w D^-1(nb)
        tab[8 + tid] = cdiv(__ldg(L.tab + 4 + tid), __ldg(L.tab + 4));   // D^-1(nb) / D^-1(0)
    }
    if (KV == KV_PAL && tid < 4 * L.npal) {
        pal_a[tid] = __ldg(L.apal + tid);
        pal_d[tid] = cscal(__ldg(L.dpal + tid), omega);
    }
    __syncthreads();

    const int c_lo = max(m0 - 1, 0), c_hi = min(m0 + WX, n3 - 1);        // staged columns
    const bool mir_l = m0 == 0 && n3 > 1;              // column -1 holds column 1
    const bool mir_r = n3 <= m0 + WX && n3 > 1;        // column n3 holds column n3 - 2
    const int row_lo = max(j0 - 1, -1), row_hi = min(j0 + T::WY, n2);   // staged rows
    const int ar = min(T::WY, n2 - j0), ac = min(WX, n3 - m0);           // active region
    const int last = min(i1, n1 - L.lo1);              // last local plane staged
    cd acc[2] = {mk(0, 0), mk(0, 0)};
    // WIDE_UP: coarse tile [cp_lo, cp_lo + ncp) x [cj_lo, cj_lo + nch) x [cm_lo, cm_lo + ncw)
    // covering every coarse vertex the block's (mirrored) fine entries interpolate from
    int cp_lo = 0, cj_lo = 0, cm_lo = 0, ncp = 0, nch = 0, ncw = 0;
    if (MODE == WIDE_UP) {
        const Lvl &C = up.C;
        const int gmin = min(gmirror(L.lo1 + i0 - 1), gmirror(L.lo1 + i0));
        const int gmax = max(gmirror(L.lo1 + i1), gmirror(L.lo1 + i1 - 1));
        cp_lo = gmin >> 1;
        ncp = min(C.n1 - 1, (gmax + 1) >> 1) - cp_lo + 1;
        cj_lo = max(0, j0 - 1) >> 1;
        nch = min(C.n2 - 1, (min(j0 + T::WY, n2 - 1) + 1) >> 1) - cj_lo + 1;
        cm_lo = max(0, m0 - 1) >> 1;
        ncw = min(C.n3 - 1, (min(m0 + WX, n3 - 1) + 1) >> 1) - cm_lo + 1;
    }
    cd *const ctile = sgen + WRING * T::SLOT;

    if (tid >= WNC) {
        // ------------------------------------------------------------------
        // producer warp: lane l copies tile rows l and l + 32 (and row l of the
        // centre-only operand) of every plane i0-1 .. last into the ring
        // ------------------------------------------------------------------
        const int lane = tid - WNC;
        const int ncol = c_hi - c_lo + 1;
        const unsigned src_bytes = (unsigned)(row_hi - row_lo + 1) *
                                   (unsigned)(ncol + (int)mir_l + (int)mir_r) * 16u;
        const unsigned aux_bytes = kAux ? (unsigned)(ar * ac) * 16u : 0u;
        int goff[2];
        bool ok[2];
#pragma unroll
        for (int t = 0; t < 2; t++) {
            const int row = lane + 32 * t;
            const int jj = j0 - 1 + row;
            ok[t] = row < T::ROWS && jj >= row_lo && jj <= row_hi;
            const int jm = jj < 0 ? -jj : (jj >= n2 ? 2 * (n2 - 1) - jj : jj);
            goff[t] = ok[t] ? jm * n3 : 0;
        }
        const bool aok = kAux && lane < ar;
        const int agoff = aok ? (j0 + lane) * n3 + m0 : 0;
        // WIDE_UP: coarse plane pl of the tile (lane r copies its row r), each on its own
        // barrier, issued a few planes ahead of the fine planes that interpolate from it
        int cp_issued = 0;
        auto issue_coarse = [&](int upto) {
            const Lvl &C = up.C;
            for (; cp_issued <= upto && cp_issued < ncp; cp_issued++) {
                const unsigned bar = b_coarse + 8 * cp_issued;
                if (lane == 0) mbar_expect_tx(bar, (unsigned)(nch * ncw) * 16u);
                __syncwarp();
                if (lane < nch)
                    bulk_g2s(sbase + (unsigned)(WRING * T::SLOT + (cp_issued * T::CH + lane) * WCW) * 16u,
                             up.e + (long long)(cp_lo + cp_issued - C.lo1) * C.plane +
                                 (long long)(cj_lo + lane) * C.n3 + cm_lo,
                             (unsigned)ncw * 16u, bar);
            }
        };
        for (int p = i0 - 1, d = 0; p <= last; p++, d++) {
            const int k = d & (WRING - 1);
            if (MODE == WIDE_UP) issue_coarse(((gmirror(L.lo1 + p) >> 1) - cp_lo) + 3);
            if (d >= WRING) mbar_wait(b_empty + 8 * k, ((d / WRING) - 1) & 1);
            // (the pre-smoothing sweep rewrote the slot through the generic proxy)
            if (kXf) asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const unsigned bar = b_full + 8 * k;
            // the centre-only operand exists on owned planes (the end planes of the
            // march may be mirrored / ghost planes: their tile is never read)
            const bool owned = p >= i0 && p < i1;
            if (lane == 0) mbar_expect_tx(bar, src_bytes + (owned ? aux_bytes : 0u));
            __syncwarp();
            const long long pb = (long long)(gmirror(L.lo1 + p) - L.lo1) * plane;
            const unsigned slot_s = sbase + (unsigned)(k * T::SLOT) * 16u;
#pragma unroll
            for (int t = 0; t < 2; t++) {
                if (!ok[t]) continue;
                const cd *g = src + pb + goff[t];
                const unsigned dst = slot_s + (unsigned)((lane + 32 * t) * WRS) * 16u;
                bulk_g2s(dst + (unsigned)(c_lo - (m0 - 1)) * 16u, g + c_lo, (unsigned)ncol * 16u, bar);
                if (mir_l) bulk_g2s(dst, g + 1, 16u, bar);
                if (mir_r) bulk_g2s(dst + (unsigned)(n3 - (m0 - 1)) * 16u, g + (n3 - 2), 16u, bar);
            }
            if (aok && owned)
                bulk_g2s(slot_s + (unsigned)(T::ENT + lane * WX) * 16u,
                         aux + (long long)p * plane + agoff, (unsigned)ac * 16u, bar);
        }
    } else {
        // ------------------------------------------------------------------
        // consumer warps
        // ------------------------------------------------------------------
        const int tx = tid & 31, wy = tid >> 5;
        const int p_top_ = n1 - L.lo1, p_bot_ = -1 - L.lo1;
        const int m = m0 + tx, js = j0 + wy * P;
        const bool act_m = m < n3;
        const int nrow = act_m ? max(0, min(P, n2 - js)) : 0;       // active rows of the strip
        const int nbm = (m == 0) + (m == n3 - 1);
        const int cf0 = (wy * P + 1) * WRS + tx + 1;               // centre entry of strip row 0
        const int af0 = T::ENT + wy * P * WX + tx;                  // centre-only operand, row 0
        // global offset of strip row 0 inside a plane (inactive strips point at vertex 0)
        const int own0 = nrow > 0 ? js * n3 + m : 0;
        int nbs = 0;                         // in-plane face count of strip row r: bits 2r, 2r+1
#pragma unroll
        for (int r = 0; r < P; r++) nbs |= (nbm + (js + r == 0) + (js + r == n2 - 1)) << (2 * r);
        auto slot = [&](int p) -> cd * { return sgen + ((p - (i0 - 1)) & (WRING - 1)) * T::SLOT; };
        auto wait_bar = [&](unsigned base, int p) {
            const int d = p - (i0 - 1);
            mbar_wait(base + 8 * (d & (WRING - 1)), (d / WRING) & 1);
        };
        auto arrive_bar = [&](unsigned base, int p) {     // one arrival per warp
            __syncwarp();
            if (tx == 0) mbar_arrive(base + 8 * ((p - (i0 - 1)) & (WRING - 1)));
        };

        // ---- WIDE_PRE / WIDE_UP: this thread's entry of the ring around the active region ----
        bool he_ok = false;
        int he_off = 0, he_goff = 0, he_nb = 0;
        int he_eo = 0, he_par = 0;           // WIDE_UP: coarse tile offset, odd i2 << 1 | odd i3
        if (kXf && tid < T::NHE) {
            int row, col;
            bool in = true;
            if (tid < WRS) { row = 0; col = tid; }
            else if (tid < 2 * WRS) { row = ar + 1; col = tid - WRS; }
            else {
                row = 1 + ((tid - 2 * WRS) >> 1);
                col = ((tid - 2 * WRS) & 1) ? ac + 1 : 0;
                in = row <= ar;
            }
            const int jj = j0 - 1 + row, mm = m0 - 1 + col;
            const bool corner = (row == 0 || row == ar + 1) && (col == 0 || col == ac + 1);
            const bool row_st = jj >= row_lo && jj <= row_hi;
            const bool col_st = (mm >= c_lo && mm <= c_hi) || (mm == -1 && mir_l) || (mm == n3 && mir_r);
            he_ok = in && col <= ac + 1 && !corner && row_st && col_st;
            const int jm = jj < 0 ? -jj : (jj >= n2 ? 2 * (n2 - 1) - jj : jj);
            const int mq = mm < 0 ? -mm : (mm >= n3 ? 2 * (n3 - 1) - mm : mm);
            he_off = row * WRS + col;
            if (he_ok) {
                he_goff = jm * n3 + mq;
                he_nb = (jm == 0) + (jm == n2 - 1) + (mq == 0) + (mq == n3 - 1);
                if (MODE == WIDE_UP) {
                    he_eo = ((jm >> 1) - cj_lo) * WCW + ((mq >> 1) - cm_lo);
                    he_par = ((jm & 1) << 1) | (mq & 1);
                }
            }
        }
        // WIDE_UP: coarse tile offsets of the strip rows (column parity is the thread's)
        int eo[P];
#pragma unroll
        for (int r = 0; r < P; r++)
            eo[r] = MODE == WIDE_UP && r < nrow ? (((js + r) >> 1) - cj_lo) * WCW + ((m >> 1) - cm_lo) : 0;
        const int opar3 = m & 1;
        // P e at an entry: bilinear (i2, i3) sums of one or two coarse planes (k_corr
        // arithmetic).  The in-plane sum of a coarse plane serves the three fine planes
        // around it, so the sums of the thread's entries are kept in registers along
        // the march (e2 / e2h, of coarse tile plane e2_c): an even fine plane reuses
        // them, an odd one adds the next coarse plane's sums and keeps those.
        auto cplane = [&](int cl, int off, bool o2, bool o3) -> cd {
            const cd *q = ctile + cl * (T::CH * WCW) + off;
            cd a = q[0];
            if (o3) a = cadd(a, q[1]);
            if (o2) {
                a = cadd(a, q[WCW]);
                if (o3) a = cadd(a, q[WCW + 1]);
            }
            return a;
        };
        auto pscale = [](bool o2, bool o3) -> double { return (o2 && o3) ? 0.25 : ((o2 || o3) ? 0.5 : 1.0); };
        cd e2[P], e2h = mk(0, 0);
#pragma unroll
        for (int r = 0; r < P; r++) e2[r] = mk(0, 0);
        int e2_c = -1;

        // local plane p mirrored at the ends of the grid (global -1 -> 1, n1 -> n1 - 2)
        const int p_top = p_top_, p_bot = p_bot_;
        auto kplane = [&](int p) -> long long {
            return (long long)(p == p_top ? p - 2 : (p == p_bot ? p + 2 : p)) * plane;
        };
        // w D^-1 factor applied to a staged entry of b (WIDE_PRE; constant medium: the
        // face rescale D^-1(nb) / D^-1(0), w D^-1(0) applied after M)
        auto dfac = [&](double kk, int ki, int nb) -> cd {
            if (KV == KV_CONST) return MODE == WIDE_UP ? tab[4 + nb] : tab[8 + nb];
            if (KV == KV_PAL) return pal_d[4 * ki + nb];
            return cscal(dinv_of(L, kk, nb), omega);
        };
        // x faces the plane touches (n1 >= 3: a mirrored plane is never a face plane)
        auto nbx_of = [&](int p) { return (p == p_bot + 1) + (p == p_top - 1); };

        // wavenumber / palette index of the thread's points: plane i (kc), plane
        // i+1 (kn) and, for WIDE_PRE, plane i+2 (kp) in flight
        double kc[P], kn[P], kp[P];
        int ic[P], in_[P], ip[P];
#pragma unroll
        for (int r = 0; r < P; r++) {
            kc[r] = kn[r] = kp[r] = L.kc;
            ic[r] = in_[r] = ip[r] = 0;
        }
        // (q: element offset of strip row 0 in the plane to read)
        auto load_k_at = [&](long long q, double (&kk)[P], int (&ii)[P]) {
            if (KV != KV_CONST) {
#pragma unroll
                for (int r = 0; r < P; r++) {
                    const long long qq = q + (r < nrow ? r * n3 : 0);
                    if (KV == KV_FIELD) kk[r] = __ldg(L.k + qq);
                    else ii[r] = (int)__ldg(L.kidx + qq);
                }
            }
        };
        auto load_k = [&](int p, double (&kk)[P], int (&ii)[P]) {
            if (KV != KV_CONST) {
                const long long q = kplane(p) + own0;
#pragma unroll
                for (int r = 0; r < P; r++) {
                    const long long qq = q + (r < nrow ? r * n3 : 0);
                    if (KV == KV_FIELD) kk[r] = __ldg(L.k + qq);
                    else ii[r] = (int)__ldg(L.kidx + qq);
                }
            }
        };
        double hk_n = L.kc, hk_p = L.kc;     // ring entry: planes i+1 / i+2
        int hi_n = 0, hi_p = 0;
        auto load_hk = [&](int p, double &kk, int &ii) {
            if (kXf && KV != KV_CONST && he_ok) {
                const long long q = kplane(p) + he_goff;
                if (KV == KV_FIELD) kk = __ldg(L.k + q);
                else ii = (int)__ldg(L.kidx + q);
            }
        };
        const int he_rel = he_goff - own0;
        auto load_hk_at = [&](long long q, double &kk, int &ii) {
            if (kXf && KV != KV_CONST && he_ok) {
                if (KV == KV_FIELD) kk = __ldg(L.k + q + he_rel);
                else ii = (int)__ldg(L.kidx + q + he_rel);
            }
        };

        // transform of plane p (WIDE_PRE): own centres -> fo[] = D^-1 b (stored when
        // `ring`), bo[] = b; the thread's ring entry
        // WIDE_UP: P e at the thread's centres and ring entry of plane p -- needs the coarse
        // tile only, so it is issued ahead of the wait for the plane itself
        int cp_have = 0;                     // coarse planes [0, cp_have) of the tile have landed
        auto prolong_all = [&](int p, cd (&pe)[P], cd &peh, bool ring) {
            if (MODE == WIDE_UP) {
                const int gm = L.lo1 + (p == p_top_ ? p - 2 : (p == p_bot_ ? p + 2 : p));
                const int cl = (gm >> 1) - cp_lo;
                const bool odd = gm & 1;
                for (; cp_have <= cl + (int)odd; cp_have++) mbar_wait(b_coarse + 8 * cp_have, 0);
                const bool hring = he_ok;        // (the ring entry's sums are carried on every plane)
                if (e2_c != cl) {                // first plane of the march, mirrored end planes
#pragma unroll
                    for (int r = 0; r < P; r++) e2[r] = cplane(cl, eo[r], (js + r) & 1, opar3);
                    if (hring) e2h = cplane(cl, he_eo, he_par & 2, he_par & 1);
                    e2_c = cl;
                }
                if (!odd) {
#pragma unroll
                    for (int r = 0; r < P; r++) {
                        const double s2 = pscale((js + r) & 1, opar3);
                        pe[r] = s2 == 1.0 ? e2[r] : cscal(e2[r], s2);
                    }
                    if (ring && hring) {
                        const double s2 = pscale(he_par & 2, he_par & 1);
                        peh = s2 == 1.0 ? e2h : cscal(e2h, s2);
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < P; r++) {
                        const cd nx = cplane(cl + 1, eo[r], (js + r) & 1, opar3);
                        pe[r] = cscal(cadd(e2[r], nx), 0.5 * pscale((js + r) & 1, opar3));
                        e2[r] = nx;
                    }
                    if (hring) {
                        const cd nx = cplane(cl + 1, he_eo, he_par & 2, he_par & 1);
                        peh = cscal(cadd(e2h, nx), 0.5 * pscale(he_par & 2, he_par & 1));
                        e2h = nx;
                    }
                    e2_c = cl + 1;
                }
            }
        };
        auto transform = [&](int p, cd (&fo)[P], cd (&bo)[P], const double (&kk)[P],
                             const int (&ii)[P], double hk, int hi, const cd (&pe)[P], cd peh,
                             bool ring) {
            cd *sl = slot(p);
            const int nbx = nbx_of(p);
            if (MODE == WIDE_UP) {
                // t = [w D^-1 b] + P e on the thread's centres and its ring entry
#pragma unroll
                for (int r = 0; r < P; r++) {
                    bo[r] = sl[cf0 + r * WRS];
                    cd t = pe[r];
                    if (up.pre) t = cadd(cmul(bo[r], dfac(kk[r], ii[r], nbx + ((nbs >> (2 * r)) & 3))), t);
                    fo[r] = t;
                    if (ring && r < nrow) sl[cf0 + r * WRS] = t;
                }
                if (ring && he_ok) {
                    cd t = peh;
                    if (up.pre) t = cadd(cmul(sl[he_off], dfac(hk, hi, nbx + he_nb)), t);
                    sl[he_off] = t;
                }
                return;
            }
            if (KV == KV_CONST) {
                // only face vertices are rescaled (b^ = b D^-1(nb) / D^-1(0))
#pragma unroll
                for (int r = 0; r < P; r++) {
                    bo[r] = fo[r] = sl[cf0 + r * WRS];
                    const int nb = nbx + ((nbs >> (2 * r)) & 3);
                    if (nb > 0 && r < nrow) {
                        fo[r] = cmul(fo[r], tab[8 + nb]);
                        if (ring) sl[cf0 + r * WRS] = fo[r];
                    }
                }
                if (ring && he_ok && nbx + he_nb > 0)
                    sl[he_off] = cmul(sl[he_off], tab[8 + nbx + he_nb]);
            } else {
#pragma unroll
                for (int r = 0; r < P; r++) {
                    bo[r] = sl[cf0 + r * WRS];
                    fo[r] = cmul(bo[r], dfac(kk[r], ii[r], nbx + ((nbs >> (2 * r)) & 3)));
                    if (ring && r < nrow) sl[cf0 + r * WRS] = fo[r];
                }
                if (ring && he_ok) sl[he_off] = cmul(sl[he_off], dfac(hk, hi, nbx + he_nb));
            }
        };

        // ---- prologue: planes i0-1 and i0 into the register sets ----
        WidePlane<P> S0, S1, S2;
        cd bc[P], bn[P];                     // WIDE_PRE / WIDE_UP: b of planes i / i+1
#pragma unroll
        for (int r = 0; r < P; r++) bc[r] = bn[r] = mk(0, 0);
        if (kXf) {
            load_k(i0 - 1, kp, ip);          // (temporarily) plane i0-1
            load_k(i0, kc, ic);
            load_k(i0 + 1, kn, in_);
            double hk0 = L.kc;
            int hi0 = 0;
            load_hk(i0, hk0, hi0);
            load_hk(i0 + 1, hk_n, hi_n);
            cd pe[P], peh = mk(0, 0);
#pragma unroll
            for (int r = 0; r < P; r++) pe[r] = mk(0, 0);
            prolong_all(i0 - 1, pe, peh, false);
            wait_bar(b_full, i0 - 1);
            transform(i0 - 1, S0.f, bn, kp, ip, 0.0, 0, pe, peh, false);
            arrive_bar(b_xf, i0 - 1);        // (keeps the slot's xf phase in step with its uses)
            arrive_bar(b_empty, i0 - 1);
            prolong_all(i0, pe, peh, true);
            wait_bar(b_full, i0);
            transform(i0, S1.f, bc, kc, ic, hk0, hi0, pe, peh, true);
            arrive_bar(b_xf, i0);
        } else {
            load_k(i0, kc, ic);
            wait_bar(b_full, i0 - 1);
            const cd *sp = slot(i0 - 1);
#pragma unroll
            for (int r = 0; r < P; r++) S0.f[r] = sp[cf0 + r * WRS];
            arrive_bar(b_empty, i0 - 1);
            wait_bar(b_full, i0);
            const cd *sc = slot(i0);
#pragma unroll
            for (int r = 0; r < P; r++) S1.f[r] = sc[cf0 + r * WRS];
        }

        long long q = (long long)i0 * plane + own0;       // strip row 0 in plane i
        // strip row 0 in the plane whose wavenumbers the next step reads (i + 2 / i + 1)
        long long kq = q + (kXf ? 2 : 1) * plane;
        const double ih2 = L.ih2;

        auto step = [&](int i, WidePlane<P> &Pm, WidePlane<P> &Cc, WidePlane<P> &Nx) {
            if (kXf) {
                if (i + 2 <= last) {             // (global plane n1 is the mirrored plane n1 - 2)
                    const long long kk2 = i + 2 == p_top ? kq - 2 * plane : kq;
                    load_k_at(kk2, kp, ip);
                    load_hk_at(kk2, hk_p, hi_p);
                }
            } else if (i + 1 < i1) {
                load_k_at(kq, kn, in_);
            }
            kq += plane;
            const cd *s0 = slot(i);
            const int nbx = nbx_of(i);
            cd nsum[P];                      // (ym + yp) + (zm + zp) of plane i
            auto inplane = [&]() {
                const cd yup = s0[cf0 - WRS], ydn = s0[cf0 + P * WRS];
                cd ylast = ydn;
                // (the row below the last active row of a partial strip is a ring entry)
                if (kXf && nrow > 0 && nrow < P) ylast = s0[cf0 + nrow * WRS];
#pragma unroll
                for (int r = 0; r < P; r++) {
                    const cd zm = s0[cf0 + r * WRS - 1], zp = s0[cf0 + r * WRS + 1];
                    const cd ym = r == 0 ? yup : Cc.f[r > 0 ? r - 1 : 0];
                    cd yp = r == P - 1 ? ydn : Cc.f[r < P - 1 ? r + 1 : 0];
                    if (kXf && r < P - 1 && r == nrow - 1) yp = ylast;
                    nsum[r] = cadd(cadd(ym, yp), cadd(zm, zp));
                }
            };
            if (kXf) {
                cd pe[P], peh = mk(0, 0);
#pragma unroll
                for (int r = 0; r < P; r++) pe[r] = mk(0, 0);
                prolong_all(i + 1, pe, peh, true);
                wait_bar(b_full, i + 1);
                transform(i + 1, Nx.f, bn, kn, in_, hk_n, hi_n, pe, peh, true);
                arrive_bar(b_xf, i + 1);
                // every warp's entries of plane i are in place (signalled one step ago: a
                // warp waits here only when it runs a whole step ahead of the slowest one;
                // waiting BEFORE the transform measured 50 % slower)
                wait_bar(b_xf, i);
                inplane();
                // plane i's slot is not read again (b of the epilogue is a register): release
                // it ahead of the arithmetic and the stores
                arrive_bar(b_empty, i);
            } else {
                wait_bar(b_full, i + 1);
                const cd *sn = slot(i + 1);
#pragma unroll
                for (int r = 0; r < P; r++) Nx.f[r] = sn[cf0 + r * WRS];
                inplane();
            }
#pragma unroll
            for (int r = 0; r < P; r++) {
                const cd fc = Cc.f[r];
                const cd av = kXf ? bc[r] : (kAux ? s0[af0 + r * WX] : mk(0, 0));
                const cd sum = cadd(cadd(Pm.f[r], Nx.f[r]), nsum[r]);
                const int nb = nbx + ((nbs >> (2 * r)) & 3);
                cd ap;
                if (KV == KV_CONST) ap = tab[nb];
                else if (KV == KV_PAL) ap = pal_a[4 * ic[r] + nb];
                else ap = ap_of(L, kc[r], nb);
                cd mf = cmul(ap, fc);
                mf.x -= ih2 * sum.x;
                mf.y -= ih2 * sum.y;
                if (MODE == WIDE_PRE) {
                    // f = w D^-1 b (staged); constant medium: f = b^ with w D^-1(0) applied after M
                    if (KV == KV_CONST) mf = cmul(tab[4], mf);
                    if (!SOMM && nb) mf = KV == KV_CONST ? cmul(tab[4], fc) : fc;
                } else if (!SOMM && nb) {
                    mf = fc;                 // Dirichlet identity row
                }
                if (r < nrow) {
                    const long long qq = q + r * n3;
                    if (EPI == WE_APPLY0 || EPI == WE_APPLY1 || EPI == WE_APPLY2) {
                        out[qq] = mf;
                        if (EPI == WE_APPLY1) acc[0] = cadd(acc[0], cjmul(av, mf));
                        if (EPI == WE_APPLY2) {
                            acc[0] = cadd(acc[0], cjmul(mf, mf));
                            acc[1] = cadd(acc[1], cjmul(mf, av));
                        }
                    } else if (EPI == WE_RESID) {
                        out[qq] = csub(av, mf);
                    } else {                 // Jacobi sweep: u = f + w D^-1 (b - M f)
                        cd wd;
                        if (KV == KV_CONST) wd = tab[4 + nb];
                        else if (KV == KV_PAL) wd = pal_d[4 * ic[r] + nb];
                        else wd = cscal(dinv_of(L, kc[r], nb), omega);
                        out[qq] = cadd(fc, cmul(wd, csub(av, mf)));
                    }
                }
            }
            if (!kXf) arrive_bar(b_empty, i);   // this warp is done with plane i's slot
            // rotation of the small per-point state (a few moves per strip)
#pragma unroll
            for (int r = 0; r < P; r++) {
                kc[r] = kn[r];
                ic[r] = in_[r];
                if (kXf) {
                    kn[r] = kp[r];
                    in_[r] = ip[r];
                    bc[r] = bn[r];
                }
            }
            if (kXf) {
                hk_n = hk_p;
                hi_n = hi_p;
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
    }
    constexpr int NR = ND > 0 ? ND : 1;
    if (ND > 0) {
        cd a2[NR];
#pragma unroll
        for (int d = 0; d < NR; d++) a2[d] = acc[d];
        reduce_finish<NR>(a2, rs);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
template <int P, int NCW = 8>
static dim3 wide_grid(const Lvl &L, int &chunk) {
    using T = WideTile<P, false, false, NCW>;
    const int gx = (L.n3 + WX - 1) / WX, gy = (L.n2 + T::WY - 1) / T::WY;
    // several short waves (sliver tiles at the 2^k + 1 edges finish early and the
    // block scheduler back-fills); every chunk re-reads two planes
    const long long cols = (long long)gx * gy;
    const long long target = 148LL * (P >= 10 ? 1 : (P >= 4 ? 2 : 3)) * 6;
    int gz = (int)std::max<long long>(1, std::min<long long>(L.nx, (target + cols - 1) / cols));
    // (the transform modes -- 7 consumer warps -- pay more per chunk: two extra planes are
    // transformed, so their marches are at least 32 planes long)
    chunk = std::max((L.nx + gz - 1) / gz, std::min(L.nx, NCW < 8 ? 32 : 8));
    gz = (L.nx + chunk - 1) / chunk;
    return dim3(gx, gy, gz);
}

template <int MODE, int EPI, int KV, bool SOMM, int P>
static void wide_launch_t(const Lvl &L, const cd *src, const cd *aux, cd *out, double omega,
                          const RedSlot &rs, cudaStream_t s, const int *done,
                          const WideUp &up = WideUp{}) {
    constexpr int NCW = wide_ncw(MODE, P);
    constexpr size_t smem = WideTile<P, EPI != WE_APPLY0 && MODE == WIDE_LOAD, MODE == WIDE_UP, NCW>::smem;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_wide<MODE, EPI, KV, SOMM, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        attr = true;
    }
    int chunk;
    dim3 g = wide_grid<P, NCW>(L, chunk);
    if (MODE == WIDE_UP) {               // the staged coarse tile covers WUP_CHUNK fine planes
        chunk = std::min(L.nx, wup_chunk(P));
        g.z = (L.nx + chunk - 1) / chunk;
    }
    launch(k_wide<MODE, EPI, KV, SOMM, P>, g, dim3(32 * (NCW + 1)), smem, s, L, src, aux ? aux : src, out, omega,
           chunk, rs, up, done);
}

template <int MODE, int EPI, int P>
static void wide_launch_kv(const Lvl &L, const cd *src, const cd *aux, cd *out, double omega,
                           const RedSlot &rs, cudaStream_t s, const int *done,
                           const WideUp &up = WideUp{}) {
    const bool somm = L.bc == HF_BC_SOMMERFELD;
    // the pre-smoothing sweep of a palette level uses the palette too (one byte per entry)
    const int kv = L.k ? (L.kidx && L.npal <= WPAL ? KV_PAL : KV_FIELD) : KV_CONST;
#define HF_WIDE_CASE(KVv)                                                                          \
    if (kv == KVv) {                                                                               \
        if (somm) wide_launch_t<MODE, EPI, KVv, true, P>(L, src, aux, out, omega, rs, s, done, up); \
        else wide_launch_t<MODE, EPI, KVv, false, P>(L, src, aux, out, omega, rs, s, done, up);     \
        return;                                                                                    \
    }
    HF_WIDE_CASE(KV_CONST)
    HF_WIDE_CASE(KV_FIELD)
    HF_WIDE_CASE(KV_PAL)
#undef HF_WIDE_CASE
}

bool wide_ok(const Lvl &L, int kind) {
    if (opt(OPT_NO_WIDE)) return false;
    if (opt(OPT_FORCE_WIDE)) return true;
    // measured inside the 513^3 solve: the family wins on the pre-smoothing sweep and
    // the plain apply; the Jacobi sweep and the applies with inner products are at the
    // HBM roofline in both families (wide_all routes them here too)
    return L.n3 > 256 && (kind >= 5 || kind == 0 || opt(OPT_WIDE_ALL));   // 6: fused up-sweep
}

// kind: 0 apply, 1 apply + conj(w) v, 2 apply + v^H v & v^H w, 3 residual, 4 Jacobi,
// 5 zero-guess pre-smoothing + residual
void launch_wide(int kind, const Lvl &L, const cd *src, const cd *aux, cd *out, double omega,
                 const RedSlot &rs, cudaStream_t s, const int *done) {
    const bool p4 = opt(OPT_WIDE_P4);   // four rows per thread (default: two)
    if (kind == 5 && opt(OPT_WIDE_P3)) {   // three rows per thread (transform modes only)
        wide_launch_kv<WIDE_PRE, WE_RESID, 3>(L, src, aux, out, omega, rs, s, done);
        return;
    }
    if (kind == 5 && opt(OPT_WIDE_BIG)) {  // one 512-thread block per SM, 15 consumer warps
        wide_launch_kv<WIDE_PRE, WE_RESID, 12>(L, src, aux, out, omega, rs, s, done);
        return;
    }
    if (kind == 5 && opt(OPT_WIDE_P1)) {   // one row per thread, 8 consumer warps, 3 blocks per SM
        wide_launch_kv<WIDE_PRE, WE_RESID, 1>(L, src, aux, out, omega, rs, s, done);
        return;
    }
#define HF_WIDE_KIND(K, MODE, EPI)                                                                 \
    if (kind == K) {                                                                               \
        if (p4) wide_launch_kv<MODE, EPI, 4>(L, src, aux, out, omega, rs, s, done);                \
        else wide_launch_kv<MODE, EPI, 2>(L, src, aux, out, omega, rs, s, done);                   \
        return;                                                                                    \
    }
    HF_WIDE_KIND(0, WIDE_LOAD, WE_APPLY0)
    HF_WIDE_KIND(1, WIDE_LOAD, WE_APPLY1)
    HF_WIDE_KIND(2, WIDE_LOAD, WE_APPLY2)
    HF_WIDE_KIND(3, WIDE_LOAD, WE_RESID)
    HF_WIDE_KIND(4, WIDE_LOAD, WE_JACOBI)
    HF_WIDE_KIND(5, WIDE_PRE, WE_RESID)
#undef HF_WIDE_KIND
}

// fused up-sweep on a whole-grid wide level: u = t + w D^-1 (b - M t), t = [w D^-1 b] + P e
void launch_wide_up(const Lvl &L, const Lvl &C, const cd *b, const cd *e, cd *u, double omega,
                    bool pre, cudaStream_t s, const int *done) {
    const WideUp up{C, e, pre ? 1 : 0};
    if (opt(OPT_WIDE_BIG)) wide_launch_kv<WIDE_UP, WE_JACOBI, 12>(L, b, b, u, omega, RedSlot{}, s, done, up);
    else if (opt(OPT_WIDE_P1)) wide_launch_kv<WIDE_UP, WE_JACOBI, 1>(L, b, b, u, omega, RedSlot{}, s, done, up);
    else if (opt(OPT_WIDE_P3)) wide_launch_kv<WIDE_UP, WE_JACOBI, 3>(L, b, b, u, omega, RedSlot{}, s, done, up);
    else if (opt(OPT_WIDE_P4)) wide_launch_kv<WIDE_UP, WE_JACOBI, 4>(L, b, b, u, omega, RedSlot{}, s, done, up);
    else wide_launch_kv<WIDE_UP, WE_JACOBI, 2>(L, b, b, u, omega, RedSlot{}, s, done, up);
}

int wide_blocks(const Lvl &L) {
    int c2, c4;
    const dim3 a = wide_grid<2>(L, c2), b = wide_grid<4>(L, c4), c = wide_grid<2, 7>(L, c2);
    const dim3 d = wide_grid<3, 5>(L, c2), e = wide_grid<4, 4>(L, c2), f = wide_grid<1, 8>(L, c2);
    const dim3 g = wide_grid<12, 15>(L, c2);
    return (int)std::max(std::max(std::max(a.x * a.y * a.z, b.x * b.y * b.z), std::max(c.x * c.y * c.z, g.x * g.y * g.z)),
                         std::max(std::max(d.x * d.y * d.z, e.x * e.y * e.z), f.x * f.y * f.z));
}

}  // namespace hf
