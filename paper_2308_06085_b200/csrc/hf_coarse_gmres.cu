// hf_coarse_gmres.cu -- the reference's coarsest-level solve on the device:
// unpreconditioned GMRES from x0 = 0 to coarsest_tol, at most coarsest_maxit
// iterations, max-iterations as a soft failure counted in coarsest_flags
// (/root/reference/pkg/src/helmfree/multigrid.py:300-323 calling
// krylov.py:111-192 gmres with Minv = identity, restart = None).
//
// ONE cooperative launch per coarsest solve, so a V-cycle that uses it is
// still a single captured CUDA graph.  Blocks own contiguous row slices of
// the coarsest grid; every reduction is per-block partials, a grid barrier,
// then every block sums the partials in the same fixed order (deterministic
// and identical in every block, so every block runs the same control flow).
// Arnoldi uses classical Gram-Schmidt applied twice (CGS2: two reductions
// per iteration instead of MGS's j + 1 sequential ones; same orthogonality to
// rounding).  The Givens rotations and g are kept redundantly in every
// block's shared memory; block 0 stores the rotated Hessenberg columns and
// solves the triangular system at the end.  The basis holds `cap` vectors:
// with cap < maxit the solve restarts from r = b - A x every cap iterations
// (cap = min(maxit, 1024, memory); the reference's full GMRES needs ~50-70
// iterations on the 17^3 coarsest grid).
#include <cooperative_groups.h>

#include <algorithm>

#include "hf_kernels.cuh"

namespace cg = cooperative_groups;

namespace hf {

__device__ __forceinline__ cd ldcg(const cd *p) { return __ldcg(p); }

// (M u)_q on a whole-grid level (operators.py:200-254): Sommerfeld ghost
// elimination = mirrored inward neighbour, Dirichlet boundary rows identities
__device__ cd apply_at(const Lvl &L, const cd *u, long long q) {
    const int i = (int)(q / L.plane);
    const int rem = (int)(q - (long long)i * L.plane);
    const int j = rem / L.n3, m = rem - j * L.n3;
    const int nb = nbnd(L, i, j, m);
    const cd uc = ldcg(u + q);
    if (L.bc == HF_BC_DIRICHLET && nb) return uc;
    const double kk = L.k ? __ldg(L.k + q) : L.kc;
    const cd ap = ap_of(L, kk, nb);
    const long long sx = L.plane, sy = L.n3;
    const long long qxm = i > 0 ? q - sx : q + sx, qxp = i < L.n1 - 1 ? q + sx : q - sx;
    const long long qym = j > 0 ? q - sy : q + sy, qyp = j < L.n2 - 1 ? q + sy : q - sy;
    const long long qzm = m > 0 ? q - 1 : q + 1, qzp = m < L.n3 - 1 ? q + 1 : q - 1;
    cd s = cadd(cadd(cadd(ldcg(u + qxm), ldcg(u + qxp)), cadd(ldcg(u + qym), ldcg(u + qyp))),
                cadd(ldcg(u + qzm), ldcg(u + qzp)));
    cd v = cmul(ap, uc);
    v.x -= L.ih2 * s.x;
    v.y -= L.ih2 * s.y;
    return v;
}

#define GM_NT 256

__device__ __forceinline__ cd warp_total(cd v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    return v;
}

__global__ void __launch_bounds__(GM_NT) k_coarse_gmres(GmArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smem[];
    const int cap = a.cap;
    cd *hs = reinterpret_cast<cd *>(smem);       // cap + 2: reduced dots
    cd *hacc = hs + (cap + 2);                   // cap + 2: h = h1 + h2 (Arnoldi column)
    cd *sn = hacc + (cap + 2);                   // cap: Givens s
    cd *g = sn + cap;                            // cap + 1
    double *cs = reinterpret_cast<double *>(g + cap + 1);   // cap: Givens c
    __shared__ cd wsum[GM_NT / 32];
    __shared__ int stop;
    if (a.done && *(volatile const int *)a.done) return;   // uniform over the grid
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nb = gridDim.x, blk = blockIdx.x;
    const long long N = a.N;
    const long long per = (N + nb - 1) / nb;
    const long long r0 = min(N, (long long)blk * per), r1 = min(N, r0 + per);
    const int stride = cap + 2;
    // partial sums double-buffered by reduction phase: a block may still be
    // reading phase p's partials while a faster one writes phase p + 1's; the
    // grid barrier between p + 1's write and p + 2's separates reuse
    int ph = 0;
    cd *part = a.part + (size_t)blk * stride;
    auto V = [&](int i) { return a.V + (size_t)i * N; };

    // block sum of one complex value per thread -> part[slot]
    auto block_part = [&](cd v, int slot) {
        v = warp_total(v);
        if (lane == 0) wsum[warp] = v;
        __syncthreads();
        if (tid == 0) {
            cd s = mk(0, 0);
            for (int w = 0; w < GM_NT / 32; w++) s = cadd(s, wsum[w]);
            part[slot] = s;
        }
        __syncthreads();
    };
    // hs[i] = sum over blocks of part[blk][i], fixed block order; flips the buffer
    auto reduce_parts = [&](int lo, int cnt) {
        const cd *pb = a.part + (size_t)ph * nb * stride;
        for (int i = lo + tid; i < lo + cnt; i += GM_NT) {
            cd s = mk(0, 0);
            for (int b2 = 0; b2 < nb; b2++) s = cadd(s, ldcg(pb + (size_t)b2 * stride + i));
            hs[i] = s;
        }
        __syncthreads();
        ph ^= 1;
        part = a.part + ((size_t)ph * nb + blk) * stride;
    };
    // part[i] = V_i^H w over this block's rows, i < cnt (one warp per vector)
    auto dots = [&](int cnt, const cd *w) {
        for (int i = warp; i < cnt; i += GM_NT / 32) {
            const cd *vi = V(i);
            cd s = mk(0, 0);
            for (long long q = r0 + lane; q < r1; q += 32) s = cadd(s, cjmul(ldcg(vi + q), ldcg(w + q)));
            s = warp_total(s);
            if (lane == 0) part[i] = s;
        }
        __syncthreads();
    };
    auto norm_part = [&](const cd *v, int slot) {
        cd s = mk(0, 0);
        for (long long q = r0 + tid; q < r1; q += GM_NT) s.x += cabs2(ldcg(v + q));
        block_part(s, slot);
    };

    for (long long q = r0 + tid; q < r1; q += GM_NT) a.x[q] = mk(0, 0);
    norm_part(a.b, cap + 1);
    grid.sync();
    reduce_parts(cap + 1, 1);
    const double denom = sqrt(fmax(hs[cap + 1].x, 0.0));
    if (denom == 0.0) return;                    // x = 0 (krylov.py:125-129)
    int iters = 0, converged = 0;
    bool first = true;
    while (true) {
        // r0 = b (first cycle) or b - A x (restart), into V_0
        if (!first) grid.sync();                 // x complete
        cd *v0 = V(0);
        for (long long q = r0 + tid; q < r1; q += GM_NT)
            v0[q] = first ? a.b[q] : csub(a.b[q], apply_at(a.L, a.x, q));
        __syncthreads();
        norm_part(v0, cap + 1);
        grid.sync();
        reduce_parts(cap + 1, 1);
        const double beta = sqrt(fmax(hs[cap + 1].x, 0.0));
        if (beta / denom <= a.tol) { converged = 1; break; }
        first = false;
        for (long long q = r0 + tid; q < r1; q += GM_NT) v0[q] = cscal(v0[q], 1.0 / beta);
        if (tid == 0) { g[0] = mk(beta, 0.0); stop = 0; }
        __syncthreads();
        int m = 0;                               // basis vectors V_0 .. V_m, columns 0 .. m-1 done
        bool breakdown = false;
        double relres = beta / denom;
        while (m < cap && iters < a.maxit) {
            grid.sync();                         // V_m complete
            cd *w = V(m + 1);
            for (long long q = r0 + tid; q < r1; q += GM_NT) w[q] = apply_at(a.L, V(m), q);
            __syncthreads();
            // CGS, twice (krylov.py:157-161 up to the orthogonalisation order)
            for (int pass = 0; pass < 2; pass++) {
                dots(m + 1, w);
                grid.sync();
                reduce_parts(0, m + 1);
                for (int i = tid; i <= m; i += GM_NT) hacc[i] = pass ? cadd(hacc[i], hs[i]) : hs[i];
                for (long long q = r0 + tid; q < r1; q += GM_NT) {
                    cd acc = ldcg(w + q);
                    for (int i = 0; i <= m; i++) acc = csub(acc, cmul(hs[i], ldcg(V(i) + q)));
                    w[q] = acc;
                }
                __syncthreads();
            }
            norm_part(w, cap + 1);
            grid.sync();
            reduce_parts(cap + 1, 1);
            const double hlast = sqrt(fmax(hs[cap + 1].x, 0.0));
            iters++;
            if (tid == 0) {                      // Givens update (krylov.py:163-177), every block
                cd *col = hacc;
                col[m + 1] = mk(hlast, 0.0);
                for (int i = 0; i < m; i++) {
                    const cd t = cadd(cscal(col[i], cs[i]), cmul(sn[i], col[i + 1]));
                    col[i + 1] = csub(cscal(col[i + 1], cs[i]), cmul(mk(sn[i].x, -sn[i].y), col[i]));
                    col[i] = t;
                }
                const cd aa = col[m], bb = col[m + 1];
                const double absa = cabsd(aa), absb = cabsd(bb);
                double c;
                cd s, r;
                if (absb == 0.0) { c = 1.0; s = mk(0, 0); r = aa; }
                else if (absa == 0.0) { c = 0.0; s = cscal(mk(bb.x, -bb.y), 1.0 / absb); r = mk(absb, 0); }
                else {
                    const double t = hypot(absa, absb);
                    c = absa / t;
                    const cd ph = cscal(aa, 1.0 / absa);
                    s = cmul(ph, cscal(mk(bb.x, -bb.y), 1.0 / t));
                    r = cscal(ph, t);
                }
                cs[m] = c;
                sn[m] = s;
                col[m] = r;
                g[m + 1] = cmul(mk(-s.x, s.y), g[m]);       // -conj(s) g_m
                g[m] = cscal(g[m], c);
                if (blk == 0)
                    for (int i = 0; i <= m; i++) a.Hm[(size_t)m * cap + i] = col[i];
                stop = (hlast <= a.btol ? 2 : 0);
                if (!stop && cabsd(g[m + 1]) / denom <= a.tol) stop = 1;
            }
            __syncthreads();
            relres = cabsd(g[m + 1]) / denom;
            if (stop == 2) { breakdown = true; m++; break; }
            for (long long q = r0 + tid; q < r1; q += GM_NT) w[q] = cscal(w[q], 1.0 / hlast);
            m++;
            if (stop == 1) break;
        }
        // y = H^-1 g (krylov.py:195-204), block 0; then x += V y
        if (blk == 0 && tid == 0) {
            for (int i = m - 1; i >= 0; i--) {
                cd acc = g[i];
                for (int j = i + 1; j < m; j++) acc = csub(acc, cmul(a.Hm[(size_t)j * cap + i], a.y[j]));
                a.y[i] = cdiv(acc, a.Hm[(size_t)i * cap + i]);
            }
        }
        grid.sync();
        for (long long q = r0 + tid; q < r1; q += GM_NT) {
            cd acc = a.x[q];
            for (int i = 0; i < m; i++) acc = cadd(acc, cmul(ldcg(a.y + i), ldcg(V(i) + q)));
            a.x[q] = acc;
        }
        if (relres <= a.tol) { converged = 1; break; }
        if (breakdown || iters >= a.maxit) break;
    }
    if (!converged && blk == 0 && tid == 0) atomicAdd(a.flags, 1);
}

size_t coarse_gmres_smem(int cap) {
    return (size_t)(cap + 2) * 16 * 2 + (size_t)cap * 16 + (size_t)(cap + 1) * 16 + (size_t)cap * 8;
}

int coarse_gmres_blocks(long long N, int cap) {
    const size_t smem = coarse_gmres_smem(cap);
    cudaFuncSetAttribute(k_coarse_gmres, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_coarse_gmres, GM_NT, smem) != cudaSuccess || occ < 1)
        return 0;
    long long want = (N + 63) / 64;
    return (int)std::min<long long>(std::min<long long>(want, (long long)sms * occ), sms);
}

cudaError_t launch_coarse_gmres(const GmArgs &a, int nblk, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nblk);
    cfg.blockDim = dim3(GM_NT);
    cfg.dynamicSmemBytes = coarse_gmres_smem(a.cap);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // every block resident: grid.sync() is safe
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_coarse_gmres, a);
}

}  // namespace hf
