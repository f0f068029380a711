// hf_runtime.cu -- native runtime behind the C ABI in include/helmfree_b200.h.
//
// Owns device memory for levels, the multigrid hierarchy and Krylov workspace;
// orchestrates kernel sequences on one CUDA stream.  The Bi-CGSTAB loop keeps
// all scalars on the device and replays one captured CUDA graph per
// iteration; the host only polls a pinned status word every few iterations.
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "hf_kernels.cuh"

using namespace hf;

// ---------------------------------------------------------------------------
// errors / stream
// ---------------------------------------------------------------------------
static thread_local std::string g_err;
static thread_local cudaStream_t g_user_stream = nullptr;

static int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}
#define CK(call)                                                                           \
    do {                                                                                   \
        cudaError_t e__ = (call);                                                          \
        if (e__ != cudaSuccess)                                                            \
            return fail(HF_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e__)); \
    } while (0)
#define CKL()                                                                              \
    do {                                                                                   \
        cudaError_t e__ = cudaGetLastError();                                              \
        if (e__ != cudaSuccess)                                                            \
            return fail(HF_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e__)); \
    } while (0)

extern "C" const char *hf_last_error(void) { return g_err.c_str(); }
extern "C" int hf_version(void) { return 2; }

// kernel-variant selection (A/B measurements and the parity tests that compare
// the variants); every variant computes the same arithmetic.  Explicit API only:
// the library reads no environment variables.
static const char *const k_opt_names[OPT_COUNT] = {
    "no_pdl", "no_flat", "no_flat_dr", "no_dr", "tiled_dr", "flat_up", "fuse_up", "no_fuse",
    "coarsest_dense", "no_palette", "no_wide", "force_wide", "wide_p4", "wide_all", "no_wide_up", "wide_p3", "wide_p1", "wide_big"};
extern "C" int hf_set_option(const char *name, int value) {
    if (!name) return fail(HF_ERR_ARG, "null option name");
    for (int i = 0; i < OPT_COUNT; i++)
        if (std::strcmp(name, k_opt_names[i]) == 0) {
            g_opt[i] = value != 0;
            return 0;
        }
    return fail(HF_ERR_ARG, std::string("unknown option ") + name);
}
extern "C" int hf_get_option(const char *name) {
    if (!name) return fail(HF_ERR_ARG, "null option name");
    for (int i = 0; i < OPT_COUNT; i++)
        if (std::strcmp(name, k_opt_names[i]) == 0) return g_opt[i];
    return fail(HF_ERR_ARG, std::string("unknown option ") + name);
}
extern "C" void hf_set_stream(void *stream) { g_user_stream = (cudaStream_t)stream; }
extern "C" int hf_device_synchronize(void) {
    CK(cudaDeviceSynchronize());
    return 0;
}

static thread_local long long g_launches = 0;
#define L1(expr) do { expr; g_launches++; } while (0)

// ---------------------------------------------------------------------------
// device allocations
// ---------------------------------------------------------------------------
struct Allocs {
    std::vector<void *> ptrs;
    ~Allocs() {
        for (void *p : ptrs) cudaFree(p);
    }
    template <class T>
    T *get(size_t count, cudaError_t &err) {
        void *p = nullptr;
        err = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
        if (err != cudaSuccess) return nullptr;
        // zero-fill, complete before any stream (incl. non-blocking ones) uses it
        err = cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T));
        if (err == cudaSuccess) err = cudaStreamSynchronize(cudaStreamLegacy);
        if (err != cudaSuccess) { cudaFree(p); return nullptr; }
        ptrs.push_back(p);
        return (T *)p;
    }
};

// complex field with HF_GHOST ghost planes on each side of the slab
static cd *new_field(Allocs &A, int nx, long long plane, cudaError_t &err) {
    cd *base = A.get<cd>((size_t)(nx + 2 * HF_GHOST) * plane, err);
    return base ? base + (size_t)HF_GHOST * plane : nullptr;
}

// ---------------------------------------------------------------------------
// levels
// ---------------------------------------------------------------------------
struct Level {
    Lvl L{};
    cd *b = nullptr, *u = nullptr, *r = nullptr, *t = nullptr;   // scratch (MGLevel)
    cd *fb = nullptr, *guess = nullptr;                          // F-cycle scratch
};

// host: minimum |diag| h^2 check (operators.py:179-182)
static bool zero_diagonal(const Lvl &L, const double *kfull) {
    const double h = L.h, h2 = h * h;
    for (int i = L.lo1; i < L.lo1 + L.nx; i++)
        for (int j = 0; j < L.n2; j++)
            for (int m = 0; m < L.n3; m++) {
                int nb = (i == 0) + (i == L.n1 - 1) + (j == 0) + (j == L.n2 - 1) + (m == 0) +
                         (m == L.n3 - 1);
                if (L.bc == HF_BC_DIRICHLET && nb) continue;
                double kk = kfull ? kfull[((size_t)i * L.n2 + j) * L.n3 + m] : L.kc;
                double k2h2 = kk * kk * h2;
                double re = 6.0 - L.sre * k2h2, im = -L.sim * k2h2;
                if (L.bc == HF_BC_SOMMERFELD) im -= nb * 2.0 * kk * h;
                if (std::hypot(re, im) < 6.0e-12) return true;
                if (!kfull) {
                    // constant k: interior value decides; boundary rows only add imaginary parts
                }
            }
    return false;
}

static int make_level(Allocs &A, Level &lv, int n1, int n2, int n3, int lo1, int nx, double h,
                      double sre, double sim, int bc, const double *kfull, double kc,
                      bool scratch, bool finest = false) {
    init_kernel_attributes();
    if (n1 < 3 || n2 < 3 || n3 < 3) return fail(HF_ERR_ARG, "grid dims must all be >= 3");
    if (!(h > 0)) return fail(HF_ERR_ARG, "grid spacing must be positive");
    if (lo1 < 0 || nx < 1 || lo1 + nx > n1) return fail(HF_ERR_ARG, "slab outside the grid");
    if (bc != HF_BC_DIRICHLET && bc != HF_BC_SOMMERFELD) return fail(HF_ERR_ARG, "bad bc");
    Lvl &L = lv.L;
    L.n1 = n1; L.n2 = n2; L.n3 = n3; L.lo1 = lo1; L.nx = nx;
    L.plane = (long long)n2 * n3;
    L.h = h; L.h2 = h * h; L.ih2 = 1.0 / (h * h); L.twoh = 2.0 / h;
    L.sre = sre; L.sim = sim; L.bc = bc;
    L.kc = kc;
    L.k = nullptr;
    if (!kfull && !(kc > 0)) return fail(HF_ERR_ARG, "wavenumber must be positive");
    if (zero_diagonal(L, kfull))
        return fail(HF_ERR_ZERO_DIAGONAL,
                    "stencil diagonal vanishes (k^2 h^2 = 6); choose a different grid");
    cudaError_t err;
    if (kfull) {
        // owned planes plus HF_GHOST ghost planes where they exist in the grid
        double *kb = A.get<double>((size_t)(nx + 2 * HF_GHOST) * L.plane, err);
        if (!kb) return fail(HF_ERR_CUDA, "cudaMalloc k");
        int g0 = std::max(0, lo1 - HF_GHOST), g1 = std::min(n1, lo1 + nx + HF_GHOST);
        double *dst = kb + (size_t)(g0 - lo1 + HF_GHOST) * L.plane;
        CK(cudaMemcpy(dst, kfull + (size_t)g0 * L.plane, (size_t)(g1 - g0) * L.plane * sizeof(double),
                      cudaMemcpyHostToDevice));
        L.k = kb + (size_t)HF_GHOST * L.plane;
    }
    {
        // a_p and D^-1 by physical-face count for a constant medium (operators.py:163-178)
        cd tab[12];
        const double kk = kc, k2h2 = kk * kk * L.h2;
        for (int nb = 0; nb < 4; nb++) {
            double re = (6.0 - sre * k2h2) * L.ih2, im = (-sim * k2h2) * L.ih2;
            if (bc == HF_BC_SOMMERFELD) im -= nb * (kk * L.twoh);
            tab[nb] = make_double2(re, im);
            double dre = re, dim = im;
            if (bc == HF_BC_DIRICHLET && nb) { dre = 1.0; dim = 0.0; }
            double inv = 1.0 / (dre * dre + dim * dim);
            tab[4 + nb] = make_double2(dre * inv, -dim * inv);
        }
        // D^-1(nb) / D^-1(0): the boundary rescale of the zero-guess pre-smoothing
        tab[8] = make_double2(1.0, 0.0);
        for (int nb = 1; nb < 4; nb++) {
            const cd a = tab[4 + nb], c = tab[4];
            const double inv = 1.0 / (c.x * c.x + c.y * c.y);
            tab[8 + nb] = make_double2((a.x * c.x + a.y * c.y) * inv, (a.y * c.x - a.x * c.y) * inv);
        }
        cd *dt = A.get<cd>(12, err);
        if (!dt) return fail(HF_ERR_CUDA, "cudaMalloc level table");
        CK(cudaMemcpy(dt, tab, sizeof(tab), cudaMemcpyHostToDevice));
        L.tab = dt;
    }
    L.kidx = nullptr; L.kpal = nullptr; L.apal = nullptr; L.dpal = nullptr; L.npal = 0;
    if (kfull && (n3 > 256 || opt(OPT_FORCE_WIDE)) && !opt(OPT_NO_PALETTE)) {
        // wide level (tiled kernels): a medium with <= 256 distinct wavenumbers over
        // this slab and its ghost planes is stored as 8-bit palette indices
        const int g0 = std::max(0, lo1 - HF_GHOST), g1 = std::min(n1, lo1 + nx + HF_GHOST);
        const size_t cnt = (size_t)(g1 - g0) * L.plane;
        const double *src = kfull + (size_t)g0 * L.plane;
        std::vector<double> pal;
        bool fits = true;
        double last = 0.0;
        bool have = false;
        for (size_t q = 0; q < cnt && fits; q++) {
            const double v = src[q];
            if (have && v == last) continue;
            last = v;
            have = true;
            auto it = std::lower_bound(pal.begin(), pal.end(), v);
            if (it == pal.end() || *it != v) {
                if (pal.size() == 256) fits = false;
                else pal.insert(it, v);
            }
        }
        if (fits) {
            std::vector<unsigned char> idx(cnt);
            size_t lastq = 0;
            for (size_t q = 0; q < cnt; q++) {
                const double v = src[q];
                if (q && v == src[lastq]) { idx[q] = idx[lastq]; lastq = q; continue; }
                idx[q] = (unsigned char)(std::lower_bound(pal.begin(), pal.end(), v) - pal.begin());
                lastq = q;
            }
            unsigned char *kb8 = A.get<unsigned char>((size_t)(nx + 2 * HF_GHOST) * L.plane, err);
            double *kp = A.get<double>(256, err);
            cd *ap = A.get<cd>(4 * 256, err), *dp = A.get<cd>(4 * 256, err);
            if (!kb8 || !kp || !ap || !dp) return fail(HF_ERR_CUDA, "cudaMalloc palette");
            CK(cudaMemcpy(kb8 + (size_t)(g0 - lo1 + HF_GHOST) * L.plane, idx.data(), cnt, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(kp, pal.data(), pal.size() * sizeof(double), cudaMemcpyHostToDevice));
            L.kpal = kp;
            launch_palette(L, (int)pal.size(), ap, dp, nullptr);
            CK(cudaDeviceSynchronize());
            L.kidx = kb8 + (size_t)HF_GHOST * L.plane;
            L.npal = (int)pal.size();
            L.apal = ap;
            L.dpal = dp;
        }
    }
    if (kfull && !L.kidx) {
        cd *dv = new_field(A, nx, L.plane, err);
        if (!dv) return fail(HF_ERR_CUDA, "cudaMalloc D^-1");
        launch_dinv(L, dv, nullptr);
        CK(cudaDeviceSynchronize());
        L.dinv = dv;
    }
    if (scratch) {
        // the finest level's cycle works on the caller's r and z: no b / u copies
        // there (17 GB at 1025 x 1025 x 513)
        if (!finest) {
            lv.b = new_field(A, nx, L.plane, err);
            lv.u = new_field(A, nx, L.plane, err);
        }
        lv.r = new_field(A, nx, L.plane, err);
        lv.t = new_field(A, nx, L.plane, err);
        if ((!finest && (!lv.b || !lv.u)) || !lv.r || !lv.t) return fail(HF_ERR_CUDA, "cudaMalloc level scratch");
    }
    return 0;
}

struct hf_operator {
    Allocs A;
    Level lv;
};

// ---------------------------------------------------------------------------
// hierarchy (multigrid.py:101-128)
// ---------------------------------------------------------------------------
struct hf_hierarchy {
    Allocs A;
    std::vector<Level> lev;
    hf_mg_config cfg{};
    int Nc = 0;
    cd *Minv = nullptr;     // row-major dense inverse of the coarsest operator (Dirichlet)
    cd *symtiles = nullptr; // Sommerfeld: packed upper triangle of M^-1 S^-1 (64 x 64 tiles)
    double *symscale = nullptr;
    cd *prow = nullptr, *pcol = nullptr;
    cd *fdm = nullptr;      // separable coarsest: [V1^-1, V2^-1, V3^-1, V1, V2, V3]
    cd *fdm_invD = nullptr; // 1 / (l1_a + l2_b + l3_c + c) on the coarsest grid
    cd *fdm_tmp = nullptr;  // 2 N scratch
    int coarsest_flags = 0;
    // coarsest GMRES (HF_COARSEST_GMRES, or the fallback when no exact
    // factorisation applies): one cooperative launch per solve
    bool gm_on = false;
    GmArgs gm{};
    int gm_nblk = 0;
};

static bool keep_coarsening(int n1, int n2, int n3, const hf_mg_config &c) {
    int th = c.coarsest_threshold;
    bool ok = c.threshold_ge ? (n1 >= th && n2 >= th && n3 >= th) : (n1 > th && n2 > th && n3 > th);
    return ok && (n1 % 2) && (n2 % 2) && (n3 % 2);
}

// ---------------------------------------------------------------------------
// separable coarsest operator: 1-D eigendecompositions (cuSOLVER geev) for
// the fast-diagonalisation solve (k_fdm_* in hf_kernels.cu)
// ---------------------------------------------------------------------------
typedef std::complex<double> zc;

// T_d of one direction (operators.py:163-172 split per axis): 2/h^2 centre,
// -1/h^2 neighbours, Sommerfeld end rows with the doubled inward neighbour and
// -2ik/h on the centre.
static std::vector<zc> op1d(int n, const Lvl &L) {
    std::vector<zc> T((size_t)n * n, 0.0);
    for (int i = 0; i < n; i++) {
        T[(size_t)i * n + i] = 2.0 * L.ih2;
        if (i > 0) T[(size_t)i * n + i - 1] += -L.ih2 * (i == n - 1 ? 2.0 : 1.0);
        if (i < n - 1) T[(size_t)i * n + i + 1] += -L.ih2 * (i == 0 ? 2.0 : 1.0);
    }
    T[0] -= zc(0.0, L.kc * L.twoh);
    T[(size_t)n * n - 1] -= zc(0.0, L.kc * L.twoh);
    return T;
}

// in-place Gauss-Jordan inverse with partial pivoting (row-major n x n)
static bool invert(std::vector<zc> &A, int n) {
    std::vector<zc> B((size_t)n * n, 0.0);
    for (int i = 0; i < n; i++) B[(size_t)i * n + i] = 1.0;
    for (int c = 0; c < n; c++) {
        int p = c;
        for (int r = c + 1; r < n; r++)
            if (std::abs(A[(size_t)r * n + c]) > std::abs(A[(size_t)p * n + c])) p = r;
        if (std::abs(A[(size_t)p * n + c]) == 0.0) return false;
        if (p != c)
            for (int k = 0; k < n; k++) {
                std::swap(A[(size_t)p * n + k], A[(size_t)c * n + k]);
                std::swap(B[(size_t)p * n + k], B[(size_t)c * n + k]);
            }
        zc inv = 1.0 / A[(size_t)c * n + c];
        for (int k = 0; k < n; k++) { A[(size_t)c * n + k] *= inv; B[(size_t)c * n + k] *= inv; }
        for (int r = 0; r < n; r++) {
            if (r == c) continue;
            zc f = A[(size_t)r * n + c];
            if (f == 0.0) continue;
            for (int k = 0; k < n; k++) {
                A[(size_t)r * n + k] -= f * A[(size_t)c * n + k];
                B[(size_t)r * n + k] -= f * B[(size_t)c * n + k];
            }
        }
    }
    A.swap(B);
    return true;
}

// Eigenvalues of a small complex upper-Hessenberg matrix (row-major, n <= ~100)
// by the shifted QR algorithm: Wilkinson shifts from the trailing 2 x 2 block,
// Givens QR steps on the active window, deflation on negligible subdiagonals.
// Host code: the 1-D operators of the separable coarsest solve are at most a
// few dozen wide, so a host solve takes microseconds (no device library setup).
static bool hessenberg_eigvals(std::vector<zc> H, int n, std::vector<zc> &lam) {
    lam.assign(n, 0.0);
    const double eps = 2.2e-16;
    int hi = n - 1, iter = 0, total = 0;
    auto h = [&](int i, int j) -> zc & { return H[(size_t)i * n + j]; };
    while (hi >= 0) {
        if (hi == 0) { lam[0] = h(0, 0); break; }
        int l = hi;
        while (l > 0 && std::abs(h(l, l - 1)) > eps * (std::abs(h(l, l)) + std::abs(h(l - 1, l - 1)))) l--;
        if (l > 0) h(l, l - 1) = 0.0;
        if (l == hi) { lam[hi] = h(hi, hi); hi--; iter = 0; continue; }
        if (++total > 100 * n) return false;
        const zc a = h(hi - 1, hi - 1), b = h(hi - 1, hi), c = h(hi, hi - 1), d = h(hi, hi);
        zc mu;
        if (iter % 11 == 10) {
            mu = d + std::abs(c);                       // exceptional shift
        } else {
            const zc tr = a + d, det = a * d - b * c;
            const zc disc = std::sqrt(tr * tr * 0.25 - det);
            const zc m1 = tr * 0.5 + disc, m2 = tr * 0.5 - disc;
            mu = std::abs(m1 - d) < std::abs(m2 - d) ? m1 : m2;
        }
        iter++;
        for (int i = l; i <= hi; i++) h(i, i) -= mu;
        std::vector<double> cs(hi - l);
        std::vector<zc> sn(hi - l);
        for (int k = l; k < hi; k++) {                  // rows: R = G^H (H - mu I)
            const zc x = h(k, k), y = h(k + 1, k);
            const double r = std::hypot(std::abs(x), std::abs(y));
            double c0 = 1.0;
            zc s0 = 0.0;
            if (r > 0) {
                c0 = std::abs(x) / r;
                const zc ph = std::abs(x) > 0 ? x / std::abs(x) : zc(1.0, 0.0);
                s0 = ph * std::conj(y) / r;
            }
            cs[k - l] = c0; sn[k - l] = s0;
            for (int j = k; j <= hi; j++) {
                const zc u = h(k, j), v = h(k + 1, j);
                h(k, j) = c0 * u + s0 * v;
                h(k + 1, j) = -std::conj(s0) * u + c0 * v;
            }
        }
        for (int k = l; k < hi; k++) {                  // columns: R Q
            const double c0 = cs[k - l];
            const zc s0 = sn[k - l];
            for (int i = l; i <= std::min(k + 1, hi); i++) {
                const zc u = h(i, k), v = h(i, k + 1);
                h(i, k) = c0 * u + std::conj(s0) * v;
                h(i, k + 1) = -s0 * u + c0 * v;
            }
        }
        for (int i = l; i <= hi; i++) h(i, i) += mu;
    }
    return true;
}

// solve (A) x = rhs in place (row-major, partial pivoting); false if singular
static bool dense_lu_solve(std::vector<zc> A, int n, std::vector<zc> &x) {
    for (int c = 0; c < n; c++) {
        int p = c;
        for (int r = c + 1; r < n; r++)
            if (std::abs(A[(size_t)r * n + c]) > std::abs(A[(size_t)p * n + c])) p = r;
        if (std::abs(A[(size_t)p * n + c]) == 0.0) return false;
        if (p != c) {
            for (int k = 0; k < n; k++) std::swap(A[(size_t)p * n + k], A[(size_t)c * n + k]);
            std::swap(x[p], x[c]);
        }
        for (int r = c + 1; r < n; r++) {
            const zc f = A[(size_t)r * n + c] / A[(size_t)c * n + c];
            if (f == 0.0) continue;
            for (int k = c; k < n; k++) A[(size_t)r * n + k] -= f * A[(size_t)c * n + k];
            x[r] -= f * x[c];
        }
    }
    for (int r = n - 1; r >= 0; r--) {
        zc acc = x[r];
        for (int k = r + 1; k < n; k++) acc -= A[(size_t)r * n + k] * x[k];
        x[r] = acc / A[(size_t)r * n + r];
    }
    return true;
}

// eigenpairs of a small matrix A (row-major, upper Hessenberg): shifted QR for
// the eigenvalues, inverse iteration for the eigenvectors (columns of X)
static bool eig_small(const std::vector<zc> &A, int n, std::vector<zc> &lam, std::vector<zc> &X) {
    if (!hessenberg_eigvals(A, n, lam)) return false;
    double an = 0;
    for (const zc &t : A) an = std::max(an, std::abs(t));
    X.assign((size_t)n * n, 0.0);
    for (int c = 0; c < n; c++) {
        std::vector<zc> M = A;
        const zc sh = lam[c] + zc(an * 1e-13, an * 1e-13);   // keep A - sh I invertible
        for (int i = 0; i < n; i++) M[(size_t)i * n + i] -= sh;
        std::vector<zc> x(n);
        for (int i = 0; i < n; i++) x[i] = zc(1.0 + 0.1 * i, 0.3 - 0.01 * i);
        for (int it = 0; it < 3; it++) {
            if (!dense_lu_solve(M, n, x)) return false;
            double nrm = 0;
            for (const zc &v : x) nrm += std::norm(v);
            nrm = std::sqrt(nrm);
            if (!(nrm > 0) || !std::isfinite(nrm)) return false;
            for (zc &v : x) v /= nrm;
        }
        for (int i = 0; i < n; i++) X[(size_t)i * n + c] = x[i];
    }
    return true;
}

// T = V diag(lam) V^-1 (row-major V, Vi) on the host.  The 1-D operator is
// symmetric under the reflection i -> n-1-i, and its eigenvalues come in
// near-degenerate even / odd pairs (gaps ~1e-12 relative at n = 33), which no
// shifted inverse iteration can separate.  So T is split into its even and odd
// blocks (orthonormal reflection-symmetric bases, each tridiagonal), each block
// is diagonalised on its own, and V = [Q_e X_e | Q_o X_o].  False unless the
// decomposition reproduces T to ~1e-12 (the hierarchy then falls back to an
// inverse-based coarsest solve).
static bool eig1d(const std::vector<zc> &T, int n, std::vector<zc> &lam, std::vector<zc> &V,
                  std::vector<zc> &Vi) {
    const int m = n / 2, ne = n - m, no = m;      // even block has the centre when n is odd
    const double r2 = std::sqrt(0.5);
    // basis vectors as (index a, index b, coefficient of b): q = c_a e_a + c_b e_b
    auto qvec = [&](bool even, int k, std::vector<zc> &q) {
        q.assign(n, 0.0);
        if (k < m) { q[k] = r2; q[n - 1 - k] = even ? r2 : -r2; }
        else q[m] = 1.0;                             // centre (even, n odd)
    };
    std::vector<zc> lamv, Vall((size_t)n * n, 0.0);
    int col = 0;
    for (int par = 0; par < 2; par++) {
        const bool even = par == 0;
        const int d = even ? ne : no;
        if (d == 0) continue;
        std::vector<std::vector<zc>> Q(d);
        for (int k = 0; k < d; k++) qvec(even, k, Q[k]);
        std::vector<zc> B((size_t)d * d, 0.0);       // Q^T T Q (real orthonormal Q)
        for (int a = 0; a < d; a++) {
            std::vector<zc> tq(n, 0.0);
            for (int i = 0; i < n; i++)
                for (int j = std::max(0, i - 1); j <= std::min(n - 1, i + 1); j++) tq[i] += T[(size_t)i * n + j] * Q[a][j];
            for (int b2 = 0; b2 < d; b2++) {
                zc acc = 0.0;
                for (int i = 0; i < n; i++) acc += Q[b2][i] * tq[i];
                B[(size_t)b2 * d + a] = acc;
            }
        }
        std::vector<zc> lb, X;
        if (!eig_small(B, d, lb, X)) return false;
        for (int c = 0; c < d; c++, col++) {
            lamv.push_back(lb[c]);
            for (int k = 0; k < d; k++)
                for (int i = 0; i < n; i++) Vall[(size_t)i * n + col] += Q[k][i] * X[(size_t)k * d + c];
        }
    }
    lam = lamv;
    V = Vall;
    double tn = 0;
    for (const zc &t : T) tn = std::max(tn, std::abs(t));
    Vi = V;
    if (!invert(Vi, n)) return false;
    double en = 0;
    for (int i = 0; i < n; i++)
        for (int j = 0; j < n; j++) {
            zc acc = 0.0;
            for (int c = 0; c < n; c++) acc += V[(size_t)i * n + c] * lam[c] * Vi[(size_t)c * n + j];
            en = std::max(en, std::abs(acc - T[(size_t)i * n + j]));
        }
    return en <= 1e-12 * tn;
}

static int build_coarsest_fdm(hf_hierarchy *H, cudaStream_t s, bool &built) {
    built = false;
    Level &C = H->lev.back();
    const Lvl &L = C.L;
    if (L.bc != HF_BC_SOMMERFELD || L.k != nullptr || opt(OPT_COARSEST_DENSE)) return 0;
    if (L.lo1 != 0 || L.nx != L.n1) return 0;
    if (fdm_smem_bytes(L.n1, L.n2, L.n3) > 200 * 1024) return 0;
    const int n[3] = {L.n1, L.n2, L.n3};
    std::vector<zc> lam[3], V[3], Vi[3];
    bool ok = true;
    for (int d = 0; d < 3 && ok; d++) ok = eig1d(op1d(n[d], L), n[d], lam[d], V[d], Vi[d]);
    if (!ok) return 0;
    const long long N = (long long)L.n1 * L.plane;
    const zc c0(-L.sre * L.kc * L.kc, -L.sim * L.kc * L.kc);
    std::vector<zc> invD((size_t)N);
    for (int a = 0; a < n[0]; a++)
        for (int b = 0; b < n[1]; b++)
            for (int c = 0; c < n[2]; c++) {
                zc dd = lam[0][a] + lam[1][b] + lam[2][c] + c0;
                if (std::abs(dd) == 0.0) return fail(HF_ERR_SOLVER, "coarsest operator is singular");
                invD[((size_t)a * n[1] + b) * n[2] + c] = 1.0 / dd;
            }
    std::vector<zc> pack;
    for (int d = 0; d < 3; d++) pack.insert(pack.end(), Vi[d].begin(), Vi[d].end());
    for (int d = 0; d < 3; d++) pack.insert(pack.end(), V[d].begin(), V[d].end());
    cudaError_t err;
    H->fdm = H->A.get<cd>(pack.size(), err);
    H->fdm_invD = H->A.get<cd>((size_t)N, err);
    H->fdm_tmp = H->A.get<cd>(2 * (size_t)N, err);
    if (!H->fdm || !H->fdm_invD || !H->fdm_tmp) return fail(HF_ERR_CUDA, "cudaMalloc fdm coarsest");
    CK(cudaMemcpy(H->fdm, pack.data(), pack.size() * sizeof(zc), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(H->fdm_invD, invD.data(), (size_t)N * sizeof(zc), cudaMemcpyHostToDevice));
    H->Nc = (int)N;
    built = true;
    return 0;
}

static int build_coarsest_direct(hf_hierarchy *H, cudaStream_t s) {
    {
        bool built = false;
        if (int rc = build_coarsest_fdm(H, s, built)) return rc;
        if (built) return 0;
    }
    Level &C = H->lev.back();
    if (C.L.lo1 != 0 || C.L.nx != C.L.n1)
        return fail(HF_ERR_UNSUPPORTED, "direct coarsest solve needs the whole coarsest grid");
    long long N = (long long)C.L.n1 * C.L.plane;
    if (N > 60000) return 1;   // no exact factorisation: the caller falls back to GMRES
    H->Nc = (int)N;
    cudaError_t err;
    cd *Amat = nullptr;
    CK(cudaMalloc(&Amat, (size_t)N * N * sizeof(cd)));
    CK(cudaMemsetAsync(Amat, 0, (size_t)N * N * sizeof(cd), s));
    launch_assemble(C.L, Amat, s);
    CKL();
    cd *Minv = nullptr;
    if (cudaMalloc(&Minv, (size_t)N * N * sizeof(cd)) != cudaSuccess) {
        cudaFree(Amat);
        return fail(HF_ERR_CUDA, "cudaMalloc coarsest inverse");
    }
    CK(cudaMemsetAsync(Minv, 0, (size_t)N * N * sizeof(cd), s));
    launch_set_identity(N, Minv, s);
    CKL();
    cusolverDnHandle_t hs;
    if (cusolverDnCreate(&hs) != CUSOLVER_STATUS_SUCCESS) {
        cudaFree(Amat);
        return fail(HF_ERR_CUDA, "cusolverDnCreate failed");
    }
    cusolverDnSetStream(hs, s);
    int lwork = 0;
    cuDoubleComplex *Ac = (cuDoubleComplex *)Amat;
    cusolverDnZgetrf_bufferSize(hs, (int)N, (int)N, Ac, (int)N, &lwork);
    cuDoubleComplex *work = nullptr;
    int *ipiv = nullptr, *info = nullptr;
    cudaMalloc(&work, (size_t)std::max(lwork, 1) * sizeof(cuDoubleComplex));
    cudaMalloc(&ipiv, (size_t)N * sizeof(int));
    cudaMalloc(&info, 2 * sizeof(int));
    // row-major A == column-major A^T; inv(A^T) column-major == inv(A) row-major
    cusolverStatus_t st1 = cusolverDnZgetrf(hs, (int)N, (int)N, Ac, (int)N, work, ipiv, info);
    cusolverStatus_t st2 = cusolverDnZgetrs(hs, CUBLAS_OP_N, (int)N, (int)N, Ac, (int)N, ipiv,
                                            (cuDoubleComplex *)Minv, (int)N, info + 1);
    int hinfo[2] = {0, 0};
    cudaMemcpyAsync(hinfo, info, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    cusolverDnDestroy(hs);
    cudaFree(work); cudaFree(ipiv); cudaFree(info); cudaFree(Amat);
    if (e != cudaSuccess) { cudaFree(Minv); return fail(HF_ERR_CUDA, std::string("coarsest factorisation: ") + cudaGetErrorString(e)); }
    if (st1 != CUSOLVER_STATUS_SUCCESS || st2 != CUSOLVER_STATUS_SUCCESS || hinfo[0] != 0 || hinfo[1] != 0) {
        cudaFree(Minv);
        return fail(HF_ERR_SOLVER, "coarsest operator is singular (getrf/getrs failed)");
    }
    if (C.L.bc == HF_BC_SOMMERFELD) {
        // symmetric form: keep only the upper triangle of B = M^-1 S^-1
        std::vector<double> sv(N);
        for (int i = 0; i < C.L.n1; i++)
            for (int j = 0; j < C.L.n2; j++)
                for (int m = 0; m < C.L.n3; m++) {
                    int nb = (i == 0) + (i == C.L.n1 - 1) + (j == 0) + (j == C.L.n2 - 1) + (m == 0) + (m == C.L.n3 - 1);
                    sv[((size_t)i * C.L.n2 + j) * C.L.n3 + m] = std::ldexp(1.0, -nb);
                }
        long long nt = sym_tiles_count((int)N);
        H->symscale = H->A.get<double>(N, err);
        H->symtiles = H->A.get<cd>((size_t)nt * 64 * 64, err);
        H->prow = H->A.get<cd>((size_t)nt * 64, err);
        H->pcol = H->A.get<cd>((size_t)nt * 64, err);
        if (!H->symscale || !H->symtiles || !H->prow || !H->pcol) {
            cudaFree(Minv);
            return fail(HF_ERR_CUDA, "cudaMalloc symmetric coarsest tiles");
        }
        CK(cudaMemcpy(H->symscale, sv.data(), N * sizeof(double), cudaMemcpyHostToDevice));
        launch_sym_pack((int)N, Minv, H->symscale, H->symtiles, s);
        e = cudaStreamSynchronize(s);
        cudaFree(Minv);
        if (e != cudaSuccess) return fail(HF_ERR_CUDA, std::string("symmetric pack: ") + cudaGetErrorString(e));
    } else {
        H->Minv = Minv;
        H->A.ptrs.push_back(Minv);
    }
    return 0;
}

static cudaStream_t work_stream() { return g_user_stream; }

// the reference's coarsest solve: GMRES to coarsest_tol (multigrid.py:300-323)
static int build_coarsest_gmres(hf_hierarchy *H) {
    Level &C = H->lev.back();
    if (C.L.lo1 != 0 || C.L.nx != C.L.n1)
        return fail(HF_ERR_UNSUPPORTED, "coarsest GMRES needs the whole coarsest grid");
    const long long N = (long long)C.L.n1 * C.L.plane;
    const long long mem_cap = (4ll << 30) / (16 * N) - 1;   // basis <= 4 GiB
    const int cap = (int)std::max<long long>(8, std::min<long long>(
                        std::min<long long>(H->cfg.coarsest_maxit, 1024), mem_cap));
    const int nblk = coarse_gmres_blocks(N, cap);
    if (nblk <= 0) return fail(HF_ERR_CUDA, "coarsest GMRES: kernel not launchable");
    cudaError_t e;
    GmArgs &g = H->gm;
    g.L = C.L;
    g.N = N;
    g.cap = cap;
    g.maxit = std::max(1, H->cfg.coarsest_maxit);
    g.tol = H->cfg.coarsest_tol;
    g.btol = 1e-30;
    g.V = H->A.get<cd>((size_t)(cap + 1) * N, e);
    g.part = H->A.get<cd>((size_t)2 * nblk * (cap + 2), e);
    g.Hm = H->A.get<cd>((size_t)cap * cap, e);
    g.y = H->A.get<cd>(cap, e);
    g.flags = H->A.get<int>(1, e);
    if (!g.V || !g.part || !g.Hm || !g.y || !g.flags) return fail(HF_ERR_CUDA, "cudaMalloc coarsest GMRES");
    H->gm_nblk = nblk;
    H->gm_on = true;
    H->Nc = (int)N;
    return 0;
}

extern "C" hf_hierarchy *hf_hierarchy_create(int n1, int n2, int n3, int lo1, int nx, double h,
                                             double beta1, double beta2, int bc,
                                             const double *k_host, double k_const,
                                             const hf_mg_config *cfg) {
    if (!cfg) { fail(HF_ERR_ARG, "null mg config"); return nullptr; }
    if (cfg->cycle != HF_CYCLE_V && cfg->cycle != HF_CYCLE_F) {
        fail(HF_ERR_ARG, "unknown cycle type");
        return nullptr;
    }
    if (cfg->coarsest_method != HF_COARSEST_DIRECT && cfg->coarsest_method != HF_COARSEST_GMRES &&
        cfg->coarsest_method != HF_COARSEST_EXTERNAL) {
        fail(HF_ERR_ARG, "coarsest_method must be HF_COARSEST_DIRECT, _GMRES or _EXTERNAL");
        return nullptr;
    }
    if (cfg->coarsest_method == HF_COARSEST_GMRES && (cfg->coarsest_maxit < 1 || !(cfg->coarsest_tol > 0))) {
        fail(HF_ERR_ARG, "coarsest GMRES needs coarsest_maxit >= 1 and coarsest_tol > 0");
        return nullptr;
    }
    if (cfg->nu1 < 0 || cfg->nu2 < 0 || !(cfg->omega > 0 && cfg->omega <= 1)) {
        fail(HF_ERR_ARG, "invalid smoother parameters");
        return nullptr;
    }
    auto *H = new hf_hierarchy();
    H->cfg = *cfg;
    double sre = beta1, sim = -beta2;
    std::vector<double> kprev, kcur;
    const double *kf = k_host;
    int a = n1, b = n2, c = n3, l0 = lo1, cnx = nx;
    double hh = h;
    for (int lvl = 0;; lvl++) {
        Level lv;
        if (make_level(H->A, lv, a, b, c, l0, cnx, hh, sre, sim, bc, kf, k_const, true, lvl == 0)) {
            delete H;
            return nullptr;
        }
        cudaError_t err;
        if (cfg->cycle == HF_CYCLE_F) {
            lv.fb = new_field(H->A, cnx, lv.L.plane, err);
            lv.guess = new_field(H->A, cnx, lv.L.plane, err);
        }
        H->lev.push_back(lv);
        if (!keep_coarsening(a, b, c, *cfg) || lvl > 30) break;
        // coarse grid: n -> (n+1)/2, h -> 2h; k subsampled at 2i (0-based) (operators.py:265-274)
        int na = (a + 1) / 2, nb = (b + 1) / 2, nc = (c + 1) / 2;
        if (kf) {
            kcur.assign((size_t)na * nb * nc, 0.0);
            for (int i = 0; i < na; i++)
                for (int j = 0; j < nb; j++)
                    for (int m = 0; m < nc; m++)
                        kcur[((size_t)i * nb + j) * nc + m] = kf[((size_t)(2 * i) * b + 2 * j) * c + 2 * m];
            kprev.swap(kcur);
            kf = kprev.data();
        }
        // derive_coarse_extent (partition.py:120-131) in 0-based form
        int clo = (l0 + 1) / 2, chi = (l0 + cnx - 1) / 2;
        if (chi < clo) {
            fail(HF_ERR_ARG, "level-incompatible: slab owns no vertices on a coarse level");
            delete H;
            return nullptr;
        }
        a = na; b = nb; c = nc; l0 = clo; cnx = chi - clo + 1; hh = 2.0 * hh;
    }
    int rc = 0;
    if (cfg->coarsest_method == HF_COARSEST_DIRECT) {
        rc = build_coarsest_direct(H, work_stream());
        if (rc == 1) rc = build_coarsest_gmres(H);   // too large for an exact factorisation
    } else if (cfg->coarsest_method == HF_COARSEST_GMRES) {
        rc = build_coarsest_gmres(H);
    }
    if (rc) {
        delete H;
        return nullptr;
    }
    return H;
}

extern "C" void hf_hierarchy_destroy(hf_hierarchy *H) { delete H; }
extern "C" int hf_hierarchy_num_levels(const hf_hierarchy *H) { return H ? (int)H->lev.size() : 0; }
extern "C" int hf_hierarchy_level_shape(const hf_hierarchy *H, int l, int *d) {
    if (!H || l < 0 || l >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    const Lvl &L = H->lev[l].L;
    d[0] = L.n1; d[1] = L.n2; d[2] = L.n3; d[3] = L.lo1; d[4] = L.nx;
    return 0;
}

// ---------------------------------------------------------------------------
// cycles (multigrid.py:326-419)
// ---------------------------------------------------------------------------
static void coarsest(hf_hierarchy *H, const cd *b, cd *x, cudaStream_t s, const int *done) {
    if (H->gm_on) {
        GmArgs a = H->gm;
        a.b = b; a.x = x; a.done = done;
        launch_coarse_gmres(a, H->gm_nblk, s);
        g_launches++;
    } else if (H->fdm) {
        const Lvl &L = H->lev.back().L;
        g_launches += launch_fdm(L.n1, L.n2, L.n3, H->fdm, H->fdm_invD, b, H->fdm_tmp, x, s, done);
    } else if (H->symtiles) {
        L1(launch_symv(H->Nc, H->symtiles, H->symscale, b, H->prow, H->pcol, x, s, done));
        g_launches++;   // tiles + reduction
    } else {
        L1(launch_gemv(H->Nc, H->Minv, b, x, s, done));
    }
}

static void smooth_sweeps(Level &lv, cd *u, const cd *b, double omega, int sweeps,
                          cudaStream_t s, const int *done) {
    for (int k = 0; k < sweeps; k++) {
        L1(launch_jacobi(lv.L, u, b, lv.t, omega, s, done));
        cudaMemcpyAsync(u, lv.t, (size_t)lv.L.nx * lv.L.plane * sizeof(cd), cudaMemcpyDeviceToDevice, s);
    }
}

static void v_cycle(hf_hierarchy *H, int li, const cd *b, cd *u, cudaStream_t s, const int *done) {
    Level &lv = H->lev[li];
    const hf_mg_config &c = H->cfg;
    if (li == (int)H->lev.size() - 1) { coarsest(H, b, u, s, done); return; }
    Level &nx = H->lev[li + 1];
    const bool fused = c.nu1 <= 1 && c.nu2 == 1;
    // fused down + restriction (k_flat_dr) where it applies; the tiled fused kernel
    // (wider planes) is opt-in (HF_DR=1): slower than the split pair there
    const bool split_dr = opt(OPT_NO_DR) || (!flat_dr_ok(lv.L) && !opt(OPT_TILED_DR));
    if (c.nu1 == 1 && fused && !split_dr) {
        L1(launch_down_restrict(lv.L, nx.L, b, nx.b, c.omega, s, done));
    } else if (c.nu1 == 1 && fused) {
        L1(launch_down1(lv.L, b, lv.r, c.omega, s, done));
        L1(launch_restrict(lv.L, nx.L, lv.r, nx.b, s, done));
    } else {
        if (c.nu1 == 0) {
            cudaMemsetAsync(u, 0, (size_t)lv.L.nx * lv.L.plane * sizeof(cd), s);
        } else {
            L1(launch_jacobi0(lv.L, b, u, c.omega, s, done));
            smooth_sweeps(lv, u, b, c.omega, c.nu1 - 1, s, done);
        }
        L1(launch_residual(lv.L, u, b, lv.r, s, done));
        L1(launch_restrict(lv.L, nx.L, lv.r, nx.b, s, done));
    }
    v_cycle(H, li + 1, nx.b, nx.u, s, done);
    if (fused) {
        g_launches += launch_up1(lv.L, nx.L, b, nx.u, u, lv.t, c.omega, c.nu1 == 1, s, done);
    } else {
        L1(launch_prolong(lv.L, nx.L, nx.u, u, true, s, done));
        smooth_sweeps(lv, u, b, c.omega, c.nu2, s, done);
    }
}

static void f_cycle(hf_hierarchy *H, int li, const cd *b, cd *u, cudaStream_t s, const int *done) {
    Level &lv = H->lev[li];
    if (li == (int)H->lev.size() - 1) { coarsest(H, b, u, s, done); return; }
    Level &nx = H->lev[li + 1];
    size_t bytes = (size_t)lv.L.nx * lv.L.plane * sizeof(cd);
    L1(launch_restrict(lv.L, nx.L, b, nx.b, s, done));
    f_cycle(H, li + 1, nx.b, nx.u, s, done);
    L1(launch_prolong(lv.L, nx.L, nx.u, u, false, s, done));
    L1(launch_residual(lv.L, u, b, lv.r, s, done));
    cudaMemcpyAsync(lv.guess, u, bytes, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(lv.fb, lv.r, bytes, cudaMemcpyDeviceToDevice, s);
    v_cycle(H, li, lv.fb, u, s, done);
    L1(launch_axpby(lv.L.nx * lv.L.plane, make_double2(1, 0), lv.guess, make_double2(1, 0), u, s));
}

static void precondition(hf_hierarchy *H, const cd *r, cd *z, cudaStream_t s, const int *done) {
    if (H->cfg.cycle == HF_CYCLE_F) f_cycle(H, 0, r, z, s, done);
    else v_cycle(H, 0, r, z, s, done);
}

extern "C" int hf_mg_precondition(hf_hierarchy *H, const double *r, double *z) {
    if (!H || !r || !z) return fail(HF_ERR_ARG, "null argument");
    cudaStream_t s = work_stream();
    precondition(H, (const cd *)r, (cd *)z, s, nullptr);
    CKL();
    return 0;
}

extern "C" int hf_restrict_fw(hf_hierarchy *H, int l, const double *r, double *out) {
    if (!H || l < 0 || l + 1 >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    L1(launch_restrict(H->lev[l].L, H->lev[l + 1].L, (const cd *)r, (cd *)out, work_stream(), nullptr));
    CKL();
    return 0;
}

extern "C" int hf_prolong_tl(hf_hierarchy *H, int l, const double *e, double *out) {
    if (!H || l < 0 || l + 1 >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    L1(launch_prolong(H->lev[l].L, H->lev[l + 1].L, (const cd *)e, (cd *)out, false, work_stream(), nullptr));
    CKL();
    return 0;
}

// fused pieces of one V-cycle level (multigrid.py:337-343), for drivers that
// exchange slab halos between them: r = b - M (w D^-1 b) ...
extern "C" int hf_level_down1(hf_hierarchy *H, int l, const double *b, double *r) {
    if (!H || l < 0 || l >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    L1(launch_down1(H->lev[l].L, (const cd *)b, (cd *)r, H->cfg.omega, work_stream(), nullptr));
    CKL();
    return 0;
}
// ... or, fused with the restriction, b_coarse = R (b - M (w D^-1 b)) (b needs
// HF_GHOST valid ghost planes at interior slab faces) ...
extern "C" int hf_level_down_restrict(hf_hierarchy *H, int l, const double *b, double *bc) {
    if (!H || l < 0 || l + 1 >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    launch_down_restrict(H->lev[l].L, H->lev[l + 1].L, (const cd *)b, (cd *)bc, H->cfg.omega,
                         work_stream(), nullptr);
    CKL();
    return 0;
}
// ... and u = u1 + w D^-1 (b - M u1), u1 = w D^-1 b + P e (t: scratch field with ghost planes;
// the caller exchanges t's halo between the two halves when the slab has interior faces)
// ... or, on whole-grid levels, correction and post-smoothing in one kernel
// (MODE_UP): u = u1 + w D^-1 (b - M u1), u1 = [w D^-1 b] + P e
extern "C" int hf_level_up(hf_hierarchy *H, int l, const double *b, const double *e, double *u) {
    if (!H || l < 0 || l + 1 >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    Level &lv = H->lev[l];
    launch_up1(lv.L, H->lev[l + 1].L, (const cd *)b, (const cd *)e, (cd *)u, lv.t, H->cfg.omega,
               H->cfg.nu1 == 1, work_stream(), nullptr);
    CKL();
    return 0;
}
extern "C" int hf_level_correct(hf_hierarchy *H, int l, const double *b, const double *e,
                                double *t) {
    if (!H || l < 0 || l + 1 >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    L1(launch_correct(H->lev[l].L, H->lev[l + 1].L, (const cd *)b, (const cd *)e, (cd *)t,
                      H->cfg.omega, H->cfg.nu1 == 1, work_stream(), nullptr));
    CKL();
    return 0;
}
// t on the owned planes AND the ghost planes at interior slab faces (needs b's
// ghost planes and one coarse ghost plane of e): the slab driver then skips the
// halo exchange of t before the post-smoothing sweep
extern "C" int hf_level_correct_ext(hf_hierarchy *H, int l, const double *b, const double *e,
                                    double *t) {
    if (!H || l < 0 || l + 1 >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    L1(launch_correct(H->lev[l].L, H->lev[l + 1].L, (const cd *)b, (const cd *)e, (cd *)t,
                      H->cfg.omega, H->cfg.nu1 == 1, work_stream(), nullptr, true));
    CKL();
    return 0;
}
extern "C" int hf_level_smooth(hf_hierarchy *H, int l, const double *t, const double *b,
                               double *u) {
    if (!H || l < 0 || l >= (int)H->lev.size()) return fail(HF_ERR_ARG, "bad level");
    L1(launch_jacobi(H->lev[l].L, (const cd *)t, (const cd *)b, (cd *)u, H->cfg.omega,
                     work_stream(), nullptr));
    CKL();
    return 0;
}

extern "C" int hf_coarsest_kind(const hf_hierarchy *H) {
    if (!H) return fail(HF_ERR_ARG, "null hierarchy");
    if (H->fdm) return HF_COARSEST_KIND_SEPARABLE;
    if (H->symtiles) return HF_COARSEST_KIND_SYMMETRIC;
    if (H->Minv) return HF_COARSEST_KIND_DENSE;
    if (H->gm_on) return HF_COARSEST_KIND_GMRES;
    return HF_COARSEST_KIND_NONE;
}

extern "C" int hf_coarsest_flags(hf_hierarchy *H, int reset) {
    if (!H) return fail(HF_ERR_ARG, "null hierarchy");
    if (!H->gm_on) return 0;
    int v = 0;
    cudaStream_t s = work_stream();
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(&v, H->gm.flags, sizeof(int), cudaMemcpyDeviceToHost));
    if (reset) CK(cudaMemset(H->gm.flags, 0, sizeof(int)));
    CK(cudaDeviceSynchronize());
    return v;
}

extern "C" int hf_coarsest_solve(hf_hierarchy *H, const double *b, double *x) {
    if (!H) return fail(HF_ERR_ARG, "null hierarchy");
    if (H->cfg.coarsest_method == HF_COARSEST_EXTERNAL)
        return fail(HF_ERR_ARG, "hierarchy was built with an external coarsest solve");
    coarsest(H, (const cd *)b, (cd *)x, work_stream(), nullptr);
    CKL();
    return 0;
}

// ---------------------------------------------------------------------------
// operators (operators.py:122-254)
// ---------------------------------------------------------------------------
extern "C" hf_operator *hf_operator_create(int n1, int n2, int n3, int lo1, int nx, double h,
                                           double shift_re, double shift_im, int bc,
                                           const double *k_host, double k_const) {
    auto *op = new hf_operator();
    // no scratch fields: only hf_jacobi_smooth needs one (allocated on first use)
    if (make_level(op->A, op->lv, n1, n2, n3, lo1, nx, h, shift_re, shift_im, bc, k_host, k_const,
                   false)) {
        delete op;
        return nullptr;
    }
    return op;
}
extern "C" void hf_operator_destroy(hf_operator *op) { delete op; }

extern "C" int hf_operator_apply(hf_operator *op, const double *u, double *v) {
    if (!op || !u || !v) return fail(HF_ERR_ARG, "null argument");
    L1(launch_apply(op->lv.L, (const cd *)u, (cd *)v, work_stream(), nullptr));
    CKL();
    return 0;
}

extern "C" int hf_operator_diag(hf_operator *op, double *d) {
    if (!op || !d) return fail(HF_ERR_ARG, "null argument");
    // D = w D^-1 b with b = D, w = 1 would divide; instead apply jacobi0 to ones:
    // diag is reported through u = 1 / (w D^-1 1) is lossy, so compute directly.
    const Lvl &L = op->lv.L;
    size_t n = (size_t)L.nx * L.plane;
    std::vector<double> kh;
    if (L.k) {
        kh.resize(n);
        CK(cudaMemcpy(kh.data(), L.k, n * sizeof(double), cudaMemcpyDeviceToHost));
    }
    std::vector<double> out(2 * n);
    for (int i = 0; i < L.nx; i++)
        for (int j = 0; j < L.n2; j++)
            for (int m = 0; m < L.n3; m++) {
                size_t q = ((size_t)i * L.n2 + j) * L.n3 + m;
                int gi = L.lo1 + i;
                int nb = (gi == 0) + (gi == L.n1 - 1) + (j == 0) + (j == L.n2 - 1) + (m == 0) + (m == L.n3 - 1);
                double kk = L.k ? kh[q] : L.kc;
                double k2h2 = kk * kk * L.h2;
                double re = (6.0 - L.sre * k2h2) * L.ih2, im = (-L.sim * k2h2) * L.ih2;
                if (L.bc == HF_BC_SOMMERFELD) im -= nb * (kk * L.twoh);
                if (L.bc == HF_BC_DIRICHLET && nb) { re = 1.0; im = 0.0; }
                out[2 * q] = re; out[2 * q + 1] = im;
            }
    CK(cudaMemcpy(d, out.data(), 2 * n * sizeof(double), cudaMemcpyHostToDevice));
    return 0;
}

extern "C" int hf_jacobi_smooth(hf_operator *op, double *u, const double *b, double omega,
                                int sweeps, int assume_zero, double *scratch) {
    if (!op || !u || !b) return fail(HF_ERR_ARG, "null argument");
    cudaStream_t s = work_stream();
    Level &lv = op->lv;
    if (!scratch && !lv.t) {
        cudaError_t err;
        lv.t = new_field(op->A, lv.L.nx, lv.L.plane, err);
        if (!lv.t) return fail(HF_ERR_CUDA, "cudaMalloc smoother scratch");
    }
    cd *tmp = scratch ? (cd *)scratch : lv.t;
    size_t bytes = (size_t)lv.L.nx * lv.L.plane * sizeof(cd);
    bool first = assume_zero != 0;
    for (int k = 0; k < sweeps; k++) {
        if (first) {
            L1(launch_jacobi0(lv.L, (const cd *)b, (cd *)u, omega, s, nullptr));
            first = false;
            continue;
        }
        L1(launch_jacobi(lv.L, (const cd *)u, (const cd *)b, tmp, omega, s, nullptr));
        CK(cudaMemcpyAsync(u, tmp, bytes, cudaMemcpyDeviceToDevice, s));
    }
    CKL();
    return 0;
}

// ---------------------------------------------------------------------------
// dot (krylov.py:67-78) -- conjugated, deterministic
// ---------------------------------------------------------------------------
struct RedBuf {
    cd *partials = nullptr;
    unsigned *counter = nullptr;
    cd *out = nullptr;
    int init(Allocs &A, size_t nblocks) {
        cudaError_t e;
        partials = A.get<cd>(nblocks * HF_MAX_DOTS, e);
        counter = A.get<unsigned>(4, e);
        out = A.get<cd>(HF_MAX_DOTS, e);
        return (partials && counter && out) ? 0 : -1;
    }
    RedSlot slot(int op, BcgState *st, const cd *gvec = nullptr, int gd = 0) const {
        RedSlot r{partials, counter, out, op, st};
        r.gvec = gvec;
        r.gd = gd;
        return r;
    }
};

extern "C" int hf_dot(int64_t n, const double *u, const double *v, double *out_host2) {
    static thread_local Allocs *A = nullptr;
    static thread_local RedBuf rb;
    if (!A) {
        A = new Allocs();
        if (rb.init(*A, 4096)) return fail(HF_ERR_CUDA, "cudaMalloc dot scratch");
    }
    cudaStream_t s = work_stream();
    L1(launch_dot(n, (const cd *)u, (const cd *)v, rb.slot(FIN_STORE, nullptr), s));
    CKL();
    CK(cudaMemcpyAsync(out_host2, rb.out, sizeof(cd), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return 0;
}

// ---------------------------------------------------------------------------
// solver: Bi-CGSTAB with device-resident scalars + CUDA graph per iteration
// ---------------------------------------------------------------------------
struct hf_solver {
    Allocs A;
    hf_operator *Aop = nullptr;
    hf_hierarchy *M = nullptr;
    long long n = 0;
    cd *x, *r, *rs, *p, *v, *ph, *s, *sh, *t;
    cd *xb = nullptr, *bb = nullptr;    // device staging for hf_solve_host
    BcgState *st = nullptr;             // device
    BcgState *st_host = nullptr;        // pinned mirror
    double *hist = nullptr;
    int hist_cap = 0;
    RedBuf red;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};   // [sparse shadow]
    int graph_kernels[2] = {0, 0};
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, evs = nullptr;
    // GMRES / IDR(s) workspace (allocated on first use)
    std::vector<cd *> basis;            // Krylov basis V (GMRES) / G, U, P (IDR)
    cd *w = nullptr, *tmp = nullptr, *tmp2 = nullptr;
    cd *hcol = nullptr;                 // device Hessenberg column / dot outputs
    int hcol_cap = 0;
    cd **vptrs = nullptr;               // device array of basis pointers
    cd *ycoef = nullptr;
    int vcap = 0;
    ~hf_solver() {
        for (cudaGraphExec_t g : graph)
            if (g) cudaGraphExecDestroy(g);
        if (st_host) cudaFreeHost(st_host);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (evs) cudaEventDestroy(evs);
        if (stream) cudaStreamDestroy(stream);
    }
};

extern "C" hf_solver *hf_solver_create(hf_operator *Aop, hf_hierarchy *M) {
    if (!Aop || !M) { fail(HF_ERR_ARG, "null operator or hierarchy"); return nullptr; }
    const Lvl &L = Aop->lv.L, &F = M->lev[0].L;
    if (L.n1 != F.n1 || L.n2 != F.n2 || L.n3 != F.n3 || L.lo1 != F.lo1 || L.nx != F.nx) {
        fail(HF_ERR_ARG, "operator and hierarchy live on different slabs");
        return nullptr;
    }
    auto *S = new hf_solver();
    S->Aop = Aop; S->M = M;
    S->n = (long long)L.nx * L.plane;
    cudaError_t e;
    cd **vecs[] = {&S->x, &S->r, &S->rs, &S->p, &S->v, &S->ph, &S->sh, &S->t};
    for (cd **pv : vecs) {
        *pv = new_field(S->A, L.nx, L.plane, e);
        if (!*pv) { fail(HF_ERR_CUDA, "cudaMalloc solver vectors"); delete S; return nullptr; }
    }
    // s = r - alpha v lives in r's buffer: r is dead once s exists (krylov.py:248-269 reads
    // only s and t until the new r), and the in-place updates stream one array less
    S->s = S->r;
    S->st = S->A.get<BcgState>(1, e);
    size_t nblk = std::max<size_t>(std::max(march_blocks(L), tile_blocks(L)), VEC_BLOCKS_HOST);
    if (!S->st || S->red.init(S->A, nblk + 64)) {
        fail(HF_ERR_CUDA, "cudaMalloc solver state");
        delete S;
        return nullptr;
    }
    if (cudaMallocHost(&S->st_host, sizeof(BcgState)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&S->ev0) != cudaSuccess || cudaEventCreate(&S->ev1) != cudaSuccess ||
        cudaEventCreateWithFlags(&S->evs, cudaEventDisableTiming) != cudaSuccess) {
        fail(HF_ERR_CUDA, "stream/event/pinned allocation failed");
        delete S;
        return nullptr;
    }
    return S;
}

extern "C" void hf_solver_destroy(hf_solver *S) { delete S; }

// one Bi-CGSTAB iteration (krylov.py:234-273), every kernel predicated on st->done

// sparse: the shadow vector has <= HF_NZ_MAX nonzeros (st->nz); the matvec's
// r~^H v and the x, r update's r~^H r are then gathered by the reductions'
// last block instead of streaming r~ (16 B per vertex, twice per iteration)
static void bcg_iteration(hf_solver *S, cudaStream_t s, bool sparse) {
    const Lvl &A = S->Aop->lv.L;
    const int *done = &S->st->done;
    long long n = S->n;
    L1(launch_bcg_p(n, S->st, S->r, S->p, S->v, s, done));
    precondition(S->M, S->p, S->ph, s, done);
    if (sparse) {
        // r~^H v = conj(r~_s) v_s over the few nonzeros of r~: a plain matvec, then a
        // one-thread gather + scalar step (same value as the last-block gather)
        L1(launch_apply(A, S->ph, S->v, s, done));
        L1(launch_bcg_gather(S->st, FIN_BCG_ALPHA, S->v, s, done));
    } else {
        L1(launch_apply_dot1(A, S->ph, S->v, S->rs, S->red.slot(FIN_BCG_ALPHA, S->st), s, done));
    }
    L1(launch_bcg_s(n, S->st, S->r, S->v, S->s, S->red.slot(FIN_BCG_S, S->st), s, done));
    precondition(S->M, S->s, S->sh, s, done);
    L1(launch_apply_dot2(A, S->sh, S->t, S->s, S->red.slot(FIN_BCG_OMEGA, S->st), s, done));
    L1(launch_bcg_xr(n, S->st, S->x, S->ph, S->sh, S->s, S->t, S->r, sparse ? nullptr : S->rs,
                     S->red.slot(FIN_BCG_RHO, S->st, sparse ? S->r : nullptr, 1), s, done));
    cudaMemcpyAsync(S->st_host, S->st, sizeof(BcgState), cudaMemcpyDeviceToHost, s);
}

static int build_graph(hf_solver *S, bool sparse) {
    if (S->graph[sparse]) return 0;
    cudaGraph_t g;
    long long before = g_launches;
    CK(cudaStreamBeginCapture(S->stream, cudaStreamCaptureModeThreadLocal));
    bcg_iteration(S, S->stream, sparse);
    cudaError_t e = cudaStreamEndCapture(S->stream, &g);
    if (e != cudaSuccess) return fail(HF_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e));
    S->graph_kernels[sparse] = (int)(g_launches - before);
    g_launches = before;
    e = cudaGraphInstantiate(&S->graph[sparse], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return fail(HF_ERR_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    return 0;
}

static int solve_bicgstab(hf_solver *S, const hf_solver_config *cfg, const cd *b, cd *x,
                          hf_report *rep) {
    cudaStream_t s = S->stream;
    if (!S->hist || S->hist_cap < cfg->maxit + 2) {
        cudaError_t e;
        S->hist = S->A.get<double>(cfg->maxit + 2, e);
        if (!S->hist) return fail(HF_ERR_CUDA, "cudaMalloc history");
        S->hist_cap = cfg->maxit + 2;
    }
    BcgState init{};
    init.tol = cfg->tol;
    init.btol = cfg->breakdown_tol > 0 ? cfg->breakdown_tol : 1e-30;
    init.maxit = cfg->maxit;
    init.hist = S->hist;
    init.hist_cap = S->hist_cap;
    *S->st_host = init;
    CK(cudaMemcpyAsync(S->st, S->st_host, sizeof(BcgState), cudaMemcpyHostToDevice, s));
    long long launches = 0;
    if (S->M->gm_on) CK(cudaMemsetAsync(S->M->gm.flags, 0, sizeof(int), s));
    CK(cudaEventRecord(S->ev0, s));
    // shadow vector r~: b (the reference, krylov.py:229), the caller's host vector,
    // or the seeded hash vector (SolverConfig.shadow)
    int shadow = cfg->shadow_kind;
    if (shadow == HF_SHADOW_RHS && cfg->shadow_host) shadow = HF_SHADOW_HOST;
    if (shadow == HF_SHADOW_HOST) {
        if (!cfg->shadow_host) return fail(HF_ERR_ARG, "HF_SHADOW_HOST needs shadow_host");
        CK(cudaMemcpyAsync(S->rs, cfg->shadow_host, (size_t)S->n * sizeof(cd), cudaMemcpyHostToDevice, s));
    }
    const Lvl &AL = S->Aop->lv.L;
    L1(launch_bcg_init(S->n, b, S->r, S->rs, S->x, S->p, S->v, S->red.slot(FIN_BCG_INIT, S->st), s,
                       shadow, cfg->shadow_seed, (long long)AL.lo1 * AL.plane));
    launch_nz_scan(S->n, S->rs, S->st, s);
    launches += 3;
    CK(cudaMemcpyAsync(S->st_host, S->st, sizeof(BcgState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const bool sparse = S->st_host->nz > 0;
    if (build_graph(S, sparse)) return HF_ERR_CUDA;
    int every = cfg->check_every > 0 ? cfg->check_every : 4;
    int graphs = 0;
    while (!S->st_host->done && graphs < cfg->maxit + every) {
        for (int k = 0; k < every; k++) {
            CK(cudaGraphLaunch(S->graph[sparse], s));
            graphs++;
        }
        CK(cudaStreamSynchronize(s));
    }
    launches += (long long)graphs * S->graph_kernels[sparse];
    if (S->st_host->s_conv) {
        L1(launch_bcg_xhalf(S->n, S->st, S->x, S->ph, s));
        launches++;
    }
    CK(cudaEventRecord(S->ev1, s));
    if (x != S->x)
        CK(cudaMemcpyAsync(x, S->x, (size_t)S->n * sizeof(cd), cudaMemcpyDeviceToDevice, s));
    CK(cudaStreamSynchronize(s));
    CKL();
    const BcgState &st = *S->st_host;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, S->ev0, S->ev1);
    rep->matvec_count = st.matvecs;
    rep->iterations = st.iter;
    rep->converged = st.converged;
    rep->breakdown = st.breakdown;
    rep->final_relres = st.relres;
    rep->solve_ms = ms;
    rep->kernel_launches = (int)launches;
    rep->coarsest_flags = 0;
    if (S->M->gm_on) CK(cudaMemcpy(&rep->coarsest_flags, S->M->gm.flags, sizeof(int), cudaMemcpyDeviceToHost));
    if (rep->history_host && rep->history_cap > 0 && st.iter > 0) {
        int cnt = std::min(st.iter, rep->history_cap);
        CK(cudaMemcpy(rep->history_host, S->hist, (size_t)cnt * sizeof(double), cudaMemcpyDeviceToHost));
    }
    return 0;
}


// ---------------------------------------------------------------------------
// host-driven Krylov loops with device vectors: GMRES (krylov.py:111-192) and
// IDR(s) (krylov.py:292-394).  Inner products are deterministic device
// reductions read back per use; the small dense work (Givens rotations, the
// s x s projection solves) runs on the host exactly as in the reference.
// ---------------------------------------------------------------------------
typedef std::complex<double> hcd;

static cd *ws_vec(hf_solver *S) {
    cudaError_t e;
    return new_field(S->A, S->Aop->lv.L.nx, S->Aop->lv.L.plane, e);
}

static int ensure_ws(hf_solver *S, int nbasis, int hcap) {
    if (!S->w) {
        S->w = ws_vec(S); S->tmp = ws_vec(S); S->tmp2 = ws_vec(S);
        if (!S->w || !S->tmp || !S->tmp2) return fail(HF_ERR_CUDA, "cudaMalloc Krylov workspace");
    }
    while ((int)S->basis.size() < nbasis) {
        cd *v = ws_vec(S);
        if (!v) return fail(HF_ERR_CUDA, "cudaMalloc Krylov basis");
        S->basis.push_back(v);
    }
    if (S->hcol_cap < hcap) {
        cudaError_t e;
        S->hcol = S->A.get<cd>(hcap, e);
        S->ycoef = S->A.get<cd>(hcap, e);
        S->vptrs = S->A.get<cd *>(hcap, e);
        if (!S->hcol || !S->ycoef || !S->vptrs) return fail(HF_ERR_CUDA, "cudaMalloc Hessenberg");
        S->hcol_cap = hcap;
    }
    return 0;
}

static hcd dot_sync(hf_solver *S, const cd *a, const cd *b, cudaStream_t s, long long &launches) {
    RedSlot rs = S->red.slot(FIN_STORE, nullptr);
    rs.out = S->hcol;
    L1(launch_dot(S->n, a, b, rs, s));
    launches++;
    cd h;
    cudaMemcpyAsync(&h, S->hcol, sizeof(cd), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    return hcd(h.x, h.y);
}
static double norm_sync(hf_solver *S, const cd *a, cudaStream_t s, long long &launches) {
    double d = dot_sync(S, a, a, s, launches).real();
    return std::sqrt(d > 0.0 ? d : 0.0);
}
static cd tod(hcd z) { return make_double2(z.real(), z.imag()); }
static void axpby_h(hf_solver *S, hcd a, const cd *x, hcd b, cd *y, cudaStream_t s, long long &l) {
    L1(launch_axpby(S->n, tod(a), x, tod(b), y, s));
    l++;
}

struct KrylovOut {
    int matvecs = 0, iters = 0, converged = 0, breakdown = 0;
    double relres = NAN;
    std::vector<double> hist;
    void record(double r) { iters++; relres = r; hist.push_back(r); }
};

static void apply_A(hf_solver *S, const cd *x, cd *y, cudaStream_t s, KrylovOut &o, long long &l) {
    L1(launch_apply(S->Aop->lv.L, x, y, s, nullptr));
    l++;
    o.matvecs++;
}
static void apply_M(hf_solver *S, const cd *x, cd *y, cudaStream_t s, long long &l) {
    long long before = g_launches;
    precondition(S->M, x, y, s, nullptr);
    l += g_launches - before;
}

// krylov.py:97-108
static void givens(hcd a, hcd b, double &c, hcd &sn, hcd &r) {
    double absa = std::abs(a), absb = std::abs(b);
    if (absb == 0.0) { c = 1.0; sn = 0.0; r = a; return; }
    if (absa == 0.0) { c = 0.0; sn = std::conj(b) / absb; r = absb; return; }
    double t = std::hypot(absa, absb);
    c = absa / t;
    sn = (a / absa) * (std::conj(b) / t);
    r = (a / absa) * t;
}

static int solve_gmres(hf_solver *S, const hf_solver_config *cfg, const cd *b, cd *x, KrylovOut &o,
                       long long &l) {
    cudaStream_t s = S->stream;
    const int maxit = cfg->maxit;
    const int restart = cfg->restart > 0 ? cfg->restart : maxit;
    const double btol = cfg->breakdown_tol > 0 ? cfg->breakdown_tol : 1e-30;
    if (ensure_ws(S, 2, std::min(restart, maxit) + 2)) return HF_ERR_CUDA;
    const size_t bytes = (size_t)S->n * sizeof(cd);
    CK(cudaMemsetAsync(x, 0, bytes, s));
    cd *r0 = S->w;   // r0 shares storage with w (r0 is consumed before w is written)
    apply_M(S, b, r0, s, l);
    double denom = norm_sync(S, r0, s, l);
    if (denom == 0.0) { o.converged = 1; o.relres = 0.0; return 0; }
    bool first = true;
    for (;;) {
        if (!first) {
            apply_A(S, x, S->tmp, s, o, l);
            axpby_h(S, 1.0, b, -1.0, S->tmp, s, l);      // tmp = b - A x
            apply_M(S, S->tmp, r0, s, l);
        }
        double beta = norm_sync(S, r0, s, l);
        if (beta / denom <= cfg->tol) { o.converged = 1; o.relres = beta / denom; return 0; }
        first = false;
        axpby_h(S, 1.0 / beta, r0, 0.0, S->basis[0], s, l);
        std::vector<std::vector<hcd>> H;
        std::vector<double> cs;
        std::vector<hcd> sn, g{hcd(beta, 0.0)};
        bool breakdown = false;
        while ((int)H.size() < restart && o.iters < maxit) {
            int m = (int)H.size() + 1;              // basis vectors so far
            apply_A(S, S->basis[m - 1], S->tmp, s, o, l);
            apply_M(S, S->tmp, S->w, s, l);
            // MGS chain: h_i = V_i^H w, w -= h_i V_i, fused pairwise; last pass |w|^2
            for (int i = 0; i <= m; i++) {
                RedSlot rs = S->red.slot(FIN_STORE, nullptr);
                rs.out = S->hcol + i;
                const cd *c = i > 0 ? S->hcol + (i - 1) : nullptr;
                const cd *vprev = i > 0 ? S->basis[i - 1] : nullptr;
                const cd *vcur = i < m ? S->basis[i] : nullptr;
                L1(launch_mgs(S->n, S->w, c, vprev, vcur, rs, s));
                l++;
            }
            std::vector<cd> hc(m + 1);
            CK(cudaMemcpyAsync(hc.data(), S->hcol, (m + 1) * sizeof(cd), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<hcd> col(m + 1);
            for (int i = 0; i < m; i++) col[i] = hcd(hc[i].x, hc[i].y);
            double ww = hc[m].x;
            double hlast = std::sqrt(ww > 0.0 ? ww : 0.0);
            col[m] = hlast;
            for (size_t i = 0; i < cs.size(); i++) {
                hcd t = cs[i] * col[i] + sn[i] * col[i + 1];
                col[i + 1] = -std::conj(sn[i]) * col[i] + cs[i] * col[i + 1];
                col[i] = t;
            }
            double c; hcd sv, r;
            givens(col[m - 1], col[m], c, sv, r);
            cs.push_back(c); sn.push_back(sv);
            col[m - 1] = r; col[m] = 0.0;
            col.resize(m);
            H.push_back(col);
            g.push_back(-std::conj(sv) * g.back());
            g[g.size() - 2] = c * g[g.size() - 2];
            double relres = std::abs(g.back()) / denom;
            o.record(relres);
            if (hlast <= btol) { breakdown = true; break; }
            if ((int)S->basis.size() < m + 1 && ensure_ws(S, m + 1, m + 2)) return HF_ERR_CUDA;
            axpby_h(S, 1.0 / hlast, S->w, 0.0, S->basis[m], s, l);
            if (relres <= cfg->tol) break;
        }
        // back substitution (krylov.py:195-204) and x += sum y_i V_i
        int mh = (int)H.size();
        std::vector<hcd> y(mh);
        for (int i = mh - 1; i >= 0; i--) {
            hcd acc = g[i];
            for (int j = i + 1; j < mh; j++) acc -= H[j][i] * y[j];
            y[i] = acc / H[i][i];
        }
        if (mh > 0) {
            std::vector<cd> yd(mh);
            for (int i = 0; i < mh; i++) yd[i] = tod(y[i]);
            CK(cudaMemcpyAsync(S->ycoef, yd.data(), mh * sizeof(cd), cudaMemcpyHostToDevice, s));
            CK(cudaMemcpyAsync(S->vptrs, S->basis.data(), mh * sizeof(cd *), cudaMemcpyHostToDevice, s));
            L1(launch_multi_axpy(S->n, mh, S->vptrs, S->ycoef, x, s));
            l++;
            CK(cudaStreamSynchronize(s));
        }
        double relres = std::abs(g.back()) / denom;
        if (relres <= cfg->tol) { o.converged = 1; return 0; }
        if (breakdown) { o.breakdown = HF_BREAKDOWN_ARNOLDI; o.converged = relres <= cfg->tol; return 0; }
        if (o.iters >= maxit) { o.converged = 0; return 0; }
    }
}

// small dense solve with partial pivoting (numpy.linalg.solve equivalent)
static bool dense_solve(std::vector<hcd> A, int m, std::vector<hcd> &rhs) {
    for (int c = 0; c < m; c++) {
        int piv = c;
        for (int r = c + 1; r < m; r++)
            if (std::abs(A[r * m + c]) > std::abs(A[piv * m + c])) piv = r;
        if (std::abs(A[piv * m + c]) == 0.0) return false;
        if (piv != c) {
            for (int k = 0; k < m; k++) std::swap(A[c * m + k], A[piv * m + k]);
            std::swap(rhs[c], rhs[piv]);
        }
        for (int r = c + 1; r < m; r++) {
            hcd f = A[r * m + c] / A[c * m + c];
            for (int k = c; k < m; k++) A[r * m + k] -= f * A[c * m + k];
            rhs[r] -= f * rhs[c];
        }
    }
    for (int r = m - 1; r >= 0; r--) {
        hcd acc = rhs[r];
        for (int k = r + 1; k < m; k++) acc -= A[r * m + k] * rhs[k];
        rhs[r] = acc / A[r * m + r];
    }
    return true;
}

static int solve_idrs(hf_solver *S, const hf_solver_config *cfg, const cd *b, cd *x, KrylovOut &o,
                      long long &l) {
    cudaStream_t s = S->stream;
    const int sdim = cfg->s;
    if (sdim < 1) return fail(HF_ERR_ARG, "IDR requires s >= 1");
    if (!cfg->shadow_host) return fail(HF_ERR_ARG, "IDR needs the shadow space (shadow_host)");
    const double btol = cfg->breakdown_tol > 0 ? cfg->breakdown_tol : 1e-30;
    // basis layout: P[0..s), G[s..2s), U[2s..3s), then r, v, u, vh
    if (ensure_ws(S, 3 * sdim + 4, 4)) return HF_ERR_CUDA;
    cd **P = &S->basis[0], **G = &S->basis[sdim], **U = &S->basis[2 * sdim];
    cd *r = S->basis[3 * sdim], *v = S->basis[3 * sdim + 1], *u = S->basis[3 * sdim + 2];
    cd *vh = S->basis[3 * sdim + 3], *gv = S->w;
    const size_t bytes = (size_t)S->n * sizeof(cd);
    for (int i = 0; i < sdim; i++)
        CK(cudaMemcpyAsync(P[i], cfg->shadow_host + 2 * (size_t)i * S->n, bytes, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(x, 0, bytes, s));
    double bnorm = norm_sync(S, b, s, l);
    if (bnorm == 0.0) { o.converged = 1; o.relres = 0.0; return 0; }
    CK(cudaMemcpyAsync(r, b, bytes, cudaMemcpyDeviceToDevice, s));
    double relres = norm_sync(S, r, s, l) / bnorm;
    if (relres <= cfg->tol) { o.converged = 1; o.relres = relres; return 0; }
    for (int i = 0; i < sdim; i++) {
        CK(cudaMemsetAsync(G[i], 0, bytes, s));
        CK(cudaMemsetAsync(U[i], 0, bytes, s));
    }
    std::vector<hcd> Mm(sdim * sdim, 0.0), f(sdim);
    for (int i = 0; i < sdim; i++) Mm[i * sdim + i] = 1.0;
    hcd om = 1.0;
    const double kappa = 0.7;
    while (o.iters < cfg->maxit) {
        for (int i = 0; i < sdim; i++) f[i] = dot_sync(S, P[i], r, s, l);
        for (int k = 0; k < sdim; k++) {
            int m = sdim - k;
            std::vector<hcd> sub(m * m), c(m);
            for (int a = 0; a < m; a++) {
                for (int bq = 0; bq < m; bq++) sub[a * m + bq] = Mm[(k + a) * sdim + (k + bq)];
                c[a] = f[k + a];
            }
            if (!dense_solve(sub, m, c)) { o.breakdown = HF_BREAKDOWN_PROJECTION; o.converged = 0; return 0; }
            CK(cudaMemcpyAsync(v, r, bytes, cudaMemcpyDeviceToDevice, s));
            for (int i = k; i < sdim; i++) axpby_h(S, -c[i - k], G[i], 1.0, v, s, l);
            apply_M(S, v, vh, s, l);
            axpby_h(S, om, vh, 0.0, u, s, l);
            for (int i = k; i < sdim; i++) axpby_h(S, c[i - k], U[i], 1.0, u, s, l);
            apply_A(S, u, gv, s, o, l);
            for (int i = 0; i < k; i++) {
                hcd alpha = dot_sync(S, P[i], gv, s, l) / Mm[i * sdim + i];
                axpby_h(S, -alpha, G[i], 1.0, gv, s, l);
                axpby_h(S, -alpha, U[i], 1.0, u, s, l);
            }
            CK(cudaMemcpyAsync(G[k], gv, bytes, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(U[k], u, bytes, cudaMemcpyDeviceToDevice, s));
            for (int i = k; i < sdim; i++) Mm[i * sdim + k] = dot_sync(S, P[i], G[k], s, l);
            if (std::abs(Mm[k * sdim + k]) < btol) { o.breakdown = HF_BREAKDOWN_PROJECTION; o.converged = 0; return 0; }
            hcd beta = f[k] / Mm[k * sdim + k];
            axpby_h(S, -beta, G[k], 1.0, r, s, l);
            axpby_h(S, beta, U[k], 1.0, x, s, l);
            relres = norm_sync(S, r, s, l) / bnorm;
            o.record(relres);
            if (relres <= cfg->tol || o.iters >= cfg->maxit) break;
            for (int i = k + 1; i < sdim; i++) f[i] = f[i] - beta * Mm[i * sdim + k];
        }
        if (relres <= cfg->tol) { o.converged = 1; return 0; }
        if (o.iters >= cfg->maxit) break;
        apply_M(S, r, vh, s, l);
        apply_A(S, vh, gv, s, o, l);
        hcd tt = dot_sync(S, gv, gv, s, l);
        if (std::abs(tt) < btol) { o.breakdown = HF_BREAKDOWN_OMEGA; break; }
        hcd tr = dot_sync(S, gv, r, s, l);
        om = tr / tt;
        double angle = std::abs(dot_sync(S, gv, r, s, l)) / (std::sqrt(std::abs(tt)) * norm_sync(S, r, s, l));
        if (angle < kappa) om = om * (kappa / angle);
        if (std::abs(om) < btol) { o.breakdown = HF_BREAKDOWN_OMEGA; break; }
        axpby_h(S, om, vh, 1.0, x, s, l);
        axpby_h(S, -om, gv, 1.0, r, s, l);
        relres = norm_sync(S, r, s, l) / bnorm;
        o.record(relres);
        if (relres <= cfg->tol) { o.converged = 1; return 0; }
    }
    o.converged = relres <= cfg->tol;
    return 0;
}

static int solve_hostloop(hf_solver *S, const hf_solver_config *cfg, const cd *b, cd *x,
                          hf_report *rep) {
    cudaStream_t s = S->stream;
    KrylovOut o;
    long long launches = 0;
    if (S->M->gm_on) CK(cudaMemsetAsync(S->M->gm.flags, 0, sizeof(int), s));
    CK(cudaEventRecord(S->ev0, s));
    int rc = cfg->method == HF_METHOD_GMRES ? solve_gmres(S, cfg, b, x, o, launches)
                                            : solve_idrs(S, cfg, b, x, o, launches);
    if (rc) return rc;
    CK(cudaEventRecord(S->ev1, s));
    CK(cudaStreamSynchronize(s));
    CKL();
    float ms = 0.f;
    cudaEventElapsedTime(&ms, S->ev0, S->ev1);
    rep->matvec_count = o.matvecs;
    rep->iterations = o.iters;
    rep->converged = o.converged;
    rep->breakdown = o.breakdown;
    rep->final_relres = o.relres;
    rep->solve_ms = ms;
    rep->kernel_launches = (int)launches;
    rep->coarsest_flags = 0;
    if (S->M->gm_on) CK(cudaMemcpy(&rep->coarsest_flags, S->M->gm.flags, sizeof(int), cudaMemcpyDeviceToHost));
    if (rep->history_host)
        for (int i = 0; i < std::min<int>((int)o.hist.size(), rep->history_cap); i++)
            rep->history_host[i] = o.hist[i];
    return 0;
}

// ---------------------------------------------------------------------------
// Device-resident Bi-CGSTAB for slab drivers (dist.SlabSolver.solve_device):
// the scalars live on the device as in the single-slab graph path; every
// reduction kernel stores this slab's partial sums (two complex) into a
// caller buffer, the driver adds them over slabs (NCCL all-reduce across
// ranks), and hf_bcg_step advances the state from the totals.  All kernels are
// predicated on the device done flag, so the host only polls the state.
// ---------------------------------------------------------------------------
struct hf_bcg {
    Allocs A;
    BcgState *st = nullptr;
    BcgState *host = nullptr;      // pinned mirror
    double *hist = nullptr;
    RedBuf red;
    ~hf_bcg() {
        if (host) cudaFreeHost(host);
    }
};

extern "C" hf_bcg *hf_bcg_create(hf_operator *Aop, double tol, int maxit, double btol) {
    if (!Aop || maxit < 1 || !(tol > 0)) { fail(HF_ERR_ARG, "bad Bi-CGSTAB state request"); return nullptr; }
    auto *B = new hf_bcg();
    cudaError_t e;
    B->st = B->A.get<BcgState>(1, e);
    B->hist = B->A.get<double>((size_t)maxit + 2, e);
    const size_t nblk = std::max<size_t>(std::max(march_blocks(Aop->lv.L), tile_blocks(Aop->lv.L)),
                                         VEC_BLOCKS_HOST);
    if (!B->st || !B->hist || B->red.init(B->A, nblk + 64) ||
        cudaMallocHost(&B->host, sizeof(BcgState)) != cudaSuccess) {
        fail(HF_ERR_CUDA, "cudaMalloc Bi-CGSTAB state");
        delete B;
        return nullptr;
    }
    BcgState init{};
    init.tol = tol;
    init.btol = btol > 0 ? btol : 1e-30;
    init.maxit = maxit;
    init.hist = B->hist;
    init.hist_cap = maxit + 2;
    *B->host = init;
    if (cudaMemcpy(B->st, B->host, sizeof(BcgState), cudaMemcpyHostToDevice) != cudaSuccess) {
        fail(HF_ERR_CUDA, "state upload");
        delete B;
        return nullptr;
    }
    return B;
}
extern "C" void hf_bcg_destroy(hf_bcg *B) { delete B; }

static RedSlot bcg_store(hf_bcg *B, double *sums) {
    RedSlot r = B->red.slot(FIN_STORE, nullptr);
    r.out = (cd *)sums;
    return r;
}
extern "C" int hf_bcg_step(hf_bcg *B, int op, const double *sums) {
    if (!B || op < FIN_BCG_INIT || op > FIN_BCG_RHO) return fail(HF_ERR_ARG, "bad step");
    launch_bcg_step(B->st, op, (const cd *)sums, work_stream());
    CKL();
    return 0;
}
// out6 = iter, done, converged, breakdown, matvecs, s_conv (synchronises)
extern "C" int hf_bcg_read(hf_bcg *B, int *out6, double *relres, double *hist, int hist_cap) {
    if (!B || !out6) return fail(HF_ERR_ARG, "bad read");
    cudaStream_t s = work_stream();
    CK(cudaMemcpyAsync(B->host, B->st, sizeof(BcgState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const BcgState &st = *B->host;
    out6[0] = st.iter; out6[1] = st.done; out6[2] = st.converged;
    out6[3] = st.breakdown; out6[4] = st.matvecs; out6[5] = st.s_conv;
    if (relres) *relres = st.relres;
    if (hist && hist_cap > 0 && st.iter > 0)
        CK(cudaMemcpy(hist, B->hist, (size_t)std::min(st.iter, hist_cap) * sizeof(double),
                      cudaMemcpyDeviceToHost));
    return 0;
}
// r = b, rs = b, x = p = v = 0; sums = |b|^2, rs^H r (this slab)
extern "C" int hf_bcg_vec_init(hf_bcg *B, int64_t n, const double *b, double *r, double *rs,
                               double *x, double *p, double *v, double *sums) {
    launch_bcg_init(n, (const cd *)b, (cd *)r, (cd *)rs, (cd *)x, (cd *)p, (cd *)v, bcg_store(B, sums),
                    work_stream());
    CKL();
    return 0;
}
// p = r + beta (p - omega v)
extern "C" int hf_bcg_vec_p(hf_bcg *B, int64_t n, const double *r, double *p, const double *v) {
    launch_bcg_p(n, B->st, (const cd *)r, (cd *)p, (const cd *)v, work_stream(), &B->st->done);
    CKL();
    return 0;
}
// s = r - alpha v; sums = |s|^2
extern "C" int hf_bcg_vec_s(hf_bcg *B, int64_t n, const double *r, const double *v, double *s,
                            double *sums) {
    launch_bcg_s(n, B->st, (const cd *)r, (const cd *)v, (cd *)s, bcg_store(B, sums), work_stream(),
                 &B->st->done);
    CKL();
    return 0;
}
// x += alpha ph + omega sh; r = s - omega t; sums = |r|^2, rs^H r
extern "C" int hf_bcg_vec_xr(hf_bcg *B, int64_t n, double *x, const double *ph, const double *sh,
                             const double *s, const double *t, double *r, const double *rs,
                             double *sums) {
    launch_bcg_xr(n, B->st, (cd *)x, (const cd *)ph, (const cd *)sh, (const cd *)s, (const cd *)t,
                  (cd *)r, (const cd *)rs, bcg_store(B, sums), work_stream(), &B->st->done);
    CKL();
    return 0;
}
// x += alpha ph (convergence at the half step)
extern "C" int hf_bcg_vec_xhalf(hf_bcg *B, int64_t n, double *x, const double *ph) {
    launch_bcg_xhalf(n, B->st, (cd *)x, (const cd *)ph, work_stream());
    CKL();
    return 0;
}
// v = A u with this slab's inner products: nd = 1: w^H v; nd = 2: v^H v, v^H w
extern "C" int hf_operator_apply_dot(hf_operator *op, hf_bcg *B, int nd, const double *u, double *v,
                                     const double *w, double *sums) {
    if (!op || !B || (nd != 1 && nd != 2)) return fail(HF_ERR_ARG, "bad apply_dot");
    if (nd == 1)
        launch_apply_dot1(op->lv.L, (const cd *)u, (cd *)v, (const cd *)w, bcg_store(B, sums), work_stream(),
                          &B->st->done);
    else
        launch_apply_dot2(op->lv.L, (const cd *)u, (cd *)v, (const cd *)w, bcg_store(B, sums), work_stream(),
                          &B->st->done);
    CKL();
    return 0;
}

// Measurement hook (bench.py kernel table): the Bi-CGSTAB vector kernels of
// one iteration (krylov.py:240, 248-249, 266-269) launched `reps` times on the
// solver's workspace, inner products into a scratch slot (the device scalar
// state is not touched).  Mean device time per launch in *ms.
extern "C" int hf_solver_bench_vec(hf_solver *S, int which, int reps, float *ms) {
    if (!S || reps < 1 || !ms || which < 0 || which > 4) return fail(HF_ERR_ARG, "bad bench request");
    cudaStream_t s = work_stream();
    const RedSlot scratch = S->red.slot(FIN_STORE, nullptr);
    auto one = [&]() {
        if (which == 0) launch_bcg_p(S->n, S->st, S->r, S->p, S->v, s, nullptr);
        else if (which == 1) launch_bcg_s(S->n, S->st, S->r, S->v, S->s, scratch, s, nullptr);
        else if (which == 4)   // the second matvec of an iteration: t = A s^ with t^H t, t^H s
            launch_apply_dot2(S->Aop->lv.L, S->sh, S->t, S->s, scratch, s, nullptr);
        else   // 3: the sparse-shadow variant (r~^H r gathered, r~ not streamed)
            launch_bcg_xr(S->n, S->st, S->x, S->ph, S->sh, S->s, S->t, S->r, which == 2 ? S->rs : nullptr,
                          scratch, s, nullptr);
    };
    if (reps > 1) one();   // warm-up (reps = 1: a single, cold launch)
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, s));
    for (int k = 0; k < reps; k++) one();
    CK(cudaEventRecord(b, s));
    CK(cudaEventSynchronize(b));
    float t = 0;
    CK(cudaEventElapsedTime(&t, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    CKL();
    *ms = t / reps;
    return 0;
}

extern "C" int hf_solve(hf_solver *S, const hf_solver_config *cfg, const double *b, double *x,
                        hf_report *rep) {
    if (!S || !cfg || !b || !x || !rep) return fail(HF_ERR_ARG, "null argument");
    if (cfg->maxit < 1 || !(cfg->tol > 0)) return fail(HF_ERR_ARG, "invalid tol/maxit");
    // order the private stream after the caller's stream and back
    CK(cudaEventRecord(S->evs, work_stream()));
    CK(cudaStreamWaitEvent(S->stream, S->evs, 0));
    int rc;
    switch (cfg->method) {
    case HF_METHOD_BICGSTAB:
        rc = solve_bicgstab(S, cfg, (const cd *)b, (cd *)x, rep);
        break;
    case HF_METHOD_GMRES:
    case HF_METHOD_IDRS:
        rc = solve_hostloop(S, cfg, (const cd *)b, (cd *)x, rep);
        break;
    default:
        return fail(HF_ERR_ARG, "unknown Krylov method");
    }
    if (rc) return rc;
    CK(cudaEventRecord(S->evs, S->stream));
    CK(cudaStreamWaitEvent(work_stream(), S->evs, 0));
    return 0;
}

extern "C" int hf_solve_host(hf_solver *S, const hf_solver_config *cfg, const double *b_host,
                             double *x_host, hf_report *rep) {
    if (!S || !b_host || !x_host) return fail(HF_ERR_ARG, "null argument");
    cudaError_t e;
    if (!S->bb) {
        S->bb = new_field(S->A, S->Aop->lv.L.nx, S->Aop->lv.L.plane, e);
        S->xb = new_field(S->A, S->Aop->lv.L.nx, S->Aop->lv.L.plane, e);
        if (!S->bb || !S->xb) return fail(HF_ERR_CUDA, "cudaMalloc staging");
    }
    size_t bytes = (size_t)S->n * sizeof(cd);
    CK(cudaMemcpyAsync(S->bb, b_host, bytes, cudaMemcpyHostToDevice, S->stream));
    CK(cudaEventRecord(S->evs, S->stream));
    CK(cudaStreamWaitEvent(work_stream(), S->evs, 0));
    int rc = hf_solve(S, cfg, (const double *)S->bb, (double *)S->xb, rep);
    if (rc) return rc;
    CK(cudaMemcpyAsync(x_host, S->xb, bytes, cudaMemcpyDeviceToHost, S->stream));
    CK(cudaStreamSynchronize(S->stream));
    return 0;
}

// ---------------------------------------------------------------------------
// Native multi-slab Bi-CGSTAB: the reference's SPMD worker body
// (runner.py:95-131) with its distributed V-cycle (multigrid.py:326-343), halo
// exchanges (partition.py:509-536) and global inner products
// (partition.py:611-621), laid out as slabs along i1.  Every step of one
// iteration -- vector updates, the slab V-cycle level kernels, the halo
// exchanges, the coarsest gather, the inner-product all-reduces and the scalar
// update -- is stream-ordered on ONE stream, and the iteration is captured once
// as a CUDA graph and replayed (no host work per level or per inner product;
// the host polls the device state every few iterations).
//   transport LOCAL: all slabs of the decomposition in this process (virtual
//     ranks on one GPU): halos are device copies, sums added in slab order.
//   transport NCCL: one slab per process/GPU: halos are ncclSend/ncclRecv
//     pairs with the two neighbours (peer to peer over NVLink), sums are one
//     ncclAllReduce of four doubles, the coarsest slabs one ncclAllGather.
//     NCCL is loaded at run time (hf_nccl_init) from the same libnccl the
//     caller's torch.distributed uses; its calls are captured in the graph.
// ---------------------------------------------------------------------------
#include <dlfcn.h>

namespace {
struct NcclId { char internal[128]; };
struct NcclApi {
    void *h = nullptr;
    int (*getUniqueId)(NcclId *) = nullptr;
    int (*commInitRank)(void **, int, NcclId, int) = nullptr;
    int (*commDestroy)(void *) = nullptr;
    int (*send)(const void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    int (*recv)(void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    int (*groupStart)() = nullptr;
    int (*groupEnd)() = nullptr;
    int (*allReduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
    int (*allGather)(const void *, void *, size_t, int, void *, cudaStream_t) = nullptr;
    const char *(*errorString)(int) = nullptr;
};
NcclApi g_nccl;
const int kNcclDouble = 8, kNcclSum = 0;
}  // namespace

extern "C" int hf_nccl_init(const char *libpath) {
    if (g_nccl.h) return 0;
    void *h = dlopen(libpath && *libpath ? libpath : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return fail(HF_ERR_UNSUPPORTED, std::string("cannot load NCCL: ") + dlerror());
    auto sym = [&](const char *n) { return dlsym(h, n); };
    g_nccl.getUniqueId = (int (*)(NcclId *))sym("ncclGetUniqueId");
    g_nccl.commInitRank = (int (*)(void **, int, NcclId, int))sym("ncclCommInitRank");
    g_nccl.commDestroy = (int (*)(void *))sym("ncclCommDestroy");
    g_nccl.send = (int (*)(const void *, size_t, int, int, void *, cudaStream_t))sym("ncclSend");
    g_nccl.recv = (int (*)(void *, size_t, int, int, void *, cudaStream_t))sym("ncclRecv");
    g_nccl.groupStart = (int (*)())sym("ncclGroupStart");
    g_nccl.groupEnd = (int (*)())sym("ncclGroupEnd");
    g_nccl.allReduce = (int (*)(const void *, void *, size_t, int, int, void *, cudaStream_t))sym("ncclAllReduce");
    g_nccl.allGather = (int (*)(const void *, void *, size_t, int, void *, cudaStream_t))sym("ncclAllGather");
    g_nccl.errorString = (const char *(*)(int))sym("ncclGetErrorString");
    if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.send || !g_nccl.recv || !g_nccl.groupStart ||
        !g_nccl.groupEnd || !g_nccl.allReduce || !g_nccl.allGather || !g_nccl.commDestroy)
        return fail(HF_ERR_UNSUPPORTED, "libnccl lacks the point-to-point / collective API");
    g_nccl.h = h;
    return 0;
}

extern "C" int hf_nccl_unique_id(void *out128) {
    if (!g_nccl.h) return fail(HF_ERR_ARG, "hf_nccl_init first");
    NcclId id;
    int r = g_nccl.getUniqueId(&id);
    if (r) return fail(HF_ERR_CUDA, "ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof(id));
    return 0;
}

struct SlabLocal {
    hf_operator *A = nullptr;
    hf_hierarchy *H = nullptr;
    long long n = 0;
    cd *x, *r, *rs, *p, *v, *ph, *s, *sh, *t;
};

struct hf_slab {
    Allocs A;
    int transport = HF_TRANSPORT_LOCAL, world = 1, rank = 0;
    std::vector<SlabLocal> sl;
    std::vector<int> clo, cnx;        // every slab's coarsest-level planes (global)
    int cmax = 0;
    long long cplane = 0;
    hf_hierarchy *Hc = nullptr;       // whole coarsest grid, exact solve, replicated
    cd *bc_full = nullptr, *xc_full = nullptr, *gpad = nullptr, *gsend = nullptr;
    std::vector<char> fuse_down;      // per level: HF_GHOST-deep halo + fused down kernel
    int nlev = 0;
    BcgState *st = nullptr, *st_host = nullptr;
    double *hist = nullptr;
    int hist_cap = 0;
    RedBuf red;
    cd *sums = nullptr;               // [nloc][3 parts][2] partial sums, then the total
    cudaStream_t cstream = nullptr;   // halo exchanges overlapped with interior planes
    cudaEvent_t evf = nullptr, evj = nullptr;
    cudaStream_t stream = nullptr;
    cudaGraphExec_t graph[2] = {nullptr, nullptr};   // [sparse shadow on this rank's slabs]
    int graph_kernels[2] = {0, 0};
    // sparse shadow: per local slab, the (<= HF_NZ_MAX) nonzeros of its part of r~ (only the
    // nz fields of the struct are used); r~ is then not streamed by the matvec / x, r update
    std::vector<BcgState *> nzst;
    BcgState *nz_host = nullptr;      // pinned, one per local slab
    bool sparse = false;
    void *comm = nullptr;
    ~hf_slab() {
        for (int k = 0; k < 2; k++)
            if (graph[k]) cudaGraphExecDestroy(graph[k]);
        if (nz_host) cudaFreeHost(nz_host);
        for (SlabLocal &q : sl) {
            if (q.H) hf_hierarchy_destroy(q.H);
            if (q.A) hf_operator_destroy(q.A);
        }
        if (Hc) hf_hierarchy_destroy(Hc);
        if (st_host) cudaFreeHost(st_host);
        if (comm && g_nccl.commDestroy) g_nccl.commDestroy(comm);
        if (evf) cudaEventDestroy(evf);
        if (evj) cudaEventDestroy(evj);
        if (cstream) cudaStreamDestroy(cstream);
        if (stream) cudaStreamDestroy(stream);
    }
};

extern "C" hf_slab *hf_slab_create(int n1, int n2, int n3, double h, double beta1, double beta2, int bc,
                                   const double *k_host, double k_const, const hf_mg_config *mg,
                                   int nloc, const int *lo1s, const int *nxs, int world, int rank,
                                   int transport, const void *nccl_id, int maxit) {
    if (!mg || nloc < 1 || !lo1s || !nxs || world < 1 || rank < 0 || rank >= world || maxit < 1) {
        fail(HF_ERR_ARG, "bad slab arguments");
        return nullptr;
    }
    if (mg->cycle != HF_CYCLE_V || mg->nu1 != 1 || mg->nu2 != 1) {
        fail(HF_ERR_UNSUPPORTED, "slab driver implements the V(1,1) cycle");
        return nullptr;
    }
    if (transport == HF_TRANSPORT_LOCAL && nloc != world) {
        fail(HF_ERR_ARG, "LOCAL transport: all slabs in this process (nloc == world)");
        return nullptr;
    }
    if (transport == HF_TRANSPORT_NCCL && (nloc != 1 || !nccl_id || !g_nccl.h)) {
        fail(HF_ERR_ARG, "NCCL transport: one slab per rank, hf_nccl_init and a unique id");
        return nullptr;
    }
    auto *S = new hf_slab();
    S->transport = transport; S->world = world; S->rank = rank;
    hf_mg_config c = *mg;
    c.coarsest_method = HF_COARSEST_EXTERNAL;
    cudaError_t e;
    for (int i = 0; i < nloc; i++) {
        SlabLocal q;
        q.A = hf_operator_create(n1, n2, n3, lo1s[i], nxs[i], h, 1.0, 0.0, bc, k_host, k_const);
        q.H = q.A ? hf_hierarchy_create(n1, n2, n3, lo1s[i], nxs[i], h, beta1, beta2, bc, k_host, k_const, &c)
                  : nullptr;
        if (!q.A || !q.H) { S->sl.push_back(q); delete S; return nullptr; }
        const Lvl &L = q.A->lv.L;
        q.n = (long long)L.nx * L.plane;
        cd **vecs[] = {&q.x, &q.r, &q.rs, &q.p, &q.v, &q.ph, &q.sh, &q.t};
        for (cd **pv : vecs) {
            *pv = new_field(S->A, L.nx, L.plane, e);
            if (!*pv) { S->sl.push_back(q); delete S; fail(HF_ERR_CUDA, "cudaMalloc slab vectors"); return nullptr; }
        }
        q.s = q.r;      // s lives in r's buffer (in-place s and x / r updates, as in hf_solver)
        S->sl.push_back(q);
    }
    S->nlev = (int)S->sl[0].H->lev.size();
    if (S->nlev < 2) {
        delete S;
        fail(HF_ERR_UNSUPPORTED, "slab driver needs at least two multigrid levels");
        return nullptr;
    }
    // every slab's extent per level (derive_coarse_extent, partition.py:120-131),
    // to decide the fused down kernel (every slab of level l owns >= HF_GHOST planes)
    // and to place the coarsest slabs
    std::vector<int> all_lo(world), all_nx(world);
    if (transport == HF_TRANSPORT_LOCAL) {
        for (int r = 0; r < world; r++) { all_lo[r] = lo1s[r]; all_nx[r] = nxs[r]; }
    } else {
        // balanced split along i1 (partition.py:103-117), the caller's decomposition
        const int base = n1 / world, rem = n1 % world;
        int lo = 0;
        for (int r = 0; r < world; r++) {
            all_lo[r] = lo;
            all_nx[r] = base + (r < rem ? 1 : 0);
            lo += all_nx[r];
        }
        if (all_lo[rank] != lo1s[0] || all_nx[rank] != nxs[0]) {
            delete S;
            fail(HF_ERR_ARG, "NCCL transport expects the balanced i1 split (slab_partition)");
            return nullptr;
        }
    }
    S->fuse_down.assign(S->nlev, 1);
    for (int l = 0; l < S->nlev; l++) {
        for (int r = 0; r < world; r++)
            if (all_nx[r] < HF_GHOST) S->fuse_down[l] = 0;
        if (l + 1 < S->nlev)
            for (int r = 0; r < world; r++) {
                const int clo = (all_lo[r] + 1) / 2, chi = (all_lo[r] + all_nx[r] - 1) / 2;
                all_lo[r] = clo;
                all_nx[r] = chi - clo + 1;
            }
    }
    S->clo = all_lo; S->cnx = all_nx;
    S->cmax = *std::max_element(all_nx.begin(), all_nx.end());
    // whole coarsest grid: exact solve replicated on every rank
    const Lvl &K = S->sl[0].H->lev.back().L;
    S->cplane = K.plane;
    std::vector<double> kc;
    const double *kcp = nullptr;
    if (k_host) {
        const int st = 1 << (S->nlev - 1);
        kc.resize((size_t)K.n1 * K.plane);
        for (int i = 0; i < K.n1; i++)
            for (int j = 0; j < K.n2; j++)
                for (int m = 0; m < K.n3; m++)
                    kc[((size_t)i * K.n2 + j) * K.n3 + m] = k_host[((size_t)(st * i) * n2 + st * j) * n3 + st * m];
        kcp = kc.data();
    }
    hf_mg_config cc = *mg;
    cc.coarsest_method = HF_COARSEST_DIRECT;
    cc.coarsest_threshold = std::max(K.n1, std::max(K.n2, K.n3)) + 1;   // one level
    cc.threshold_ge = 0;
    S->Hc = hf_hierarchy_create(K.n1, K.n2, K.n3, 0, K.n1, K.h, beta1, beta2, bc, kcp, k_const, &cc);
    if (!S->Hc) { delete S; return nullptr; }
    S->bc_full = S->A.get<cd>((size_t)K.n1 * K.plane, e);
    S->xc_full = S->A.get<cd>((size_t)K.n1 * K.plane, e);
    if (transport == HF_TRANSPORT_NCCL) {
        S->gsend = S->A.get<cd>((size_t)S->cmax * K.plane, e);
        S->gpad = S->A.get<cd>((size_t)world * S->cmax * K.plane, e);
    }
    S->st = S->A.get<BcgState>(1, e);
    S->hist = S->A.get<double>((size_t)maxit + 2, e);
    S->hist_cap = maxit + 2;
    S->sums = S->A.get<cd>((size_t)(3 * nloc + 1) * 2, e);
    size_t nblk = VEC_BLOCKS_HOST;
    for (SlabLocal &q : S->sl)
        nblk = std::max<size_t>(nblk, std::max(march_blocks(q.A->lv.L), tile_blocks(q.A->lv.L)));
    if (!S->bc_full || !S->xc_full || !S->st || !S->hist || !S->sums || S->red.init(S->A, nblk + 64) ||
        (transport == HF_TRANSPORT_NCCL && (!S->gsend || !S->gpad)) ||
        cudaMallocHost(&S->st_host, sizeof(BcgState)) != cudaSuccess ||
        cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&S->cstream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&S->evf, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&S->evj, cudaEventDisableTiming) != cudaSuccess) {
        delete S;
        fail(HF_ERR_CUDA, "slab workspace allocation");
        return nullptr;
    }
    if (transport == HF_TRANSPORT_NCCL) {
        NcclId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        const int r = g_nccl.commInitRank(&S->comm, world, id, rank);
        if (r) {
            S->comm = nullptr;
            delete S;
            fail(HF_ERR_CUDA, std::string("ncclCommInitRank: ") + (g_nccl.errorString ? g_nccl.errorString(r) : "?"));
            return nullptr;
        }
    }
    return S;
}

extern "C" void hf_slab_destroy(hf_slab *S) { delete S; }

// fill `planes` ghost planes of level-l fields f[i] (owned plane 0) at interior faces
static int slab_halo(hf_slab *S, int l, const std::vector<cd *> &f, int planes, cudaStream_t s) {
    const int nloc = (int)S->sl.size();
    if (S->transport == HF_TRANSPORT_LOCAL) {
        for (int i = 0; i + 1 < nloc; i++) {
            const Lvl &a = S->sl[i].H->lev[l].L, &b = S->sl[i + 1].H->lev[l].L;
            const size_t bytes = (size_t)planes * a.plane * sizeof(cd);
            CK(cudaMemcpyAsync(f[i] + (size_t)a.nx * a.plane, f[i + 1], bytes, cudaMemcpyDeviceToDevice, s));
            CK(cudaMemcpyAsync(f[i + 1] - (size_t)planes * b.plane, f[i] + (size_t)(a.nx - planes) * a.plane,
                               bytes, cudaMemcpyDeviceToDevice, s));
        }
        return 0;
    }
    if (S->world == 1) return 0;
    const Lvl &L = S->sl[0].H->lev[l].L;
    const size_t cnt = (size_t)planes * L.plane * 2;   // doubles
    cd *o = f[0];
    int r = g_nccl.groupStart();
    if (S->rank > 0) {
        r |= g_nccl.send(o, cnt, kNcclDouble, S->rank - 1, S->comm, s);
        r |= g_nccl.recv(o - (size_t)planes * L.plane, cnt, kNcclDouble, S->rank - 1, S->comm, s);
    }
    if (S->rank < S->world - 1) {
        r |= g_nccl.send(o + (size_t)(L.nx - planes) * L.plane, cnt, kNcclDouble, S->rank + 1, S->comm, s);
        r |= g_nccl.recv(o + (size_t)L.nx * L.plane, cnt, kNcclDouble, S->rank + 1, S->comm, s);
    }
    r |= g_nccl.groupEnd();
    return r ? fail(HF_ERR_CUDA, "NCCL halo exchange") : 0;
}

// sum the partials of `parts` slots per slab (fixed slab, then part order) into
// `out`: the global total (LOCAL) or this rank's partial (NCCL, all-reduced next)
__global__ void k_sum_slabs(int nloc, int parts, const cd *sums, cd *out) {
    if (threadIdx.x >= 2) return;
    cd a = mk(0, 0);
    for (int i = 0; i < nloc; i++)
        for (int k = 0; k < parts; k++) a = cadd(a, sums[2 * (3 * i + k) + threadIdx.x]);
    out[threadIdx.x] = a;
}

// global sums of the slabs' partials (all local slabs, all ranks) -> scalar step `op`
static int slab_reduce_step(hf_slab *S, int op, cudaStream_t s, int parts = 1) {
    const int nloc = (int)S->sl.size();
    cd *tot = S->sums + 2 * 3 * nloc;
    if (S->transport == HF_TRANSPORT_LOCAL) {
        k_sum_slabs<<<1, 32, 0, s>>>(nloc, parts, S->sums, tot);
    } else {
        const cd *src = S->sums;
        if (parts > 1) {
            k_sum_slabs<<<1, 32, 0, s>>>(nloc, parts, S->sums, S->sums + 2);   // into part 1 of slab 0
            src = S->sums + 2;
        }
        if (g_nccl.allReduce(src, tot, 4, kNcclDouble, kNcclSum, S->comm, s))
            return fail(HF_ERR_CUDA, "NCCL all-reduce");
    }
    launch_bcg_step(S->st, op, tot, s);
    g_launches += 2;
    return 0;
}

static RedSlot slab_store(hf_slab *S, int i, int part = 0) {
    RedSlot r = S->red.slot(FIN_STORE, nullptr);
    r.out = S->sums + 2 * (3 * i + part);
    return r;
}

// planes [p0, p1) of a slab level as a slab of its own: the kernels read the
// planes either side of the range as ghost planes, so a range of interior
// planes needs no halo
static Lvl sub_slab(const Lvl &L, int p0, int p1) {
    Lvl o = L;
    o.lo1 = L.lo1 + p0;
    o.nx = p1 - p0;
    if (L.k) o.k = L.k + (size_t)p0 * L.plane;
    if (L.dinv) o.dinv = L.dinv + (size_t)p0 * L.plane;
    if (L.kidx) o.kidx = L.kidx + (size_t)p0 * L.plane;
    return o;
}

// halo exchange on the comm stream, overlapped with `interior` on the main
// stream; `boundary` runs after both (the ghost planes have arrived)
template <class FI, class FB>
static int overlapped(hf_slab *S, int l, const std::vector<cd *> &f, int planes, cudaStream_t s,
                      FI &&interior, FB &&boundary) {
    CK(cudaEventRecord(S->evf, s));
    CK(cudaStreamWaitEvent(S->cstream, S->evf, 0));
    if (slab_halo(S, l, f, planes, S->cstream)) return HF_ERR_CUDA;
    CK(cudaEventRecord(S->evj, S->cstream));
    interior();
    CK(cudaStreamWaitEvent(s, S->evj, 0));
    boundary();
    return 0;
}

// coarse planes [c0, c1) (local) of slab level C whose fine planes [2gc - rad,
// 2gc + rad] (global) all lie in the owned fine planes of F
static void coarse_interior(const Lvl &F, const Lvl &C, int rad, int &c0, int &c1) {
    const int flo = F.lo1, fhi = F.lo1 + F.nx - 1;
    int g0 = (flo + rad + 1) / 2, g1 = (fhi - rad) / 2;       // ceil, floor
    g0 = std::max(g0, C.lo1);
    g1 = std::min(g1, C.lo1 + C.nx - 1);
    c0 = g0 - C.lo1;
    c1 = std::max(c0, g1 - C.lo1 + 1);
}

// one V(1,1) cycle over the slabs: dst[i] ~= M^-1 src[i] (multigrid.py:326-343).
// Each level's halo exchange overlaps the part of the level kernel that needs
// no ghost planes (interior planes launched as a sub-slab); the face planes
// follow once the ghost planes have arrived.
static int slab_cycle(hf_slab *S, const std::vector<cd *> &src, const std::vector<cd *> &dst, cudaStream_t s) {
    const int nloc = (int)S->sl.size(), nl = S->nlev;
    const int *done = &S->st->done;
    const double om = S->sl[0].H->cfg.omega;
    auto bl = [&](int i, int l) { return l == 0 ? src[i] : S->sl[i].H->lev[l].b; };
    auto ul = [&](int i, int l) { return l == 0 ? dst[i] : S->sl[i].H->lev[l].u; };
    std::vector<cd *> f(nloc);
    for (int l = 0; l < nl - 1; l++) {
        for (int i = 0; i < nloc; i++) f[i] = bl(i, l);
        const bool fuse = S->fuse_down[l] && (flat_dr_ok(S->sl[0].H->lev[l].L) || opt(OPT_TILED_DR)) &&
                          !opt(OPT_NO_DR);
        if (fuse) {
            // b_c = R (b - M (w D^-1 b)): coarse planes reading fine planes 2gc-2 .. 2gc+2
            auto part = [&](bool inner) {
                for (int i = 0; i < nloc; i++) {
                    Level &lv = S->sl[i].H->lev[l], &nx = S->sl[i].H->lev[l + 1];
                    int c0, c1;
                    coarse_interior(lv.L, nx.L, 2, c0, c1);
                    auto run = [&](int a, int b2) {
                        if (b2 <= a) return;
                        launch_down_restrict(lv.L, sub_slab(nx.L, a, b2), f[i], nx.b + (size_t)a * nx.L.plane,
                                             om, s, done);
                        g_launches++;
                    };
                    if (inner) run(c0, c1);
                    else { run(0, c0); run(std::max(c1, c0), nx.L.nx); }
                }
            };
            if (overlapped(S, l, f, HF_GHOST, s, [&] { part(true); }, [&] { part(false); })) return HF_ERR_CUDA;
            continue;
        }
        // split pair: r = b - M (w D^-1 b) on fine planes, then b_c = R r
        std::vector<cd *> rr(nloc);
        for (int i = 0; i < nloc; i++) rr[i] = S->sl[i].H->lev[l].r;
        auto down = [&](bool inner) {
            for (int i = 0; i < nloc; i++) {
                Level &lv = S->sl[i].H->lev[l];
                const int nx = lv.L.nx;
                auto run = [&](int a, int b2) {
                    if (b2 <= a) return;
                    const size_t o = (size_t)a * lv.L.plane;
                    launch_down1(sub_slab(lv.L, a, b2), f[i] + o, lv.r + o, om, s, done);
                    g_launches++;
                };
                if (nx > 2) {
                    if (inner) run(1, nx - 1);
                    else { run(0, 1); run(nx - 1, nx); }
                } else if (!inner) {
                    run(0, nx);
                }
            }
        };
        if (overlapped(S, l, f, 1, s, [&] { down(true); }, [&] { down(false); })) return HF_ERR_CUDA;
        auto restr = [&](bool inner) {
            for (int i = 0; i < nloc; i++) {
                Level &lv = S->sl[i].H->lev[l], &nx = S->sl[i].H->lev[l + 1];
                int c0, c1;
                coarse_interior(lv.L, nx.L, 1, c0, c1);
                auto run = [&](int a, int b2) {
                    if (b2 <= a) return;
                    launch_restrict(lv.L, sub_slab(nx.L, a, b2), lv.r, nx.b + (size_t)a * nx.L.plane, s, done);
                    g_launches++;
                };
                if (inner) run(c0, c1);
                else { run(0, c0); run(std::max(c1, c0), nx.L.nx); }
            }
        };
        if (overlapped(S, l, rr, 1, s, [&] { restr(true); }, [&] { restr(false); })) return HF_ERR_CUDA;
    }
    // coarsest: gather every slab's planes into the whole grid, exact solve, scatter
    const size_t cpb = (size_t)S->cplane * sizeof(cd);
    if (S->transport == HF_TRANSPORT_LOCAL) {
        for (int i = 0; i < nloc; i++)
            CK(cudaMemcpyAsync(S->bc_full + (size_t)S->clo[i] * S->cplane, S->sl[i].H->lev[nl - 1].b,
                               S->cnx[i] * cpb, cudaMemcpyDeviceToDevice, s));
    } else {
        CK(cudaMemcpyAsync(S->gsend, S->sl[0].H->lev[nl - 1].b, S->cnx[S->rank] * cpb, cudaMemcpyDeviceToDevice, s));
        if (g_nccl.allGather(S->gsend, S->gpad, (size_t)S->cmax * S->cplane * 2, kNcclDouble, S->comm, s))
            return fail(HF_ERR_CUDA, "NCCL all-gather");
        for (int r = 0; r < S->world; r++)
            CK(cudaMemcpyAsync(S->bc_full + (size_t)S->clo[r] * S->cplane, S->gpad + (size_t)r * S->cmax * S->cplane,
                               S->cnx[r] * cpb, cudaMemcpyDeviceToDevice, s));
    }
    coarsest(S->Hc, S->bc_full, S->xc_full, s, done);
    for (int i = 0; i < nloc; i++) {
        const int r = S->transport == HF_TRANSPORT_LOCAL ? i : S->rank;
        CK(cudaMemcpyAsync(S->sl[i].H->lev[nl - 1].u, S->xc_full + (size_t)S->clo[r] * S->cplane,
                           S->cnx[r] * cpb, cudaMemcpyDeviceToDevice, s));
    }
    for (int l = nl - 2; l >= 0; l--) {
        for (int i = 0; i < nloc; i++) f[i] = S->sl[i].H->lev[l + 1].u;
        // t = w D^-1 b + P e: fine planes whose coarse planes (gi >> 1, + 1 when odd)
        // are owned need no ghost plane of e; the rest (and t on the interior-face
        // ghost planes, so the sweep needs no halo of t) after the exchange
        auto corr = [&](bool inner) {
            for (int i = 0; i < nloc; i++) {
                Level &lv = S->sl[i].H->lev[l], &nx = S->sl[i].H->lev[l + 1];
                const int nxf = lv.L.nx;
                int a = 0, b2 = nxf;                              // interior fine planes [a, b2)
                while (a < nxf && ((lv.L.lo1 + a) >> 1) < nx.L.lo1) a++;
                while (b2 > a && (((lv.L.lo1 + b2 - 1) >> 1) + ((lv.L.lo1 + b2 - 1) & 1)) > nx.L.lo1 + nx.L.nx - 1) b2--;
                auto run = [&](int p0, int p1, bool ghosts) {
                    if (p1 <= p0) return;
                    const size_t o = (size_t)p0 * lv.L.plane;
                    launch_correct(sub_slab(lv.L, p0, p1), nx.L, bl(i, l) + o, nx.u, lv.t + o, om, true, s, done,
                                   ghosts);
                    g_launches++;
                };
                if (inner) {
                    run(a, b2, false);
                } else {
                    // the face ranges; ghost planes only where the slab face is interior
                    const bool glo = lv.L.lo1 > 0, ghi = lv.L.lo1 + nxf < lv.L.n1;
                    if (a > 0) run(0, a, glo);
                    else if (glo) run(0, std::min(1, nxf), true);   // ghost plane below (and plane 0 again)
                    if (b2 < nxf) run(std::max(b2, a), nxf, ghi);
                    else if (ghi) run(nxf - 1, nxf, true);
                }
            }
        };
        // wide levels: prolongation + correction + Jacobi sweep in ONE pass of the wide family
        // (hf_wide.cu WIDE_UP; the correction t is never written).  The sweep transforms one
        // plane beyond each end of its range, so the planes [a + 1, b2 - 1) need no ghost
        // plane of e and overlap its exchange; the two face ranges follow.
        const bool wide_up = wide_ok(S->sl[0].H->lev[l].L, 6) && !opt(OPT_NO_WIDE_UP) && !opt(OPT_NO_FUSE);
        auto upw = [&](bool inner) {
            for (int i = 0; i < nloc; i++) {
                Level &lv = S->sl[i].H->lev[l], &nx = S->sl[i].H->lev[l + 1];
                const int nxf = lv.L.nx;
                const bool glo = lv.L.lo1 > 0, ghi = lv.L.lo1 + nxf < lv.L.n1;
                int a = 0, b2 = nxf;
                while (a < nxf && ((lv.L.lo1 + a) >> 1) < nx.L.lo1) a++;
                while (b2 > a && (((lv.L.lo1 + b2 - 1) >> 1) + ((lv.L.lo1 + b2 - 1) & 1)) > nx.L.lo1 + nx.L.nx - 1) b2--;
                const int p0 = glo ? std::min(a + 1, nxf) : 0, p1 = ghi ? std::max(b2 - 1, p0) : nxf;
                auto run = [&](int q0, int q1) {
                    if (q1 <= q0) return;
                    const size_t o = (size_t)q0 * lv.L.plane;
                    launch_wide_up(sub_slab(lv.L, q0, q1), nx.L, bl(i, l) + o, nx.u, ul(i, l) + o, om, true, s, done);
                    g_launches++;
                };
                if (inner) {
                    run(p0, p1);
                } else {
                    run(0, p0);
                    run(p1, nxf);
                }
            }
        };
        if (wide_up) {
            if (overlapped(S, l + 1, f, 1, s, [&] { upw(true); }, [&] { upw(false); })) return HF_ERR_CUDA;
            continue;
        }
        if (overlapped(S, l + 1, f, 1, s, [&] { corr(true); }, [&] { corr(false); })) return HF_ERR_CUDA;
        for (int i = 0; i < nloc; i++) {
            Level &lv = S->sl[i].H->lev[l];
            launch_jacobi(lv.L, lv.t, bl(i, l), ul(i, l), om, s, done);
        }
        g_launches += nloc;
    }
    return 0;
}

// v = A u with this slab's inner products, the halo exchange of u overlapped
// with the interior planes: the exchange runs on the comm stream while the
// interior planes [1, nx-1) (which read only owned planes) are swept on the main
// stream; the two face planes follow once the ghost planes have arrived.  The
// three launches store separate partial sums (parts 0..2).
static int slab_matvec(hf_slab *S, int nd, const std::vector<cd *> &u, cudaStream_t s) {
    const int nloc = (int)S->sl.size();
    const int *done = &S->st->done;
    auto mv = [&](int i, int p0, int p1, int part) {
        SlabLocal &q = S->sl[i];
        const Lvl &L = q.A->lv.L;
        const size_t off = (size_t)p0 * L.plane;
        const Lvl Ls = sub_slab(L, p0, p1);
        if (nd == 1 && S->sparse)      // r~^H v gathered below: a plain matvec
            launch_apply(Ls, u[i] + off, q.v + off, s, done);
        else if (nd == 1)
            launch_apply_dot1(Ls, u[i] + off, q.v + off, q.rs + off, slab_store(S, i, part), s, done);
        else
            launch_apply_dot2(Ls, u[i] + off, q.t + off, q.s + off, slab_store(S, i, part), s, done);
        g_launches++;
    };
    CK(cudaMemsetAsync(S->sums, 0, (size_t)3 * nloc * sizeof(cd) * 2, s));
    CK(cudaEventRecord(S->evf, s));
    CK(cudaStreamWaitEvent(S->cstream, S->evf, 0));
    if (slab_halo(S, 0, u, 1, S->cstream)) return HF_ERR_CUDA;
    CK(cudaEventRecord(S->evj, S->cstream));
    for (int i = 0; i < nloc; i++) {
        const int nx = S->sl[i].A->lv.L.nx;
        if (nx > 2) mv(i, 1, nx - 1, 0);
    }
    CK(cudaStreamWaitEvent(s, S->evj, 0));
    for (int i = 0; i < nloc; i++) {
        const int nx = S->sl[i].A->lv.L.nx;
        if (nx > 2) {
            mv(i, 0, 1, 1);
            mv(i, nx - 1, nx, 2);
        } else {
            mv(i, 0, nx, 1);
        }
    }
    if (nd == 1 && S->sparse)
        for (int i = 0; i < nloc; i++) {
            launch_gather_store(S->nzst[i], S->sl[i].v, S->sums + 2 * (3 * i), s, done);
            g_launches++;
        }
    return 0;
}

static int slab_iteration(hf_slab *S, cudaStream_t s) {
    const int nloc = (int)S->sl.size();
    const int *done = &S->st->done;
    std::vector<cd *> src(nloc), dst(nloc);
    for (int i = 0; i < nloc; i++) {
        SlabLocal &q = S->sl[i];
        L1(launch_bcg_p(q.n, S->st, q.r, q.p, q.v, s, done));
        src[i] = q.p; dst[i] = q.ph;
    }
    if (slab_cycle(S, src, dst, s)) return HF_ERR_CUDA;
    if (slab_matvec(S, 1, dst, s)) return HF_ERR_CUDA;
    if (slab_reduce_step(S, FIN_BCG_ALPHA, s, 3)) return HF_ERR_CUDA;
    for (int i = 0; i < nloc; i++) {
        SlabLocal &q = S->sl[i];
        L1(launch_bcg_s(q.n, S->st, q.r, q.v, q.s, slab_store(S, i), s, done));
        src[i] = q.s; dst[i] = q.sh;
    }
    if (slab_reduce_step(S, FIN_BCG_S, s)) return HF_ERR_CUDA;
    if (slab_cycle(S, src, dst, s)) return HF_ERR_CUDA;
    if (slab_matvec(S, 2, dst, s)) return HF_ERR_CUDA;
    if (slab_reduce_step(S, FIN_BCG_OMEGA, s, 3)) return HF_ERR_CUDA;
    for (int i = 0; i < nloc; i++) {
        SlabLocal &q = S->sl[i];
        L1(launch_bcg_xr(q.n, S->st, q.x, q.ph, q.sh, q.s, q.t, q.r, S->sparse ? nullptr : q.rs,
                         slab_store(S, i), s, done));
        if (S->sparse) L1(launch_gather_store(S->nzst[i], q.r, S->sums + 2 * (3 * i) + 1, s, done));
    }
    if (slab_reduce_step(S, FIN_BCG_RHO, s)) return HF_ERR_CUDA;
    CK(cudaMemcpyAsync(S->st_host, S->st, sizeof(BcgState), cudaMemcpyDeviceToHost, s));
    return 0;
}

// b_slabs / x_slabs: per local slab, device pointers to the owned planes
extern "C" int hf_slab_solve(hf_slab *S, const hf_solver_config *cfg, const double *const *b_slabs,
                             double *const *x_slabs, hf_report *rep) {
    if (!S || !cfg || !b_slabs || !x_slabs || !rep) return fail(HF_ERR_ARG, "null argument");
    if (cfg->method != HF_METHOD_BICGSTAB) return fail(HF_ERR_UNSUPPORTED, "slab driver runs Bi-CGSTAB");
    if (cfg->maxit + 2 > S->hist_cap) return fail(HF_ERR_ARG, "maxit above the slab solver's capacity");
    cudaStream_t s = S->stream, us = work_stream();
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaEventRecord(ev, us));                 // order after the caller's stream
    CK(cudaStreamWaitEvent(s, ev, 0));
    const int nloc = (int)S->sl.size();
    BcgState init{};
    init.tol = cfg->tol;
    init.btol = cfg->breakdown_tol > 0 ? cfg->breakdown_tol : 1e-30;
    init.maxit = cfg->maxit;
    init.hist = S->hist;
    init.hist_cap = S->hist_cap;
    *S->st_host = init;
    CK(cudaMemcpyAsync(S->st, S->st_host, sizeof(BcgState), cudaMemcpyHostToDevice, s));
    long long launches = 0;
    const int shadow = cfg->shadow_kind == HF_SHADOW_HASH ? HF_SHADOW_HASH : HF_SHADOW_RHS;
    for (int i = 0; i < nloc; i++) {
        SlabLocal &q = S->sl[i];
        const Lvl &L = q.A->lv.L;
        launch_bcg_init(q.n, (const cd *)b_slabs[i], q.r, q.rs, q.x, q.p, q.v, slab_store(S, i), s, shadow,
                        cfg->shadow_seed, (long long)L.lo1 * L.plane);
        launches++;
    }
    if (slab_reduce_step(S, FIN_BCG_INIT, s)) return HF_ERR_CUDA;
    CK(cudaMemcpyAsync(S->st_host, S->st, sizeof(BcgState), cudaMemcpyDeviceToHost, s));
    // nonzeros of this rank's parts of r~ (a point source with r~ = b: at most one slab has any)
    if (S->nzst.empty()) {
        cudaError_t e2;
        for (int i = 0; i < nloc; i++) {
            S->nzst.push_back(S->A.get<BcgState>(1, e2));
            if (!S->nzst.back()) return fail(HF_ERR_CUDA, "cudaMalloc slab nonzero list");
        }
        if (cudaMallocHost(&S->nz_host, nloc * sizeof(BcgState)) != cudaSuccess)
            return fail(HF_ERR_CUDA, "cudaMallocHost slab nonzero list");
    }
    for (int i = 0; i < nloc; i++) {
        CK(cudaMemsetAsync(S->nzst[i], 0, sizeof(BcgState), s));
        launch_nz_scan(S->sl[i].n, S->sl[i].rs, S->nzst[i], s);
        CK(cudaMemcpyAsync(S->nz_host + i, S->nzst[i], sizeof(BcgState), cudaMemcpyDeviceToHost, s));
        launches += 2;
    }
    CK(cudaStreamSynchronize(s));
    S->sparse = true;
    for (int i = 0; i < nloc; i++) S->sparse = S->sparse && S->nz_host[i].nz_count <= HF_NZ_MAX;
    const int gi = S->sparse ? 1 : 0;
    if (!S->graph[gi]) {
        cudaGraph_t g;
        long long before = g_launches;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const int rc = slab_iteration(S, s);
        cudaError_t e = cudaStreamEndCapture(s, &g);
        if (rc) return rc;
        if (e != cudaSuccess) return fail(HF_ERR_CUDA, std::string("slab graph capture: ") + cudaGetErrorString(e));
        S->graph_kernels[gi] = (int)(g_launches - before);
        g_launches = before;
        e = cudaGraphInstantiate(&S->graph[gi], g, 0);
        cudaGraphDestroy(g);
        if (e != cudaSuccess) return fail(HF_ERR_CUDA, std::string("slab graph instantiate: ") + cudaGetErrorString(e));
    }
    const int every = cfg->check_every > 0 ? cfg->check_every : 4;
    int graphs = 0;
    while (!S->st_host->done && graphs < cfg->maxit + every) {
        for (int k = 0; k < every; k++) {
            CK(cudaGraphLaunch(S->graph[gi], s));
            graphs++;
        }
        CK(cudaStreamSynchronize(s));
    }
    launches += (long long)graphs * S->graph_kernels[gi];
    for (int i = 0; i < nloc; i++) {
        SlabLocal &q = S->sl[i];
        if (S->st_host->s_conv) {
            launch_bcg_xhalf(q.n, S->st, q.x, q.ph, s);
            launches++;
        }
        CK(cudaMemcpyAsync(x_slabs[i], q.x, (size_t)q.n * sizeof(cd), cudaMemcpyDeviceToDevice, s));
    }
    CK(cudaStreamSynchronize(s));
    CK(cudaEventRecord(ev, s));
    CK(cudaStreamWaitEvent(us, ev, 0));
    cudaEventDestroy(ev);
    CKL();
    const BcgState &st = *S->st_host;
    rep->matvec_count = st.matvecs;
    rep->iterations = st.iter;
    rep->converged = st.converged;
    rep->breakdown = st.breakdown;
    rep->final_relres = st.relres;
    rep->solve_ms = 0;
    rep->kernel_launches = (int)launches;
    rep->coarsest_flags = 0;
    if (rep->history_host && rep->history_cap > 0 && st.iter > 0)
        CK(cudaMemcpy(rep->history_host, S->hist, (size_t)std::min(st.iter, rep->history_cap) * sizeof(double),
                      cudaMemcpyDeviceToHost));
    return 0;
}
