/*
 * helmfree_oracle.c -- CPU restatement of the reference CSLP/multigrid/Krylov
 * path (arxiv 2308.06085, reference package `helmfree`).
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path and the `cpu_baseline` / `--impl reference` arm of bench.py.
 * Nothing in paper_2308_06085_b200/ may link, import or call it.
 *
 * Every routine restates one reference function (file:line under
 * /root/reference/pkg/src/helmfree/).  Layout: full-grid arrays of shape
 * (n1, n2, n3), C order (i3 fastest) -- the same as the reference's numpy
 * arrays.  Complex values are C99 `double complex` (re, im interleaved).
 *
 * Deterministic reductions: dot products are summed over a fixed number of
 * contiguous chunks (independent of the OpenMP thread count), then the chunk
 * partials are summed in order.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef double complex cplx;

#define BC_DIRICHLET 0
#define BC_SOMMERFELD 1

/* ------------------------------------------------------------------------ */
/* level description                                                         */
/* ------------------------------------------------------------------------ */
typedef struct {
    int n1, n2, n3;
    double h;
    cplx shift;          /* beta1 - i*beta2  (operators.py:95-99) */
    int bc;
    double *k;           /* per-vertex wavenumber, owned by this struct */
    cplx *diag;          /* Jacobi diagonal (operators.py:163-183) */
    cplx *ap;            /* stencil centre incl. Sommerfeld terms */
    /* scratch, like MGLevel (multigrid.py:54-71) */
    cplx *u, *b, *r, *tmp;
} or_level;

static inline size_t idx3(const or_level *L, int i, int j, int m) {
    return ((size_t)i * L->n2 + j) * L->n3 + m;
}
static inline size_t npts(const or_level *L) {
    return (size_t)L->n1 * L->n2 * L->n3;
}

static void *xcalloc(size_t n, size_t sz) {
    void *p = calloc(n ? n : 1, sz);
    if (!p) abort();
    return p;
}

/* operators.py:163-183: ap = (6 - s k^2 h^2)/h^2, Sommerfeld subtracts 2ik/h
 * once per adjacent physical face; Dirichlet diag = 1 on boundary planes. */
static void level_build_diag(or_level *L) {
    size_t n = npts(L);
    L->ap = (cplx *)xcalloc(n, sizeof(cplx));
    L->diag = (cplx *)xcalloc(n, sizeof(cplx));
    const double h = L->h, h2 = L->h * L->h;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < L->n1; i++)
        for (int j = 0; j < L->n2; j++)
            for (int m = 0; m < L->n3; m++) {
                size_t q = idx3(L, i, j, m);
                double kk = L->k[q];
                double k2 = kk * kk;
                cplx ap = (6.0 - L->shift * k2 * h2) / h2;
                int nb = (i == 0) + (i == L->n1 - 1) + (j == 0) + (j == L->n2 - 1) +
                         (m == 0) + (m == L->n3 - 1);
                if (L->bc == BC_SOMMERFELD) {
                    /* sequential per-face subtraction as in the reference loop */
                    for (int f = 0; f < nb; f++) ap -= 2.0 * I * kk / h;
                    L->ap[q] = ap;
                    L->diag[q] = ap;
                } else {
                    L->ap[q] = ap;
                    L->diag[q] = nb ? 1.0 : ap;
                }
            }
}

/* operators.py:200-254 (StencilOperator.apply): v = M u on the full grid.
 * Physical ghosts are zero; Sommerfeld rows add the doubled inward neighbour;
 * Dirichlet boundary rows are identities. */
void or_apply_level(const or_level *L, const cplx *u, cplx *v) {
    const int n1 = L->n1, n2 = L->n2, n3 = L->n3;
    const double ih2 = 1.0 / (L->h * L->h);
    const int dir = L->bc == BC_DIRICHLET;
    #pragma omp parallel for schedule(static)
    for (int i = 0; i < n1; i++)
        for (int j = 0; j < n2; j++)
            for (int m = 0; m < n3; m++) {
                size_t q = idx3(L, i, j, m);
                cplx xm = i > 0 ? u[q - (size_t)n2 * n3] : 0.0;
                cplx xp = i < n1 - 1 ? u[q + (size_t)n2 * n3] : 0.0;
                cplx ym = j > 0 ? u[q - n3] : 0.0;
                cplx yp = j < n2 - 1 ? u[q + n3] : 0.0;
                cplx zm = m > 0 ? u[q - 1] : 0.0;
                cplx zp = m < n3 - 1 ? u[q + 1] : 0.0;
                cplx nb = (xm + xp) + (ym + yp) + (zm + zp);
                cplx val = L->ap[q] * u[q];
                val -= ih2 * nb;
                int onb = (i == 0) || (i == n1 - 1) || (j == 0) || (j == n2 - 1) ||
                          (m == 0) || (m == n3 - 1);
                if (onb) {
                    if (dir) {
                        val = u[q];
                    } else {
                        /* faces in the reference's order: dim0 lo/hi, dim1, dim2 */
                        if (i == 0) val -= ih2 * u[q + (size_t)n2 * n3];
                        if (i == n1 - 1) val -= ih2 * u[q - (size_t)n2 * n3];
                        if (j == 0) val -= ih2 * u[q + n3];
                        if (j == n2 - 1) val -= ih2 * u[q - n3];
                        if (m == 0) val -= ih2 * u[q + 1];
                        if (m == n3 - 1) val -= ih2 * u[q - 1];
                    }
                }
                v[q] = val;
            }
}

/* ------------------------------------------------------------------------ */
/* vector helpers and deterministic dot (partition.py:611-621)               */
/* ------------------------------------------------------------------------ */
#define OR_DOT_CHUNKS_MAX 4096
static int or_dot_chunks = 256;
void or_set_dot_chunks(int c) {
    or_dot_chunks = c < 1 ? 1 : (c > OR_DOT_CHUNKS_MAX ? OR_DOT_CHUNKS_MAX : c);
}

cplx or_vdot(size_t n, const cplx *a, const cplx *b) {
    const int OR_DOT_CHUNKS = or_dot_chunks;
    cplx part[OR_DOT_CHUNKS_MAX];
    size_t chunk = (n + OR_DOT_CHUNKS - 1) / OR_DOT_CHUNKS;
    #pragma omp parallel for schedule(static)
    for (int c = 0; c < OR_DOT_CHUNKS; c++) {
        size_t lo = (size_t)c * chunk, hi = lo + chunk;
        if (hi > n) hi = n;
        cplx s = 0.0;
        for (size_t q = lo; q < hi; q++) s += conj(a[q]) * b[q];
        part[c] = s;
    }
    cplx s = 0.0;
    for (int c = 0; c < OR_DOT_CHUNKS; c++) s += part[c];
    return s;
}

static double or_norm(size_t n, const cplx *a) {
    double d = creal(or_vdot(n, a, a));
    return sqrt(d > 0.0 ? d : 0.0);
}

/* ------------------------------------------------------------------------ */
/* multigrid kernels                                                         */
/* ------------------------------------------------------------------------ */

/* multigrid.py:138-157: damped Jacobi, u <- u + w D^-1 (b - M u). */
void or_jacobi_level(const or_level *L, cplx *u, const cplx *b, double omega, int sweeps,
                     cplx *scratch, int assume_zero) {
    size_t n = npts(L);
    int first = assume_zero;
    for (int s = 0; s < sweeps; s++) {
        if (first) {
            #pragma omp parallel for schedule(static)
            for (size_t q = 0; q < n; q++) u[q] = omega * (b[q] / L->diag[q]);
            first = 0;
            continue;
        }
        or_apply_level(L, u, scratch);
        #pragma omp parallel for schedule(static)
        for (size_t q = 0; q < n; q++) {
            cplx resid = b[q] - scratch[q];
            u[q] += omega * (resid / L->diag[q]);
        }
    }
}

/* multigrid.py:171-221: 27-point full weighting; out-of-domain taps dropped;
 * coarse physical boundary planes zeroed (Dirichlet) or scaled by 64/48 per
 * boundary direction (Sommerfeld). */
void or_restrict_level(const or_level *F, const or_level *C, const cplx *rf, cplx *out) {
    static const double w1[3] = {1.0, 2.0, 1.0};
    const int dir = C->bc == BC_DIRICHLET;
    #pragma omp parallel for schedule(static)
    for (int ci = 0; ci < C->n1; ci++)
        for (int cj = 0; cj < C->n2; cj++)
            for (int cm = 0; cm < C->n3; cm++) {
                cplx acc = 0.0;
                for (int o1 = -1; o1 <= 1; o1++)
                    for (int o2 = -1; o2 <= 1; o2++)
                        for (int o3 = -1; o3 <= 1; o3++) {
                            int fi = 2 * ci + o1, fj = 2 * cj + o2, fm = 2 * cm + o3;
                            double w = w1[o1 + 1] * w1[o2 + 1] * w1[o3 + 1];
                            cplx val = 0.0;
                            if (fi >= 0 && fi < F->n1 && fj >= 0 && fj < F->n2 && fm >= 0 &&
                                fm < F->n3)
                                val = rf[idx3(F, fi, fj, fm)];
                            acc += w * val;
                        }
                acc /= 64.0;
                int on[3] = {ci == 0 || ci == C->n1 - 1, cj == 0 || cj == C->n2 - 1,
                             cm == 0 || cm == C->n3 - 1};
                /* lo and hi of the same dim are separate passes in the reference
                 * (only matters for n==1 which cannot occur: n >= 3) */
                for (int d = 0; d < 3; d++) {
                    if (!on[d]) continue;
                    if (dir) acc = 0.0;
                    else acc *= 64.0 / 48.0;
                }
                out[idx3(C, ci, cj, cm)] = acc;
            }
}

/* multigrid.py:238-297: trilinear prolongation; coincident fine vertices copy,
 * others average 2/4/8 coarse neighbours (sum, then divide by the count). */
void or_prolong_level(const or_level *C, const or_level *F, const cplx *ec, cplx *out) {
    #pragma omp parallel for schedule(static)
    for (int fi = 0; fi < F->n1; fi++)
        for (int fj = 0; fj < F->n2; fj++)
            for (int fm = 0; fm < F->n3; fm++) {
                int odd1 = (fi % 2) == 0, odd2 = (fj % 2) == 0, odd3 = (fm % 2) == 0;
                int c1 = fi / 2, c2 = fj / 2, c3 = fm / 2;
                int e1 = odd1 ? 1 : 2, e2 = odd2 ? 1 : 2, e3 = odd3 ? 1 : 2;
                cplx acc = 0.0;
                int first = 1;
                for (int d1 = 0; d1 < e1; d1++)
                    for (int d2 = 0; d2 < e2; d2++)
                        for (int d3 = 0; d3 < e3; d3++) {
                            cplx v = ec[idx3(C, c1 + d1, c2 + d2, c3 + d3)];
                            if (first) { acc = v; first = 0; }
                            else acc = acc + v;
                        }
                int ns = e1 * e2 * e3;
                if (ns > 1) acc = acc / (double)ns;
                out[idx3(F, fi, fj, fm)] = acc;
            }
}

/* ------------------------------------------------------------------------ */
/* Krylov solvers (krylov.py)                                                */
/* ------------------------------------------------------------------------ */
typedef void (*or_op_fn)(void *ctx, const cplx *x, cplx *y);

typedef struct {
    int matvec_count;
    int iterations;
    int converged;
    int breakdown;        /* 0 none, 1 arnoldi, 2 rho, 3 omega, 4 projection */
    double final_relres;
    double *history;      /* caller-provided, length >= maxit + 1 (may be NULL) */
    int history_cap;
} or_report;

static void rep_record(or_report *rep, double relres) {
    if (rep->history && rep->iterations < rep->history_cap)
        rep->history[rep->iterations] = relres;
    rep->iterations++;
    rep->final_relres = relres;
}

/* krylov.py:97-108 complex Givens rotation */
static void givens(cplx a, cplx b, double *c, cplx *s, cplx *r) {
    double absa = cabs(a), absb = cabs(b);
    if (absb == 0.0) { *c = 1.0; *s = 0.0; *r = a; return; }
    if (absa == 0.0) { *c = 0.0; *s = conj(b) / absb; *r = absb; return; }
    double t = hypot(absa, absb);
    *c = absa / t;
    *s = (a / absa) * (conj(b) / t);
    *r = (a / absa) * t;
}

/* krylov.py:111-192: full (restartable) left-preconditioned GMRES, MGS Arnoldi,
 * Givens least squares; zero initial guess.  minv == NULL means identity. */
void or_gmres(size_t n, or_op_fn A, void *actx, or_op_fn minv, void *mctx, const cplx *b,
              cplx *x, double tol, int maxit, int restart, double breakdown_tol,
              or_report *rep) {
    memset(x, 0, n * sizeof(cplx));
    rep->matvec_count = rep->iterations = rep->converged = rep->breakdown = 0;
    rep->final_relres = NAN;
    if (restart <= 0) restart = maxit;
    cplx *r0 = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *w = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *tmp = (cplx *)xcalloc(n, sizeof(cplx));
    if (minv) minv(mctx, b, r0); else memcpy(r0, b, n * sizeof(cplx));
    double denom = or_norm(n, r0);
    if (denom == 0.0) {
        rep->converged = 1; rep->final_relres = 0.0;
        free(r0); free(w); free(tmp); return;
    }
    int cap = restart + 1;
    cplx **V = (cplx **)xcalloc(cap, sizeof(cplx *));
    cplx *H = (cplx *)xcalloc((size_t)cap * cap, sizeof(cplx));  /* column-major H[j*cap+i] */
    double *cs = (double *)xcalloc(cap, sizeof(double));
    cplx *sn = (cplx *)xcalloc(cap, sizeof(cplx));
    cplx *g = (cplx *)xcalloc(cap + 1, sizeof(cplx));
    cplx *col = (cplx *)xcalloc(cap + 1, sizeof(cplx));
    cplx *y = (cplx *)xcalloc(cap, sizeof(cplx));
    int first = 1;
    for (;;) {
        if (!first) {
            A(actx, x, tmp); rep->matvec_count++;
            for (size_t q = 0; q < n; q++) tmp[q] = b[q] - tmp[q];
            if (minv) minv(mctx, tmp, r0); else memcpy(r0, tmp, n * sizeof(cplx));
        }
        double beta = or_norm(n, r0);
        if (beta / denom <= tol) {
            rep->converged = 1; rep->final_relres = beta / denom; break;
        }
        first = 0;
        int nv = 0;
        if (!V[0]) V[0] = (cplx *)xcalloc(n, sizeof(cplx));
        for (size_t q = 0; q < n; q++) V[0][q] = r0[q] / beta;
        nv = 1;
        int nh = 0;
        g[0] = beta;
        int breakdown = 0;
        while (nh < restart && rep->iterations < maxit) {
            A(actx, V[nv - 1], tmp); rep->matvec_count++;
            if (minv) minv(mctx, tmp, w); else memcpy(w, tmp, n * sizeof(cplx));
            int m = nv;
            for (int i = 0; i <= m; i++) col[i] = 0.0;
            for (int i = 0; i < m; i++) {
                cplx hij = or_vdot(n, V[i], w);
                #pragma omp parallel for schedule(static)
                for (size_t q = 0; q < n; q++) w[q] = w[q] - hij * V[i][q];
                col[i] = hij;
            }
            double hlast = or_norm(n, w);
            col[m] = hlast;
            for (int i = 0; i < nh; i++) {
                cplx t = cs[i] * col[i] + sn[i] * col[i + 1];
                col[i + 1] = -conj(sn[i]) * col[i] + cs[i] * col[i + 1];
                col[i] = t;
            }
            double c; cplx s, r;
            givens(col[m - 1], col[m], &c, &s, &r);
            cs[nh] = c; sn[nh] = s;
            col[m - 1] = r; col[m] = 0.0;
            for (int i = 0; i < m; i++) H[(size_t)nh * cap + i] = col[i];
            nh++;
            g[nh] = -conj(s) * g[nh - 1];
            g[nh - 1] = c * g[nh - 1];
            double relres = cabs(g[nh]) / denom;
            rep_record(rep, relres);
            if (hlast <= breakdown_tol) { breakdown = 1; break; }
            if (!V[nv]) V[nv] = (cplx *)xcalloc(n, sizeof(cplx));
            #pragma omp parallel for schedule(static)
            for (size_t q = 0; q < n; q++) V[nv][q] = w[q] / hlast;
            nv++;
            if (relres <= tol) break;
        }
        /* krylov.py:195-204 back substitution */
        for (int i = nh - 1; i >= 0; i--) {
            cplx acc = g[i];
            for (int j = i + 1; j < nh; j++) acc = acc - H[(size_t)j * cap + i] * y[j];
            y[i] = acc / H[(size_t)i * cap + i];
        }
        for (int i = 0; i < nh; i++) {
            #pragma omp parallel for schedule(static)
            for (size_t q = 0; q < n; q++) x[q] = x[q] + y[i] * V[i][q];
        }
        double relres = cabs(g[nh]) / denom;
        if (relres <= tol) { rep->converged = 1; break; }
        if (breakdown) { rep->breakdown = 1; rep->converged = relres <= tol; break; }
        if (rep->iterations >= maxit) { rep->converged = 0; break; }
    }
    for (int i = 0; i < cap; i++) free(V[i]);
    free(V); free(H); free(cs); free(sn); free(g); free(col); free(y);
    free(r0); free(w); free(tmp);
}

/* Bi-CGSTAB shadow vector (the B200 path's SolverConfig.shadow): 0 = r~ = b as in
 * the reference (krylov.py:229); 2 = seeded hash vector, the same splitmix64
 * formula as hf_device.cuh shadow_hash (an extension the reference does not
 * have; parity of the extension is checked against this restatement). */
static int or_shadow_mode = 0;
static unsigned long long or_shadow_seed = 0;
void or_set_bicgstab_shadow(int mode, unsigned long long seed) {
    or_shadow_mode = mode; or_shadow_seed = seed;
}
static unsigned long long or_splitmix64(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static cplx or_shadow_hash(unsigned long long seed, unsigned long long q) {
    unsigned long long a = or_splitmix64(seed * 0x632be59bd9b4e019ull + 2 * q);
    unsigned long long b = or_splitmix64(seed * 0x632be59bd9b4e019ull + 2 * q + 1);
    const double s = 1.0 / 9007199254740992.0;
    return ((double)(a >> 11) * s - 0.5) + I * ((double)(b >> 11) * s - 0.5);
}

/* krylov.py:207-276: right-preconditioned Bi-CGSTAB, true-residual stopping. */
void or_bicgstab(size_t n, or_op_fn A, void *actx, or_op_fn minv, void *mctx, const cplx *b,
                 cplx *x, double tol, int maxit, double breakdown_tol, or_report *rep) {
    memset(x, 0, n * sizeof(cplx));
    rep->matvec_count = rep->iterations = rep->converged = rep->breakdown = 0;
    rep->final_relres = NAN;
    double bnorm = or_norm(n, b);
    if (bnorm == 0.0) { rep->converged = 1; rep->final_relres = 0.0; return; }
    cplx *r = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *rs = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *v = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *p = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *ph = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *s = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *sh = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *t = (cplx *)xcalloc(n, sizeof(cplx));
    memcpy(r, b, n * sizeof(cplx));
    if (or_norm(n, r) / bnorm <= tol) {
        rep->converged = 1; rep->final_relres = or_norm(n, r) / bnorm; goto done;
    }
    if (or_shadow_mode == 2) {
        for (size_t q = 0; q < n; q++) rs[q] = or_shadow_hash(or_shadow_seed, q);
    } else {
        memcpy(rs, r, n * sizeof(cplx));
    }
    cplx rho = 1.0, alpha = 1.0, omega = 1.0;
    while (rep->iterations < maxit) {
        cplx rho_new = or_vdot(n, rs, r);
        if (cabs(rho_new) < breakdown_tol) { rep->breakdown = 2; break; }
        cplx beta = (rho_new / rho) * (alpha / omega);
        #pragma omp parallel for schedule(static)
        for (size_t q = 0; q < n; q++) p[q] = r[q] + beta * (p[q] - omega * v[q]);
        if (minv) minv(mctx, p, ph); else memcpy(ph, p, n * sizeof(cplx));
        A(actx, ph, v); rep->matvec_count++;
        cplx den = or_vdot(n, rs, v);
        if (cabs(den) < breakdown_tol) { rep->breakdown = 2; break; }
        alpha = rho_new / den;
        #pragma omp parallel for schedule(static)
        for (size_t q = 0; q < n; q++) s[q] = r[q] - alpha * v[q];
        double snorm = or_norm(n, s);
        if (snorm / bnorm <= tol) {
            #pragma omp parallel for schedule(static)
            for (size_t q = 0; q < n; q++) x[q] = x[q] + alpha * ph[q];
            memcpy(r, s, n * sizeof(cplx));
            rep_record(rep, snorm / bnorm);
            rep->converged = 1;
            goto done;
        }
        if (minv) minv(mctx, s, sh); else memcpy(sh, s, n * sizeof(cplx));
        A(actx, sh, t); rep->matvec_count++;
        cplx tt = or_vdot(n, t, t);
        if (cabs(tt) < breakdown_tol) { rep->breakdown = 3; break; }
        omega = or_vdot(n, t, s) / tt;
        if (cabs(omega) < breakdown_tol) { rep->breakdown = 3; break; }
        #pragma omp parallel for schedule(static)
        for (size_t q = 0; q < n; q++) {
            x[q] = x[q] + alpha * ph[q] + omega * sh[q];
            r[q] = s[q] - omega * t[q];
        }
        rho = rho_new;
        double relres = or_norm(n, r) / bnorm;
        rep_record(rep, relres);
        if (relres <= tol) { rep->converged = 1; goto done; }
    }
    rep->converged = 0;
done:
    free(r); free(rs); free(v); free(p); free(ph); free(s); free(sh); free(t);
}

/* small dense solve (partial pivoting) for the IDR projection system */
static int dense_solve(int m, cplx *Mat, int ld, cplx *rhs) {
    for (int c = 0; c < m; c++) {
        int piv = c;
        for (int r = c + 1; r < m; r++)
            if (cabs(Mat[r * ld + c]) > cabs(Mat[piv * ld + c])) piv = r;
        if (cabs(Mat[piv * ld + c]) == 0.0) return -1;
        if (piv != c) {
            for (int k = 0; k < m; k++) {
                cplx t = Mat[c * ld + k]; Mat[c * ld + k] = Mat[piv * ld + k]; Mat[piv * ld + k] = t;
            }
            cplx t = rhs[c]; rhs[c] = rhs[piv]; rhs[piv] = t;
        }
        for (int r = c + 1; r < m; r++) {
            cplx f = Mat[r * ld + c] / Mat[c * ld + c];
            for (int k = c; k < m; k++) Mat[r * ld + k] -= f * Mat[c * ld + k];
            rhs[r] -= f * rhs[c];
        }
    }
    for (int r = m - 1; r >= 0; r--) {
        cplx acc = rhs[r];
        for (int k = r + 1; k < m; k++) acc -= Mat[r * ld + k] * rhs[k];
        rhs[r] = acc / Mat[r * ld + r];
    }
    return 0;
}

/* krylov.py:292-394: IDR(s) biorthogonal variant, right preconditioning.
 * P holds the s orthonormal shadow vectors (krylov.py:279-289), generated by
 * the caller from numpy's default_rng(seed) exactly as the reference does. */
void or_idrs(size_t n, or_op_fn A, void *actx, or_op_fn minv, void *mctx, const cplx *b,
             cplx *x, int s, const cplx *P, double tol, int maxit, double breakdown_tol,
             or_report *rep) {
    memset(x, 0, n * sizeof(cplx));
    rep->matvec_count = rep->iterations = rep->converged = rep->breakdown = 0;
    rep->final_relres = NAN;
    double bnorm = or_norm(n, b);
    if (bnorm == 0.0) { rep->converged = 1; rep->final_relres = 0.0; return; }
    cplx *r = (cplx *)xcalloc(n, sizeof(cplx));
    memcpy(r, b, n * sizeof(cplx));
    double relres = or_norm(n, r) / bnorm;
    if (relres <= tol) { rep->converged = 1; rep->final_relres = relres; free(r); return; }
    cplx *G = (cplx *)xcalloc((size_t)s * n, sizeof(cplx));
    cplx *U = (cplx *)xcalloc((size_t)s * n, sizeof(cplx));
    cplx *v = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *vh = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *u = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *gv = (cplx *)xcalloc(n, sizeof(cplx));
    cplx *Mm = (cplx *)xcalloc((size_t)s * s, sizeof(cplx));
    cplx *f = (cplx *)xcalloc(s, sizeof(cplx));
    cplx *cc = (cplx *)xcalloc(s, sizeof(cplx));
    cplx *sub = (cplx *)xcalloc((size_t)s * s, sizeof(cplx));
    for (int i = 0; i < s; i++) Mm[i * s + i] = 1.0;
    cplx om = 1.0;
    const double kappa = 0.7;
    while (rep->iterations < maxit) {
        for (int i = 0; i < s; i++) f[i] = or_vdot(n, P + (size_t)i * n, r);
        for (int k = 0; k < s; k++) {
            int m = s - k;
            for (int a = 0; a < m; a++) {
                for (int c2 = 0; c2 < m; c2++) sub[a * m + c2] = Mm[(k + a) * s + (k + c2)];
                cc[a] = f[k + a];
            }
            if (dense_solve(m, sub, m, cc) != 0) {
                rep->breakdown = 4; rep->converged = 0; goto done;
            }
            memcpy(v, r, n * sizeof(cplx));
            for (int i = k; i < s; i++) {
                cplx ci = cc[i - k];
                const cplx *Gi = G + (size_t)i * n;
                #pragma omp parallel for schedule(static)
                for (size_t q = 0; q < n; q++) v[q] = v[q] - ci * Gi[q];
            }
            if (minv) minv(mctx, v, vh); else memcpy(vh, v, n * sizeof(cplx));
            #pragma omp parallel for schedule(static)
            for (size_t q = 0; q < n; q++) u[q] = om * vh[q];
            for (int i = k; i < s; i++) {
                cplx ci = cc[i - k];
                const cplx *Ui = U + (size_t)i * n;
                #pragma omp parallel for schedule(static)
                for (size_t q = 0; q < n; q++) u[q] = u[q] + ci * Ui[q];
            }
            A(actx, u, gv); rep->matvec_count++;
            for (int i = 0; i < k; i++) {
                cplx al = or_vdot(n, P + (size_t)i * n, gv) / Mm[i * s + i];
                const cplx *Gi = G + (size_t)i * n;
                const cplx *Ui = U + (size_t)i * n;
                #pragma omp parallel for schedule(static)
                for (size_t q = 0; q < n; q++) {
                    gv[q] = gv[q] - al * Gi[q];
                    u[q] = u[q] - al * Ui[q];
                }
            }
            memcpy(G + (size_t)k * n, gv, n * sizeof(cplx));
            memcpy(U + (size_t)k * n, u, n * sizeof(cplx));
            for (int i = k; i < s; i++) Mm[i * s + k] = or_vdot(n, P + (size_t)i * n, gv);
            if (cabs(Mm[k * s + k]) < breakdown_tol) {
                rep->breakdown = 4; rep->converged = 0; goto done;
            }
            cplx beta = f[k] / Mm[k * s + k];
            {
                const cplx *Gk = G + (size_t)k * n;
                const cplx *Uk = U + (size_t)k * n;
                #pragma omp parallel for schedule(static)
                for (size_t q = 0; q < n; q++) {
                    r[q] = r[q] - beta * Gk[q];
                    x[q] = x[q] + beta * Uk[q];
                }
            }
            relres = or_norm(n, r) / bnorm;
            rep_record(rep, relres);
            if (relres <= tol || rep->iterations >= maxit) break;
            for (int i = k + 1; i < s; i++) f[i] = f[i] - beta * Mm[i * s + k];
        }
        if (relres <= tol) { rep->converged = 1; goto done; }
        if (rep->iterations >= maxit) break;
        if (minv) minv(mctx, r, vh); else memcpy(vh, r, n * sizeof(cplx));
        A(actx, vh, gv); rep->matvec_count++;
        cplx tt = or_vdot(n, gv, gv);
        if (cabs(tt) < breakdown_tol) { rep->breakdown = 3; break; }
        cplx tr = or_vdot(n, gv, r);
        om = tr / tt;
        double angle = cabs(or_vdot(n, gv, r)) / (sqrt(cabs(tt)) * or_norm(n, r));
        if (angle < kappa) om = om * (kappa / angle);
        if (cabs(om) < breakdown_tol) { rep->breakdown = 3; break; }
        #pragma omp parallel for schedule(static)
        for (size_t q = 0; q < n; q++) {
            x[q] = x[q] + om * vh[q];
            r[q] = r[q] - om * gv[q];
        }
        relres = or_norm(n, r) / bnorm;
        rep_record(rep, relres);
        if (relres <= tol) { rep->converged = 1; goto done; }
    }
    rep->converged = relres <= tol;
done:
    free(r); free(G); free(U); free(v); free(vh); free(u); free(gv); free(Mm); free(f);
    free(cc); free(sub);
}

/* ------------------------------------------------------------------------ */
/* hierarchy + cycles (multigrid.py:90-128, 300-419)                          */
/* ------------------------------------------------------------------------ */
typedef struct {
    int nlev;
    or_level lev[32];
    int nu1, nu2;
    double omega;
    int cycle_f;          /* 0 V, 1 F */
    double coarsest_tol;
    int coarsest_maxit;
    int coarsest_fail;    /* count of coarsest GMRES non-convergences */
    int coarsest_iters;   /* total coarsest GMRES iterations (diagnostic) */
    int coarsest_calls;
} or_hier;

static void coarse_apply(void *ctx, const cplx *x, cplx *y) {
    or_apply_level((const or_level *)ctx, x, y);
}

/* multigrid.py:90-98 stop rule: continue while all dims satisfy the
 * threshold ("gt" or "ge") and every dim is odd. */
static int keep_coarsening(int n1, int n2, int n3, int th, int ge) {
    int ok = ge ? (n1 >= th && n2 >= th && n3 >= th) : (n1 > th && n2 > th && n3 > th);
    return ok && (n1 % 2 == 1) && (n2 % 2 == 1) && (n3 % 2 == 1);
}

/* k: finest k field (n1*n2*n3); coarse k subsampled at 2i-1 (operators.py:265-274). */
or_hier *or_hier_create(int n1, int n2, int n3, double h, double beta1, double beta2,
                        int bc, const double *k, int nu1, int nu2, double omega, int cycle_f,
                        int threshold, int threshold_ge, double coarsest_tol,
                        int coarsest_maxit) {
    or_hier *H = (or_hier *)xcalloc(1, sizeof(or_hier));
    H->nu1 = nu1; H->nu2 = nu2; H->omega = omega; H->cycle_f = cycle_f;
    H->coarsest_tol = coarsest_tol; H->coarsest_maxit = coarsest_maxit;
    int a = n1, b2 = n2, c = n3;
    double hh = h;
    const double *kprev = k;
    int pb = 0, pc = 0;
    for (;;) {
        or_level *L = &H->lev[H->nlev];
        L->n1 = a; L->n2 = b2; L->n3 = c; L->h = hh;
        L->shift = beta1 - I * beta2;
        L->bc = bc;
        size_t n = (size_t)a * b2 * c;
        L->k = (double *)xcalloc(n, sizeof(double));
        if (H->nlev == 0) {
            memcpy(L->k, k, n * sizeof(double));
        } else {
            for (int i = 0; i < a; i++)
                for (int j = 0; j < b2; j++)
                    for (int m = 0; m < c; m++)
                        L->k[((size_t)i * b2 + j) * c + m] =
                            kprev[((size_t)(2 * i) * pb + 2 * j) * pc + 2 * m];
        }
        level_build_diag(L);
        L->u = (cplx *)xcalloc(n, sizeof(cplx));
        L->b = (cplx *)xcalloc(n, sizeof(cplx));
        L->r = (cplx *)xcalloc(n, sizeof(cplx));
        L->tmp = (cplx *)xcalloc(n, sizeof(cplx));
        H->nlev++;
        if (!keep_coarsening(a, b2, c, threshold, threshold_ge) || H->nlev >= 32) break;
        kprev = L->k; pb = b2; pc = c;
        a = (a + 1) / 2; b2 = (b2 + 1) / 2; c = (c + 1) / 2; hh = 2.0 * hh;
    }
    return H;
}

void or_hier_free(or_hier *H) {
    if (!H) return;
    for (int l = 0; l < H->nlev; l++) {
        or_level *L = &H->lev[l];
        free(L->k); free(L->diag); free(L->ap); free(L->u); free(L->b); free(L->r); free(L->tmp);
    }
    free(H);
}

int or_hier_nlev(const or_hier *H) { return H->nlev; }
void or_hier_level_dims(const or_hier *H, int l, int *dims) {
    dims[0] = H->lev[l].n1; dims[1] = H->lev[l].n2; dims[2] = H->lev[l].n3;
}
void or_hier_stats(const or_hier *H, int *out) {
    out[0] = H->coarsest_calls; out[1] = H->coarsest_iters; out[2] = H->coarsest_fail;
}

/* Optional exact coarsest solve (row-major dense inverse supplied by the test
 * harness): the B200 path's coarsest_method="direct".  NULL = reference GMRES. */
static const cplx *or_coarse_inverse = NULL;
static size_t or_coarse_n = 0;
void or_set_coarse_inverse(const cplx *Minv, size_t n) { or_coarse_inverse = Minv; or_coarse_n = n; }

/* multigrid.py:300-323 */
static void coarsest_solve(or_hier *H, const cplx *b, cplx *x) {
    or_level *L = &H->lev[H->nlev - 1];
    if (or_coarse_inverse && or_coarse_n == npts(L)) {
        size_t n = or_coarse_n;
        #pragma omp parallel for schedule(static)
        for (size_t i = 0; i < n; i++) {
            cplx acc = 0.0;
            const cplx *row = or_coarse_inverse + i * n;
            for (size_t j = 0; j < n; j++) acc += row[j] * b[j];
            x[i] = acc;
        }
        H->coarsest_calls++;
        return;
    }
    or_report rep = {0};
    or_gmres(npts(L), coarse_apply, L, NULL, NULL, b, x, H->coarsest_tol, H->coarsest_maxit, 0,
             1e-30, &rep);
    H->coarsest_calls++;
    H->coarsest_iters += rep.iterations;
    if (!rep.converged) H->coarsest_fail++;
}

static void residual(or_level *L) {   /* multigrid.py:383-386 */
    size_t n = npts(L);
    or_apply_level(L, L->u, L->tmp);
    #pragma omp parallel for schedule(static)
    for (size_t q = 0; q < n; q++) L->r[q] = L->b[q] - L->tmp[q];
}

static void v_cycle(or_hier *H, int li) {   /* multigrid.py:326-343 */
    or_level *L = &H->lev[li];
    size_t n = npts(L);
    if (li == H->nlev - 1) { coarsest_solve(H, L->b, L->u); return; }
    or_level *N = &H->lev[li + 1];
    if (H->nu1 == 0) memset(L->u, 0, n * sizeof(cplx));
    else or_jacobi_level(L, L->u, L->b, H->omega, H->nu1, L->tmp, 1);
    residual(L);
    or_restrict_level(L, N, L->r, N->b);
    v_cycle(H, li + 1);
    or_prolong_level(N, L, N->u, L->tmp);       /* multigrid.py:389-392 */
    #pragma omp parallel for schedule(static)
    for (size_t q = 0; q < n; q++) L->u[q] += L->tmp[q];
    or_jacobi_level(L, L->u, L->b, H->omega, H->nu2, L->tmp, 0);
}

static void f_cycle(or_hier *H, int li) {   /* multigrid.py:346-370 */
    or_level *L = &H->lev[li];
    size_t n = npts(L);
    if (li == H->nlev - 1) { coarsest_solve(H, L->b, L->u); return; }
    or_level *N = &H->lev[li + 1];
    or_restrict_level(L, N, L->b, N->b);
    f_cycle(H, li + 1);
    or_prolong_level(N, L, N->u, L->u);
    residual(L);
    cplx *guess = (cplx *)xcalloc(n, sizeof(cplx));
    memcpy(guess, L->u, n * sizeof(cplx));
    memcpy(L->b, L->r, n * sizeof(cplx));
    v_cycle(H, li);
    #pragma omp parallel for schedule(static)
    for (size_t q = 0; q < n; q++) L->u[q] += guess[q];
    free(guess);
}

/* multigrid.py:395-419: z = one cycle applied to r with zero initial guess. */
void or_mg_precondition(or_hier *H, const cplx *r, cplx *z) {
    or_level *T = &H->lev[0];
    size_t n = npts(T);
    memcpy(T->b, r, n * sizeof(cplx));
    if (H->cycle_f) f_cycle(H, 0); else v_cycle(H, 0);
    memcpy(z, T->u, n * sizeof(cplx));
}

/* level-indexed wrappers for kernel-level parity tests */
void or_hier_apply(or_hier *H, int l, const cplx *u, cplx *v) { or_apply_level(&H->lev[l], u, v); }
void or_hier_diag(or_hier *H, int l, cplx *d) {
    memcpy(d, H->lev[l].diag, npts(&H->lev[l]) * sizeof(cplx));
}
void or_hier_jacobi(or_hier *H, int l, cplx *u, const cplx *b, double omega, int sweeps,
                    int assume_zero) {
    cplx *scratch = (cplx *)xcalloc(npts(&H->lev[l]), sizeof(cplx));
    or_jacobi_level(&H->lev[l], u, b, omega, sweeps, scratch, assume_zero);
    free(scratch);
}
void or_hier_restrict(or_hier *H, int l, const cplx *rf, cplx *out) {
    or_restrict_level(&H->lev[l], &H->lev[l + 1], rf, out);
}
void or_hier_prolong(or_hier *H, int l, const cplx *ec, cplx *out) {
    or_prolong_level(&H->lev[l + 1], &H->lev[l], ec, out);
}
void or_hier_coarsest(or_hier *H, const cplx *b, cplx *x) { coarsest_solve(H, b, x); }

/* ------------------------------------------------------------------------ */
/* full solve: Helmholtz operator A (kind helmholtz: shift 1) + CSLP cycle   */
/* (runner.py:95-131)                                                        */
/* ------------------------------------------------------------------------ */
typedef struct {
    or_level A;          /* finest Helmholtz operator */
    or_hier *H;
} or_solver;

static void solver_apply_a(void *ctx, const cplx *x, cplx *y) {
    or_apply_level(&((or_solver *)ctx)->A, x, y);
}
static void solver_minv(void *ctx, const cplx *x, cplx *y) {
    or_mg_precondition(((or_solver *)ctx)->H, x, y);
}

/* method: 0 gmres, 1 bicgstab, 2 idrs.  P: s shadow vectors for IDR (else NULL).
 * stats_out (may be NULL): coarsest calls, coarsest iterations, coarsest failures. */
int or_solve(int n1, int n2, int n3, double h, int bc, const double *k, const cplx *b,
             cplx *x, int method, double tol, int maxit, int restart, int s, const cplx *P,
             double beta1, double beta2, int nu1, int nu2, double omega, int cycle_f,
             int threshold, int threshold_ge, double coarsest_tol, int coarsest_maxit,
             int *matvecs, int *iterations, int *converged, int *breakdown,
             double *final_relres, double *history, int history_cap, int *stats_out) {
    or_solver S;
    memset(&S, 0, sizeof(S));
    S.A.n1 = n1; S.A.n2 = n2; S.A.n3 = n3; S.A.h = h; S.A.shift = 1.0; S.A.bc = bc;
    size_t n = (size_t)n1 * n2 * n3;
    S.A.k = (double *)xcalloc(n, sizeof(double));
    memcpy(S.A.k, k, n * sizeof(double));
    level_build_diag(&S.A);
    S.H = or_hier_create(n1, n2, n3, h, beta1, beta2, bc, k, nu1, nu2, omega, cycle_f,
                         threshold, threshold_ge, coarsest_tol, coarsest_maxit);
    or_report rep = {0};
    rep.history = history; rep.history_cap = history_cap;
    if (method == 0)
        or_gmres(n, solver_apply_a, &S, solver_minv, &S, b, x, tol, maxit, restart, 1e-30, &rep);
    else if (method == 1)
        or_bicgstab(n, solver_apply_a, &S, solver_minv, &S, b, x, tol, maxit, 1e-30, &rep);
    else
        or_idrs(n, solver_apply_a, &S, solver_minv, &S, b, x, s, P, tol, maxit, 1e-30, &rep);
    *matvecs = rep.matvec_count; *iterations = rep.iterations; *converged = rep.converged;
    *breakdown = rep.breakdown; *final_relres = rep.final_relres;
    if (stats_out) or_hier_stats(S.H, stats_out);
    or_hier_free(S.H);
    free(S.A.k); free(S.A.diag); free(S.A.ap);
    return 0;
}

/* Persistent solver (bench.py's CPU legs time solves without the hierarchy
 * setup, like the native arm): or_solver_create builds A and the CSLP hierarchy
 * once; or_solver_solve runs one Krylov solve (runner.py:95-131 minus setup). */
void *or_solver_create(int n1, int n2, int n3, double h, int bc, const double *k, double beta1,
                       double beta2, int nu1, int nu2, double omega, int cycle_f, int threshold,
                       int threshold_ge, double coarsest_tol, int coarsest_maxit) {
    or_solver *S = (or_solver *)xcalloc(1, sizeof(or_solver));
    S->A.n1 = n1; S->A.n2 = n2; S->A.n3 = n3; S->A.h = h; S->A.shift = 1.0; S->A.bc = bc;
    size_t n = (size_t)n1 * n2 * n3;
    S->A.k = (double *)xcalloc(n, sizeof(double));
    memcpy(S->A.k, k, n * sizeof(double));
    level_build_diag(&S->A);
    S->H = or_hier_create(n1, n2, n3, h, beta1, beta2, bc, k, nu1, nu2, omega, cycle_f,
                          threshold, threshold_ge, coarsest_tol, coarsest_maxit);
    return S;
}
void or_solver_free(void *p) {
    or_solver *S = (or_solver *)p;
    or_hier_free(S->H);
    free(S->A.k); free(S->A.diag); free(S->A.ap);
    free(S);
}
int or_solver_solve(void *p, const cplx *b, cplx *x, int method, double tol, int maxit,
                    int *iterations, int *converged, int *breakdown, double *final_relres) {
    or_solver *S = (or_solver *)p;
    size_t n = (size_t)S->A.n1 * S->A.n2 * S->A.n3;
    or_report rep = {0};
    if (method == 1)
        or_bicgstab(n, solver_apply_a, S, solver_minv, S, b, x, tol, maxit, 1e-30, &rep);
    else
        or_gmres(n, solver_apply_a, S, solver_minv, S, b, x, tol, maxit, 0, 1e-30, &rep);
    *iterations = rep.iterations; *converged = rep.converged; *breakdown = rep.breakdown;
    *final_relres = rep.final_relres;
    return 0;
}

/* plain Helmholtz/CSLP apply on a full grid (for kernel-level parity) */
void or_apply(int n1, int n2, int n3, double h, double shift_re, double shift_im, int bc,
              const double *k, const cplx *u, cplx *v) {
    or_level L;
    memset(&L, 0, sizeof(L));
    L.n1 = n1; L.n2 = n2; L.n3 = n3; L.h = h; L.shift = shift_re + I * shift_im; L.bc = bc;
    L.k = (double *)k;
    level_build_diag(&L);
    or_apply_level(&L, u, v);
    free(L.diag); free(L.ap);
}

int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
