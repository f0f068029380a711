/*
 * helmfree_b200.h -- C ABI of the B200-native CSLP / multigrid / Krylov path.
 *
 * Drop-in boundary for the reference package `helmfree`
 * (/root/reference/pkg/src/helmfree).  Every entry point names the reference
 * interface it replaces (file:line).  Plain C: opaque handles, plain pointers
 * and sizes, no torch types.  Build: paper_2308_06085_b200/_lib/libhelmfree_b200.so
 *
 * Conventions
 *  - Fields are complex128, stored as interleaved (re, im) doubles, shape
 *    (nx, n2, n3) in C order (i3 fastest) -- the reference's numpy layout.
 *    `double *` field arguments point at the first owned value.
 *  - Blocks are slabs along i1: a worker owns global planes [lo1, lo1 + nx).
 *    When a slab face is interior (not a physical boundary) the caller
 *    guarantees HF_GHOST planes of valid neighbour data directly before /
 *    after the owned planes (the halo exchange fills them).
 *  - Device pointers unless a name ends in _host.
 *  - Return codes: 0 on success, negative on error (hf_last_error() explains).
 *    Errors never fall back to another implementation.
 */
#ifndef HELMFREE_B200_H
#define HELMFREE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HF_GHOST 2

#define HF_BC_DIRICHLET 0
#define HF_BC_SOMMERFELD 1

#define HF_CYCLE_V 0
#define HF_CYCLE_F 1

#define HF_METHOD_GMRES 0
#define HF_METHOD_BICGSTAB 1
#define HF_METHOD_IDRS 2

#define HF_COARSEST_DIRECT 0   /* exact: fast diagonalisation, packed symmetric or dense inverse */
#define HF_COARSEST_GMRES 1    /* the reference's unpreconditioned full GMRES to coarsest_tol,
                                  at most coarsest_maxit iterations (multigrid.py:300-323) */
#define HF_COARSEST_EXTERNAL 2 /* no coarsest solve: the caller gathers the
                                  coarse RHS and solves it (multi-GPU slabs)  */

/* Bi-CGSTAB shadow vector r~ (B200 addition; the reference always takes r~ = b,
 * krylov.py:229, which breaks down on the rho test for a point source on large
 * wedge grids -- see DESIGN.md section 4) */
#define HF_SHADOW_RHS 0
#define HF_SHADOW_HOST 1
#define HF_SHADOW_HASH 2   /* r~_q = splitmix64 hash of (seed, global index q), uniform in
                              [-1/2, 1/2)^2 -- identical on any slab layout */

#define HF_BREAKDOWN_NONE 0
#define HF_BREAKDOWN_ARNOLDI 1
#define HF_BREAKDOWN_RHO 2
#define HF_BREAKDOWN_OMEGA 3
#define HF_BREAKDOWN_PROJECTION 4

#define HF_ERR_ARG -1
#define HF_ERR_CUDA -2
#define HF_ERR_ZERO_DIAGONAL -3
#define HF_ERR_UNSUPPORTED -4
#define HF_ERR_SOLVER -5

typedef struct hf_operator hf_operator;
typedef struct hf_hierarchy hf_hierarchy;
typedef struct hf_solver hf_solver;
typedef struct hf_bcg hf_bcg;

/* multigrid.py:42-51 MGConfig */
typedef struct hf_mg_config {
    int nu1, nu2;
    double omega;
    int cycle;               /* HF_CYCLE_V | HF_CYCLE_F */
    int coarsest_threshold;  /* coarsen while all dims > (or >=) this */
    int threshold_ge;        /* 0: "gt" (default), 1: "ge" */
    double coarsest_tol;
    int coarsest_maxit;
    int coarsest_method;     /* HF_COARSEST_DIRECT | HF_COARSEST_GMRES */
} hf_mg_config;

/* krylov.py:34-43 SolverConfig */
typedef struct hf_solver_config {
    int method;              /* HF_METHOD_* */
    double tol;
    int maxit;
    int s;                   /* IDR shadow dimension */
    int restart;             /* GMRES restart length, 0 = full */
    double breakdown_tol;
    const double *shadow_host;  /* IDR: s orthonormal vectors (s * N complex), host;
                                   Bi-CGSTAB: one shadow vector r~ (N complex), host */
    int check_every;         /* Bi-CGSTAB: iterations per host convergence poll */
    int shadow_kind;         /* Bi-CGSTAB r~: HF_SHADOW_RHS (reference, r~ = b),
                                HF_SHADOW_HOST (shadow_host), HF_SHADOW_HASH (seeded) */
    uint64_t shadow_seed;    /* HF_SHADOW_HASH seed */
} hf_solver_config;

/* krylov.py:46-64 ConvergenceReport (phase_times reduced to device times) */
typedef struct hf_report {
    int matvec_count;
    int iterations;
    int converged;
    int breakdown;           /* HF_BREAKDOWN_* */
    double final_relres;
    double *history_host;    /* caller buffer, >= maxit + 1 entries, may be NULL */
    int history_cap;
    int coarsest_flags;      /* coarsest solves that missed coarsest_tol */
    double solve_ms;         /* device time of the Krylov loop (CUDA events) */
    int kernel_launches;     /* kernels this library enqueued for the solve */
} hf_report;

/* ---- library ----------------------------------------------------------- */
const char *hf_last_error(void);
int hf_version(void);
/* Kernel-variant selection for A/B measurements and the parity tests that compare
 * variants (process-wide; every variant computes the same arithmetic; all off is the
 * measured-fastest default).  Names: "no_pdl", "no_flat", "no_flat_dr", "no_dr",
 * "tiled_dr", "flat_up", "fuse_up", "no_fuse", "coarsest_dense", "no_palette" (the
 * last applies to hierarchies / operators created after it is set).  The library reads
 * no environment variables. */
int hf_set_option(const char *name, int value);
int hf_get_option(const char *name);   /* 0/1, or HF_ERR_ARG for an unknown name */
/* Stream used by all subsequent calls of this thread (cudaStream_t, NULL = default). */
void hf_set_stream(void *stream);
int hf_device_synchronize(void);

/* ---- operators.py:122-254 StencilOperator / apply_operator -------------- */
/* k_host: full global wavenumber field (n1*n2*n3, C order) or NULL for the
 * constant k_const.  shift = beta1 - i*beta2 (Helmholtz: 1 + 0i). */
hf_operator *hf_operator_create(int n1, int n2, int n3, int lo1, int nx, double h,
                                double shift_re, double shift_im, int bc,
                                const double *k_host, double k_const);
void hf_operator_destroy(hf_operator *op);
/* v = A u on the owned slab (operators.py:200-223). */
int hf_operator_apply(hf_operator *op, const double *u, double *v);
/* Jacobi diagonal (operators.py:163-183), nx*n2*n3 complex. */
int hf_operator_diag(hf_operator *op, double *d);
/* multigrid.py:138-157 jacobi_smooth; scratch: one field (with ghost planes
 * when the slab has interior faces). */
int hf_jacobi_smooth(hf_operator *op, double *u, const double *b, double omega, int sweeps,
                     int assume_zero, double *scratch);

/* ---- multigrid.py:101-128 build_hierarchy ------------------------------ */
hf_hierarchy *hf_hierarchy_create(int n1, int n2, int n3, int lo1, int nx, double h,
                                  double beta1, double beta2, int bc, const double *k_host,
                                  double k_const, const hf_mg_config *cfg);
void hf_hierarchy_destroy(hf_hierarchy *hier);
int hf_hierarchy_num_levels(const hf_hierarchy *hier);
/* dims5 = {n1, n2, n3, lo1, nx} of level l */
int hf_hierarchy_level_shape(const hf_hierarchy *hier, int level, int *dims5);
/* multigrid.py:171-202 restrict_fw: fine level `level` -> level+1 */
int hf_restrict_fw(hf_hierarchy *hier, int level, const double *r_fine, double *b_coarse);
/* multigrid.py:238-297 prolong_tl: coarse level `level`+1 -> fine `level` */
int hf_prolong_tl(hf_hierarchy *hier, int level, const double *e_coarse, double *out_fine);
/* multigrid.py:300-323 coarsest_solve */
int hf_coarsest_solve(hf_hierarchy *hier, const double *b, double *x);
/* Which exact coarsest solve the hierarchy set up (B200 addition; the
   reference always iterates GMRES to coarsest_tol, multigrid.py:300-323). */
#define HF_COARSEST_KIND_NONE 0        /* external (slab drivers) */
#define HF_COARSEST_KIND_DENSE 1       /* dense inverse, GEMV */
#define HF_COARSEST_KIND_SYMMETRIC 2   /* packed symmetric M^-1 S^-1 */
#define HF_COARSEST_KIND_SEPARABLE 3   /* fast diagonalisation (constant k) */
#define HF_COARSEST_KIND_GMRES 4       /* GMRES to coarsest_tol (HF_COARSEST_GMRES, or the
                                          direct method's fallback on coarsest grids over
                                          60000 vertices without a separable factorisation) */
int hf_coarsest_kind(const hf_hierarchy *hier);
/* multigrid.py:320-322 hier.coarsest_flags: coarsest GMRES solves that stopped at
   coarsest_maxit above coarsest_tol since the last reset (always 0 for exact solves). */
int hf_coarsest_flags(hf_hierarchy *hier, int reset);
/* multigrid.py:395-419 mg_precondition: z ~= M^-1 r, one V/F cycle */
int hf_mg_precondition(hf_hierarchy *hier, const double *r, double *z);
/* Fused pieces of one V(1,1) level (multigrid.py:337-343) for slab drivers that
 * exchange halos in between.  down1: r = b - M (w D^-1 b) (pre-smooth from zero +
 * residual).  correct: t = w D^-1 b + P e (nu1 = 1; t = P e when nu1 = 0).
 * smooth: u = t + w D^-1 (b - M t) (post-smoothing sweep). */
int hf_level_down1(hf_hierarchy *hier, int level, const double *b, double *r);
/* down1 fused with restrict_fw: b_coarse = R (b - M (w D^-1 b)) without the fine
 * residual (multigrid.py:383-386 + 171-221); b needs HF_GHOST valid ghost planes
 * at interior slab faces.  b_coarse is the next level's owned block. */
int hf_level_down_restrict(hf_hierarchy *hier, int level, const double *b, double *b_coarse);
int hf_level_correct(hf_hierarchy *hier, int level, const double *b, const double *e_coarse,
                     double *t);
int hf_level_smooth(hf_hierarchy *hier, int level, const double *t, const double *b, double *u);
/* correct on the owned planes and on the ghost planes at interior slab faces (b's
 * HF_GHOST-deep halo and one coarse ghost plane of e must be valid), so the
 * smoothing sweep needs no halo exchange of t. */
int hf_level_correct_ext(hf_hierarchy *hier, int level, const double *b, const double *e_coarse,
                         double *t);
/* correct + smooth in one pass (whole-grid levels; split kernels on slabs):
 * u = t + w D^-1 (b - M t), t = [w D^-1 b] + P e (multigrid.py:389-392, 153-156). */
int hf_level_up(hf_hierarchy *hier, int level, const double *b, const double *e_coarse, double *u);

/* ---- krylov.py:111-407 + runner.py:95-131 ------------------------------ */
/* A: Helmholtz operator (shift 1) on the same slab as the hierarchy's finest level. */
hf_solver *hf_solver_create(hf_operator *A, hf_hierarchy *M);
void hf_solver_destroy(hf_solver *s);
/* Device-resident solve: x = A^-1 b preconditioned by one MG cycle. */
/* ---- device-resident Bi-CGSTAB for slab drivers (krylov.py:207-276) ----
 * The scalars (rho, alpha, omega, beta, norms, history, stop flags) live on the
 * device.  Each reduction stores THIS slab's partial sums (two complex, device
 * `sums`); the driver adds them over slabs / ranks (NCCL all-reduce) and calls
 * hf_bcg_step with the op that consumed them: 1 init (|b|^2, r~^H r),
 * 2 alpha (r~^H v), 3 s-norm (|s|^2), 4 omega (t^H t, t^H s), 5 rho (|r|^2,
 * r~^H r).  Every kernel is a no-op once the device state is done. */
hf_bcg *hf_bcg_create(hf_operator *A, double tol, int maxit, double breakdown_tol);
void hf_bcg_destroy(hf_bcg *state);
int hf_bcg_step(hf_bcg *state, int op, const double *sums);
int hf_bcg_read(hf_bcg *state, int *out6, double *relres, double *history_host, int history_cap);
int hf_bcg_vec_init(hf_bcg *state, int64_t n, const double *b, double *r, double *rs, double *x,
                    double *p, double *v, double *sums);
int hf_bcg_vec_p(hf_bcg *state, int64_t n, const double *r, double *p, const double *v);
int hf_bcg_vec_s(hf_bcg *state, int64_t n, const double *r, const double *v, double *s, double *sums);
int hf_bcg_vec_xr(hf_bcg *state, int64_t n, double *x, const double *ph, const double *sh,
                  const double *s, const double *t, double *r, const double *rs, double *sums);
int hf_bcg_vec_xhalf(hf_bcg *state, int64_t n, double *x, const double *ph);
int hf_operator_apply_dot(hf_operator *A, hf_bcg *state, int nd, const double *u, double *v,
                          const double *w, double *sums);

/* Measurement hook (bench.py): mean device ms of the Bi-CGSTAB vector kernel
 * `which` (0: p update, 1: s update + |s|^2, 2: x, r update + |r|^2, r~^H r,
 * 3: the same with a sparse shadow vector (r~ not streamed); krylov.py:240,
 * 248-249, 266-269; 4: the second matvec of an iteration with its inner
 * products, t = A s^, t^H t, t^H s, krylov.py:256-258) over `reps` launches
 * on the solver's workspace; the device scalar state is not modified. */
int hf_solver_bench_vec(hf_solver *solver, int which, int reps, float *ms);
int hf_solve(hf_solver *s, const hf_solver_config *cfg, const double *b, double *x,
             hf_report *rep);
/* Same, from HOST buffers (pinned or pageable): H2D of b, solve, D2H of x. */
int hf_solve_host(hf_solver *s, const hf_solver_config *cfg, const double *b_host,
                  double *x_host, hf_report *rep);

/* ---- native multi-slab Bi-CGSTAB (runner.py:95-131 over i1 slabs) --------
 * One iteration -- vector updates, the slab V(1,1) cycle, halo exchanges
 * (partition.py:509-536), the coarsest gather, the inner-product all-reduces
 * (partition.py:611-621) and the scalar update -- stream-ordered on one stream
 * and replayed as one CUDA graph.  LOCAL: all slabs of the decomposition in this
 * process (nloc == world; halos are device copies).  NCCL: one slab per rank,
 * the balanced i1 split; halos ncclSend/ncclRecv with the neighbours, sums one
 * ncclAllReduce, coarsest slabs one ncclAllGather (captured in the graph). */
#define HF_TRANSPORT_LOCAL 0
#define HF_TRANSPORT_NCCL 1
typedef struct hf_slab hf_slab;
/* load libnccl (path, or NULL for the already-loaded libnccl.so.2) */
int hf_nccl_init(const char *libpath);
/* rank 0 draws the 128-byte ncclUniqueId the caller broadcasts */
int hf_nccl_unique_id(void *out128);
/* lo1s / nxs: this process's slabs (global first plane, plane count) */
hf_slab *hf_slab_create(int n1, int n2, int n3, double h, double beta1, double beta2, int bc,
                        const double *k_host, double k_const, const hf_mg_config *cfg, int nloc,
                        const int *lo1s, const int *nxs, int world, int rank, int transport,
                        const void *nccl_id, int maxit);
void hf_slab_destroy(hf_slab *slab);
/* b_slabs / x_slabs: device pointers to each local slab's owned planes */
int hf_slab_solve(hf_slab *slab, const hf_solver_config *cfg, const double *const *b_slabs,
                  double *const *x_slabs, hf_report *rep);

/* ---- krylov.py:67-78 dot (owned region, conjugated) --------------------- */
int hf_dot(int64_t n, const double *u, const double *v, double *out_host2);

#ifdef __cplusplus
}
#endif
#endif
