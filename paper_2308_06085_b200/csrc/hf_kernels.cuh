// hf_kernels.cuh -- host-side launchers of the kernels in hf_kernels.cu.
#pragma once
#include "hf_device.cuh"

namespace hf {

// kernel-variant options (hf_set_option in the C ABI); all off = the default
enum HfOpt { OPT_NO_PDL = 0, OPT_NO_FLAT, OPT_NO_FLAT_DR, OPT_NO_DR, OPT_TILED_DR, OPT_FLAT_UP,
             OPT_FUSE_UP, OPT_NO_FUSE, OPT_COARSEST_DENSE, OPT_NO_PALETTE, OPT_NO_WIDE, OPT_FORCE_WIDE,
             OPT_WIDE_P4, OPT_WIDE_ALL, OPT_NO_WIDE_UP, OPT_WIDE_P3, OPT_WIDE_P1, OPT_WIDE_BIG, OPT_COUNT };
extern int g_opt[OPT_COUNT];
inline bool opt(int o) { return g_opt[o] != 0; }

int march_blocks(const Lvl &L);
int tile_blocks(const Lvl &L);
// wide-plane sweeps (hf_wide.cu): kind 0 apply, 1 apply + conj(w) v, 2 apply + v^H v & v^H w,
// 3 residual, 4 Jacobi sweep, 5 zero-guess pre-smoothing + residual
bool wide_ok(const Lvl &L, int kind);
int wide_blocks(const Lvl &L);
void launch_wide_up(const Lvl &L, const Lvl &C, const cd *b, const cd *e, cd *u, double omega,
                    bool pre, cudaStream_t s, const int *done);
void launch_wide(int kind, const Lvl &L, const cd *src, const cd *aux, cd *out, double omega,
                 const RedSlot &rs, cudaStream_t s, const int *done);
void init_kernel_attributes();
void launch_apply(const Lvl &L, const cd *u, cd *v, cudaStream_t s, const int *done);
void launch_apply_dot1(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done);
void launch_apply_dot2(const Lvl &L, const cd *u, cd *v, const cd *w, const RedSlot &rs,
                       cudaStream_t s, const int *done);
void launch_residual(const Lvl &L, const cd *u, const cd *b, cd *r, cudaStream_t s,
                     const int *done);
void launch_jacobi(const Lvl &L, const cd *u, const cd *b, cd *uo, double omega,
                   cudaStream_t s, const int *done);
void launch_jacobi0(const Lvl &L, const cd *b, cd *u, double omega, cudaStream_t s,
                    const int *done);
void launch_down1(const Lvl &L, const cd *b, cd *r, double omega, cudaStream_t s,
                  const int *done);
void launch_restrict(const Lvl &F, const Lvl &C, const cd *r, cd *out, cudaStream_t s,
                     const int *done);
// b_coarse = R (b - M (w D^-1 b)): fused pre-smooth + residual + restriction
void launch_down_restrict(const Lvl &F, const Lvl &C, const cd *b, cd *out, double omega,
                          cudaStream_t s, const int *done);
bool flat_dr_ok(const Lvl &F);   // the flat fused kernel (k_flat_dr) covers this level
void launch_prolong(const Lvl &F, const Lvl &C, const cd *e, cd *out, bool add, cudaStream_t s,
                    const int *done);
// returns the number of kernels launched (1 fused, 2 split)
int launch_up1(const Lvl &L, const Lvl &C, const cd *b, const cd *e, cd *u, cd *t, double omega,
               bool pre, cudaStream_t s, const int *done);
void launch_palette(const Lvl &L, int np, cd *apal, cd *dpal, cudaStream_t s);
void launch_dinv(const Lvl &L, cd *out_owned, cudaStream_t s);
// ghosts: also the ghost planes at interior slab faces (b and e halos must be valid)
void launch_correct(const Lvl &L, const Lvl &C, const cd *b, const cd *e, cd *t, double omega,
                    bool pre, cudaStream_t s, const int *done, bool ghosts = false);
void launch_gemv(int N, const cd *Minv, const cd *b, cd *x, cudaStream_t s, const int *done);
void launch_sym_pack(int N, const cd *Minv, const double *sv, cd *tiles, cudaStream_t s);
void launch_symv(int N, const cd *tiles, const double *sv, const cd *b, cd *prow, cd *pcol, cd *x,
                 cudaStream_t s, const int *done);
long long sym_tiles_count(int N);
size_t fdm_smem_bytes(int n1, int n2, int n3);
void fdm_groups(int n1, int n2, int n3, int &R, int &C);
// returns the number of kernels launched
int launch_fdm(int n1, int n2, int n3, const cd *fdm, const cd *invD, const cd *b, cd *tmp,
               cd *x, cudaStream_t s, const int *done);
void launch_assemble(const Lvl &L, cd *A, cudaStream_t s);
void launch_set_identity(long long N, cd *B, cudaStream_t s);
void launch_zero(long long n, cd *y, cudaStream_t s);
void launch_axpby(long long n, cd a, const cd *x, cd b, cd *y, cudaStream_t s);
void launch_mgs(long long n, cd *w, const cd *c, const cd *vprev, const cd *vcur,
                const RedSlot &rs, cudaStream_t s);
void launch_multi_axpy(long long n, int m, const cd *const *V, const cd *y, cd *x, cudaStream_t s);
void launch_dot(long long n, const cd *a, const cd *b, const RedSlot &rs, cudaStream_t s);
void launch_bcg_init(long long n, const cd *b, cd *r, cd *rs, cd *x, cd *p, cd *v,
                     const RedSlot &red, cudaStream_t s, int shadow = HF_SHADOW_RHS,
                     unsigned long long seed = 0, long long q0 = 0);
void launch_bcg_p(long long n, const BcgState *st, const cd *r, cd *p, const cd *v,
                  cudaStream_t s, const int *done);
void launch_bcg_s(long long n, const BcgState *st, const cd *r, const cd *v, cd *sv,
                  const RedSlot &red, cudaStream_t s, const int *done);
void launch_bcg_xr(long long n, const BcgState *st, cd *x, const cd *ph, const cd *sh,
                   const cd *sv, const cd *t, cd *r, const cd *rs, const RedSlot &red,
                   cudaStream_t s, const int *done);
void launch_bcg_xhalf(long long n, const BcgState *st, cd *x, const cd *ph, cudaStream_t s);
void launch_bcg_step(BcgState *st, int op, const cd *sums, cudaStream_t s);
// slab drivers: *out = this slab's share of r~^H g over its own nonzeros of r~ (list in nz)
void launch_gather_store(const BcgState *nz, const cd *g, cd *out, cudaStream_t s, const int *done);
// sparse shadow: sums[0] = r~^H g gathered over the nonzeros of r~, then scalar step `op`
void launch_bcg_gather(BcgState *st, int op, const cd *g, cudaStream_t s, const int *done);
// find the (<= HF_NZ_MAX) nonzeros of the shadow vector: st->nz = count, or -1 (dense)
void launch_nz_scan(long long n, const cd *rs, BcgState *st, cudaStream_t s);

#define VEC_BLOCKS_HOST 592

// coarsest GMRES in one cooperative launch (hf_coarse_gmres.cu)
struct GmArgs {
    Lvl L;                 // coarsest level (whole grid)
    long long N;
    int cap, maxit;        // basis vectors, iteration limit (multigrid.py:48-49)
    double tol, btol;
    const cd *b;
    cd *x;
    cd *V;                 // (cap + 1) * N basis
    cd *part;              // 2 * blocks * (cap + 2) partial sums (double-buffered)
    cd *Hm;                // cap * cap rotated Hessenberg columns (block 0)
    cd *y;                 // cap
    int *flags;            // solves that missed tol (coarsest_flags)
    const int *done;
};
size_t coarse_gmres_smem(int cap);
int coarse_gmres_blocks(long long N, int cap);
cudaError_t launch_coarse_gmres(const GmArgs &a, int nblk, cudaStream_t s);

}  // namespace hf
