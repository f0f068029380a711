// hf_stencil.cuh -- device / launch building blocks shared by the kernel
// translation units (hf_kernels.cu, hf_wide.cu): programmatic dependent launch,
// mbarrier / bulk-copy wrappers, the stencil epilogues and the launch helper.
#pragma once
#include <utility>

#include "hf_kernels.cuh"

namespace hf {

// Programmatic dependent launch: every kernel is launched with the
// programmatic-stream-serialization attribute.  On entry a CTA waits for the
// previous grid to complete (its writes are then visible).  A SMALL grid (the
// coarse levels, the scalar steps) then signals at once that the next grid may
// launch: that happens once every CTA of this grid is resident, so the next
// kernel's CTAs fill SMs as this grid's last wave drains and start the moment
// it completes -- the launch latency is hidden.  A LARGE grid (many waves: the
// 513^3 sweeps) does not signal: the next grid launches when this one exits.
// Its early-resident CTAs would only take shared memory and warp slots from the
// running sweep (measured at 513^3: 18.9 -> 18.2 ms per iteration for the tiled
// sweeps, 19.0 -> 17.6 for the wide family).  Waiting before anything else
// keeps the chain transitive (no grid can finish before its predecessor).
#define HF_PDL_EARLY_BLOCKS (148 * 8)
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    if (gridDim.x * gridDim.y * gridDim.z <= HF_PDL_EARLY_BLOCKS)
        asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ bool is_done(const int *done) {
    pdl_enter();
    return done && *(volatile const int *)done;
}

__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// epilogues: epi(q, f_centre, (M f)_centre, w D^-1 at the centre, staged operand, acc)
// v = M f (+ inner products), DOT: 0 none, 1 conj(w) v, 2 conj(v) v & conj(v) w
template <int DOT>
struct EpiApply {
    cd *v;
    static constexpr bool kAux = DOT > 0;   // w
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

// u = f + w D^-1 (b - M f) (one damped Jacobi sweep, multigrid.py:153-156)
struct EpiJacobi {
    cd *u;
    static constexpr bool kAux = true;      // b
    static constexpr bool kDinv = true;
    __device__ __forceinline__ void operator()(long long q, cd fc, cd mf, cd wd, cd b,
                                               cd (&)[2]) const {
        u[q] = cadd(fc, cmul(wd, csub(b, mf)));
    }
};

// every launch carries the programmatic-stream-serialization attribute (PDL)
template <class... KArgs, class... Args>
static inline void launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                   Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    const bool pdl = !opt(OPT_NO_PDL);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}


}  // namespace hf
