// Device helpers shared by the OSP kernels. Every fp32/fp64 operation that the
// reference rounds separately is written with an explicit _rn intrinsic, so no
// FMA contraction can change a bit (SURVEY.md §7 hard part 3); the library is
// also compiled with --fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include "../osp_internal.h"

namespace osp {

// Checked build (make checked -> libosp_b200_checked.so, OSP_LIB_VARIANT=checked):
// every kernel's indices are bounds-checked against the group geometry and a
// violation prints its site and traps. compute-sanitizer is not available on
// the GPU pool, so the test suite runs against this build instead
// (tools/gpu_r2_checked.sh). Compiles to nothing in the product build.
#ifdef OSP_CHECKED
#define OSP_DCHECK(cond, what)                                                          \
    do {                                                                                \
        if (!(cond)) {                                                                  \
            printf("OSP_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, \
                   __LINE__, static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x)); \
            __trap();                                                                   \
        }                                                                               \
    } while (0)
#else
#define OSP_DCHECK(cond, what) \
    do {                       \
    } while (0)
#endif

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled while its predecessor in the stream drains; it must call pdl_wait()
// before touching anything the predecessor wrote (a no-op without the
// attribute), and pdl_trigger() lets its own successor start launching early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ float4 ld_stream4(const float* p) {
    float4 r;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
        : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
        : "l"(p));
    return r;
}

__device__ __forceinline__ float ld_stream1(const float* p) {
    float r;
    asm("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(r) : "l"(p));
    return r;
}

// Loads from peer GPUs' HBM over NVLink (CUDA IPC mappings): mode 0 = nc /
// no_allocate (as local streaming), 1 = .cg (L2 only), 2 = default caching.
__device__ __forceinline__ float4 ld_peer4(const float* p, int mode) {
    float4 r;
    if (mode == 1) {
        asm volatile("ld.global.cg.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "l"(p));
    } else if (mode == 2) {
        asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                     : "l"(p));
    } else {
        r = ld_stream4(p);
    }
    return r;
}

__device__ __forceinline__ void st_stream4(float* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// sgd_delta (learner.cpp:395): float(-lr * (double)g)
__device__ __forceinline__ float sgd_conv(double neg_lr, float g) {
    return __double2float_rn(__dmul_rn(neg_lr, static_cast<double>(g)));
}

// One step of aggregate_layer's inner loop (protocol.cpp:24):
// sum += weights[w] * (double)x  — mul rounded, then add rounded.
__device__ __forceinline__ double agg_acc(double sum, double w, float x) {
    return __dadd_rn(sum, __dmul_rn(w, static_cast<double>(x)));
}

// out[e] = static_cast<float>(sum / total_weight) (protocol.cpp:26); x/1.0 == x.
__device__ __forceinline__ float agg_finish(const AggParams& ap, double sum) {
    return __double2float_rn(ap.divide ? __ddiv_rn(sum, ap.total) : sum);
}

// One PGP term |(double)g * (double)p| (importance.cpp:21-23); exact in double.
__device__ __forceinline__ double pgp_term(float g, float p) {
    return fabs(__dmul_rn(static_cast<double>(g), static_cast<double>(p)));
}

// Deterministic block reduction (fixed shuffle tree, then warps in order).
// Depth contributed: 5 (shuffle) + nwarps - 1 (sequential over warps).
template <int THREADS>
__device__ __forceinline__ double block_sum_fixed(double v, double* red) {
    constexpr int W = THREADS / 32;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < W; ++k) s = __dadd_rn(s, red[k]);
    }
    __syncthreads();
    return s;  // valid in thread 0
}

}  // namespace osp
