// Helpers shared by the sharded exchange kernels (shard_x.cu, shard_chain.cu).
#pragma once

#include "common.cuh"
#include "tma.cuh"

namespace osp {
namespace {

// position u of a tile sequence given as layer prefixes lp[0..n] (layer ids ll,
// or the identity when null): the layer l and the tile index k inside it
__device__ __forceinline__ void xseq_lookup(const int* lp, const int* ll, int n, int u, int& l,
                                            int& k) {
    int a = 0, b = n - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (lp[m] <= u) a = m;
        else b = m - 1;
    }
    l = ll ? ll[a] : a;
    k = u - lp[a];
}

__device__ __forceinline__ bool xspin(const unsigned* p, unsigned want, unsigned* error) {
    if (static_cast<int>(ld_acquire_sys(p) - want) >= 0) return true;
    const uint64_t t0 = now_ns();
    while (static_cast<int>(ld_acquire_sys(p) - want) < 0) {
        __nanosleep(64);
        if (now_ns() - t0 > 20000000000ull) {
            atomicExch(error, 1u);
            return false;
        }
    }
    return true;
}

__device__ __forceinline__ float4 cvt4x(const AggParams& ap, float4 v) {
    if (ap.sgd) {
        v.x = sgd_conv(ap.neg_lr, v.x);
        v.y = sgd_conv(ap.neg_lr, v.y);
        v.z = sgd_conv(ap.neg_lr, v.z);
        v.w = sgd_conv(ap.neg_lr, v.w);
    }
    return v;
}

__device__ __forceinline__ float4 add4x(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                       __fadd_rn(a.w, b.w));
}

}  // namespace
}  // namespace osp
