// Element-wise device primitives behind the per-function C-ABI entry points
// (the reference free functions, one kernel each). The group step (stage.cu)
// fuses these; here they stand alone so the C++ façade can replay the
// reference's message-by-message engine on the device.

#include "common.cuh"

namespace osp {
namespace {

struct Contribs {
    const float* p[OSP_MAX_WORKERS];
};

constexpr int kEwThreads = 256;

int ew_grid(uint64_t n) {
    const uint64_t want = (n + kEwThreads - 1) / kEwThreads;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
    return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

// aggregate_layer (protocol.cpp:9-30)
__global__ void k_aggregate(Contribs c, AggParams ap, uint64_t n, float* __restrict__ out) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int w = 0; w < ap.n; ++w) s = agg_acc(s, ap.w[w], c.p[w][e]);
        out[e] = agg_finish(ap, s);
    }
}

// finish_layer over segments (protocol.cpp:292-307): agg, global += agg.
__global__ void k_aggregate_apply(Contribs c, AggParams ap, const uint64_t* __restrict__ seg_off,
                                  const uint64_t* __restrict__ seg_cnt, float* __restrict__ global,
                                  float* __restrict__ agg_out) {
    const int sg = blockIdx.y;
    const uint64_t off = seg_off[sg], cnt = seg_cnt[sg];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = off + i;
        double s = 0.0;
        for (int w = 0; w < ap.n; ++w) s = agg_acc(s, ap.w[w], c.p[w][e]);
        const float a = agg_finish(ap, s);
        global[e] = __fadd_rn(global[e], a);
        if (agg_out) agg_out[e] = a;
    }
}

// apply_delta (param.cpp:127-150): p += scale * d, fp32 mul then add.
__global__ void k_apply_delta(float* __restrict__ p, const float* __restrict__ d, uint64_t n,
                              float scale) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x)
        p[e] = __fadd_rn(p[e], __fmul_rn(scale, d[e]));
}

// sgd_delta (learner.cpp:391-398)
__global__ void k_sgd(const float* __restrict__ g, uint64_t n, double neg_lr,
                      float* __restrict__ out) {
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n;
         e += uint64_t(gridDim.x) * blockDim.x)
        out[e] = sgd_conv(neg_lr, g[e]);
}

// ---- synthetic deltas (runner.cpp:312-321, rng.hpp:16-61) ------------------
constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t splitmix(uint64_t& s) {
    s += kGamma;
    return mix64(s);
}

__device__ uint64_t derive_seed_dev(uint64_t root, uint64_t tag, uint64_t a, uint64_t b) {
    uint64_t s = root;
    splitmix(s);
    s ^= 0x6a09e667f3bcc908ull + tag;
    splitmix(s);
    s ^= 0xbb67ae8584caa73bull + a;
    splitmix(s);
    s ^= 0x3c6ef372fe94f82bull + b;
    return splitmix(s);
}

// Rng(seed) warms up with two draws, so draw k uses state seed + (k+3)*gamma;
// uniform(lo, hi) = lo + (hi - lo) * u53, then float (runner.cpp:318-320).
__global__ void k_synth(uint64_t seed, uint64_t iteration, uint64_t worker0, uint64_t first,
                        uint64_t n, float* __restrict__ out, uint64_t ld) {
    const uint64_t w = worker0 + blockIdx.y;
    const uint64_t s = derive_seed_dev(seed, 6, w, iteration);
    const double lo = -1e-3;
    const double span = __dsub_rn(1e-3, -1e-3);
    float* row = out + static_cast<uint64_t>(blockIdx.y) * ld;
    for (uint64_t k = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t x = mix64(s + (first + k + 3) * kGamma);
        const double u = __dmul_rn(__ull2double_rn(x >> 11), 0x1.0p-53);
        row[k] = __double2float_rn(__dadd_rn(lo, __dmul_rn(span, u)));
    }
}

// lgp_partial (protocol.cpp:69-97) over segments: local -> base = p; p += local,
// else p += 1.0f * global.
__global__ void k_lgp_partial(float* __restrict__ p, const float* __restrict__ gd,
                              const float* __restrict__ ld_, float* __restrict__ base,
                              const uint64_t* __restrict__ seg_off,
                              const uint64_t* __restrict__ seg_cnt,
                              const uint8_t* __restrict__ seg_local) {
    const int sg = blockIdx.y;
    const uint64_t off = seg_off[sg], cnt = seg_cnt[sg];
    const bool local = seg_local[sg] != 0;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = off + i;
        const float v = p[e];
        if (local) {
            base[e] = v;
            p[e] = __fadd_rn(v, ld_[e]);
        } else {
            p[e] = __fadd_rn(v, __fmul_rn(1.0f, gd[e]));
        }
    }
}

// lgp_correct (protocol.cpp:99-116): p = base + global
__global__ void k_lgp_correct(float* __restrict__ p, const float* __restrict__ base,
                              const float* __restrict__ gd, const uint64_t* __restrict__ seg_off,
                              const uint64_t* __restrict__ seg_cnt) {
    const int sg = blockIdx.y;
    const uint64_t off = seg_off[sg], cnt = seg_cnt[sg];
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < cnt;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t e = off + i;
        p[e] = __fadd_rn(base[e], gd[e]);
    }
}

Contribs pack(const float* const* contribs, int n) {
    Contribs c{};
    for (int w = 0; w < n; ++w) c.p[w] = contribs[w];
    return c;
}

}  // namespace

cudaError_t launch_aggregate_layer(const float* const* contribs, const AggParams& ap, uint64_t n,
                                   float* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_aggregate<<<ew_grid(n), kEwThreads, 0, s>>>(pack(contribs, ap.n), ap, n, out);
    return cudaGetLastError();
}

cudaError_t launch_aggregate_apply_segments(const float* const* contribs, const AggParams& ap,
                                            const uint64_t* seg_off, const uint64_t* seg_cnt,
                                            int n_seg, float* global, float* agg_out,
                                            cudaStream_t s) {
    if (n_seg == 0) return cudaSuccess;
    // grid.x sized for the largest segment would need it on the host; 64 blocks
    // per segment row with a grid-stride loop covers any size.
    k_aggregate_apply<<<dim3(64, n_seg), kEwThreads, 0, s>>>(pack(contribs, ap.n), ap, seg_off,
                                                             seg_cnt, global, agg_out);
    return cudaGetLastError();
}

cudaError_t launch_apply_delta(float* p, const float* d, uint64_t n, float scale, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_apply_delta<<<ew_grid(n), kEwThreads, 0, s>>>(p, d, n, scale);
    return cudaGetLastError();
}

cudaError_t launch_sgd_delta(const float* g, uint64_t n, double lr, float* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_sgd<<<ew_grid(n), kEwThreads, 0, s>>>(g, n, -lr, out);
    return cudaGetLastError();
}

cudaError_t launch_synth(uint64_t seed, int n_workers, uint64_t iteration, uint64_t first,
                         uint64_t n, float* out, uint64_t ld, uint64_t worker0, cudaStream_t s) {
    if (n == 0 || n_workers == 0) return cudaSuccess;
    uint64_t bx = (n + kEwThreads - 1) / kEwThreads;
    const uint64_t cap = static_cast<uint64_t>(sm_count()) * 8;
    if (bx > cap) bx = cap;
    k_synth<<<dim3(static_cast<unsigned>(bx), n_workers), kEwThreads, 0, s>>>(
        seed, iteration, worker0, first, n, out, ld);
    return cudaGetLastError();
}

cudaError_t launch_lgp_partial_segments(float* p, const float* global_delta,
                                        const float* local_delta, float* base,
                                        const uint64_t* seg_off, const uint64_t* seg_cnt,
                                        const uint8_t* seg_local, int n_seg, cudaStream_t s) {
    if (n_seg == 0) return cudaSuccess;
    k_lgp_partial<<<dim3(64, n_seg), kEwThreads, 0, s>>>(p, global_delta, local_delta, base,
                                                         seg_off, seg_cnt, seg_local);
    return cudaGetLastError();
}

cudaError_t launch_lgp_correct_segments(float* p, const float* base, const float* global_delta,
                                        const uint64_t* seg_off, const uint64_t* seg_cnt,
                                        int n_seg, cudaStream_t s) {
    if (n_seg == 0) return cudaSuccess;
    k_lgp_correct<<<dim3(64, n_seg), kEwThreads, 0, s>>>(p, base, global_delta, seg_off, seg_cnt);
    return cudaGetLastError();
}

}  // namespace osp
