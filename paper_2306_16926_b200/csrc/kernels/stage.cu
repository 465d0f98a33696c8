// Stage kernels of the group step: the HBM-bound streaming passes.
//
// stage 1 (the iteration barrier; OspServer::try_close_barrier + finish_layer,
//   protocol.cpp:292-307, 361-382, and the pull on every co-resident worker,
//   OspWorker::apply_pull -> lgp_partial, protocol.cpp:69-97, 212-228):
//   RS layer element:  agg = float(sum_w w_k*(double)x_k / W)   (fixed worker order)
//                      G' = G + agg;  P_w = G'  for every worker  (p + 1.0f*agg, p == G)
//                      PGP partial += |(double)agg * (double)G'|
//   ICS layer element: P_w = G + x_w                              (base + local estimate)
// stage 2 (one ICS chunk; on_push_ics_chunk -> finish_layer, protocol.cpp:326-353,
//   and lgp_correct, protocol.cpp:99-116):
//   element of a chunk layer: agg as above; G' = G + agg; P_w = G' (base + global,
//   base == G by gradient conservation); PGP partial.
//
// Worker parameters are written, not read: at an iteration boundary every
// worker's parameters equal the global vector bit-for-bit (the reference's
// conservation check, checks.cpp:126-184), so `p` in lgp_partial is G and the
// per-worker `base` copies of the reference are never materialised.
//
// Work decomposition: the flat vector is cut into tiles of T elements that
// never straddle a layer (tile -> layer table built once per partition). A
// persistent grid walks tiles; each tile is a 128-bit vectorised streaming pass
// (two quads in flight per thread, nc/no_allocate loads of the deltas,
// evict-first stores of the worker rows) with scalar head/tail for layers whose
// offset is not 16-byte aligned. The PGP partial of a tile is reduced in a fixed
// order and written to partials[tile], so the per-layer sum is deterministic.

#include "common.cuh"

namespace osp {
namespace {

// ---------------------------------------------------------------------------
// per-element bodies
// ---------------------------------------------------------------------------

__device__ __forceinline__ float ldx1(const AggParams& ap, const float* X, uint64_t ldX, int w,
                                      uint64_t f) {
    float v = ld_stream1(X + static_cast<uint64_t>(w) * ldX + f);
    return ap.sgd ? sgd_conv(ap.neg_lr, v) : v;
}

__device__ __forceinline__ float4 cvt4(const AggParams& ap, float4 v) {
    if (ap.sgd) {
        v.x = sgd_conv(ap.neg_lr, v.x);
        v.y = sgd_conv(ap.neg_lr, v.y);
        v.z = sgd_conv(ap.neg_lr, v.z);
        v.w = sgd_conv(ap.neg_lr, v.w);
    }
    return v;
}

template <int NS>
__device__ __forceinline__ int nworkers(const AggParams& ap) {
    return NS > 0 ? NS : ap.n;
}

// Aggregate + apply one scalar element.
template <int NS>
__device__ __forceinline__ void agg_scalar(const GroupView& g, const AggParams& ap,
                                           const float* X, uint64_t ldX, uint64_t f,
                                           double& acc) {
    const int n = nworkers<NS>(ap);
    double s = 0.0;
    for (int w = 0; w < n; ++w) s = agg_acc(s, ap.w[w], ldx1(ap, X, ldX, w, f));
    const float a = agg_finish(ap, s);
    const float gn = __fadd_rn(g.G[f], a);
    g.G[f] = gn;
    for (int w = 0; w < n; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
    acc = __dadd_rn(acc, pgp_term(a, gn));
}

template <int NS>
__device__ __forceinline__ void local_scalar(const GroupView& g, const AggParams& ap,
                                             const float* X, uint64_t ldX, uint64_t f) {
    const int n = nworkers<NS>(ap);
    const float go = g.G[f];
    for (int w = 0; w < n; ++w)
        g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, ldx1(ap, X, ldX, w, f));
}

// Finish one quad whose deltas are already in registers.
template <int NS>
__device__ __forceinline__ void agg_quad_finish(const GroupView& g, const AggParams& ap,
                                                const float4* x, float4 go, uint64_t f,
                                                double& acc) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int w = 0; w < NS; ++w) {
        const float4 v = cvt4(ap, x[w]);
        const double wt = ap.w[w];
        s0 = agg_acc(s0, wt, v.x);
        s1 = agg_acc(s1, wt, v.y);
        s2 = agg_acc(s2, wt, v.z);
        s3 = agg_acc(s3, wt, v.w);
    }
    float4 a, gn;
    a.x = agg_finish(ap, s0);
    a.y = agg_finish(ap, s1);
    a.z = agg_finish(ap, s2);
    a.w = agg_finish(ap, s3);
    gn.x = __fadd_rn(go.x, a.x);
    gn.y = __fadd_rn(go.y, a.y);
    gn.z = __fadd_rn(go.z, a.z);
    gn.w = __fadd_rn(go.w, a.w);
    *reinterpret_cast<float4*>(g.G + f) = gn;
#pragma unroll
    for (int w = 0; w < NS; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
    acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
    acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
    acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
    acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
}

// Dynamic worker count: accumulate while loading (no register arrays).
__device__ __forceinline__ void agg_quad_dyn(const GroupView& g, const AggParams& ap,
                                             const float* X, uint64_t ldX, uint64_t f,
                                             double& acc) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    const float4 go = *reinterpret_cast<const float4*>(g.G + f);
    for (int w = 0; w < ap.n; ++w) {
        const float4 v = cvt4(ap, ld_stream4(X + static_cast<uint64_t>(w) * ldX + f));
        const double wt = ap.w[w];
        s0 = agg_acc(s0, wt, v.x);
        s1 = agg_acc(s1, wt, v.y);
        s2 = agg_acc(s2, wt, v.z);
        s3 = agg_acc(s3, wt, v.w);
    }
    float4 a, gn;
    a.x = agg_finish(ap, s0);
    a.y = agg_finish(ap, s1);
    a.z = agg_finish(ap, s2);
    a.w = agg_finish(ap, s3);
    gn.x = __fadd_rn(go.x, a.x);
    gn.y = __fadd_rn(go.y, a.y);
    gn.z = __fadd_rn(go.z, a.z);
    gn.w = __fadd_rn(go.w, a.w);
    *reinterpret_cast<float4*>(g.G + f) = gn;
    for (int w = 0; w < ap.n; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
    acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
    acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
    acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
    acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                       __fadd_rn(a.w, b.w));
}

// ---------------------------------------------------------------------------
// tile bodies
// ---------------------------------------------------------------------------

// RS (stage 1) / ICS chunk (stage 2): aggregate + apply + broadcast to workers.
template <int NS>
__device__ void tile_agg(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                         uint64_t s, uint64_t e, bool vec, double& acc) {
    const int tid = threadIdx.x;
    const int B = blockDim.x;
    uint64_t hs = s, he = s, be = s;
    if (vec) {
        he = min(e, (s + 3) & ~uint64_t(3));
        be = he + ((e - he) & ~uint64_t(3));
    } else {
        he = e;
        be = e;
    }
    for (uint64_t f = hs + tid; f < he; f += B) agg_scalar<NS>(g, ap, X, ldX, f, acc);
    if constexpr (NS > 0) {
        const uint64_t step = 4ull * B;
        for (uint64_t f0 = he + 4ull * tid; f0 < be; f0 += 2 * step) {
            const uint64_t f1 = f0 + step;
            const bool has1 = f1 < be;
            float4 xa[NS], xb[NS];
#pragma unroll
            for (int w = 0; w < NS; ++w) {
                xa[w] = ld_stream4(X + static_cast<uint64_t>(w) * ldX + f0);
                if (has1) xb[w] = ld_stream4(X + static_cast<uint64_t>(w) * ldX + f1);
            }
            const float4 ga = *reinterpret_cast<const float4*>(g.G + f0);
            float4 gb = make_float4(0.f, 0.f, 0.f, 0.f);
            if (has1) gb = *reinterpret_cast<const float4*>(g.G + f1);
            agg_quad_finish<NS>(g, ap, xa, ga, f0, acc);
            if (has1) agg_quad_finish<NS>(g, ap, xb, gb, f1, acc);
        }
    } else {
        for (uint64_t f0 = he + 4ull * tid; f0 < be; f0 += 4ull * B)
            agg_quad_dyn(g, ap, X, ldX, f0, acc);
    }
    for (uint64_t f = be + tid; f < e; f += B) agg_scalar<NS>(g, ap, X, ldX, f, acc);
}

// ICS layer at the barrier: each worker takes its own delta on top of G.
template <int NS>
__device__ void tile_local(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                           uint64_t s, uint64_t e, bool vec) {
    const int tid = threadIdx.x;
    const int B = blockDim.x;
    uint64_t he = e, be = e;
    if (vec) {
        he = min(e, (s + 3) & ~uint64_t(3));
        be = he + ((e - he) & ~uint64_t(3));
    }
    for (uint64_t f = s + tid; f < he; f += B) local_scalar<NS>(g, ap, X, ldX, f);
    if constexpr (NS > 0) {
        const uint64_t step = 4ull * B;
        for (uint64_t f0 = he + 4ull * tid; f0 < be; f0 += 2 * step) {
            const uint64_t f1 = f0 + step;
            const bool has1 = f1 < be;
            float4 xa[NS], xb[NS];
#pragma unroll
            for (int w = 0; w < NS; ++w) {
                xa[w] = ld_stream4(X + static_cast<uint64_t>(w) * ldX + f0);
                if (has1) xb[w] = ld_stream4(X + static_cast<uint64_t>(w) * ldX + f1);
            }
            const float4 ga = *reinterpret_cast<const float4*>(g.G + f0);
            float4 gb = make_float4(0.f, 0.f, 0.f, 0.f);
            if (has1) gb = *reinterpret_cast<const float4*>(g.G + f1);
#pragma unroll
            for (int w = 0; w < NS; ++w)
                st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f0, add4(ga, cvt4(ap, xa[w])));
            if (has1) {
#pragma unroll
                for (int w = 0; w < NS; ++w)
                    st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f1,
                               add4(gb, cvt4(ap, xb[w])));
            }
        }
    } else {
        for (uint64_t f0 = he + 4ull * tid; f0 < be; f0 += 4ull * B) {
            const float4 go = *reinterpret_cast<const float4*>(g.G + f0);
            for (int w = 0; w < ap.n; ++w) {
                const float4 v = cvt4(ap, ld_stream4(X + static_cast<uint64_t>(w) * ldX + f0));
                st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f0, add4(go, v));
            }
        }
    }
    for (uint64_t f = be + tid; f < e; f += B) local_scalar<NS>(g, ap, X, ldX, f);
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

template <int NS>
__global__ void __launch_bounds__(kStageThreads) k_stage1(GroupView g, AggParams ap,
                                                          const float* __restrict__ X,
                                                          uint64_t ldX, int vec) {
    __shared__ double red[kStageThreads / 32];
    for (int t = blockIdx.x; t < g.NT; t += gridDim.x) {
        const int l = g.tile_layer[t];
        const uint64_t lo = g.offsets[l];
        const uint64_t s = lo + static_cast<uint64_t>(t - g.tile_base[l]) * g.T;
        const uint64_t e = min(s + static_cast<uint64_t>(g.T), lo + g.counts[l]);
        if (g.flags[l]) {
            tile_local<NS>(g, ap, X, ldX, s, e, vec != 0);
        } else {
            double acc = 0.0;
            tile_agg<NS>(g, ap, X, ldX, s, e, vec != 0, acc);
            const double tot = block_sum_fixed<kStageThreads>(acc, red);
            if (threadIdx.x == 0) g.partials[t] = tot;
        }
    }
}

template <int NS>
__global__ void __launch_bounds__(kStageThreads) k_stage2(GroupView g, AggParams ap,
                                                          const float* __restrict__ X,
                                                          uint64_t ldX, int chunk, int vec) {
    __shared__ double red[kStageThreads / 32];
    if (chunk >= g.meta[META_N_USED]) return;
    const int jb = g.chunk_begin[chunk], je = g.chunk_begin[chunk + 1];
    const int u0 = g.ics_tile_prefix[jb], u1 = g.ics_tile_prefix[je];
    for (int u = u0 + blockIdx.x; u < u1; u += gridDim.x) {
        // layer j of the chunk with ics_tile_prefix[j] <= u < ics_tile_prefix[j+1]
        int a = jb, b = je - 1;
        while (a < b) {
            const int m = (a + b + 1) >> 1;
            if (g.ics_tile_prefix[m] <= u) a = m;
            else b = m - 1;
        }
        const int l = g.ics_layers[a];
        const int k = u - g.ics_tile_prefix[a];
        const uint64_t lo = g.offsets[l];
        const uint64_t s = lo + static_cast<uint64_t>(k) * g.T;
        const uint64_t e = min(s + static_cast<uint64_t>(g.T), lo + g.counts[l]);
        double acc = 0.0;
        tile_agg<NS>(g, ap, X, ldX, s, e, vec != 0, acc);
        const double tot = block_sum_fixed<kStageThreads>(acc, red);
        if (threadIdx.x == 0) g.partials[g.tile_base[l] + k] = tot;
    }
}

bool vec_ok(const GroupView& g, const float* X, uint64_t ldX) {
    return (ldX % 4 == 0) && (g.ldP % 4 == 0) &&
           (reinterpret_cast<uintptr_t>(X) % 16 == 0) &&
           (reinterpret_cast<uintptr_t>(g.G) % 16 == 0) &&
           (reinterpret_cast<uintptr_t>(g.P) % 16 == 0);
}

template <typename K1>
cudaError_t dispatch_n(int n, K1&& k) {
    switch (n) {
        case 1: return k(std::integral_constant<int, 1>{});
        case 2: return k(std::integral_constant<int, 2>{});
        case 4: return k(std::integral_constant<int, 4>{});
        case 8: return k(std::integral_constant<int, 8>{});
        default: return k(std::integral_constant<int, 0>{});
    }
}

}  // namespace

int stage_blocks_per_sm(int n_workers) {
    int blocks = 0;
    cudaError_t e = dispatch_n(n_workers, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_stage1<NS>,
                                                             kStageThreads, 0);
    });
    if (e != cudaSuccess || blocks < 1) blocks = 1;
    return blocks;
}

cudaError_t launch_stage1(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int grid, cudaStream_t s) {
    const int vec = vec_ok(g, X, ldX) ? 1 : 0;
    grid = grid < g.NT ? grid : g.NT;
    if (grid < 1) return cudaSuccess;
    return dispatch_n(ap.n, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        k_stage1<NS><<<grid, kStageThreads, 0, s>>>(g, ap, X, ldX, vec);
        return cudaGetLastError();
    });
}

cudaError_t launch_stage2(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int chunk, int grid, cudaStream_t s) {
    const int vec = vec_ok(g, X, ldX) ? 1 : 0;
    grid = grid < g.NT ? grid : g.NT;
    if (grid < 1) return cudaSuccess;
    return dispatch_n(ap.n, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        k_stage2<NS><<<grid, kStageThreads, 0, s>>>(g, ap, X, ldX, chunk, vec);
        return cudaGetLastError();
    });
}

}  // namespace osp
