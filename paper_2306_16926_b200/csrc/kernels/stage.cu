// Stage kernels of the group step: the HBM-bound streaming passes.
//
// stage 1 (the iteration barrier; OspServer::try_close_barrier + finish_layer,
//   protocol.cpp:292-307, 361-382, and the pull on every co-resident worker,
//   OspWorker::apply_pull -> lgp_partial, protocol.cpp:69-97, 212-228):
//   RS layer element:  agg = float(sum_w w_k*(double)x_k / W)   (fixed worker order)
//                      G' = G + agg;  P_w = G'  for every worker  (p + 1.0f*agg, p == G)
//                      PGP partial += |(double)agg * (double)G'|
//   ICS layer element: P_w = G + x_w                              (base + local estimate)
// stage 2 (ICS chunks [c0, c1); on_push_ics_chunk -> finish_layer,
//   protocol.cpp:326-353, and lgp_correct, protocol.cpp:99-116):
//   element of a chunk layer: agg as above; G' = G + agg; P_w = G' (base + global,
//   base == G by gradient conservation); PGP partial.
//
// Worker parameters are written, not read: at an iteration boundary every
// worker's parameters equal the global vector bit-for-bit (the reference's
// conservation check, checks.cpp:126-184), so `p` in lgp_partial is G and the
// per-worker `base` copies of the reference are never materialised.
//
// Work decomposition. The flat vector is cut into tiles of T elements that never
// straddle a layer. A tile is owned by ONE WARP: lanes stream it with 128-bit
// loads (two quads per lane in flight per iteration, nc/no_allocate loads of the
// deltas, evict-first stores of the worker rows; scalar head/tail when a layer
// offset is not 16-byte aligned) and reduce the tile's PGP partial with a fixed
// shuffle tree — no block barrier anywhere in the streaming loop. Warps take
// tiles from a device work counter (one atomic per tile, prefetched one tile
// ahead), so the tail is a fraction of one tile however ragged the layer table
// is; the last warp out resets the counter for the next launch.

#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"

namespace osp {
namespace {

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

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
    return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                       __fadd_rn(a.w, b.w));
}

template <int NS>
__device__ __forceinline__ int nworkers(const AggParams& ap) {
    return NS > 0 ? NS : ap.n;
}

// ---- aggregate + apply ------------------------------------------------------

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

__device__ __forceinline__ void agg_finish4(const GroupView& g, const AggParams& ap, double s0,
                                            double s1, double s2, double s3, float4 go,
                                            uint64_t f, int n, double& acc) {
    float4 a, gn;
    a.x = agg_finish(ap, s0);
    a.y = agg_finish(ap, s1);
    a.z = agg_finish(ap, s2);
    a.w = agg_finish(ap, s3);
    gn = add4(go, a);
    *reinterpret_cast<float4*>(g.G + f) = gn;
    for (int w = 0; w < n; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
    acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
    acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
    acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
    acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
}

template <int NS>
__device__ __forceinline__ void agg_quad_regs(const GroupView& g, const AggParams& ap,
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
    agg_finish4(g, ap, s0, s1, s2, s3, go, f, NS, acc);
}

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
    agg_finish4(g, ap, s0, s1, s2, s3, go, f, ap.n, acc);
}

// One warp aggregates [s, e) of one layer.
template <int NS>
__device__ void warp_tile_agg(const GroupView& g, const AggParams& ap, const float* X,
                              uint64_t ldX, uint64_t s, uint64_t e, bool vec, int lane,
                              double& acc) {
    uint64_t he = e, be = e;
    if (vec) {
        he = min(e, (s + 3) & ~uint64_t(3));
        be = he + ((e - he) & ~uint64_t(3));
    }
    for (uint64_t f = s + lane; f < he; f += 32) agg_scalar<NS>(g, ap, X, ldX, f, acc);
    if constexpr (NS > 0) {
        for (uint64_t f0 = he + 4ull * lane; f0 < be; f0 += 256) {
            const uint64_t f1 = f0 + 128;
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
            agg_quad_regs<NS>(g, ap, xa, ga, f0, acc);
            if (has1) agg_quad_regs<NS>(g, ap, xb, gb, f1, acc);
        }
    } else {
        for (uint64_t f0 = he + 4ull * lane; f0 < be; f0 += 128) agg_quad_dyn(g, ap, X, ldX, f0, acc);
    }
    for (uint64_t f = be + lane; f < e; f += 32) agg_scalar<NS>(g, ap, X, ldX, f, acc);
}

// ---- local estimate (ICS layers at the barrier) -------------------------------

template <int NS>
__device__ __forceinline__ void local_scalar(const GroupView& g, const AggParams& ap,
                                             const float* X, uint64_t ldX, uint64_t f) {
    const int n = nworkers<NS>(ap);
    const float go = g.G[f];
    for (int w = 0; w < n; ++w)
        g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, ldx1(ap, X, ldX, w, f));
}

template <int NS>
__device__ void warp_tile_local(const GroupView& g, const AggParams& ap, const float* X,
                                uint64_t ldX, uint64_t s, uint64_t e, bool vec, int lane) {
    uint64_t he = e, be = e;
    if (vec) {
        he = min(e, (s + 3) & ~uint64_t(3));
        be = he + ((e - he) & ~uint64_t(3));
    }
    for (uint64_t f = s + lane; f < he; f += 32) local_scalar<NS>(g, ap, X, ldX, f);
    if constexpr (NS > 0) {
        for (uint64_t f0 = he + 4ull * lane; f0 < be; f0 += 256) {
            const uint64_t f1 = f0 + 128;
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
        for (uint64_t f0 = he + 4ull * lane; f0 < be; f0 += 128) {
            const float4 go = *reinterpret_cast<const float4*>(g.G + f0);
            for (int w = 0; w < ap.n; ++w) {
                const float4 v = cvt4(ap, ld_stream4(X + static_cast<uint64_t>(w) * ldX + f0));
                st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f0, add4(go, v));
            }
        }
    }
    for (uint64_t f = be + lane; f < e; f += 32) local_scalar<NS>(g, ap, X, ldX, f);
}

// ---- dynamic tile scheduler ------------------------------------------------------

__device__ __forceinline__ int grab(int* next, int lane) {
    int t = 0;
    if (lane == 0) t = atomicAdd(next, 1);
    return __shfl_sync(0xffffffffu, t, 0);
}

__device__ __forceinline__ void retire(int* next, int* done, int lane) {
    if (lane == 0) {
        const int total = static_cast<int>(gridDim.x * (blockDim.x >> 5));
        if (atomicAdd(done, 1) == total - 1) {  // every warp has made its last grab
            atomicExch(next, 0);
            atomicExch(done, 0);
        }
    }
}

__device__ __forceinline__ double warp_sum_fixed(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;
}

// Publish a tile's PGP partial (fixed shuffle tree); resolve.cu reduces the
// layer's partials in a fixed order.
__device__ __forceinline__ void finish_tile(const GroupView& g, int t, double acc, int lane) {
    acc = warp_sum_fixed(acc);
    if (lane == 0) g.partials[t] = acc;
}

// ---- per-block layer tables ----------------------------------------------------
// Each tile needs its layer's offset, size, first tile and flag, and (stage 2)
// its position in the ICS list. Loading those from global memory is a chain of
// dependent L2 round trips per tile (~1-2 us against ~13 us of streaming per
// tile), so every block first copies the tables into shared memory (layouts up
// to kSmemLayers layers) and resolves tiles there; larger layouts read global.

constexpr int kSmemLayers = 2048;

struct Tab {
    const uint64_t* off;  // [L]
    const uint64_t* cnt;  // [L]
    const int* tb;        // [L+1] first tile of each layer
    const uint8_t* flag;  // [L]
    const int* sl;        // sequence layers [n]
    const int* sp;        // sequence tile prefix [n+1]
    int n;                // sequence length
    int L;
};

size_t tab_smem_bytes(int L) {
    return L <= kSmemLayers ? static_cast<size_t>(L) * 29 + 64 : 0;
}

// seq: layer list + tile prefix for positions [jb, je) (stage 2 / shard), or null.
__device__ Tab load_tab(const GroupView& g, unsigned char* sm, const int* seq_layers,
                        const int* seq_pref, int jb, int je) {
    Tab t;
    t.L = g.L;
    t.n = je - jb;
    if (g.L > kSmemLayers) {
        t.off = g.offsets;
        t.cnt = g.counts;
        t.tb = g.tile_base;
        t.flag = g.flags;
        t.sl = seq_layers ? seq_layers + jb : nullptr;
        t.sp = seq_pref ? seq_pref + jb : nullptr;
        return t;
    }
    const int L = g.L;
    uint64_t* off = reinterpret_cast<uint64_t*>(sm);
    uint64_t* cnt = off + L;
    int* tb = reinterpret_cast<int*>(cnt + L);
    int* sl = tb + L + 1;
    int* sp = sl + L;
    uint8_t* flag = reinterpret_cast<uint8_t*>(sp + L + 1);
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
        off[i] = g.offsets[i];
        cnt[i] = g.counts[i];
        tb[i] = g.tile_base[i];
        flag[i] = g.flags[i];
    }
    if (threadIdx.x == 0) tb[L] = g.tile_base[L];
    if (seq_layers)
        for (int i = threadIdx.x; i < t.n; i += blockDim.x) sl[i] = seq_layers[jb + i];
    if (seq_pref)
        for (int i = threadIdx.x; i <= t.n; i += blockDim.x) sp[i] = seq_pref[jb + i];
    __syncthreads();
    t.off = off;
    t.cnt = cnt;
    t.tb = tb;
    t.flag = flag;
    t.sl = sl;
    t.sp = sp;
    return t;
}

// global tile index -> layer (largest l with tb[l] <= t)
__device__ __forceinline__ int tab_layer_of_tile(const Tab& tab, int t) {
    int a = 0, b = tab.L - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (tab.tb[m] <= t) a = m;
        else b = m - 1;
    }
    return a;
}

// sequence tile u (absolute prefix value) -> (layer, tile within layer)
__device__ __forceinline__ void tab_seq_tile(const Tab& tab, int u, int& l, int& k) {
    int a = 0, b = tab.n - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (tab.sp[m] <= u) a = m;
        else b = m - 1;
    }
    l = tab.sl[a];
    k = u - tab.sp[a];
}

__device__ __forceinline__ void tab_range(const Tab& tab, const GroupView& g, int l, int k,
                                          uint64_t& s, uint64_t& e) {
    const uint64_t lo = tab.off[l];
    s = lo + static_cast<uint64_t>(k) * g.T;
    e = min(s + static_cast<uint64_t>(g.T), lo + tab.cnt[l]);
}

// ---- kernels -------------------------------------------------------------------

template <int NS>
__global__ void __launch_bounds__(kStageThreads) k_stage1(GroupView g, AggParams ap,
                                                          const float* __restrict__ X,
                                                          uint64_t ldX, int vec) {
    extern __shared__ __align__(16) unsigned char smem_tab[];
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const Tab tab = load_tab(g, smem_tab, nullptr, nullptr, 0, 0);
    int* next = g.sched + SCHED_S1_NEXT;
    int t = grab(next, lane);
    while (t < g.NT) {
        const int tn = grab(next, lane);  // prefetch the next tile id
        const int l = tab_layer_of_tile(tab, t);
        uint64_t s, e;
        tab_range(tab, g, l, t - tab.tb[l], s, e);
        if (tab.flag[l]) {
            warp_tile_local<NS>(g, ap, X, ldX, s, e, vec != 0, lane);
        } else {
            double acc = 0.0;
            warp_tile_agg<NS>(g, ap, X, ldX, s, e, vec != 0, lane, acc);
            finish_tile(g, t, acc, lane);
        }
        t = tn;
    }
    retire(next, g.sched + SCHED_S1_DONE, lane);
}

// Chunks [c0, c1) of the current ICS list (clamped to the non-empty chunks).
template <int NS>
__global__ void __launch_bounds__(kStageThreads) k_stage2(GroupView g, AggParams ap,
                                                          const float* __restrict__ X,
                                                          uint64_t ldX, int c0, int c1, int vec) {
    extern __shared__ __align__(16) unsigned char smem_tab[];
    pdl_wait();
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    int* next = g.sched + SCHED_S2_NEXT;
    const int used = g.meta[META_N_USED];
    if (c1 > used) c1 = used;
    int jb = 0, je = 0;
    if (c0 < c1) {
        jb = g.chunk_begin[c0];
        je = g.chunk_begin[c1];
    }
    const Tab tab = load_tab(g, smem_tab, g.ics_layers, g.ics_tile_prefix, jb, je);
    const int u0 = tab.n > 0 ? tab.sp[0] : 0, u1 = tab.n > 0 ? tab.sp[tab.n] : 0;
    int u = u0 + grab(next, lane);
    while (u < u1) {
        const int un = u0 + grab(next, lane);
        int l, k;
        tab_seq_tile(tab, u, l, k);
        uint64_t s, e;
        tab_range(tab, g, l, k, s, e);
        double acc = 0.0;
        warp_tile_agg<NS>(g, ap, X, ldX, s, e, vec != 0, lane, acc);
        finish_tile(g, tab.tb[l] + k, acc, lane);
        u = un;
    }
    retire(next, g.sched + SCHED_S2_DONE, lane);
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

// Opt a kernel into the largest table size once per context (dynamic smem
// above 48 KB; the attribute belongs to the context).
cudaError_t allow_tab_smem(const void* fn) {
    static std::mutex mu;
    static std::set<std::pair<unsigned long long, const void*>> done;
    const auto key = std::make_pair(current_ctx_id(), fn);
    std::lock_guard<std::mutex> lock(mu);
    if (done.count(key)) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(tab_smem_bytes(kSmemLayers)));
    if (e == cudaSuccess) done.insert(key);
    return e;
}

int stage_blocks_per_sm(int n_workers, int n_layers) {
    int blocks = 0;
    cudaError_t e = dispatch_n(n_workers, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        cudaError_t r = allow_tab_smem(reinterpret_cast<const void*>(k_stage1<NS>));
        if (r != cudaSuccess) return r;
        return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, k_stage1<NS>, kStageThreads,
                                                             tab_smem_bytes(n_layers));
    });
    if (e != cudaSuccess || blocks < 1) blocks = 1;
    return blocks;
}

cudaError_t launch_stage1(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int grid, cudaStream_t s) {
    const int vec = vec_ok(g, X, ldX) ? 1 : 0;
    if (grid < 1) return cudaSuccess;
    const size_t sm = tab_smem_bytes(g.L);
    return dispatch_n(ap.n, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        cudaError_t e = allow_tab_smem(reinterpret_cast<const void*>(k_stage1<NS>));
        if (e != cudaSuccess) return e;
        return launch_pdl(k_stage1<NS>, dim3(grid), dim3(kStageThreads), sm, s, g, ap, X, ldX, vec);
    });
}

cudaError_t launch_stage2(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int c0, int c1, int grid, cudaStream_t s) {
    const int vec = vec_ok(g, X, ldX) ? 1 : 0;
    if (grid < 1) return cudaSuccess;
    const size_t sm = tab_smem_bytes(g.L);
    return dispatch_n(ap.n, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        cudaError_t e = allow_tab_smem(reinterpret_cast<const void*>(k_stage2<NS>));
        if (e != cudaSuccess) return e;
        return launch_pdl(k_stage2<NS>, dim3(grid), dim3(kStageThreads), sm, s, g, ap, X, ldX, c0,
                          c1, vec);
    });
}

}  // namespace osp
