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

// ===========================================================================
// Sharded path (one process per GPU, PS sharded one shard per GPU).
//
// push = reduce-scatter fused into k_shard_agg: the owner of a tile range reads
//   every worker's delta rows straight out of the peers' HBM over NVLink
//   (CUDA IPC mappings, 128-bit loads), aggregates in the reference's fixed
//   ascending worker order in fp64 (bit-exact, unlike an fp32 NCCL
//   reduce-scatter), and
// pull = all-gather fused into the same kernel: the fp32 aggregate is stored
//   into every rank's agg_full buffer (NVLink stores).
// Then each rank applies locally (k_shard_apply): G' = G + agg, its workers'
// rows, PGP partials — so every rank holds an identical G replica and computes
// the identical next GIB with no further exchange.
// A stage's tile sequence (RS list for stage 1, ICS chunks [c0,c1) for stage 2)
// is split into P equal tile-count ranges, one per rank.
// ===========================================================================

// The stage's (layer list, tile prefix, positions [jb, je)): RS layers
// ascending for stage 1, ICS chunks [c0, c1) in rank order for stage 2.
__device__ __forceinline__ Tab stage_tab(const GroupView& g, unsigned char* sm, int stage, int c0,
                                         int c1) {
    if (stage == 1) return load_tab(g, sm, g.rs_layers, g.rs_tile_prefix, 0, g.meta[META_N_RS]);
    const int used = g.meta[META_N_USED];
    if (c1 > used) c1 = used;
    int jb = 0, je = 0;
    if (c0 < c1) {
        jb = g.chunk_begin[c0];
        je = g.chunk_begin[c1];
    }
    return load_tab(g, sm, g.ics_layers, g.ics_tile_prefix, jb, je);
}

// Pipelined sharded step: the stage-1 (RS) tile sequence is exchanged in two
// halves so the first half's apply overlaps the second half's exchange.
// part 0 = the whole sequence [U0, U0+U), 1 = its first half, 2 = its second.
__device__ __forceinline__ void seq_part(int part, int& U0, int& U) {
    if (part == 1) {
        U = U / 2;
    } else if (part == 2) {
        U0 += U / 2;
        U -= U / 2;
    }
}

// Global index of the tile at the middle of the RS sequence (RS layers ascend
// by id, so "RS position < middle" <=> "global tile index < this"). NT when
// there is no RS tile.
__device__ int rs_mid_tile(const GroupView& g) {
    const int n_rs = g.meta[META_N_RS];
    const int U = n_rs > 0 ? g.rs_tile_prefix[n_rs] : 0;
    if (U == 0) return g.NT;
    const int mid = U / 2;
    int a = 0, b = n_rs - 1;  // last p with prefix[p] <= mid
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (g.rs_tile_prefix[m] <= mid) a = m;
        else b = m - 1;
    }
    return g.tile_base[g.rs_layers[a]] + (mid - g.rs_tile_prefix[a]);
}

// The owner's part of the push/pull for elements [s, e): read every worker's
// row (local or peer HBM over NVLink), aggregate in the fixed worker order,
// store the fp32 aggregate into every rank's agg buffer.
template <int NS>
__device__ void peer_agg_range(const AggParams& ap, const PeerTable& pt, uint64_t s, uint64_t e,
                               bool vec, int lane) {
    const int n = nworkers<NS>(ap);
    uint64_t he = e, be = e;
    if (vec) {
        he = min(e, (s + 3) & ~uint64_t(3));
        be = he + ((e - he) & ~uint64_t(3));
    }
    for (uint64_t f = s + lane; f < he; f += 32) {
        double acc = 0.0;
        for (int w = 0; w < n; ++w) {
            float x = ld_stream1(pt.xrow[w] + f);
            if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
            acc = agg_acc(acc, ap.w[w], x);
        }
        const float a = agg_finish(ap, acc);
        for (int r = 0; r < pt.world; ++r) pt.agg[r][f] = a;
    }
    if constexpr (NS > 0) {
        // two quads per lane in flight: NVLink peer loads have ~2 us latency
        for (uint64_t f0 = he + 4ull * lane; f0 < be; f0 += 256) {
            const uint64_t f1 = f0 + 128;
            const bool has1 = f1 < be;
            float4 xa[NS], xb[NS];
#pragma unroll
            for (int w = 0; w < NS; ++w) {
                xa[w] = ld_peer4(pt.xrow[w] + f0, pt.ldmode);
                if (has1) xb[w] = ld_peer4(pt.xrow[w] + f1, pt.ldmode);
            }
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (q == 1 && !has1) break;
                const float4* xs = q == 0 ? xa : xb;
                const uint64_t f = q == 0 ? f0 : f1;
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
                for (int w = 0; w < NS; ++w) {
                    const float4 v = cvt4(ap, xs[w]);
                    s0 = agg_acc(s0, ap.w[w], v.x);
                    s1 = agg_acc(s1, ap.w[w], v.y);
                    s2 = agg_acc(s2, ap.w[w], v.z);
                    s3 = agg_acc(s3, ap.w[w], v.w);
                }
                const float4 a = make_float4(agg_finish(ap, s0), agg_finish(ap, s1),
                                             agg_finish(ap, s2), agg_finish(ap, s3));
                for (int r = 0; r < pt.world; ++r)
                    *reinterpret_cast<float4*>(pt.agg[r] + f) = a;
            }
        }
    }
    for (uint64_t f = he + 4ull * lane; NS == 0 && f < be; f += 128) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        {
            for (int w = 0; w < n; ++w) {
                const float4 v = cvt4(ap, ld_stream4(pt.xrow[w] + f));
                s0 = agg_acc(s0, ap.w[w], v.x);
                s1 = agg_acc(s1, ap.w[w], v.y);
                s2 = agg_acc(s2, ap.w[w], v.z);
                s3 = agg_acc(s3, ap.w[w], v.w);
            }
        }
        const float4 a = make_float4(agg_finish(ap, s0), agg_finish(ap, s1),
                                     agg_finish(ap, s2), agg_finish(ap, s3));
        for (int r = 0; r < pt.world; ++r) *reinterpret_cast<float4*>(pt.agg[r] + f) = a;
    }
    for (uint64_t f = be + lane; f < e; f += 32) {
        double acc = 0.0;
        for (int w = 0; w < n; ++w) {
            float x = ld_stream1(pt.xrow[w] + f);
            if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
            acc = agg_acc(acc, ap.w[w], x);
        }
        const float a = agg_finish(ap, acc);
        for (int r = 0; r < pt.world; ++r) pt.agg[r][f] = a;
    }
}

// ---- in-kernel cross-GPU ordering (replaces separate barrier launches) --------
// Slot [kind][q] of rank r's flag array holds the last epoch rank q signalled
// for that kind. A kernel may wait at its start for every peer's slot to reach
// its epoch, signal at its start (every CTA; idempotent), and/or signal when
// its last CTA finishes (after every CTA's system-scope fence). Waits are
// bounded (20 s) and record pt.error instead of hanging.
__device__ __forceinline__ void xsync_signal(const PeerTable& pt, int kind, unsigned ep) {
    for (int q = 0; q < pt.world; ++q) {
        volatile unsigned* slot = pt.flags[q] + kind * kMaxRanks + pt.rank;
        *slot = ep;
    }
}

__device__ void xsync_start(const PeerTable& pt, const XSync& sy) {
    if (threadIdx.x == 0) {
        if (sy.signal_start >= 0) {
            __threadfence_system();
            xsync_signal(pt, sy.signal_start, sy.ep_start);
        }
        if (sy.wait >= 0) {
            const unsigned ep = sy.ep_wait;
            for (int q = 0; q < pt.world; ++q) {
                volatile unsigned* mine = pt.flags[pt.rank] + sy.wait * kMaxRanks + q;
                if (static_cast<int>(*mine - ep) >= 0) continue;
                uint64_t t0;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                while (static_cast<int>(*mine - ep) < 0) {
                    __nanosleep(128);
                    uint64_t t;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                    if (t - t0 > 20000000000ull) {
                        atomicExch(pt.error, 1u);
                        break;
                    }
                }
            }
            __threadfence_system();
        }
    }
    __syncthreads();
}

// Call with every thread of the block after its last memory operation.
__device__ void xsync_end(const GroupView& g, const PeerTable& pt, const XSync& sy) {
    if (sy.signal_end < 0) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        int* ticket = g.sched + SCHED_XSYNC_TICKET;
        if (atomicAdd(ticket, 1) == static_cast<int>(gridDim.x) - 1) {
            atomicExch(ticket, 0);
            __threadfence_system();
            xsync_signal(pt, sy.signal_end, sy.ep_end);
        }
    }
}

template <int NS>
__global__ void __launch_bounds__(kStageThreads) k_shard_agg(GroupView g, AggParams ap,
                                                             PeerTable pt, int stage, int c0,
                                                             int c1, int vec, XSync sy, int part) {
    extern __shared__ __align__(16) unsigned char smem_tab[];
    xsync_start(pt, sy);
    const int lane = threadIdx.x & 31;
    int* next = g.sched + SCHED_AGG_NEXT;
    const Tab tab = stage_tab(g, smem_tab, stage, c0, c1);
    int U0 = tab.n > 0 ? tab.sp[0] : 0;
    int U = tab.n > 0 ? tab.sp[tab.n] - U0 : 0;
    seq_part(part, U0, U);
    const int lo = U0 + static_cast<int>((static_cast<int64_t>(U) * pt.rank) / pt.world);
    const int hi = U0 + static_cast<int>((static_cast<int64_t>(U) * (pt.rank + 1)) / pt.world);
    int u = lo + grab(next, lane);
    while (u < hi) {
        const int un = lo + grab(next, lane);
        int l, k;
        tab_seq_tile(tab, u, l, k);
        uint64_t s, e;
        tab_range(tab, g, l, k, s, e);
        peer_agg_range<NS>(ap, pt, s, e, vec != 0, lane);
        u = un;
    }
    __threadfence_system();  // peer stores visible before the signal
    retire(next, g.sched + SCHED_AGG_DONE, lane);
    xsync_end(g, pt, sy);
}

// Apply one element range from agg_full: G' = G + a; local worker rows = G'; PGP.
__device__ void warp_tile_apply(const GroupView& g, int n_loc, uint64_t s, uint64_t e, bool vec,
                                int lane, double& acc) {
    uint64_t he = e, be = e;
    if (vec) {
        he = min(e, (s + 3) & ~uint64_t(3));
        be = he + ((e - he) & ~uint64_t(3));
    }
    for (uint64_t f = s + lane; f < he; f += 32) {
        const float a = g.agg_full[f];
        const float gn = __fadd_rn(g.G[f], a);
        g.G[f] = gn;
        for (int w = 0; w < n_loc; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
        acc = __dadd_rn(acc, pgp_term(a, gn));
    }
    for (uint64_t f = he + 4ull * lane; f < be; f += 128) {
        const float4 a = *reinterpret_cast<const float4*>(g.agg_full + f);
        const float4 go = *reinterpret_cast<const float4*>(g.G + f);
        const float4 gn = add4(go, a);
        *reinterpret_cast<float4*>(g.G + f) = gn;
        for (int w = 0; w < n_loc; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
        acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
        acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
        acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
        acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
    }
    for (uint64_t f = be + lane; f < e; f += 32) {
        const float a = g.agg_full[f];
        const float gn = __fadd_rn(g.G[f], a);
        g.G[f] = gn;
        for (int w = 0; w < n_loc; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
        acc = __dadd_rn(acc, pgp_term(a, gn));
    }
}

// stage 1 apply: RS tiles from agg_full, ICS tiles = local estimate of the
// local workers (same body as k_stage1's ICS path).
__global__ void __launch_bounds__(kStageThreads) k_shard_apply1(GroupView g, AggParams ap_loc,
                                                                PeerTable pt,
                                                                const float* __restrict__ X,
                                                                uint64_t ldX, int vec, XSync sy) {
    extern __shared__ __align__(16) unsigned char smem_tab[];
    xsync_start(pt, sy);
    const int lane = threadIdx.x & 31;
    int* next = g.sched + SCHED_S1_NEXT;
    const Tab tab = load_tab(g, smem_tab, nullptr, nullptr, 0, 0);
    int t = grab(next, lane);
    while (t < g.NT) {
        const int tn = grab(next, lane);
        const int l = tab_layer_of_tile(tab, t);
        uint64_t s, e;
        tab_range(tab, g, l, t - tab.tb[l], s, e);
        if (tab.flag[l]) {
            warp_tile_local<0>(g, ap_loc, X, ldX, s, e, vec != 0, lane);
        } else {
            double acc = 0.0;
            warp_tile_apply(g, ap_loc.n, s, e, vec != 0, lane, acc);
            finish_tile(g, t, acc, lane);
        }
        t = tn;
    }
    retire(next, g.sched + SCHED_S1_DONE, lane);
}

__global__ void __launch_bounds__(kStageThreads) k_shard_apply2(GroupView g, PeerTable pt,
                                                                int n_loc, int c0, int c1,
                                                                int vec, XSync sy) {
    extern __shared__ __align__(16) unsigned char smem_tab[];
    xsync_start(pt, sy);
    const int lane = threadIdx.x & 31;
    int* next = g.sched + SCHED_S2_NEXT;
    const Tab tab = stage_tab(g, smem_tab, 2, c0, c1);
    const int U0 = tab.n > 0 ? tab.sp[0] : 0;
    const int U1 = tab.n > 0 ? tab.sp[tab.n] : 0;
    int u = U0 + grab(next, lane);
    while (u < U1) {
        const int un = U0 + grab(next, lane);
        int l, k;
        tab_seq_tile(tab, u, l, k);
        uint64_t s, e;
        tab_range(tab, g, l, k, s, e);
        double acc = 0.0;
        warp_tile_apply(g, n_loc, s, e, vec != 0, lane, acc);
        finish_tile(g, tab.tb[l] + k, acc, lane);
        u = un;
    }
    retire(next, g.sched + SCHED_S2_DONE, lane);
}

// Stage-1 apply fused with the stage-2 push/pull. The two are independent
// (disjoint elements of agg_full and G; both only read the deltas), and one is
// HBM-bound (apply) while the other is NVLink-bound (peer aggregate), so one
// launch runs both: three warps in four start on the apply tiles, the fourth
// on this rank's stage-2 aggregate tiles (measured split), and a warp whose
// list runs dry switches to the other. The last warp out resets both work
// counters.
template <int NS>
__global__ void __launch_bounds__(kStageThreads) k_shard_fused(GroupView g, AggParams ap_all,
                                                               AggParams ap_loc, PeerTable pt,
                                                               const float* __restrict__ X,
                                                               uint64_t ldX, int c0, int c1,
                                                               int vec_apply, int vec_agg,
                                                               int apply_every, XSync sy,
                                                               FusedLists fl) {
    extern __shared__ __align__(16) unsigned char smem_tab[];
    xsync_start(pt, sy);
    const int lane = threadIdx.x & 31;
    const Tab tab = stage_tab(g, smem_tab, fl.agg_stage, c0, c1);
    int U0 = tab.n > 0 ? tab.sp[0] : 0;
    int U = tab.n > 0 ? tab.sp[tab.n] - U0 : 0;
    seq_part(fl.agg_part, U0, U);
    // apply list: mode 0 every tile; 1 RS tiles before the RS middle + every
    // deferred tile (local estimate); 2 RS tiles from the middle on
    const int t_mid = fl.apply_mode ? rs_mid_tile(g) : 0;
    const int t_first = fl.apply_mode == 2 ? t_mid : 0;
    const int lo = U0 + static_cast<int>((static_cast<int64_t>(U) * pt.rank) / pt.world);
    const int hi = U0 + static_cast<int>((static_cast<int64_t>(U) * (pt.rank + 1)) / pt.world);
    int* next_apply = g.sched + SCHED_S1_NEXT;
    int* next_agg = g.sched + SCHED_AGG_NEXT;
    auto fetch = [&](int list) -> int {
        if (list == 0) {
            const int t = t_first + grab(next_apply, lane);
            return t < g.NT ? t : -1;
        }
        const int u = lo + grab(next_agg, lane);
        return u < hi ? u : -1;
    };
    // apply_every > 0: one warp in apply_every starts on the (HBM-bound) apply
    // list, the rest on the (NVLink-bound) aggregate list; < 0: one warp in
    // -apply_every starts on the aggregate list. A warp whose list runs dry
    // switches to the other.
    const int gw = (blockIdx.x * (blockDim.x >> 5)) + (threadIdx.x >> 5);
    int list = apply_every > 0 ? (gw % apply_every == 0 ? 0 : 1) : (gw % -apply_every == 0 ? 1 : 0);
    int dry = 0;
    int cur = fetch(list);
    while (true) {
        if (cur < 0) {
            dry |= 1 << list;
            if (dry == 3) break;
            list ^= 1;
            cur = fetch(list);
            continue;
        }
        const int nxt = fetch(list);
        if (list == 0) {
            const int t = cur;
            const int l = tab_layer_of_tile(tab, t);
            uint64_t s, e;
            tab_range(tab, g, l, t - tab.tb[l], s, e);
            const bool skip = (fl.apply_mode == 1 && !tab.flag[l] && t >= t_mid) ||
                              (fl.apply_mode == 2 && tab.flag[l]);
            if (skip) {
            } else if (tab.flag[l]) {
                warp_tile_local<0>(g, ap_loc, X, ldX, s, e, vec_apply != 0, lane);
            } else {
                double acc = 0.0;
                warp_tile_apply(g, ap_loc.n, s, e, vec_apply != 0, lane, acc);
                finish_tile(g, t, acc, lane);
            }
        } else {
            int l, k;
            tab_seq_tile(tab, cur, l, k);
            uint64_t s, e;
            tab_range(tab, g, l, k, s, e);
            peer_agg_range<NS>(ap_all, pt, s, e, vec_agg != 0, lane);
        }
        cur = nxt;
    }
    __threadfence_system();
    if (lane == 0) {
        const int total = static_cast<int>(gridDim.x * (blockDim.x >> 5));
        if (atomicAdd(g.sched + SCHED_S1_DONE, 1) == total - 1) {
            atomicExch(next_apply, 0);
            atomicExch(next_agg, 0);
            atomicExch(g.sched + SCHED_S1_DONE, 0);
        }
    }
    xsync_end(g, pt, sy);
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

cudaError_t launch_shard_agg(const GroupView& g, const AggParams& ap, const PeerTable& pt,
                             int stage, int c0, int c1, int grid, const XSync& sy, cudaStream_t s,
                             int part) {
    bool vec = (g.ldP % 4 == 0);
    for (int w = 0; w < ap.n; ++w) vec = vec && (reinterpret_cast<uintptr_t>(pt.xrow[w]) % 16 == 0);
    for (int r = 0; r < pt.world; ++r) vec = vec && (reinterpret_cast<uintptr_t>(pt.agg[r]) % 16 == 0);
    if (grid < 1) return cudaSuccess;
    const size_t sm = tab_smem_bytes(g.L);
    return dispatch_n(ap.n, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        cudaError_t e = allow_tab_smem(reinterpret_cast<const void*>(k_shard_agg<NS>));
        if (e != cudaSuccess) return e;
        k_shard_agg<NS><<<grid, kStageThreads, sm, s>>>(g, ap, pt, stage, c0, c1, vec ? 1 : 0, sy,
                                                        part);
        return cudaGetLastError();
    });
}

cudaError_t launch_shard_apply(const GroupView& g, const AggParams& ap_loc, const PeerTable& pt,
                               const float* Xloc, uint64_t ldX, int stage, int c0, int c1, int grid,
                               const XSync& sy, cudaStream_t s) {
    const bool vec = vec_ok(g, Xloc, ldX) && (reinterpret_cast<uintptr_t>(g.agg_full) % 16 == 0);
    if (grid < 1) return cudaSuccess;
    const size_t sm = tab_smem_bytes(g.L);
    cudaError_t e;
    if (stage == 1) {
        if ((e = allow_tab_smem(reinterpret_cast<const void*>(k_shard_apply1))) != cudaSuccess) return e;
        k_shard_apply1<<<grid, kStageThreads, sm, s>>>(g, ap_loc, pt, Xloc, ldX, vec ? 1 : 0, sy);
    } else {
        if ((e = allow_tab_smem(reinterpret_cast<const void*>(k_shard_apply2))) != cudaSuccess) return e;
        k_shard_apply2<<<grid, kStageThreads, sm, s>>>(g, pt, ap_loc.n, c0, c1, vec ? 1 : 0, sy);
    }
    return cudaGetLastError();
}

cudaError_t launch_shard_fused(const GroupView& g, const AggParams& ap_all, const AggParams& ap_loc,
                               const PeerTable& pt, const float* Xloc, uint64_t ldX, int c0, int c1,
                               int grid, const XSync& sy, cudaStream_t s, FusedLists fl) {
    const bool vec_apply =
        vec_ok(g, Xloc, ldX) && (reinterpret_cast<uintptr_t>(g.agg_full) % 16 == 0);
    bool vec_agg = true;
    for (int w = 0; w < ap_all.n; ++w)
        vec_agg = vec_agg && (reinterpret_cast<uintptr_t>(pt.xrow[w]) % 16 == 0);
    for (int r = 0; r < pt.world; ++r)
        vec_agg = vec_agg && (reinterpret_cast<uintptr_t>(pt.agg[r]) % 16 == 0);
    if (grid < 1) return cudaSuccess;
    const size_t sm = tab_smem_bytes(g.L);
    return dispatch_n(ap_all.n, [&](auto nc) -> cudaError_t {
        constexpr int NS = decltype(nc)::value;
        cudaError_t e = allow_tab_smem(reinterpret_cast<const void*>(k_shard_fused<NS>));
        if (e != cudaSuccess) return e;
        // measured (tools/fused_split.sh, ResNet-50): one warp in 4 starting on
        // the aggregate: 0.608 -> 0.575 ms (P=2), 0.577 -> 0.514 ms (P=4)
        static const int every = [] {
            const char* v = std::getenv("OSP_FUSED_APPLY_EVERY");
            const int e = v && *v ? std::atoi(v) : -4;
            return e != 0 ? e : -4;
        }();
        k_shard_fused<NS><<<grid, kStageThreads, sm, s>>>(g, ap_all, ap_loc, pt, Xloc, ldX, c0, c1,
                                                          vec_apply ? 1 : 0, vec_agg ? 1 : 0, every, sy,
                                                          fl);
        return cudaGetLastError();
    });
}


}  // namespace osp
