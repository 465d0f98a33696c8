// TMA-staged variant of the group stage kernels (same math and results as
// stage.cu; selected with OSP_GROUP_TMA).
//
// One CTA = CW = T/128 consumer warps + 1 producer warp, kStages-deep ring in
// shared memory (each stage: the tile's N delta rows and its G slice).
// Producer (one elected lane): grabs the next tile (dynamic counter), resolves
// it through the per-block layer tables, arms full[s] with the byte count and
// issues N+1 1-D bulk copies (cp.async.bulk global->shared, SASS UBLKCP) of the
// tile's delta rows and G slice. Consumers: wait full[s], read their quad of
// every row from shared memory, aggregate in fp64 in the fixed worker order,
// write G and the N worker rows with 128-bit streaming stores, leave their warp
// PGP partial in the stage slot and arrive on empty[s]. The producer, when it
// reclaims stage s, sums the CW warp partials in order and publishes the tile
// partial (depth: 4 terms per thread + 5 shuffles + CW warps, within the T/32+13
// bound resolve.cu assumes). Tiles whose layer offset or size is not 16-byte
// granular are streamed by the consumers straight from global memory.
// Every mbarrier wait is bounded (20 s) and traps instead of hanging.

#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "common.cuh"
#include "tma.cuh"

namespace osp {
// Opt the kernel into its shared-memory size and query its occupancy once per
// (context, kernel, smem bytes): both are host API calls the launch-bound small
// layouts would otherwise pay on every launch. Keyed on the context, not the
// device: a recreated context starts without the opt-in.
cudaError_t tma_blocks_per_sm(const void* kern, int threads, size_t sm, int* per_sm) {
    static std::mutex mu;
    static std::map<std::tuple<unsigned long long, const void*, size_t>, int> cache;
    static std::map<std::pair<unsigned long long, const void*>, size_t> opted;  // attribute = max asked
    cudaError_t e = cudaSuccess;
    const unsigned long long dev = current_ctx_id();
    const auto key = std::make_tuple(dev, kern, sm);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *per_sm = it->second;
        return cudaSuccess;
    }
    // never lower the opt-in: a smaller layout must not break a cached larger one
    size_t& cur = opted[std::make_pair(dev, kern)];
    if (sm > cur) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sm));
        if (e != cudaSuccess) return e;
        cur = sm;
    }
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, threads, sm);
    if (e != cudaSuccess) return e;
    if (*per_sm < 1) return cudaErrorInvalidConfiguration;
    cache.emplace(key, *per_sm);
    return cudaSuccess;
}

namespace {

// Shapes: CW consumer warps (each thread T/(CW*128) quads per tile) and a KS-deep
// ring. Default min(T/128, 8) warps and 2 stages; OSP_TMA_CW /
// OSP_TMA_STAGES override for experiments.

// Per-stage descriptor written by the producer, read by the consumers.
struct StageMeta {
    uint64_t s, e;  // element range
    int t;          // global tile index (partials slot), -1 = stop
    int kind;       // 0 = aggregate (RS / stage 2), 1 = local estimate (stage-1 ICS)
    int staged;     // 1 = data in shared memory, 0 = consumers read global memory
    int pad;
};

struct TileTab {  // per-block layer tables (as stage.cu's Tab)
    const uint64_t* off;
    const uint64_t* cnt;
    const int* tb;
    const uint8_t* flag;
    const int* sl;
    const int* sp;
    int n;
    int L;
};

__device__ int tab_layer(const TileTab& tab, int t) {
    int a = 0, b = tab.L - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (tab.tb[m] <= t) a = m;
        else b = m - 1;
    }
    return a;
}

__device__ void tab_seq(const TileTab& tab, int u, int& l, int& k) {
    int a = 0, b = tab.n - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (tab.sp[m] <= u) a = m;
        else b = m - 1;
    }
    l = tab.sl[a];
    k = u - tab.sp[a];
}

// ---- consumer bodies ----------------------------------------------------------

// staged form: v read from shared memory, v' streamed out
__device__ __forceinline__ float4 momentum4s(const GroupView& g, int w, uint64_t f, float4 v,
                                             float4 x) {
    const float4 vn = make_float4(__fadd_rn(__fmul_rn(g.mu, v.x), x.x), __fadd_rn(__fmul_rn(g.mu, v.y), x.y),
                                  __fadd_rn(__fmul_rn(g.mu, v.z), x.z), __fadd_rn(__fmul_rn(g.mu, v.w), x.w));
    st_stream4(g.V + static_cast<uint64_t>(w) * g.ldP + f, vn);
    return vn;
}

__device__ __forceinline__ float momentum1(const GroupView& g, int w, uint64_t f, float x) {
    float* vp = g.V + static_cast<uint64_t>(w) * g.ldP + f;
    const float vn = __fadd_rn(__fmul_rn(g.mu, *vp), x);
    *vp = vn;
    return vn;
}

template <int NS>
__device__ __forceinline__ void consume_agg_quad(const GroupView& g, const AggParams& ap,
                                                 const float4* xs, float4 go, uint64_t f,
                                                 double& acc) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int w = 0; w < NS; ++w) {
        float4 v = xs[w];
        if (ap.sgd) {
            v.x = sgd_conv(ap.neg_lr, v.x);
            v.y = sgd_conv(ap.neg_lr, v.y);
            v.z = sgd_conv(ap.neg_lr, v.z);
            v.w = sgd_conv(ap.neg_lr, v.w);
        }
        s0 = agg_acc(s0, ap.w[w], v.x);
        s1 = agg_acc(s1, ap.w[w], v.y);
        s2 = agg_acc(s2, ap.w[w], v.z);
        s3 = agg_acc(s3, ap.w[w], v.w);
    }
    float4 a;
    a.x = agg_finish(ap, s0);
    a.y = agg_finish(ap, s1);
    a.z = agg_finish(ap, s2);
    a.w = agg_finish(ap, s3);
    const float4 gn = make_float4(__fadd_rn(go.x, a.x), __fadd_rn(go.y, a.y), __fadd_rn(go.z, a.z),
                                  __fadd_rn(go.w, a.w));
    *reinterpret_cast<float4*>(g.G + f) = gn;
#pragma unroll
    for (int w = 0; w < NS; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
    acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
    acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
    acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
    acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
}

template <int NS>
__device__ __forceinline__ void consume_local_quad(const GroupView& g, const AggParams& ap,
                                                   const float4* xs, float4 go, uint64_t f) {
#pragma unroll
    for (int w = 0; w < NS; ++w) {
        float4 v = xs[w];
        if (ap.sgd) {
            v.x = sgd_conv(ap.neg_lr, v.x);
            v.y = sgd_conv(ap.neg_lr, v.y);
            v.z = sgd_conv(ap.neg_lr, v.z);
            v.w = sgd_conv(ap.neg_lr, v.w);
        }
        st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f,
                   make_float4(__fadd_rn(go.x, v.x), __fadd_rn(go.y, v.y), __fadd_rn(go.z, v.z),
                               __fadd_rn(go.w, v.w)));
    }
}

// Stage-1 ICS quad with the carry: the local estimates (as consume_local_quad)
// and, from the same shared-memory rows, the aggregate the stage-2 kernel will
// apply: C = G_old + agg (G itself keeps G_old until stage 2), PGP term now.
template <int NS>
__device__ __forceinline__ void consume_split_quad(const GroupView& g, const AggParams& ap,
                                                   const float4* xs, float4 go, uint64_t f,
                                                   double& acc) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
    for (int w = 0; w < NS; ++w) {
        float4 v = xs[w];
        if (ap.sgd) {
            v.x = sgd_conv(ap.neg_lr, v.x);
            v.y = sgd_conv(ap.neg_lr, v.y);
            v.z = sgd_conv(ap.neg_lr, v.z);
            v.w = sgd_conv(ap.neg_lr, v.w);
        }
        st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f,
                   make_float4(__fadd_rn(go.x, v.x), __fadd_rn(go.y, v.y), __fadd_rn(go.z, v.z),
                               __fadd_rn(go.w, v.w)));
        s0 = agg_acc(s0, ap.w[w], v.x);
        s1 = agg_acc(s1, ap.w[w], v.y);
        s2 = agg_acc(s2, ap.w[w], v.z);
        s3 = agg_acc(s3, ap.w[w], v.w);
    }
    float4 a;
    a.x = agg_finish(ap, s0);
    a.y = agg_finish(ap, s1);
    a.z = agg_finish(ap, s2);
    a.w = agg_finish(ap, s3);
    const float4 gn = make_float4(__fadd_rn(go.x, a.x), __fadd_rn(go.y, a.y), __fadd_rn(go.z, a.z),
                                  __fadd_rn(go.w, a.w));
    st_stream4(g.C + f, gn);
    acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
    acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
    acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
    acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
}

// Stage-2 quad with the carry: G' = C, every worker row = C (lgp_correct:
// base + agg == G_old + agg, protocol.cpp:99-116 with base == G_old).
template <int NS>
__device__ __forceinline__ void consume_bcast_quad(const GroupView& g, float4 gn, uint64_t f) {
    *reinterpret_cast<float4*>(g.G + f) = gn;
#pragma unroll
    for (int w = 0; w < NS; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
}

// Unstaged tile (unaligned layer): per-element from global memory.
template <int NS, int CW>
__device__ void consume_direct(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                               const StageMeta& m, int ctid, double& acc, bool mom) {
    for (uint64_t f = m.s + ctid; f < m.e; f += CW * 32) {
        if (m.kind == 2) {
            const float gn = g.C[f];
            g.G[f] = gn;
            for (int w = 0; w < NS; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
        } else if (m.kind == 1) {
            const float go = g.G[f];
            double s = 0.0;
            for (int w = 0; w < NS; ++w) {
                float x = X[static_cast<uint64_t>(w) * ldX + f];
                if (mom) x = momentum1(g, w, f, x);
                if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x);
                s = agg_acc(s, ap.w[w], x);
            }
            if (g.C) {
                const float a = agg_finish(ap, s);
                const float gn = __fadd_rn(go, a);
                g.C[f] = gn;
                acc = __dadd_rn(acc, pgp_term(a, gn));
            }
        } else {
            double s = 0.0;
            for (int w = 0; w < NS; ++w) {
                float x = X[static_cast<uint64_t>(w) * ldX + f];
                if (mom) x = momentum1(g, w, f, x);
                if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                s = agg_acc(s, ap.w[w], x);
            }
            const float a = agg_finish(ap, s);
            const float gn = __fadd_rn(g.G[f], a);
            g.G[f] = gn;
            for (int w = 0; w < NS; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
            acc = __dadd_rn(acc, pgp_term(a, gn));
        }
    }
}

// STAGE 1: all tiles (RS aggregate / ICS local estimate, + the ICS carry when
// g.C is set); STAGE 2: ICS chunks [c0, c1) from the deltas; STAGE 3: ICS
// chunks [c0, c1) from the carry (one staged row per tile instead of N + 1).
template <int NS, int STAGE, int CW, int kStages, bool MOM>
__global__ void __launch_bounds__((CW + 1) * 32) k_stage_tma(GroupView g, AggParams ap,
                                                           const float* __restrict__ X,
                                                           uint64_t ldX, int c0, int c1, int ovl) {
    extern __shared__ __align__(128) unsigned char smem[];
    // ovl (stage 3 only): launched after this iteration's resolve, which waited
    // for stage 1 before letting this grid launch; run beside the resolve (no
    // wait on it) from the stage-1 snapshot of the ICS lists, join at the end
    if (!(STAGE == 3 && ovl)) pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int T = g.T;
    // slot rows: N delta rows + G (+ N velocity rows with momentum); 1 for stage 3
    constexpr int kRows = STAGE == 3 ? 1 : (MOM ? 2 * NS + 1 : NS + 1);
    const size_t stage_floats = static_cast<size_t>(kRows) * T;
    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + kStages * stage_floats);
    uint64_t* empty = full + kStages;
    StageMeta* meta = reinterpret_cast<StageMeta*>(empty + kStages);
    double* red = reinterpret_cast<double*>(meta + kStages);  // [kStages][CW]
    unsigned char* tabmem = reinterpret_cast<unsigned char*>(red + kStages * CW);

    // layer tables (+ the stage-2 sequence) in shared memory
    const int L = g.L;
    uint64_t* t_off = reinterpret_cast<uint64_t*>(tabmem);
    uint64_t* t_cnt = t_off + L;
    int* t_tb = reinterpret_cast<int*>(t_cnt + L);
    uint8_t* t_flag = reinterpret_cast<uint8_t*>(t_tb + L + 1);
    int* t_sl = reinterpret_cast<int*>(t_flag + ((L + 15) & ~15));
    int* t_sp = t_sl + L;
    // stage 1 with the carry: block 0 snapshots the ICS lists stage 3 will use
    const int n_ch = g.n_chunks;
    int* snap_cb = g.snap ? g.snap + kSnapHead : nullptr;
    int* snap_il = g.snap ? snap_cb + n_ch + 1 : nullptr;
    int* snap_tp = g.snap ? snap_il + L : nullptr;
    if (STAGE == 1 && g.snap && blockIdx.x == 0) {
        const int n_ics = g.meta[META_N_ICS];
        if (tid == 0) {
            g.snap[0] = g.meta[META_N_USED];
            g.snap[1] = static_cast<int>(g.meta64[META64_RESOLVED] + 1);
        }
        for (int i = tid; i <= n_ch; i += blockDim.x) snap_cb[i] = g.chunk_begin[i];
        for (int i = tid; i < n_ics; i += blockDim.x) snap_il[i] = g.ics_layers[i];
        for (int i = tid; i <= n_ics; i += blockDim.x) snap_tp[i] = g.ics_tile_prefix[i];
    }
    const int* l_cb = STAGE == 3 ? snap_cb : g.chunk_begin;
    const int* l_il = STAGE == 3 ? snap_il : g.ics_layers;
    const int* l_tp = STAGE == 3 ? snap_tp : g.ics_tile_prefix;
    int jb = 0, je = 0;
    if (STAGE >= 2) {
        const int used = STAGE == 3 ? g.snap[0] : g.meta[META_N_USED];
        const int cc1 = c1 > used ? used : c1;
        if (c0 < cc1) {
            jb = l_cb[c0];
            je = l_cb[cc1];
        }
    }
    for (int i = tid; i < L; i += blockDim.x) {
        t_off[i] = g.offsets[i];
        t_cnt[i] = g.counts[i];
        t_tb[i] = g.tile_base[i];
        t_flag[i] = g.flags[i];
    }
    if (tid == 0) t_tb[L] = g.tile_base[L];
    if (STAGE >= 2) {
        for (int i = tid; i < je - jb; i += blockDim.x) t_sl[i] = l_il[jb + i];
        for (int i = tid; i <= je - jb; i += blockDim.x) t_sp[i] = l_tp[jb + i];
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        mbar_init_fence();
    }
    __syncthreads();
    TileTab tab{t_off, t_cnt, t_tb, t_flag, t_sl, t_sp, je - jb, L};

    if (warp == CW) {
        // ---------------- producer ----------------
        int* next = g.sched + (STAGE == 1 ? SCHED_S1_NEXT : SCHED_S2_NEXT);
        const int lim = STAGE == 1 ? g.NT : (tab.n > 0 ? tab.sp[tab.n] : 0);
        const int base = STAGE == 1 ? 0 : (tab.n > 0 ? tab.sp[0] : 0);
        // tile partial published for RS tiles, and for ICS tiles when stage 1
        // carries their aggregate; never by the stage-3 broadcast
        const bool carry = STAGE == 1 && g.C != nullptr;
        int pending_t[kStages];
        bool pending_pub[kStages];
        for (int s = 0; s < kStages; ++s) pending_t[s] = -1;
        if (lane == 0) {
            for (int i = 0;; ++i) {
                const int s = i % kStages;
                const int use = i / kStages;
                if (use > 0) {
                    mbar_wait(&empty[s], (use - 1) & 1);
                    if (pending_t[s] >= 0 && pending_pub[s]) {
                        double tot = 0.0;
                        for (int w = 0; w < CW; ++w)
                            tot = __dadd_rn(tot, red[s * CW + w]);
                        g.partials[pending_t[s]] = tot;
                    }
                    pending_t[s] = -1;
                }
                const int u = base + atomicAdd(next, 1);
                StageMeta m{};
                if (u >= lim) {
                    m.t = -1;
                    meta[s] = m;
                    mbar_arrive(&full[s]);
                    // drain the stages still in flight
                    for (int j = 1; j < kStages; ++j) {
                        const int i2 = i + j;
                        const int s2 = i2 % kStages;
                        const int use2 = i2 / kStages;
                        if (use2 > 0 && pending_t[s2] >= 0) {
                            mbar_wait(&empty[s2], (use2 - 1) & 1);
                            if (pending_pub[s2]) {
                                double tot = 0.0;
                                for (int w = 0; w < CW; ++w)
                                    tot = __dadd_rn(tot, red[s2 * CW + w]);
                                g.partials[pending_t[s2]] = tot;
                            }
                            pending_t[s2] = -1;
                        }
                    }
                    break;
                }
                int l, k;
                if (STAGE == 1) {
                    l = tab_layer(tab, u);
                    k = u - tab.tb[l];
                    m.kind = tab.flag[l] ? 1 : 0;
                    m.t = u;
                } else {
                    tab_seq(tab, u, l, k);
                    m.kind = STAGE == 3 ? 2 : 0;
                    m.t = tab.tb[l] + k;
                }
                const uint64_t lo = tab.off[l];
                m.s = lo + static_cast<uint64_t>(k) * T;
                m.e = min(m.s + static_cast<uint64_t>(T), lo + tab.cnt[l]);
                const uint64_t n = m.e - m.s;
                OSP_DCHECK(l >= 0 && l < tab.L, "stage tile layer out of range");
                OSP_DCHECK(m.t >= 0 && m.t < g.NT, "stage tile id out of range");
                OSP_DCHECK(m.s < m.e && m.e <= tab.off[tab.L - 1] + tab.cnt[tab.L - 1],
                           "stage tile range outside the partition");
                OSP_DCHECK(n <= static_cast<uint64_t>(T), "stage tile longer than the ring slot");
                m.staged = (m.s % 4 == 0) && (n % 4 == 0) &&
                           (STAGE == 3 || ((ldX % 4 == 0) &&
                                           (reinterpret_cast<uintptr_t>(X) % 16 == 0)));
                meta[s] = m;
                pending_t[s] = m.t;
                pending_pub[s] = m.kind == 0 || (m.kind == 1 && carry);
                if (m.staged) {
                    const unsigned bytes = static_cast<unsigned>(n * 4);
                    mbar_arrive_tx(&full[s], bytes * kRows);
                    float* dst = ring + s * stage_floats;
                    if (STAGE == 3) {
                        bulk_g2s(dst, g.C + m.s, bytes, &full[s]);
                    } else {
                        for (int w = 0; w < NS; ++w)
                            bulk_g2s(dst + static_cast<size_t>(w) * T,
                                     X + static_cast<uint64_t>(w) * ldX + m.s, bytes, &full[s]);
                        bulk_g2s(dst + static_cast<size_t>(NS) * T, g.G + m.s, bytes, &full[s]);
                        if (MOM)
                            for (int w = 0; w < NS; ++w)
                                bulk_g2s(dst + static_cast<size_t>(NS + 1 + w) * T,
                                         g.V + static_cast<uint64_t>(w) * g.ldP + m.s, bytes,
                                         &full[s]);
                    }
                } else {
                    mbar_arrive(&full[s]);
                }
            }
            // every producer out: reset the counter for the next launch
            const int total = static_cast<int>(gridDim.x);
            int* done = g.sched + (STAGE == 1 ? SCHED_S1_DONE : SCHED_S2_DONE);
            if (atomicAdd(done, 1) == total - 1) {
                atomicExch(next, 0);
                atomicExch(done, 0);
                if (STAGE == 3 && ovl) {
                    // join: this grid (and so the next kernel in the stream) ends
                    // only once the overlapped resolve has published its lists
                    const unsigned long long want = static_cast<unsigned>(g.snap[1]);
                    volatile unsigned long long* dn =
                        reinterpret_cast<volatile unsigned long long*>(g.meta64 + META64_RESOLVE_DONE);
                    uint64_t t0;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                    // reached or passed (a repeated stage2_resolve must not hang)
                    while (static_cast<int>(static_cast<unsigned>(*dn) - static_cast<unsigned>(want)) < 0) {
                        __nanosleep(64);
                        uint64_t t;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                        if (t - t0 > 20000000000ull) __trap();
                    }
                    __threadfence();
                }
            }
        }
        return;
    }

    // ---------------- consumers ----------------
    const int ctid = tid;  // 0 .. CW*32-1
    for (int i = 0;; ++i) {
        const int s = i % kStages;
        mbar_wait(&full[s], (i / kStages) & 1);
        const StageMeta m = meta[s];
        if (m.t < 0) break;
        double acc = 0.0;
        if (m.staged) {
            const float* buf = ring + s * stage_floats;
            const int nq = static_cast<int>((m.e - m.s) >> 2);
            if (STAGE == 3) {
                for (int q = ctid; q < nq; q += CW * 32)
                    consume_bcast_quad<NS>(g, *reinterpret_cast<const float4*>(buf + 4 * q),
                                           m.s + 4ull * q);
            } else for (int q = ctid; q < nq; q += CW * 32) {
                float4 xs[NS];
#pragma unroll
                for (int w = 0; w < NS; ++w)
                    xs[w] = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(w) * T + 4 * q);
                const float4 go = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(NS) * T + 4 * q);
                const uint64_t f = m.s + 4ull * q;
                if (MOM) {  // velocities staged in the slot after G
#pragma unroll
                    for (int w = 0; w < NS; ++w) {
                        const float4 v = *reinterpret_cast<const float4*>(
                            buf + static_cast<size_t>(NS + 1 + w) * T + 4 * q);
                        xs[w] = momentum4s(g, w, f, v, xs[w]);
                    }
                }
                if (m.kind == 0) consume_agg_quad<NS>(g, ap, xs, go, f, acc);
                else if (g.C) consume_split_quad<NS>(g, ap, xs, go, f, acc);
                else consume_local_quad<NS>(g, ap, xs, go, f);
            }
        } else {
            consume_direct<NS, CW>(g, ap, X, ldX, m, ctid, acc, MOM);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        if (lane == 0) {
            red[s * CW + warp] = acc;
            mbar_arrive(&empty[s]);
        }
        __syncwarp();
    }
}

size_t tma_smem_bytes(int rows, int T, int L, int CW, int kStages) {
    const size_t ring = static_cast<size_t>(kStages) * rows * T * sizeof(float);
    const size_t bars = 2 * kStages * sizeof(uint64_t);
    const size_t metas = kStages * sizeof(StageMeta);
    const size_t red = kStages * CW * sizeof(double);
    const size_t tab = static_cast<size_t>(L) * 16 + (L + 1) * 4 + ((L + 15) & ~15) + L * 4 +
                       (L + 1) * 4 + 64;
    return ring + bars + metas + red + tab;
}

template <int STAGE, int NS, int CW, int KS>
cudaError_t launch_tma_cw(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int c0, int c1, int ovl, cudaStream_t s) {
    size_t sm = tma_smem_bytes(STAGE == 3 ? 1 : NS + 1, g.T, g.L, CW, KS);
    // momentum is a separate stage-1 instantiation (velocity rows staged in the
    // ring too): its traffic would otherwise cost the default kernel registers
    void (*kern)(GroupView, AggParams, const float*, uint64_t, int, int, int) =
        k_stage_tma<NS, STAGE, CW, KS, false>;
    if constexpr (STAGE == 1) {
        if (g.V) {
            kern = k_stage_tma<NS, STAGE, CW, KS, true>;
            sm = tma_smem_bytes(2 * NS + 1, g.T, g.L, CW, KS);
        }
    }
    int per_sm = 0;
    cudaError_t e = tma_blocks_per_sm(reinterpret_cast<const void*>(kern), (CW + 1) * 32, sm,
                                      &per_sm);
    if (e != cudaSuccess) return e;
    // grid stays one wave even when a small layout has fewer tiles: clamping it
    // to the tile count measured no faster for the 420-parameter MLP (18.4 ->
    // 20.5 us per graph-replayed step; profiles/r1_mlp_launch_notes.md)
    const int grid = sm_count() * per_sm;
    return launch_pdl(kern, dim3(grid), dim3((CW + 1) * 32), sm, s, g, ap, X, ldX, c0, c1, ovl);
}

struct TmaShape {
    int cw, ks;
};

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

TmaShape tma_shape(int T) {
    static const int cw_env = env_int("OSP_TMA_CW", 0);
    static const int ks_env = env_int("OSP_TMA_STAGES", 0);
    // measured (resnet50, N=8): 2 stages beat 3-4 (more CTAs per SM), T=1024
    TmaShape sh{T / 128 > 8 ? 8 : T / 128, 2};
    if (cw_env == 4 || cw_env == 8 || cw_env == 16) sh.cw = cw_env;
    if (ks_env >= 2 && ks_env <= 4) sh.ks = ks_env;
    if (sh.cw * 128 > T) sh.cw = T / 128;
    return sh;
}

template <int STAGE, int NS, int CW>
cudaError_t launch_tma_ks(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int c0, int c1, int ovl, int ks, cudaStream_t s) {
    switch (ks) {
        case 2: return launch_tma_cw<STAGE, NS, CW, 2>(g, ap, X, ldX, c0, c1, ovl, s);
        case 3: return launch_tma_cw<STAGE, NS, CW, 3>(g, ap, X, ldX, c0, c1, ovl, s);
        default: return launch_tma_cw<STAGE, NS, CW, 4>(g, ap, X, ldX, c0, c1, ovl, s);
    }
}

template <int STAGE, int NS>
cudaError_t launch_tma_n(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                         int c0, int c1, int ovl, cudaStream_t s) {
    const TmaShape sh = tma_shape(g.T);
    switch (sh.cw) {
        case 4: return launch_tma_ks<STAGE, NS, 4>(g, ap, X, ldX, c0, c1, ovl, sh.ks, s);
        case 8: return launch_tma_ks<STAGE, NS, 8>(g, ap, X, ldX, c0, c1, ovl, sh.ks, s);
        case 16: return launch_tma_ks<STAGE, NS, 16>(g, ap, X, ldX, c0, c1, ovl, sh.ks, s);
        default: return cudaErrorNotSupported;
    }
}

// N in {3, 5, 6, 7}: the default shape only (2-slot ring, T/128 <= 8 consumer
// warps), no sweep overrides, to bound the number of instantiations
int default_cw(int T) { return T / 128 > 8 ? 8 : T / 128; }

template <int STAGE, int NS>
cudaError_t launch_tma_n_default(const GroupView& g, const AggParams& ap, const float* X,
                                 uint64_t ldX, int c0, int c1, int ovl, cudaStream_t s) {
    switch (default_cw(g.T)) {
        case 4: return launch_tma_cw<STAGE, NS, 4, 2>(g, ap, X, ldX, c0, c1, ovl, s);
        case 8: return launch_tma_cw<STAGE, NS, 8, 2>(g, ap, X, ldX, c0, c1, ovl, s);
        default: return cudaErrorNotSupported;
    }
}

template <int STAGE>
cudaError_t launch_tma(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                       int c0, int c1, int ovl, cudaStream_t s) {
    switch (ap.n) {
        case 1: return launch_tma_n<STAGE, 1>(g, ap, X, ldX, c0, c1, ovl, s);
        case 2: return launch_tma_n<STAGE, 2>(g, ap, X, ldX, c0, c1, ovl, s);
        case 3: return launch_tma_n_default<STAGE, 3>(g, ap, X, ldX, c0, c1, ovl, s);
        case 4: return launch_tma_n<STAGE, 4>(g, ap, X, ldX, c0, c1, ovl, s);
        case 5: return launch_tma_n_default<STAGE, 5>(g, ap, X, ldX, c0, c1, ovl, s);
        case 6: return launch_tma_n_default<STAGE, 6>(g, ap, X, ldX, c0, c1, ovl, s);
        case 7: return launch_tma_n_default<STAGE, 7>(g, ap, X, ldX, c0, c1, ovl, s);
        case 8: return launch_tma_n<STAGE, 8>(g, ap, X, ldX, c0, c1, ovl, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace

namespace {
TmaShape shape_for(int n_workers, int T) {
    const bool pow2 = n_workers == 1 || n_workers == 2 || n_workers == 4 || n_workers == 8;
    return pow2 ? tma_shape(T) : TmaShape{default_cw(T), 2};
}
}  // namespace

bool tma_supported(int n_workers, int T, int L) {
    if (n_workers < 1 || n_workers > 8) return false;
    if (T < 512 || T > 4096) return false;
    const TmaShape sh = shape_for(n_workers, T);
    return tma_smem_bytes(n_workers + 1, T, L, sh.cw, sh.ks) <= 220 * 1024;
}

bool tma_momentum_supported(int n_workers, int T, int L) {
    if (!tma_supported(n_workers, T, L)) return false;
    const TmaShape sh = shape_for(n_workers, T);
    return tma_smem_bytes(2 * n_workers + 1, T, L, sh.cw, sh.ks) <= 220 * 1024;
}

cudaError_t launch_stage1_tma(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                              cudaStream_t s) {
    return launch_tma<1>(g, ap, X, ldX, 0, 0, 0, s);
}

cudaError_t launch_stage2_tma(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                              int c0, int c1, cudaStream_t s, int overlap) {
    if (g.C) return launch_tma<3>(g, ap, X, ldX, c0, c1, overlap, s);
    if (overlap) return cudaErrorInvalidValue;
    return launch_tma<2>(g, ap, X, ldX, c0, c1, 0, s);
}

}  // namespace osp
