// Whole OSP iteration in ONE launch of ONE CTA for launch-bound layouts (the
// small MLP of BASELINE config #1: L <= 32 layers, a few thousand parameters).
// The big-layout step is three launches (stage 1 over every SM, the resolve,
// the stage-2 broadcast); for a 420-parameter model those launches, their
// table loads and the resolve's ~15 block-wide phases are the whole cost, so
// here every phase of the iteration runs in one 512-thread CTA and the
// resolve is done by a single warp with shuffles (one layer per lane):
//
//   stage 1   (OspServer::try_close_barrier + finish_layer, protocol.cpp:292-307,
//             361-382; OspWorker::apply_pull -> lgp_partial, protocol.cpp:69-97):
//             per element agg = float(sum_w w_k*(double)x_k / W) in the fixed worker
//             order; RS layers: G' = G + agg, every worker row = G'; ICS layers:
//             every worker row = G + x_w (the LGP local estimate) and the carry
//             C = G + agg.
//   stage 2   (on_push_ics_chunk / lgp_correct, protocol.cpp:99-116, 326-353),
//             after a block barrier: ICS layers G = C, every worker row = C
//             (base + agg, base == G_old).
//   resolve   (check_resolution, protocol.cpp:384-439): PGP per layer
//             (importance.cpp:11-28) as tile partials summed in a fixed tree,
//             certified against the reference's sequential sum (resolve.cu's
//             interval rule; touching intervals are recomputed sequentially),
//             rank (importance.cpp:30-40), prefix rule (importance.cpp:42-59),
//             chunk map (split_for_sync, protocol.cpp:145-164), and every device
//             list / counter / GIB byte the regular kernels keep, so the group
//             can continue on either path.
//
// Latency is the cost here, not bytes: every warp maps its own tiles from the
// layer table held in registers and keeps kBatch tiles' loads in flight; block
// barriers after stage 1, stage 2, the layer sums and the certificate.
// Results are bit-identical to stage1 + stage2_resolve (tests/test_gpu_parity.py).

#include "common.cuh"

namespace osp {
namespace {

constexpr int kSmallThreads = 512;
constexpr int kSmallWarps = kSmallThreads / 32;
constexpr int kSmallTile = 32;  // PGP tile: one term per lane, then 5 shuffles
constexpr double kU = 1.1102230246251565404e-16;  // 2^-53

struct SmallSmem {
    uint64_t off[kSmallMaxLayers + 1];
    uint64_t cnt[kSmallMaxLayers];
    int tb[kSmallMaxLayers + 1];       // the group's tile geometry (lists for the big kernels)
    int ptb[kSmallMaxLayers + 1];      // PGP tiles of this kernel per layer (prefix)
    int flag[kSmallMaxLayers];         // current GIB
    double part[kSmallMaxTiles];       // PGP tile partials
    double exact[kSmallMaxLayers];     // exact sequential sums of marked layers
    double lsum[kSmallMaxLayers];      // per-layer tree sums of the tile partials
    uint64_t budget, resolved;
    int n_marked;
};

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T u = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += u;
    }
    return v;
}

// rank of lane l's (key, id) among lanes 0..L-1 (stable: ties by id); every
// lane of the warp must call it
__device__ __forceinline__ int warp_rank(double key, int lane, int L) {
    int r = 0;
    for (int j = 0; j < L; ++j) {
        const double kj = __shfl_sync(0xffffffffu, key, j);
        r += (kj < key) || (kj == key && j < lane);
    }
    return r;
}

template <int NS>
constexpr int kRowsOf() { return NS > 0 ? NS : 1; }

// Stage 1 of one element: fixed-order aggregate, G' = G + agg; a barrier layer
// ends there (G and every worker row = G'), a deferred one gets the local
// estimates and the carry. Returns the PGP term. xs: the NS deltas (NS > 0) or
// read here (NS == 0).
template <int NS>
__device__ __forceinline__ double small_elem(const GroupView& g, const AggParams& ap,
                                             const float* __restrict__ X, uint64_t ldX,
                                             uint64_t f, float go, const float* xs, bool ics,
                                             float& gn_out) {
    const int n = NS > 0 ? NS : ap.n;
    double sum = 0.0;
#pragma unroll
    for (int w = 0; w < (NS > 0 ? NS : 1); ++w) {
        if (NS > 0) {
            float x = xs[w];
            if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
            sum = agg_acc(sum, ap.w[w], x);
        }
    }
    if (NS == 0) {
        for (int w = 0; w < n; ++w) {
            float x = X[static_cast<uint64_t>(w) * ldX + f];
            if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
            sum = agg_acc(sum, ap.w[w], x);
        }
    }
    const float a = agg_finish(ap, sum);
    const float gn = __fadd_rn(go, a);
    gn_out = gn;
    if (ics) {  // LGP local estimate now, the carry for stage 2
        for (int w = 0; w < n; ++w) {
            float x = NS > 0 ? xs[w < kRowsOf<NS>() ? w : 0] : X[static_cast<uint64_t>(w) * ldX + f];
            if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
            g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x);
        }
        g.C[f] = gn;
    } else {
        g.G[f] = gn;
        for (int w = 0; w < n; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
    }
    return pgp_term(a, gn);
}

template <int NS>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_step_small(GroupView g, AggParams ap, const float* __restrict__ X, uint64_t ldX) {
    __shared__ SmallSmem s;
    pdl_wait();
    pdl_trigger();
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int L = g.L;
    // every warp: the layer table in registers (lane = layer) and this kernel's
    // PGP tile prefix by a warp scan, so each warp maps its own tiles and issues
    // its loads at once; warp 0 also stages the tables and the resolve's scalars
    // in shared memory (read after the stage-1 barrier)
    uint64_t off = 0, cnt = 0;
    int fl = 0;
    if (lane < L) {
        off = g.offsets[lane];
        cnt = g.counts[lane];
        fl = g.flags[lane];
    }
    const int nt = lane < L ? static_cast<int>((cnt + kSmallTile - 1) / kSmallTile) : 0;
    const int incl = warp_incl_scan<int>(nt, lane);
    const int n_ptiles = __shfl_sync(0xffffffffu, incl, L - 1);
    if (warp == 0) {
        int tb = 0;
        if (lane < L) tb = g.tile_base[lane];
        const int tb_end = g.tile_base[L];  // lane L does not exist when L == 32
        const uint64_t budget = g.meta64[META64_BUDGET], resolved = g.meta64[META64_RESOLVED];
        const uint64_t end = warp_incl_scan<unsigned long long>(cnt, lane);
        if (lane < L) {
            s.off[lane] = off;
            s.cnt[lane] = cnt;
            s.flag[lane] = fl;
            s.ptb[lane] = incl - nt;
            s.tb[lane] = tb;
        }
        if (lane == L - 1) {
            s.ptb[L] = incl;
            s.off[L] = end;
            s.tb[L] = tb_end;
        }
        if (lane == 0) {
            s.budget = budget;
            s.resolved = resolved;
            s.n_marked = 0;
        }
    }
    OSP_DCHECK(L >= 1 && L <= kSmallMaxLayers && n_ptiles <= kSmallMaxTiles,
               "small step: layout above the single-launch limits");
    // tile t -> (first element of the lane's element, layer end, deferred?)
    auto locate = [&](int t, uint64_t& f, uint64_t& end, bool& ics) {
        const int l = __popc(__ballot_sync(0xffffffffu, lane < L && incl <= t));
        const uint64_t lo = __shfl_sync(0xffffffffu, off, l);
        const uint64_t ln = __shfl_sync(0xffffffffu, cnt, l);
        const int first = __shfl_sync(0xffffffffu, incl - nt, l);
        ics = __shfl_sync(0xffffffffu, fl, l) != 0;
        f = lo + static_cast<uint64_t>(t - first) * kSmallTile + lane;
        end = lo + ln;
    };

    // ---- stage 1: one warp per 32-element PGP tile, kBatch tiles in flight
    constexpr int kBatch = 4;
    constexpr int kRows = NS > 0 ? NS : 1;
    const float* xrow[kRows];  // row bases, computed once
#pragma unroll
    for (int w = 0; w < kRows; ++w) xrow[w] = X + static_cast<uint64_t>(w) * ldX;
    float gkeep[kBatch];  // this warp's first batch of G' values, kept for stage 2
#pragma unroll
    for (int j = 0; j < kBatch; ++j) gkeep[j] = 0.f;
    for (int t0 = warp; t0 < n_ptiles; t0 += kSmallWarps * kBatch) {
        float go[kBatch], xs[kBatch][kRows];
        uint64_t fe[kBatch];
        bool ok[kBatch], ics[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const int t = t0 + j * kSmallWarps;
            ok[j] = false;
            fe[j] = 0;
            ics[j] = false;
            if (t < n_ptiles) {  // warp-uniform
                uint64_t f, e;
                bool dfr;
                locate(t, f, e, dfr);
                ok[j] = f < e;
                fe[j] = f;
                ics[j] = dfr;
            }
            if (ok[j]) {
                go[j] = g.G[fe[j]];
#pragma unroll
                for (int w = 0; w < kRows; ++w)
                    if (NS > 0) xs[j][w] = xrow[w][fe[j]];
            }
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const int t = t0 + j * kSmallWarps;
            if (t >= n_ptiles) break;  // warp-uniform
            float gn = 0.f;
            double acc = ok[j] ? small_elem<NS>(g, ap, X, ldX, fe[j], go[j], xs[j], ics[j], gn) : 0.0;
            if (t0 == warp) gkeep[j] = gn;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
            if (lane == 0) s.part[t] = acc;
        }
    }
    __syncthreads();  // stage 1 complete: local estimates and the carry written

    // ---- stage 2: the carry broadcast on the deferred layers, in stage 1's
    // element mapping (the first batch's values are still in registers, later
    // batches read the carry back, kBatch loads in flight)
    for (int t0 = warp; t0 < n_ptiles; t0 += kSmallWarps * kBatch) {
        float cv[kBatch];
        uint64_t fe[kBatch];
        bool on[kBatch];
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            const int t = t0 + j * kSmallWarps;
            on[j] = false;
            fe[j] = 0;
            if (t < n_ptiles) {  // warp-uniform
                uint64_t f, e;
                bool dfr;
                locate(t, f, e, dfr);
                on[j] = dfr && f < e;
                fe[j] = f;
            }
            cv[j] = t0 == warp ? gkeep[j] : (on[j] ? g.C[fe[j]] : 0.f);
        }
#pragma unroll
        for (int j = 0; j < kBatch; ++j) {
            if (!on[j]) continue;
            g.G[fe[j]] = cv[j];
            for (int w = 0; w < (NS > 0 ? NS : ap.n); ++w)
                g.P[static_cast<uint64_t>(w) * g.ldP + fe[j]] = cv[j];
        }
    }
    __syncthreads();  // G final (the exact fallback reads it), tile partials in shared memory
    // per-layer sums of the tile partials, warp l for layer l: lane-strided in
    // order, then the fixed shuffle tree (depth <= ceil(nt / 32) + 5)
    for (int l = warp; l < L; l += kSmallWarps) {
        double acc = 0.0;
        for (int t = s.ptb[l] + lane; t < s.ptb[l + 1]; t += 32) acc = __dadd_rn(acc, s.part[t]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        if (lane == 0) s.lsum[l] = acc;
    }
    __syncthreads();

    // ---- resolve (warp 0; lane = layer for the per-layer values)
    double key = __longlong_as_double(0x7ff0000000000000ll);
    bool marked = false;
    if (warp == 0) {
        double rad = 0.0;
        if (lane < L) key = s.lsum[lane];
        if (lane < L) {
            const double nt = static_cast<double>(s.ptb[lane + 1] - s.ptb[lane]);
            // depth: 5 (tile tree) + ceil(nt / 32) + 5 (layer tree) + slack
            const double D = 5.0 + floor((nt + 31.0) / 32.0) + 5.0 + 2.0;
            rad = key * (kU * (1.01 * (static_cast<double>(s.cnt[lane]) - 1.0 + D) + 8.0));
            g.scores[lane] = key;
            g.lscore[lane] = key;
        }
        for (int j = 0; j < L; ++j) {
            const double kj = __shfl_sync(0xffffffffu, key, j);
            const double rj = __shfl_sync(0xffffffffu, rad, j);
            if (lane < L && j != lane && key != 0.0 && kj + rj >= key - rad && kj - rj <= key + rad)
                marked = true;
        }
        if (lane < L) g.marked[lane] = marked ? 1 : 0;
        const unsigned mm = __ballot_sync(0xffffffffu, marked);
        if (lane == 0) s.n_marked = __popc(mm);
    }
    // warp 0 decides whether the exact fallback (every warp) runs
    __syncthreads();
    const int n_marked = s.n_marked;
    if (n_marked > 0) {
        // exact sequential PGP of the marked layers (importance.cpp:20-25 order),
        // one warp each, against the final G, with agg recomputed as above
        int slot = 0;
        for (int l = 0; l < L; ++l) {
            if (!g.marked[l]) continue;
            if (slot++ % kSmallWarps != warp) continue;
            const uint64_t b0 = s.off[l], e0 = b0 + s.cnt[l];
            double sum = 0.0;
            for (uint64_t b = b0; b < e0; b += 32) {
                const uint64_t f = b + lane;
                double t = 0.0;
                if (f < e0) {
                    double a = 0.0;
                    for (int w = 0; w < ap.n; ++w) {
                        float x = X[static_cast<uint64_t>(w) * ldX + f];
                        if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                        a = agg_acc(a, ap.w[w], x);
                    }
                    t = pgp_term(agg_finish(ap, a), g.G[f]);
                }
                const int valid = static_cast<int>((e0 - b) < 32 ? (e0 - b) : 32);
                for (int i = 0; i < valid; ++i) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, t, i));
            }
            if (lane == 0) {
                g.exact[l] = sum;
                s.exact[l] = sum;
            }
        }
        __syncthreads();
        if (warp == 0 && marked) key = s.exact[lane];
        if (tid == 0) {
            g.meta64[META64_FB_LAYERS] += static_cast<uint64_t>(n_marked);
            g.meta64[META64_FB_RESOLVES] += 1;
        }
    }
    if (warp != 0) return;

    // rank, prefix rule, chunk map, lists (lane = rank position r or layer id)
    const int rk = warp_rank(key, lane, L);
    const int my_rank = lane < L ? rk : 32;
    int sorted = 0;  // sorted[r]: the lane whose rank is r
    for (int j = 0; j < L; ++j) {
        const int rj = __shfl_sync(0xffffffffu, my_rank, j);
        if (rj == lane) sorted = j;
    }
    const uint64_t bpe = g.bpe;
    const uint64_t bytes_r = lane < L ? s.cnt[sorted] * bpe : 0ull;
    const uint64_t pre = warp_incl_scan<unsigned long long>(bytes_r, lane);
    const uint64_t budget = s.budget;
    const unsigned fit = __ballot_sync(0xffffffffu, lane < L && pre <= budget);
    const int k = __popc(fit);  // pre is nondecreasing: the fitting ranks are a prefix
    const uint64_t total = __shfl_sync(0xffffffffu, pre, k > 0 ? k - 1 : 0);
    const uint64_t tot = k > 0 ? total : 0ull;
    const uint64_t nc = static_cast<uint64_t>(g.n_chunks);
    const bool in_ics = lane < k;
    uint64_t idx = 0;
    if (in_ics) {
        const uint64_t cum = pre - bytes_r;
        idx = tot == 0 ? 0 : (cum * nc) / tot;
        if (idx > nc - 1) idx = nc - 1;
    }
    const uint64_t prev_idx = __shfl_up_sync(0xffffffffu, idx, 1);
    const int is_new = in_ics && (lane == 0 || idx != prev_idx) ? 1 : 0;
    const int chunk_no = warp_incl_scan<int>(is_new, lane);  // 1-based in the compacted map
    const int n_used_all = __shfl_sync(0xffffffffu, chunk_no, k > 0 ? k - 1 : 0);
    const int n_used = k > 0 ? n_used_all : 0;
    const int ics_tiles = in_ics ? s.tb[sorted + 1] - s.tb[sorted] : 0;
    const int ics_tp = warp_incl_scan<int>(ics_tiles, lane);
    const int deferred = lane < L && my_rank < k ? 1 : 0;
    const int rs = lane < L && !deferred ? 1 : 0;
    const int rs_pos = warp_incl_scan<int>(rs, lane);
    const int rs_tiles = rs ? s.tb[lane + 1] - s.tb[lane] : 0;
    const int rs_tp = warp_incl_scan<int>(rs_tiles, lane);
    const uint32_t tag = static_cast<uint32_t>(s.resolved + 1);
    if (in_ics) {
        g.chunk_of[sorted] = chunk_no - 1;
        g.ics_layers[lane] = sorted;
        if (is_new) g.chunk_begin[chunk_no - 1] = lane;
        g.ics_tile_prefix[lane + 1] = ics_tp;
    }
    if (lane < L) {
        g.flags[lane] = static_cast<uint8_t>(deferred);
        if (rs) {
            g.chunk_of[lane] = -1;
            if (g.rs_layers) {
                g.rs_layers[rs_pos - 1] = lane;
                g.rs_tile_prefix[rs_pos] = rs_tp;
            }
        }
    }
    const unsigned dmask = __ballot_sync(0xffffffffu, deferred);
    uint8_t* gb = g.gib_bytes;
    const int nbm = (L + 7) / 8;
    if (lane < 4) {
        gb[lane] = (tag >> (8 * lane)) & 0xff;
        gb[4 + lane] = (static_cast<uint32_t>(L) >> (8 * lane)) & 0xff;
        gb[8 + nbm + lane] = (static_cast<uint32_t>(k) >> (8 * lane)) & 0xff;
    }
    if (lane < nbm) gb[8 + lane] = static_cast<uint8_t>((dmask >> (8 * lane)) & 0xffu);
    if (in_ics)
        for (int i = 0; i < 4; ++i)
            gb[8 + nbm + 4 + 4 * lane + i] = (static_cast<uint32_t>(sorted) >> (8 * i)) & 0xff;
    if (lane == 0) {
        g.ics_tile_prefix[0] = 0;
        if (g.rs_layers) g.rs_tile_prefix[0] = 0;
        g.chunk_begin[n_used] = k;
        g.meta[META_N_ICS] = k;
        g.meta[META_N_USED] = n_used;
        g.meta[META_N_RS] = L - k;
        g.meta64[META64_DEFERRED] = tot;
        g.meta64[META64_TAG] = tag;
        if (g.hist) g.hist[tag % kHist] = tot;
        g.meta64[META64_RESOLVED] = tag;
    }
    // the resolve epoch the regular path's overlapped stage 2 joins on; nothing
    // runs beside this kernel, so kernel completion publishes it (no fence)
    if (lane == 0) g.meta64[META64_RESOLVE_DONE] = tag;
}

}  // namespace

bool small_step_supported(int n_workers, int L, uint64_t M) {
    return n_workers >= 1 && n_workers <= OSP_MAX_WORKERS && L >= 1 && L <= kSmallMaxLayers &&
           M <= static_cast<uint64_t>(kSmallMaxTiles - kSmallMaxLayers) * kSmallTile;
}

cudaError_t launch_step_small(const GroupView& g, const AggParams& ap, const float* X,
                              uint64_t ldX, cudaStream_t s) {
    const dim3 grid(1), block(kSmallThreads);
    switch (ap.n) {
        case 1: return launch_pdl(k_step_small<1>, grid, block, 0, s, g, ap, X, ldX);
        case 2: return launch_pdl(k_step_small<2>, grid, block, 0, s, g, ap, X, ldX);
        case 3: return launch_pdl(k_step_small<3>, grid, block, 0, s, g, ap, X, ldX);
        case 4: return launch_pdl(k_step_small<4>, grid, block, 0, s, g, ap, X, ldX);
        case 5: return launch_pdl(k_step_small<5>, grid, block, 0, s, g, ap, X, ldX);
        case 6: return launch_pdl(k_step_small<6>, grid, block, 0, s, g, ap, X, ldX);
        case 7: return launch_pdl(k_step_small<7>, grid, block, 0, s, g, ap, X, ldX);
        case 8: return launch_pdl(k_step_small<8>, grid, block, 0, s, g, ap, X, ldX);
        default: return launch_pdl(k_step_small<0>, grid, block, 0, s, g, ap, X, ldX);
    }
}

}  // namespace osp
