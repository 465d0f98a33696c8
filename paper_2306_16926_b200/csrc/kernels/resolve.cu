// Resolution of an iteration on the device (OspServer::check_resolution,
// protocol.cpp:384-439): per-layer PGP (importance.cpp:11-28) -> rank
// (importance.cpp:30-40) -> prefix-rule GIB (importance.cpp:42-59) -> the
// rank-ordered ICS list, its byte-balanced chunk map (split_for_sync,
// protocol.cpp:122-166) and the tile lists the next iteration's stage-2
// kernels walk. One CTA of 1024 threads, one launch; ~60 B per layer of
// shared memory up to kSmemResolveLayers layers, a global scratch buffer above.
//
// Bit-exact ranking from a parallel sum (SURVEY.md §7 hard part 1). The
// reference sums |g*p| sequentially in double; a parallel tree rounds
// differently. Every term is exact in double and non-negative, so
//   CPU:  |c - s| <= gamma(n-1) * s        (n = layer elements)
//   GPU:  |s^ - s| <= gamma(D) * s          (D = adds on any term's path)
// and c lies in [s^ - E, s^ + E] with E = s^ * u * (1.01 * (n - 1 + D) + 8)
// (u = 2^-53; the slack absorbs gamma's second-order term and the rounding of
// the interval ends). Layers whose interval touches another layer's interval
// are "marked"; their scores are recomputed in the reference's exact
// sequential order (one warp per marked layer, inside this kernel), and the
// ranking is redone with exact keys for them. Unmarked intervals are disjoint
// from every other interval, so the resulting order equals the reference's
// stable (score, id) order. Exact zeros (s^ == 0 <=> every term is 0) are
// exact and never marked.

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace osp {
namespace {

constexpr double kU = 1.1102230246251565404e-16;  // 2^-53
constexpr int kWarps = kResolveThreads / 32;

// Depth of the stage kernels' per-tile reduction (stage.cu): per-lane
// sequential terms (<= T/32 + head/tail), then 5 shuffle levels.
__device__ __forceinline__ double tile_depth(int T) { return static_cast<double>(T / 32 + 8 + 5); }

struct Smem {
    double* key;
    double* rad;
    double* a1;
    double* a2;
    int* sorted;
    int* pos;
    int* i1;
    int* i2;
    double* wtot;  // [4 * kWarps] scan scratch (8-byte slots), always shared memory
    uint64_t* cnt; // [L] layer element counts (staged from global)
    int* tb;       // [L+1] tile_base (staged from global)
    int* flag;     // [8], always shared memory
};

// Per-layer arrays of the single-CTA phases: dynamic shared memory up to
// kSmemResolveLayers layers, above that a global scratch buffer owned by the
// group (g.rscratch) — one CTA reads it, so block barriers order it as well.
// The scan scratch and the flags stay in shared memory either way (every block
// of k_resolve's first phase uses them).
__device__ Smem carve(char* base, int L, double* wtot, int* flag) {
    Smem s;
    s.key = reinterpret_cast<double*>(base);
    s.rad = s.key + L;
    s.a1 = s.rad + L;
    s.a2 = s.a1 + L;
    s.cnt = reinterpret_cast<uint64_t*>(s.a2 + L);
    s.sorted = reinterpret_cast<int*>(s.cnt + L);
    s.pos = s.sorted + L;
    s.i1 = s.pos + L;
    s.i2 = s.i1 + L;
    s.tb = s.i2 + L;
    s.wtot = wtot;
    s.flag = flag;
    return s;
}

}  // namespace

size_t resolve_scratch_bytes(int L) {
    return static_cast<size_t>(L) * (5 * sizeof(double) + 5 * sizeof(int)) + sizeof(int) + 16;
}

namespace {

// dynamic shared memory of the single-CTA kernels (0 when the arrays are global)
size_t smem_bytes(int L) { return L <= kSmemResolveLayers ? resolve_scratch_bytes(L) : 0; }

// One coalesced load of the layer geometry into shared memory; everything the
// single-CTA phases need per layer is then a shared-memory read.
__device__ void stage_geometry(const GroupView& g, const Smem& s) {
    for (int l = threadIdx.x; l < g.L; l += blockDim.x) {
        s.cnt[l] = g.counts[l];
        s.tb[l] = g.tile_base[l];
    }
    if (threadIdx.x == 0) s.tb[g.L] = g.tile_base[g.L];
    __syncthreads();
}

// Block-wide inclusive scan of a[0..n) in shared memory (associative,
// commutative op): per-thread contiguous segment, warp shuffle scan of the
// segment totals, one warp over the warp totals. Three barriers.
template <typename T, typename Op>
__device__ void block_scan(T* a, int n, T ident, Op op, double* wtot_raw) {
    T* wtot = reinterpret_cast<T*>(wtot_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = min(n, tid * per), e = min(n, b + per);
    T run = ident;
    for (int i = b; i < e; ++i) run = op(run, a[i]);
    T incl = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = op(v, incl);
    }
    if (lane == 31) wtot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        T w = lane < kWarps ? wtot[lane] : ident;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w = op(v, w);
        }
        if (lane < kWarps) wtot[lane] = w;
    }
    __syncthreads();
    const T excl_in_warp = __shfl_up_sync(0xffffffffu, incl, 1);
    T pre = warp > 0 ? wtot[warp - 1] : ident;
    if (lane > 0) pre = op(pre, excl_in_warp);
    for (int i = b; i < e; ++i) {
        pre = op(pre, a[i]);
        a[i] = pre;
    }
    __syncthreads();
}

// K independent inclusive scans of a[j][0..n), j < K, with one op, sharing the
// three barriers of block_scan (wtot_raw needs K * kWarps 8-byte slots).
template <int K, typename T, typename Op>
__device__ void block_scan_multi(T* const* a, int n, T ident, Op op, double* wtot_raw) {
    T* wtot = reinterpret_cast<T*>(wtot_raw);  // [K][kWarps]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int b = min(n, tid * per), e = min(n, b + per);
    T incl[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        T run = ident;
        for (int i = b; i < e; ++i) run = op(run, a[j][i]);
        incl[j] = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T v = __shfl_up_sync(0xffffffffu, incl[j], o);
            if (lane >= o) incl[j] = op(v, incl[j]);
        }
        if (lane == 31) wtot[j * kWarps + warp] = incl[j];
    }
    __syncthreads();
    if (warp < K) {
        T w = lane < kWarps ? wtot[warp * kWarps + lane] : ident;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T v = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w = op(v, w);
        }
        if (lane < kWarps) wtot[warp * kWarps + lane] = w;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const T excl_in_warp = __shfl_up_sync(0xffffffffu, incl[j], 1);
        T pre = warp > 0 ? wtot[j * kWarps + warp - 1] : ident;
        if (lane > 0) pre = op(pre, excl_in_warp);
        for (int i = b; i < e; ++i) {
            pre = op(pre, a[j][i]);
            a[j][i] = pre;
        }
    }
    __syncthreads();
}

// Rank by (key, id): the reference's stable_sort by score with id tie-break
// (importance.cpp:30-40). Small L: counting rank. Larger L: bitonic sort of
// (key, id) pairs padded to a power of two with (+inf, INT_MAX); a1..a2 (2L
// doubles) and i1..i2 (2L ints) are free at every call site and hold the
// pairs. Scores are non-negative sums, so the comparison is a plain total
// order. (Measured crossover: counting 13.7 us vs bitonic 18.4 us resolve at
// L = 161; 24.0 vs 22.5 us at L = 467.)
constexpr int kCountRankMax = 320;
__device__ void rank_layers_block(const Smem& s, int L) {
    if (L <= kCountRankMax) {
        // small L: rank(l) = #{j : (key_j, j) < (key_l, l)}, G = 2^k lanes of a
        // warp share one layer's count (xor-shuffle sum inside the group)
        int G = 1;
        while (G < 32 && 2 * G * L <= static_cast<int>(blockDim.x)) G *= 2;
        const int sub = threadIdx.x % G;
        const int lanes = blockDim.x / G;
        for (int base = 0; base < L; base += lanes) {
            const int l = base + static_cast<int>(threadIdx.x) / G;
            int r = 0;
            if (l < L) {
                const double kl = s.key[l];
#pragma unroll 4
                for (int j = sub; j < L; j += G) {
                    const double kj = s.key[j];
                    r += (kj < kl) || (kj == kl && j < l);
                }
            }
            for (int o = 1; o < G; o <<= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
            if (l < L && sub == 0) s.sorted[r] = l;
        }
        __syncthreads();
        return;
    }
    int P2 = 1;
    while (P2 < L) P2 <<= 1;
    double* sk = s.a1;  // [2L] (a1 then a2)
    int* si = s.i1;     // [2L] (i1 then i2)
    for (int i = threadIdx.x; i < P2; i += blockDim.x) {
        sk[i] = i < L ? s.key[i] : __longlong_as_double(0x7ff0000000000000ll);
        si[i] = i < L ? i : 0x7fffffff;
    }
    __syncthreads();
    for (int k = 2; k <= P2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const double a = sk[i], b = sk[p];
                    const int ia = si[i], ib = si[p];
                    const bool gt = a > b || (a == b && ia > ib);
                    if (gt == ((i & k) == 0)) {
                        sk[i] = b;
                        sk[p] = a;
                        si[i] = ib;
                        si[p] = ia;
                    }
                }
            }
            __syncthreads();
        }
    }
    for (int r = threadIdx.x; r < L; r += blockDim.x) s.sorted[r] = si[r];
    __syncthreads();
}

// Given the ICS list ord[0..k) (rank order) and the inclusive byte prefix over
// it in a1 (uint64 bit patterns), write flags, ICS list, compacted chunk map,
// tile prefixes, RS list, meta and the encoded GIB. Mirrors split_for_sync's
// chunking (protocol.cpp:145-164): idx = min(n-1, cum*n/total) in u64, empty
// chunks dropped. key / rad are free here and hold the four scanned arrays.
__device__ void finalize_lists(const GroupView& g, const Smem& s, const int* ord, int k,
                               uint32_t tag) {
    const int tid = threadIdx.x, B = blockDim.x, L = g.L;
    uint64_t* pre = reinterpret_cast<uint64_t*>(s.a1);
    const uint64_t total = k > 0 ? pre[k - 1] : 0;
    const uint64_t nc = static_cast<uint64_t>(g.n_chunks);
    int* fl = s.pos;
    for (int l = tid; l < L; l += B) fl[l] = 0;
    for (int r = tid; r < k; r += B) {
        const uint64_t bytes = s.cnt[ord[r]] * static_cast<uint64_t>(g.bpe);
        const uint64_t cum = pre[r] - bytes;
        uint64_t idx = total == 0 ? 0 : (cum * nc) / total;
        if (idx > nc - 1) idx = nc - 1;
        s.i1[r] = static_cast<int>(idx);
    }
    __syncthreads();
    for (int r = tid; r < k; r += B) fl[ord[r]] = 1;
    __syncthreads();
    // scans: new-chunk flags and ICS tile counts in rank order, RS flags and RS
    // tile counts in id order
    int* sc_new = reinterpret_cast<int*>(s.key);
    int* sc_icst = sc_new + L;
    int* sc_rsf = reinterpret_cast<int*>(s.rad);
    int* sc_rst = sc_rsf + L;
    for (int i = tid; i < L; i += B) {
        const bool ics = i < k;
        sc_new[i] = ics && (i == 0 || s.i1[i] != s.i1[i - 1]) ? 1 : 0;
        sc_icst[i] = ics ? s.tb[ord[i] + 1] - s.tb[ord[i]] : 0;
        sc_rsf[i] = fl[i] ? 0 : 1;
        sc_rst[i] = fl[i] ? 0 : s.tb[i + 1] - s.tb[i];
    }
    __syncthreads();
    int* arrs[4] = {sc_new, sc_icst, sc_rsf, sc_rst};
    block_scan_multi<4, int>(arrs, L, 0, [](int a, int b) { return a + b; }, s.wtot);
    const int n_used = k > 0 ? sc_new[k - 1] : 0;
    OSP_DCHECK(k >= 0 && k <= L, "resolve: deferred count outside [0, L]");
    for (int r = tid; r < k; r += B) {
        const int l = ord[r];
        const int c = sc_new[r] - 1;
        OSP_DCHECK(l >= 0 && l < L, "resolve: ICS list id out of range");
        OSP_DCHECK(c >= 0 && c < g.n_chunks, "resolve: chunk index out of range");
        g.chunk_of[l] = c;
        g.ics_layers[r] = l;
        if (r == 0 || sc_new[r] != sc_new[r - 1]) g.chunk_begin[c] = r;
        g.ics_tile_prefix[r + 1] = sc_icst[r];
    }
    const int n_rs = L - k;
    for (int l = tid; l < L; l += B) {
        g.flags[l] = static_cast<uint8_t>(fl[l]);
        if (!fl[l]) {
            g.chunk_of[l] = -1;
            if (g.rs_layers) {
                const int p = sc_rsf[l] - 1;
                g.rs_layers[p] = l;
                g.rs_tile_prefix[p + 1] = sc_rst[l];
            }
        }
    }
    if (tid == 0) {
        g.ics_tile_prefix[0] = 0;
        if (g.rs_layers) g.rs_tile_prefix[0] = 0;
        g.chunk_begin[n_used] = k;
        g.meta[META_N_ICS] = k;
        g.meta[META_N_USED] = n_used;
        g.meta[META_N_RS] = n_rs;
        g.meta64[META64_DEFERRED] = total;
        g.meta64[META64_TAG] = tag;
        if (g.hist) g.hist[tag % kHist] = total;
        const uint32_t ul = static_cast<uint32_t>(L);
        for (int i = 0; i < 4; ++i) {
            g.gib_bytes[i] = (tag >> (8 * i)) & 0xff;
            g.gib_bytes[4 + i] = (ul >> (8 * i)) & 0xff;
        }
    }
    for (int byte = tid; byte < (L + 7) / 8; byte += B) {
        uint8_t v = 0;
        for (int b = 0; b < 8; ++b) {
            const int l = byte * 8 + b;
            if (l < L && fl[l]) v |= static_cast<uint8_t>(1u << b);
        }
        g.gib_bytes[8 + byte] = v;
    }
    // rank-order side channel after the bitmap: n u32 LE, then the deferred ids
    // least important first (osp_gib_wire_encode's layout)
    uint8_t* tail = g.gib_bytes + 8 + (L + 7) / 8;
    if (tid == 0)
        for (int i = 0; i < 4; ++i) tail[i] = (static_cast<uint32_t>(k) >> (8 * i)) & 0xff;
    for (int r = tid; r < k; r += B) {
        const uint32_t id = static_cast<uint32_t>(ord[r]);
        for (int i = 0; i < 4; ++i) tail[4 + 4 * r + i] = (id >> (8 * i)) & 0xff;
    }
}

// Exact sequential PGP of one layer (importance.cpp:20-25 order) by one warp,
// with the aggregated delta recomputed from the worker deltas exactly as the
// stage kernels computed it, against the post-update global vector.
__device__ double exact_layer_pgp(const GroupView& g, const AggParams& ap, const float* X,
                                  uint64_t ldX, int l, int lane) {
    const uint64_t off = g.offsets[l], end = off + g.counts[l];
    double sum = 0.0;
    for (uint64_t b = off; b < end; b += 32) {
        const uint64_t f = b + lane;
        double t = 0.0;
        if (f < end) {
            float agg;
            if (g.agg_full) {  // sharded path: the applied aggregate is resident
                agg = g.agg_full[f];
            } else {
                double a = 0.0;
                for (int w = 0; w < ap.n; ++w) {
                    float x = X[static_cast<uint64_t>(w) * ldX + f];
                    if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                    a = agg_acc(a, ap.w[w], x);
                }
                agg = agg_finish(ap, a);
            }
            // carry: the deferred layers' post-update values are in C (G may
            // still be being written by the overlapped stage 2)
            t = pgp_term(agg, (g.C && g.flags[l]) ? g.C[f] : g.G[f]);
        }
        const int valid = static_cast<int>((end - b) < 32 ? (end - b) : 32);
        for (int i = 0; i < valid; ++i) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, t, i));
    }
    return sum;
}

__global__ void __launch_bounds__(kResolveThreads) k_resolve(GroupView g, AggParams ap,
                                                             const float* __restrict__ X,
                                                             uint64_t ldX) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ double sh_wtot[4 * kWarps];
    __shared__ int sh_flag[8];
    pdl_wait();
    pdl_trigger();
    const int L = g.L;
    const Smem s = carve(g.rscratch ? g.rscratch : smem_raw, L, sh_wtot, sh_flag);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // 0. every block: tree sums of the tile partials per sum item (<= kSumChunk
    //    tiles of one layer; fixed order: thread-strided sequential, shuffle
    //    tree, warps in order)
    for (int it = blockIdx.x; it < g.n_sum_items; it += gridDim.x) {
        const int t0 = g.sum_items[3 * it + 1], t1 = g.sum_items[3 * it + 2];
        OSP_DCHECK(t0 >= 0 && t0 <= t1 && t1 <= g.NT, "resolve: sum item outside the tiles");
        double acc = 0.0;
        for (int t = t0 + tid; t < t1; t += blockDim.x) acc = __dadd_rn(acc, g.partials[t]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        if (lane == 0) s.wtot[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            double tot = 0.0;
            for (int w = 0; w < kWarps; ++w) tot = __dadd_rn(tot, s.wtot[w]);
            g.item_sums[it] = tot;
        }
        __syncthreads();
    }
    // the last block to finish does the single-CTA part
    if (tid == 0) {
        __threadfence();
        s.flag[2] = atomicAdd(g.sched + SCHED_RESOLVE_DONE, 1) == static_cast<int>(gridDim.x) - 1;
    }
    __syncthreads();
    if (!s.flag[2]) return;
    __threadfence();
    if (tid == 0) g.sched[SCHED_RESOLVE_DONE] = 0;

    stage_geometry(g, s);
    // 1. per-layer scores (items summed in order) and certificate radii. Depth
    //    of any term: tile tree + item tree (<= ceil(kSumChunk/threads) strided
    //    terms, 5 shuffles, kWarps warps) + the sequential item sum + slack
    for (int l = tid; l < L; l += blockDim.x) {
        const int i0 = g.layer_items[l], i1 = g.layer_items[l + 1];
        double acc = 0.0;
        for (int it = i0; it < i1; ++it) acc = __dadd_rn(acc, __ldcg(g.item_sums + it));
        g.lscore[l] = acc;
        const int nt = s.tb[l + 1] - s.tb[l];
        const int per_item = nt < kSumChunk ? nt : kSumChunk;
        const double D = tile_depth(g.T) + (per_item + kResolveThreads - 1) / kResolveThreads + 5 +
                         kWarps + (i1 - i0) + 2;
        const double n = static_cast<double>(s.cnt[l]);
        s.key[l] = acc;
        s.rad[l] = acc * (kU * (1.01 * (n - 1.0 + D) + 8.0));
        g.scores[l] = acc;
    }
    if (tid == 0) {
        s.flag[0] = 0;
        s.flag[1] = 0;
    }
    __syncthreads();
    rank_layers_block(s, L);

    // 2. certificate: any interval overlap between two layers marks both
    for (int r = tid; r < L; r += blockDim.x) {
        const int l = s.sorted[r];
        s.a1[r] = s.key[l] + s.rad[l];             // hi, prefix max
        s.a2[L - 1 - r] = -(s.key[l] - s.rad[l]);  // -lo, reversed: suffix min of lo
    }
    __syncthreads();
    {
        double* arrs[2] = {s.a1, s.a2};
        block_scan_multi<2, double>(arrs, L, -1e308, [](double a, double b) { return a > b ? a : b; },
                                    s.wtot);
    }
    int my_marks = 0;
    for (int r = tid; r < L; r += blockDim.x) {
        const int l = s.sorted[r];
        const double k = s.key[l], rd = s.rad[l];
        const double premax = r > 0 ? s.a1[r - 1] : -1.0;
        const double sufmin = r < L - 1 ? -s.a2[L - 2 - r] : 1e308;
        const bool m = (k != 0.0) && (k + rd >= sufmin || k - rd <= premax);
        g.marked[l] = m ? 1 : 0;
        s.i1[r] = m ? 1 : 0;
        my_marks += m ? 1 : 0;
    }
    if (my_marks) atomicAdd(&s.flag[0], my_marks);
    __syncthreads();
    const int n_marked = s.flag[0];
    if (n_marked > 0) {
        // 3. exact sequential scores for the marked layers, one warp each, then re-rank
        block_scan<int>(s.i1, L, 0, [](int a, int b) { return a + b; }, s.wtot);
        for (int r = tid; r < L; r += blockDim.x)
            if (g.marked[s.sorted[r]]) s.i2[s.i1[r] - 1] = s.sorted[r];
        __syncthreads();
        for (int m = warp; m < n_marked; m += kWarps) {
            const int l = s.i2[m];
            const double ex = exact_layer_pgp(g, ap, X, ldX, l, lane);
            if (lane == 0) {
                g.exact[l] = ex;
                s.key[l] = ex;
            }
        }
        if (tid == 0) {
            g.meta64[META64_FB_LAYERS] += static_cast<uint64_t>(n_marked);
            g.meta64[META64_FB_RESOLVES] += 1;
        }
        __syncthreads();
        rank_layers_block(s, L);
    }

    // 4. prefix rule: inclusive byte scan in rank order, k = #prefix <= budget
    uint64_t* pre = reinterpret_cast<uint64_t*>(s.a1);
    for (int r = tid; r < L; r += blockDim.x)
        pre[r] = s.cnt[s.sorted[r]] * static_cast<uint64_t>(g.bpe);
    __syncthreads();
    block_scan<uint64_t>(pre, L, 0ull, [](uint64_t a, uint64_t b) { return a + b; }, s.wtot);
    const uint64_t budget = g.meta64[META64_BUDGET];
    int cnt = 0;
    for (int r = tid; r < L; r += blockDim.x) cnt += pre[r] <= budget ? 1 : 0;
    if (cnt) atomicAdd(&s.flag[1], cnt);
    __syncthreads();
    const int k = s.flag[1];
    const uint32_t tag = static_cast<uint32_t>(g.meta64[META64_RESOLVED] + 1);
    __syncthreads();
    if (tid == 0) g.meta64[META64_RESOLVED] += 1;
    finalize_lists(g, s, s.sorted, k, tag);
    // publish: every list written (block barrier, then a cumulative fence)
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        atomicExch(reinterpret_cast<unsigned long long*>(g.meta64 + META64_RESOLVE_DONE),
                   static_cast<unsigned long long>(g.meta64[META64_RESOLVED]));
    }
}

// Install a host-provided GIB: g.flags already written; order (device) is the
// rank list. Deferred order = order filtered by the bitmap, then missing
// flagged ids ascending (split_for_sync, protocol.cpp:133-142).
__global__ void __launch_bounds__(kResolveThreads) k_install(GroupView g, const int* order,
                                                             int n_order, uint32_t tag) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ double sh_wtot[4 * kWarps];
    __shared__ int sh_flag[8];
    const int L = g.L;
    const Smem s = carve(g.rscratch ? g.rscratch : smem_raw, L, sh_wtot, sh_flag);
    stage_geometry(g, s);
    if (threadIdx.x == 0) {
        int k = 0;
        for (int l = 0; l < L; ++l) s.pos[l] = 0;  // seen
        for (int i = 0; i < n_order; ++i) {
            const int id = order[i];
            if (id >= 0 && id < L && g.flags[id] && !s.pos[id]) {
                s.sorted[k++] = id;
                s.pos[id] = 1;
            }
        }
        for (int l = 0; l < L; ++l)
            if (g.flags[l] && !s.pos[l]) s.sorted[k++] = l;
        s.flag[1] = k;
        uint64_t* pre = reinterpret_cast<uint64_t*>(s.a1);
        uint64_t run = 0;
        for (int r = 0; r < k; ++r) {
            run += s.cnt[s.sorted[r]] * static_cast<uint64_t>(g.bpe);
            pre[r] = run;
        }
        if (g.meta64) {
            g.meta64[META64_RESOLVED] = tag;
            g.meta64[META64_RESOLVE_DONE] = tag;
        }
    }
    __syncthreads();
    finalize_lists(g, s, s.sorted, s.flag[1], tag);
}

__global__ void k_set_budget(uint64_t* meta64, uint64_t budget) { meta64[META64_BUDGET] = budget; }

// Per-tile PGP partials of (params, grads) in the group's tile geometry for the
// certified resolve of arbitrary vectors: one warp per tile, lane-strided terms
// summed in order, then the fixed shuffle tree (depth <= T/32 + 5, inside
// tile_depth's bound).
__global__ void __launch_bounds__(256) k_pgp_tiles(GroupView g, const float* __restrict__ params,
                                                   const float* __restrict__ grads) {
    const int lane = threadIdx.x & 31;
    const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int t = gw; t < g.NT; t += nw) {
        const int l = g.tile_layer[t];
        const uint64_t s = g.offsets[l] + static_cast<uint64_t>(t - g.tile_base[l]) * g.T;
        const uint64_t e = min(s + static_cast<uint64_t>(g.T), g.offsets[l] + g.counts[l]);
        double acc = 0.0;
        for (uint64_t f = s + lane; f < e; f += 32) acc = __dadd_rn(acc, pgp_term(grads[f], params[f]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        if (lane == 0) g.partials[t] = acc;
    }
}

// Per-function API: exact sequential PGP of (params, grads) per layer.
__global__ void k_pgp_exact(const float* __restrict__ P, const float* __restrict__ Gr,
                            const uint64_t* offsets, const uint64_t* counts, double* scores) {
    const int l = blockIdx.x;
    const int lane = threadIdx.x;
    const uint64_t off = offsets[l], end = off + counts[l];
    double sum = 0.0;
    for (uint64_t b = off; b < end; b += 32) {
        const uint64_t f = b + lane;
        const double t = f < end ? pgp_term(Gr[f], P[f]) : 0.0;
        const int valid = static_cast<int>((end - b) < 32 ? (end - b) : 32);
        for (int i = 0; i < valid; ++i) sum = __dadd_rn(sum, __shfl_sync(0xffffffffu, t, i));
    }
    if (lane == 0) scores[l] = sum;
}

// Per-function API: rank + prefix-rule GIB of given scores.
__global__ void __launch_bounds__(kResolveThreads) k_rank_gib(const double* scores,
                                                              const uint64_t* counts, uint32_t bpe,
                                                              int L, uint64_t budget, int* order,
                                                              uint8_t* flags, char* scratch) {
    extern __shared__ __align__(16) char smem_raw[];
    __shared__ double sh_wtot[4 * kWarps];
    __shared__ int sh_flag[8];
    const Smem s = carve(scratch ? scratch : smem_raw, L, sh_wtot, sh_flag);
    for (int l = threadIdx.x; l < L; l += blockDim.x) s.key[l] = scores[l];
    __syncthreads();
    rank_layers_block(s, L);
    uint64_t* pre = reinterpret_cast<uint64_t*>(s.a1);
    for (int r = threadIdx.x; r < L; r += blockDim.x) pre[r] = counts[s.sorted[r]] * uint64_t(bpe);
    __syncthreads();
    block_scan<uint64_t>(pre, L, 0ull, [](uint64_t a, uint64_t b) { return a + b; }, s.wtot);
    for (int r = threadIdx.x; r < L; r += blockDim.x) {
        order[r] = s.sorted[r];
        flags[s.sorted[r]] = pre[r] <= budget ? 1 : 0;
    }
}

// Raise a kernel's dynamic shared-memory opt-in only when a launch needs more
// than any before it in this context (never lowered, so groups of different L
// can interleave): saves a host API call per launch on the launch-bound layouts.
// Keyed on the context (attributes do not survive a recreated context).
cudaError_t set_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<unsigned long long, const void*>, size_t> opted;
    cudaError_t e = cudaSuccess;
    const unsigned long long ctx = current_ctx_id();
    std::lock_guard<std::mutex> lock(mu);
    size_t& cur = opted[std::make_pair(ctx, fn)];
    if (bytes <= cur) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(bytes));
    if (e == cudaSuccess) cur = bytes;
    return e;
}

}  // namespace

cudaError_t launch_resolve(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                           cudaStream_t st) {
    const size_t sm = smem_bytes(g.L);
    cudaError_t e = set_smem(reinterpret_cast<const void*>(k_resolve), sm);
    if (e != cudaSuccess) return e;
    const int items = g.n_sum_items > 0 ? g.n_sum_items : 1;
    const int blocks = items < sm_count() ? items : sm_count();
    return launch_pdl(k_resolve, dim3(blocks), dim3(kResolveThreads), sm, st, g, ap, X, ldX);
}

cudaError_t launch_install_gib(const GroupView& g, const int* order, int n_order, uint32_t tag,
                               cudaStream_t st) {
    const size_t sm = smem_bytes(g.L);
    cudaError_t e = set_smem(reinterpret_cast<const void*>(k_install), sm);
    if (e != cudaSuccess) return e;
    k_install<<<1, kResolveThreads, sm, st>>>(g, order, n_order, tag);
    return cudaGetLastError();
}

cudaError_t launch_pgp_tiles(const GroupView& g, const float* params, const float* grads,
                             cudaStream_t st) {
    if (g.NT < 1) return cudaSuccess;
    const int blocks = min((g.NT + 7) / 8, sm_count() * 8);
    k_pgp_tiles<<<blocks, 256, 0, st>>>(g, params, grads);
    return cudaGetLastError();
}

cudaError_t launch_set_budget(const GroupView& g, uint64_t budget, cudaStream_t st) {
    k_set_budget<<<1, 1, 0, st>>>(g.meta64, budget);
    return cudaGetLastError();
}

cudaError_t launch_pgp_exact(const float* params, const float* grads, const uint64_t* offsets,
                             const uint64_t* counts, int L, double* scores, cudaStream_t st) {
    if (L < 1) return cudaSuccess;
    k_pgp_exact<<<L, 32, 0, st>>>(params, grads, offsets, counts, scores);
    return cudaGetLastError();
}

cudaError_t launch_rank_gib(const double* scores, const uint64_t* counts, uint32_t bpe, int L,
                            uint64_t budget, int* order, uint8_t* flags, cudaStream_t st) {
    if (L < 1) return cudaSuccess;
    const size_t sm = smem_bytes(L);
    char* scratch = nullptr;
    if (sm == 0) {  // above kSmemResolveLayers: the per-layer arrays in global memory
        cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), resolve_scratch_bytes(L), st);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = set_smem(reinterpret_cast<const void*>(k_rank_gib), sm);
    if (e == cudaSuccess) {
        k_rank_gib<<<1, kResolveThreads, sm, st>>>(scores, counts, bpe, L, budget, order, flags,
                                                   scratch);
        e = cudaGetLastError();
    }
    if (scratch) cudaFreeAsync(scratch, st);
    return e;
}

}  // namespace osp
