// The sharded (multi-GPU) exchange kernel: one launch does a stage's push
// (reduce-scatter), fixed-order aggregation, pull (all-gather) and the local
// apply, with per-tile ready flags over NVLink peer memory instead of grid-wide
// cross-GPU barriers (one process per GPU, CUDA-IPC mappings).
//
// The exchanged tile sequence (mode SINGLE: every tile, the ICS payload split at
// stage-1 time as split_for_sync copies it, protocol.cpp:122-166; mode RS: the
// barrier layers; mode ICS: the deferred layers of chunks [c0, c1)) is cut into
// P contiguous owner ranges, and each owner range into one slice per CTA. Three
// kinds of work item per CTA:
//
//   A  a tile of this rank's own slice: bulk-copy (cp.async.bulk, SASS UBLKCP)
//      every worker's delta rows into shared memory — the local ones from HBM,
//      the others straight out of the peers' HBM over NVLink — plus the G slice;
//      aggregate in fp64 in the reference's ascending worker order
//      (protocol.cpp:9-30, bit-exact, unlike an fp32 NCCL reduce-scatter);
//      apply locally (RS: G' = G + agg, local rows = G'; ICS in SINGLE mode:
//      local rows = G + x_w, the LGP local estimate, and the carry C = G + agg);
//      store agg into every rank's pull buffer (NVLink stores); the publisher
//      warp then writes the tile's PGP partial into every rank's partials and,
//      after a system-scope fence, the tile's flag on every peer.
//   B  the same slice position of a peer's range: wait for its flag, bulk-copy
//      agg (written by the owner into the local pull buffer), the G slice and,
//      for a deferred layer in SINGLE mode, the local delta rows; apply as A.
//   L  (mode RS) a deferred layer's tile: the local estimate only, no exchange.
//
// CTA c of every rank works on slice c of every owner range at the same pace,
// so B items are scheduled by due time a few A items behind (lag): the peer's
// CTA c has published them by then. A merge by due time interleaves the
// NVLink-bound A items with the HBM-bound B / L items so both links stay busy.
//
// Ordering across GPUs: at launch every CTA signals "this iteration's delta rows
// are ready" (epoch) into every peer's ready slots and waits for every peer's
// before its first A item (or, with none, before it ends); a rank at iteration i has finished iteration i-1's
// kernels, so the pull buffer, partials and flags need no double buffering.
// Tile flags carry the iteration number (each tile is exchanged once per
// iteration) and are never reset. Every wait is bounded (20 s) and records an
// error instead of hanging.

#include "common.cuh"
#include "tma.cuh"
#include "shard_common.cuh"

namespace osp {
namespace {

enum XItem { XI_A = 0, XI_B = 1, XI_L = 2 };
constexpr int kPQ = 16;  // publication queue entries per CTA

struct XMeta {
    uint64_t s, e;  // element range
    int t;          // global tile id, -1 = stop
    int kind;       // XItem
    int staged;     // rows in shared memory (else consumers read global memory)
    int ics;        // tile of a deferred layer
};

// Per-CTA item order: A items at due time i, the peers' B items
// (j + 1) * nA / nB + lag - 1 (behind the A item the peer's CTA is on), L items
// spread evenly; ties go to A. A B item whose flag has not landed yet is passed
// over while A / L items remain (the producer never blocks the ring on a peer
// while it has local work to issue). Identical on every lane: the readiness
// probe is lane 0's, broadcast.
struct XSched {
    int nA, nL, nB[kMaxRanks];
    int ia, il, ib[kMaxRanks];
    int P, R, lag;
    int pace;  // A items of this slice (or of the peers' slices when this CTA has none)

    __device__ double dueA() const { return ia < nA ? static_cast<double>(ia) : 1e30; }
    __device__ double dueL() const {
        if (il >= nL) return 1e30;
        return (static_cast<double>(il) + 0.5) * pace / nL;
    }
    __device__ double dueB(int q) const {
        if (ib[q] >= nB[q]) return 1e30;
        return (static_cast<double>(ib[q]) + 1.0) * pace / nB[q] + lag - 1;
    }
    // the earliest-due B item: (peer, index) or q = -1
    __device__ void headB(int& q, int& k, double& due) const {
        q = -1;
        due = 1e30;
        for (int p = 0; p < P; ++p) {
            if (p == R) continue;
            const double d = dueB(p);
            if (d < due) {
                due = d;
                q = p;
            }
        }
        k = q >= 0 ? ib[q] : 0;
    }
    // next (kind, peer, index) given whether the head B item is ready; kind -1 = done
    __device__ void next(bool b_ready, int& kind, int& q, int& k) {
        int bq, bk;
        double bd;
        headB(bq, bk, bd);
        const double da = dueA(), dl = dueL();
        const bool local_left = ia < nA || il < nL;
        kind = -1;
        if (bq >= 0 && (b_ready || !local_left) && bd < da && bd < dl) {
            kind = XI_B;
            q = bq;
            k = bk;
            ++ib[bq];
            return;
        }
        if (ia < nA && da <= dl) {
            kind = XI_A;
            q = R;
            k = ia++;
            return;
        }
        if (il < nL) {
            kind = XI_L;
            q = R;
            k = il++;
            return;
        }
        if (bq >= 0) {
            kind = XI_B;
            q = bq;
            k = bk;
            ++ib[bq];
        }
    }
};

// Slot layout: A: rows 0..N-1 = every worker's deltas, row N = G.
//              B: row 0 = agg, row 1 = G, rows 2.. = local deltas (ICS, SINGLE).
//              L: rows 0..NL-1 = local deltas, row NL = G.
template <int NS, int CW, int KS>
__global__ void __launch_bounds__((CW + 2) * 32) k_shard_x(GroupView g, AggParams ap, XArgs xa) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int T = g.T;
    const int P = xa.world, R = xa.rank, NL = xa.n_loc, N = ap.n;
    const size_t SF = static_cast<size_t>(xa.slot_rows) * T;

    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + KS * SF);
    uint64_t* empty = full + KS;
    uint64_t* pdone = empty + KS;                       // [kPQ] publication entries complete
    XMeta* meta = reinterpret_cast<XMeta*>(pdone + kPQ);
    double* red = reinterpret_cast<double*>(meta + KS);  // [kPQ][CW] warp partials
    int* pq_t = reinterpret_cast<int*>(red + kPQ * CW);  // [kPQ] tile id (-1 stop, -2 no flag)
    int* pub_head = pq_t + kPQ;                         // [1] entries the publisher consumed
    unsigned char* tabmem = reinterpret_cast<unsigned char*>(pub_head + 4);

    // ---- tables: layer geometry, exchange sequence, local-estimate sequence
    const int L = g.L;
    uint64_t* t_off = reinterpret_cast<uint64_t*>(tabmem);
    uint64_t* t_cnt = t_off + L;
    int* t_tb = reinterpret_cast<int*>(t_cnt + L);
    uint8_t* t_flag = reinterpret_cast<uint8_t*>(t_tb + L + 1);
    int* xl = reinterpret_cast<int*>(t_flag + ((L + 15) & ~15));
    int* xp = xl + L;
    int* cl = xp + L + 1;
    int* cp = cl + L;
    int nx = 0, nc = 0, xb = 0;
    const int* XL = nullptr;
    const int* XP = g.tile_base;
    const int used = g.meta[META_N_USED];
    if (xa.mode == XM_SINGLE) {
        nx = L;
    } else if (xa.mode == XM_RS) {
        XL = g.rs_layers;
        XP = g.rs_tile_prefix;
        nx = g.meta[META_N_RS];
        nc = used > 0 ? g.chunk_begin[used] : 0;
    } else {
        XL = g.ics_layers;
        XP = g.ics_tile_prefix;
        const int cc1 = xa.c1 > used ? used : xa.c1;
        if (xa.c0 < cc1) {
            xb = g.chunk_begin[xa.c0];
            nx = g.chunk_begin[cc1] - xb;
        }
    }
    for (int i = tid; i < L; i += blockDim.x) {
        t_off[i] = g.offsets[i];
        t_cnt[i] = g.counts[i];
        t_tb[i] = g.tile_base[i];
        t_flag[i] = g.flags[i];
    }
    if (tid == 0) t_tb[L] = g.tile_base[L];
    if (XL)
        for (int i = tid; i < nx; i += blockDim.x) xl[i] = XL[xb + i];
    for (int i = tid; nx > 0 && i <= nx; i += blockDim.x) xp[i] = XP[xb + i];
    for (int i = tid; i < nc; i += blockDim.x) cl[i] = g.ics_layers[i];
    for (int i = tid; nc > 0 && i <= nc; i += blockDim.x) cp[i] = g.ics_tile_prefix[i];
    // SINGLE mode is this iteration's stage 1: block 0 snapshots the ICS lists
    // the stage-3 broadcast walks (as k_stage_tma's stage 1 does)
    if (xa.mode == XM_SINGLE && g.snap && blockIdx.x == 0 && !xa.solo) {
        const int n_ics = g.meta[META_N_ICS];
        int* snap_cb = g.snap + kSnapHead;
        int* snap_il = snap_cb + g.n_chunks + 1;
        int* snap_tp = snap_il + L;
        if (tid == 0) {
            g.snap[0] = used;
            g.snap[1] = static_cast<int>(g.meta64[META64_RESOLVED] + 1);
        }
        for (int i = tid; i <= g.n_chunks; i += blockDim.x) snap_cb[i] = g.chunk_begin[i];
        for (int i = tid; i < n_ics; i += blockDim.x) snap_il[i] = g.ics_layers[i];
        for (int i = tid; i <= n_ics; i += blockDim.x) snap_tp[i] = g.ics_tile_prefix[i];
    }
    if (tid == 0) {
        for (int s = 0; s < KS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        for (int j = 0; j < kPQ; ++j) mbar_init(&pdone[j], CW);
        *pub_head = 0;
        mbar_init_fence();
    }
    __syncthreads();

    // role split (xa.split): even CTAs take the own slices (A items, NVLink-bound),
    // odd CTAs the peers' slices and the local estimates (B / L items, HBM-bound),
    // so waiting on a peer never takes a ring slot from the exchange
    const bool split = xa.split != 0 && gridDim.x >= 2;
    const int C = split ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
    const int c = split ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
    const int role = split ? (static_cast<int>(blockIdx.x) & 1) + 1 : 0;  // 0 all, 1 A, 2 B/L
    const int U0 = nx > 0 ? xp[0] : 0;
    const int U = nx > 0 ? xp[nx] - U0 : 0;
    const int V = nc > 0 ? cp[nc] - cp[0] : 0;
    // owner range of rank q, and CTA c's slice of it
    auto range_lo = [&](int q) { return static_cast<int>((static_cast<int64_t>(U) * q) / P); };
    auto slice_lo = [&](int q, int cc) {
        const int lo = range_lo(q), len = range_lo(q + 1) - lo;
        return lo + static_cast<int>((static_cast<int64_t>(len) * cc) / C);
    };
    const int lcl_lo = static_cast<int>((static_cast<int64_t>(V) * c) / C);

    auto locate = [&](int kind, int u, XMeta& m) {
        int l, kk;
        if (kind == XI_L) xseq_lookup(cp, cl, nc, (nc > 0 ? cp[0] : 0) + u, l, kk);
        else xseq_lookup(xp, XL ? xl : nullptr, nx, U0 + u, l, kk);
        m.t = t_tb[l] + kk;
        m.s = t_off[l] + static_cast<uint64_t>(kk) * T;
        const uint64_t le = t_off[l] + t_cnt[l];
        m.e = m.s + static_cast<uint64_t>(T) < le ? m.s + static_cast<uint64_t>(T) : le;
        m.kind = kind;
        m.ics = t_flag[l];
        OSP_DCHECK(l >= 0 && l < L, "shard: tile layer out of range");
        OSP_DCHECK(m.t >= 0 && m.t < g.NT, "shard: tile id out of range");
        OSP_DCHECK(m.s < m.e && m.e - m.s <= static_cast<uint64_t>(T), "shard: tile range");
        m.staged = xa.vec && NS > 0 && (m.s % 4 == 0) && ((m.e - m.s) % 4 == 0);
    };

    if (warp == CW + 1) {
        // ================= publisher =================
        // Consumers hand every item to this warp through a kPQ-entry queue
        // (warp partials + tile id) and free the ring slot themselves, so the
        // system-scope fence below never holds a slot. A tiles' partials go out
        // as their entries complete; their flags are published in batches under
        // one fence (cumulative over the consumers' pull stores, acquired through
        // the entry barrier, and the partials): when kPubBatch are pending or no
        // further entry is complete yet.
        constexpr int kPubMax = 16;
        const int batch = xa.pub_batch < 1 ? 1 : (xa.pub_batch > kPubMax ? kPubMax : xa.pub_batch);
        int pend[kPubMax];
        int np = 0;
        long long t_fence = 0, n_flush = 0;
        auto flush = [&]() {
            if (np == 0) return;
            if (lane == 0 && !xa.solo && xa.phase == 0) {
                const long long f0 = clock64();
                // acq_rel (not sc): a release pattern for the flag stores below
                asm volatile("fence.acq_rel.sys;" ::: "memory");
                for (int j = 0; j < np; ++j)
                    for (int r = 0; r < P; ++r)
                        if (r != R) *reinterpret_cast<volatile unsigned*>(xa.tflag[r] + pend[j]) = xa.epoch;
                t_fence += clock64() - f0;
                ++n_flush;
            }
            np = 0;
            __syncwarp();
        };
        for (int i = 0;; ++i) {
            const int j = i % kPQ;
            const unsigned par = (i / kPQ) & 1;
            if (!mbar_try(&pdone[j], par)) {
                // nothing else to do: publish what is pending — at once when at
                // least pub_min flags wait, else after 2 us (a peer may be
                // blocked on exactly these tiles)
                if (np >= xa.pub_min) flush();
                const uint64_t w0 = now_ns();
                while (!mbar_try(&pdone[j], par)) {
                    const uint64_t dt = now_ns() - w0;
                    if (np > 0 && dt > 2000) flush();
                    if (dt > 20000000000ull) __trap();
                }
            }
            const int t = pq_t[j];
            double tot = 0.0;
            if (t >= 0)
                for (int w = 0; w < CW; ++w) tot = __dadd_rn(tot, red[j * CW + w]);
            __syncwarp();
            if (lane == 0) st_release_cta_s32(pub_head, i + 1);  // entry j may be reused
            if (t == -1) {
                flush();
                if (xa.phase == 1 && !xa.solo && lane == 0) {
                    // this CTA's pull stores (acquired through the queue) are
                    // visible system-wide; the last CTA out signals every peer
                    __threadfence_system();
                    if (atomicAdd(xa.ticket, 1u) == gridDim.x - 1) {
                        atomicExch(xa.ticket, 0u);
                        __threadfence_system();
                        for (int q = 0; q < P; ++q)
                            if (q != R) st_release_sys(xa.ready[q] + kMaxRanks + R, xa.done_epoch);
                    }
                }
                break;
            }
            if (t < 0) continue;  // B / L item: nothing to publish
            if (lane == 0)
                for (int r = 0; r < P; ++r) xa.part[r][t] = tot;
            pend[np++] = t;
            if (np >= batch) flush();
        }
        if (xa.dbg && lane == 0) {
            atomicAdd(xa.dbg + 3, static_cast<unsigned long long>(t_fence));
            atomicAdd(xa.dbg + 9, static_cast<unsigned long long>(n_flush));
        }
        return;
    }

    if (warp == CW) {
        // ================= producer (whole warp; lane j issues row j) =================
        XSched sc;
        sc.P = P;
        sc.R = R;
        sc.lag = xa.lag;
        sc.ia = sc.il = 0;
        // xa.phase: 0 = A, B and L items with per-tile flags; 1 = A and L items
        // only (then a cross-GPU "own tiles done" signal); 2 = B items only,
        // after every peer's signal (no per-tile waits)
        const bool do_a = role != 2 && (c < C) && xa.phase != 2;
        const bool do_bl = role != 1 && (c < C);
        const bool do_b = do_bl && xa.phase != 1, do_l = do_bl && xa.phase != 2;
        sc.nA = do_a ? slice_lo(R, c + 1) - slice_lo(R, c) : 0;
        sc.nL = do_l && xa.mode == XM_RS
                    ? static_cast<int>((static_cast<int64_t>(V) * (c + 1)) / C) - lcl_lo : 0;
        int pace = sc.nA;
        for (int q = 0; q < kMaxRanks; ++q) {
            sc.ib[q] = 0;
            sc.nB[q] = (do_b && q < P && q != R && !xa.solo) ? slice_lo(q, c + 1) - slice_lo(q, c) : 0;
            if (q < P && q != R) pace = max(pace, slice_lo(q, c + 1) - slice_lo(q, c));
        }
        sc.pace = pace > 0 ? pace : 1;
        // this iteration's delta rows are ready here; peers' before the first A item
        if (xa.phase == 2 && lane == 0)  // every peer's own tiles are in the pull buffer
            for (int q = 0; q < P; ++q)
                if (q != R) xspin(xa.ready[R] + kMaxRanks + q, xa.done_epoch, xa.error);
        if (lane == 0 && xa.mode != XM_ICS && !xa.solo && role != 2 && xa.phase != 2) {
            __threadfence_system();
            for (int q = 0; q < P; ++q)
                if (q != R) st_release_sys(xa.ready[q] + R, xa.epoch);
        }
        bool peers_ready = xa.mode == XM_ICS || xa.solo;
        long long t_bspin = 0, t_empty = 0, n_block = 0, n_it[3] = {0, 0, 0};
        const long long t_start = clock64();
        for (int i = 0;; ++i) {
            const int s = i % KS;
            const int use = i / KS;
            if (use > 0) {
                const long long e0 = clock64();
                mbar_wait(&empty[s], (use - 1) & 1);
                t_empty += clock64() - e0;
            }
            // probe the head B item's flag (lane 0), then choose
            int bq, bk;
            double bd;
            sc.headB(bq, bk, bd);
            int ready = xa.phase == 2 ? 1 : 0;
            if (bq >= 0 && xa.phase != 2) {
                XMeta mb{};
                locate(XI_B, slice_lo(bq, c) + bk, mb);
                if (lane == 0)
                    ready = static_cast<int>(ld_relaxed_sys(xa.tflag[R] + mb.t) - xa.epoch) >= 0 ? 1 : 0;
                ready = __shfl_sync(0xffffffffu, ready, 0);
            }
            int kind, q, k;
            sc.next(ready != 0, kind, q, k);  // every lane, same result
            XMeta m{};
            if (kind < 0) {
                // A CTA that exchanged nothing still waits for every peer's
                // deltas-ready epoch before it ends: the stage-2 (ICS) launch of
                // the same iteration reads the peers' rows on the strength of
                // this launch's wait (a budget of the whole model leaves stage 1
                // without barrier tiles), and a rank must not run ahead into the
                // next iteration's rows while a peer still reads this one's.
                if (!peers_ready && do_a) {
                    if (lane == 0)
                        for (int p = 0; p < P; ++p)
                            if (p != R) xspin(xa.ready[R] + p, xa.epoch, xa.error);
                    __syncwarp();
                    peers_ready = true;
                }
                if (lane == 0) {
                    m.t = -1;
                    meta[s] = m;
                    mbar_arrive(&full[s]);
                }
                break;
            }
            ++n_it[kind];
            const int u = kind == XI_A ? slice_lo(R, c) + k
                        : kind == XI_B ? slice_lo(q, c) + k
                                       : lcl_lo + k;
            locate(kind, u, m);
            if (kind == XI_A && !peers_ready) {
                if (lane == 0)
                    for (int p = 0; p < P; ++p)
                        if (p != R) xspin(xa.ready[R] + p, xa.epoch, xa.error);
                __syncwarp();
                fence_proxy_async();
                peers_ready = true;
            }
            if (kind == XI_B) {
                const long long b0 = clock64();
                if (lane == 0 && xa.phase != 2) xspin(xa.tflag[R] + m.t, xa.epoch, xa.error);
                __syncwarp();
                fence_proxy_async();
                if (!ready) {
                    t_bspin += clock64() - b0;
                    ++n_block;
                }
            }
            const bool local_rows = kind == XI_L || (kind == XI_B && m.ics && xa.mode == XM_SINGLE);
            const int nrows = kind == XI_A ? N + 1 : kind == XI_L ? NL + 1 : (local_rows ? 2 + NL : 2);
            OSP_DCHECK(!m.staged || nrows <= xa.slot_rows, "shard: item rows exceed the ring slot");
            OSP_DCHECK(u >= 0 && u < (kind == XI_L ? V : U), "shard: sequence position out of range");
            const unsigned bytes = static_cast<unsigned>((m.e - m.s) * 4);
            if (lane == 0) {
                meta[s] = m;
                if (m.staged) mbar_arrive_tx(&full[s], bytes * nrows);
            }
            __syncwarp();
            if (m.staged) {
                float* dst = ring + s * SF;
                for (int r = lane; r < nrows; r += 32) {
                    const float* src;
                    if (kind == XI_A) src = r < N ? xa.xrow[r] + m.s : g.G + m.s;
                    else if (kind == XI_L) src = r < NL ? xa.xrow[R * NL + r] + m.s : g.G + m.s;
                    else src = r == 0 ? xa.agg[R] + m.s : r == 1 ? g.G + m.s : xa.xrow[R * NL + r - 2] + m.s;
                    bulk_g2s(dst + static_cast<size_t>(r) * T, src, bytes, &full[s]);
                }
            } else if (lane == 0) {
                mbar_arrive(&full[s]);
            }
        }
        if (xa.dbg && lane == 0) {
            atomicAdd(xa.dbg + 0, static_cast<unsigned long long>(t_bspin));
            atomicAdd(xa.dbg + 1, static_cast<unsigned long long>(t_empty));
            atomicAdd(xa.dbg + 4, static_cast<unsigned long long>(clock64() - t_start));
            atomicAdd(xa.dbg + 5, static_cast<unsigned long long>(n_block));
            for (int j = 0; j < 3; ++j) atomicAdd(xa.dbg + 6 + j, static_cast<unsigned long long>(n_it[j]));
        }
        return;
    }

    // ================= consumers =================
    const int ctid = tid;
    long long t_full = 0;
    for (int i = 0;; ++i) {
        const int s = i % KS;
        const long long f0 = clock64();
        mbar_wait(&full[s], (i / KS) & 1);
        t_full += clock64() - f0;
        const XMeta m = meta[s];
        const int j = i % kPQ;
        if (m.t < 0) {
            if (lane == 0) {
                // queue entry j is free once the publisher consumed item i - kPQ
                while (ld_acquire_cta_s32(pub_head) < i - kPQ + 1) __nanosleep(32);
                if (warp == 0) pq_t[j] = -1;
                mbar_arrive(&pdone[j]);
            }
            break;
        }
        const float* buf = ring + s * SF;
        // ICS tile of SINGLE mode: local estimate + carry; otherwise G' and rows
        const bool carry = m.ics && xa.mode == XM_SINGLE;
        double acc = 0.0;
        if (m.staged) {
            const int nq = static_cast<int>((m.e - m.s) >> 2);
            for (int qd = ctid; qd < nq; qd += CW * 32) {
                const uint64_t f = m.s + 4ull * qd;
                if (m.kind == XI_A) {
                    if constexpr (NS > 0) {
                        const float4 go = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(NS) * T + 4 * qd);
                        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
                        for (int w = 0; w < NS; ++w) {
                            const float4 v = cvt4x(ap, *reinterpret_cast<const float4*>(
                                                           buf + static_cast<size_t>(w) * T + 4 * qd));
                            s0 = agg_acc(s0, ap.w[w], v.x);
                            s1 = agg_acc(s1, ap.w[w], v.y);
                            s2 = agg_acc(s2, ap.w[w], v.z);
                            s3 = agg_acc(s3, ap.w[w], v.w);
                        }
                        const float4 a = make_float4(agg_finish(ap, s0), agg_finish(ap, s1),
                                                     agg_finish(ap, s2), agg_finish(ap, s3));
                        const float4 gn = add4x(go, a);
                        for (int r = 0; r < P; ++r) *reinterpret_cast<float4*>(xa.agg[r] + f) = a;
                        if (carry) {
                            st_stream4(g.C + f, gn);
                            for (int w = 0; w < NL; ++w) {
                                const float4 v = cvt4x(ap, *reinterpret_cast<const float4*>(
                                                               buf + static_cast<size_t>(R * NL + w) * T + 4 * qd));
                                st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, add4x(go, v));
                            }
                        } else {
                            *reinterpret_cast<float4*>(g.G + f) = gn;
                            for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
                        }
                        acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
                        acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
                        acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
                        acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
                    }
                } else if (m.kind == XI_B) {
                    const float4 a = *reinterpret_cast<const float4*>(buf + 4 * qd);
                    const float4 go = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(T) + 4 * qd);
                    const float4 gn = add4x(go, a);
                    if (carry) {
                        st_stream4(g.C + f, gn);
                        for (int w = 0; w < NL; ++w) {
                            const float4 v = cvt4x(ap, *reinterpret_cast<const float4*>(
                                                           buf + static_cast<size_t>(2 + w) * T + 4 * qd));
                            st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, add4x(go, v));
                        }
                    } else {
                        *reinterpret_cast<float4*>(g.G + f) = gn;
                        for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
                    }
                } else {
                    const float4 go = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(NL) * T + 4 * qd);
                    for (int w = 0; w < NL; ++w) {
                        const float4 v = cvt4x(ap, *reinterpret_cast<const float4*>(
                                                       buf + static_cast<size_t>(w) * T + 4 * qd));
                        st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, add4x(go, v));
                    }
                }
            }
        } else {
            // unstaged tile (unaligned layer, or more workers than the slot holds):
            // per element from global memory (peer rows over NVLink)
            for (uint64_t f = m.s + ctid; f < m.e; f += CW * 32) {
                const float go = g.G[f];
                if (m.kind == XI_L) {
                    for (int w = 0; w < NL; ++w) {
                        float x = xa.xrow[R * NL + w][f];
                        if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                        g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x);
                    }
                    continue;
                }
                float a;
                if (m.kind == XI_A) {
                    double sum = 0.0;
                    for (int w = 0; w < N; ++w) {
                        float x = xa.xrow[w][f];
                        if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                        sum = agg_acc(sum, ap.w[w], x);
                    }
                    a = agg_finish(ap, sum);
                    for (int r = 0; r < P; ++r) xa.agg[r][f] = a;
                } else {
                    a = __ldcg(xa.agg[R] + f);
                }
                const float gn = __fadd_rn(go, a);
                if (carry) {
                    g.C[f] = gn;
                    for (int w = 0; w < NL; ++w) {
                        float x = xa.xrow[R * NL + w][f];
                        if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                        g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x);
                    }
                } else {
                    g.G[f] = gn;
                    for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
                }
                if (m.kind == XI_A) acc = __dadd_rn(acc, pgp_term(a, gn));
            }
        }
        if (m.kind == XI_A) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&empty[s]);  // the slot's data has been read
            while (ld_acquire_cta_s32(pub_head) < i - kPQ + 1) __nanosleep(32);
            red[j * CW + warp] = acc;
            if (warp == 0) pq_t[j] = m.kind == XI_A ? m.t : -2;
            mbar_arrive(&pdone[j]);  // release: this warp's stores and partial
        }
    }
    if (xa.dbg && tid == 0) atomicAdd(xa.dbg + 2, static_cast<unsigned long long>(t_full));
}

constexpr int kXCW = 8;

size_t x_smem_bytes(int slot_rows, int T, int L, int ks) {
    const size_t ring = static_cast<size_t>(ks) * slot_rows * T * sizeof(float);
    const size_t ctl = 2 * ks * sizeof(uint64_t) + kPQ * sizeof(uint64_t) + ks * sizeof(XMeta) +
                       kPQ * kXCW * sizeof(double) + kPQ * sizeof(int) + 16;
    const size_t tab = static_cast<size_t>(L) * 16 + (L + 1) * 4 + ((L + 15) & ~15) + L * 4 +
                       (L + 1) * 4 + L * 4 + (L + 1) * 4 + 128;
    return ring + ctl + tab;
}

template <int NS, int KS>
cudaError_t launch_x_ks(const GroupView& g, const AggParams& ap, const XArgs& xa, cudaStream_t s) {
    auto kern = k_shard_x<NS, kXCW, KS>;
    const size_t sm = x_smem_bytes(xa.slot_rows, g.T, g.L, KS);
    int per_sm = 0;
    cudaError_t e = tma_blocks_per_sm(reinterpret_cast<const void*>(kern), (kXCW + 2) * 32, sm, &per_sm);
    if (e != cudaSuccess) return e;
    const int grid = sm_count() * (per_sm > 2 ? 2 : per_sm);
    kern<<<grid, (kXCW + 2) * 32, sm, s>>>(g, ap, xa);
    return cudaGetLastError();
}

template <int NS>
cudaError_t launch_x_ns(const GroupView& g, const AggParams& ap, const XArgs& xa, cudaStream_t s) {
    return launch_x_ks<NS, 2>(g, ap, xa, s);  // 3 stages measured slower (r2_multi_gpu_notes.md)
}

// Phase 2 of the barrier form: the peers' tiles of the exchanged sequence,
// applied straight from the pull buffer with 128-bit loads (HBM-bound: one
// warp per tile, two quads per lane in flight, no shared-memory staging), after
// every peer has signalled that its own tiles are in this rank's pull buffer.
__global__ void __launch_bounds__(256) k_shard_peer_apply(GroupView g, AggParams ap, XArgs xa) {
    extern __shared__ __align__(16) unsigned char smem_tab[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int P = xa.world, R = xa.rank, NL = xa.n_loc;
    const int L = g.L;
    uint64_t* t_off = reinterpret_cast<uint64_t*>(smem_tab);
    uint64_t* t_cnt = t_off + L;
    int* t_tb = reinterpret_cast<int*>(t_cnt + L);
    uint8_t* t_flag = reinterpret_cast<uint8_t*>(t_tb + L + 1);
    int* xl = reinterpret_cast<int*>(t_flag + ((L + 15) & ~15));
    int* xp = xl + L;
    int nx = 0, xb = 0;
    const int* XL = nullptr;
    const int* XP = g.tile_base;
    const int used = g.meta[META_N_USED];
    if (xa.mode == XM_SINGLE) {
        nx = L;
    } else if (xa.mode == XM_RS) {
        XL = g.rs_layers;
        XP = g.rs_tile_prefix;
        nx = g.meta[META_N_RS];
    } else {
        XL = g.ics_layers;
        XP = g.ics_tile_prefix;
        const int cc1 = xa.c1 > used ? used : xa.c1;
        if (xa.c0 < cc1) {
            xb = g.chunk_begin[xa.c0];
            nx = g.chunk_begin[cc1] - xb;
        }
    }
    for (int i = tid; i < L; i += blockDim.x) {
        t_off[i] = g.offsets[i];
        t_cnt[i] = g.counts[i];
        t_tb[i] = g.tile_base[i];
        t_flag[i] = g.flags[i];
    }
    if (XL)
        for (int i = tid; i < nx; i += blockDim.x) xl[i] = XL[xb + i];
    for (int i = tid; nx > 0 && i <= nx; i += blockDim.x) xp[i] = XP[xb + i];
    if (tid == 0) {
        for (int q = 0; q < P; ++q)
            if (q != R) xspin(xa.ready[R] + kMaxRanks + q, xa.done_epoch, xa.error);
    }
    __syncthreads();
    const int U0 = nx > 0 ? xp[0] : 0;
    const int U = nx > 0 ? xp[nx] - U0 : 0;
    const int lo = static_cast<int>((static_cast<int64_t>(U) * R) / P);
    const int hi = static_cast<int>((static_cast<int64_t>(U) * (R + 1)) / P);
    const int n_peer = U - (hi - lo);
    const bool carry_mode = xa.mode == XM_SINGLE;
    const float* aggR = xa.agg[R];
    const int gw = static_cast<int>((blockIdx.x * blockDim.x + tid) >> 5);
    const int nw = static_cast<int>((gridDim.x * blockDim.x) >> 5);
    for (int k = gw; k < n_peer; k += nw) {
        const int u = U0 + (k < lo ? k : k + (hi - lo));
        OSP_DCHECK(u >= U0 && u < U0 + U && (u < U0 + lo || u >= U0 + hi), "peer apply: position");
        int l, kk;
        xseq_lookup(xp, XL ? xl : nullptr, nx, u, l, kk);
        OSP_DCHECK(l >= 0 && l < L && kk >= 0, "peer apply: tile lookup");
        const uint64_t b = t_off[l] + static_cast<uint64_t>(kk) * g.T;
        const uint64_t e = min(b + static_cast<uint64_t>(g.T), t_off[l] + t_cnt[l]);
        const bool carry = carry_mode && t_flag[l];
        const bool vec = xa.vec && (b % 4 == 0) && ((e - b) % 4 == 0);
        if (vec) {
            for (uint64_t f0 = b + 4ull * lane; f0 < e; f0 += 256) {
                const uint64_t f1 = f0 + 128;
                const bool has1 = f1 < e;
                const float4 a0 = ld_stream4(aggR + f0), g0 = *reinterpret_cast<const float4*>(g.G + f0);
                float4 a1 = a0, g1 = g0;
                if (has1) {
                    a1 = ld_stream4(aggR + f1);
                    g1 = *reinterpret_cast<const float4*>(g.G + f1);
                }
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                    if (q == 1 && !has1) break;
                    const uint64_t f = q == 0 ? f0 : f1;
                    const float4 go = q == 0 ? g0 : g1;
                    const float4 gn = add4x(go, q == 0 ? a0 : a1);
                    if (carry) {
                        st_stream4(g.C + f, gn);
                        for (int w = 0; w < NL; ++w) {
                            const float4 x = cvt4x(ap, ld_stream4(xa.xrow[R * NL + w] + f));
                            st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, add4x(go, x));
                        }
                    } else {
                        *reinterpret_cast<float4*>(g.G + f) = gn;
                        for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
                    }
                }
            }
        } else {
            for (uint64_t f = b + lane; f < e; f += 32) {
                const float go = g.G[f];
                const float gn = __fadd_rn(go, aggR[f]);
                if (carry) {
                    g.C[f] = gn;
                    for (int w = 0; w < NL; ++w) {
                        float x = xa.xrow[R * NL + w][f];
                        if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                        g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x);
                    }
                } else {
                    g.G[f] = gn;
                    for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
                }
            }
        }
    }
}

size_t peer_apply_smem(int L) {
    return static_cast<size_t>(L) * 16 + (L + 1) * 4 + ((L + 15) & ~15) + L * 4 + (L + 1) * 4 + 64;
}

}  // namespace

int x_slot_rows(int n_workers) { return n_workers <= kXMaxStagedWorkers ? n_workers + 1 : 2; }

bool shard_x_supported(int n_workers, int T, int L) {
    if (T < 512 || T > 4096) return false;
    return x_smem_bytes(x_slot_rows(n_workers), T, L, 2) <= 220 * 1024;
}

cudaError_t launch_shard_peer_apply(const GroupView& g, const AggParams& ap, const XArgs& xa,
                                    cudaStream_t s) {
    const size_t sm = peer_apply_smem(g.L);
    int per_sm = 0;
    cudaError_t e = tma_blocks_per_sm(reinterpret_cast<const void*>(k_shard_peer_apply), 256, sm,
                                      &per_sm);
    if (e != cudaSuccess) return e;
    k_shard_peer_apply<<<sm_count() * (per_sm < 4 ? per_sm : 4), 256, sm, s>>>(g, ap, xa);
    return cudaGetLastError();
}

cudaError_t launch_shard_x(const GroupView& g, const AggParams& ap, const XArgs& xa, cudaStream_t s) {
    switch (ap.n <= kXMaxStagedWorkers ? ap.n : 0) {
        case 1: return launch_x_ns<1>(g, ap, xa, s);
        case 2: return launch_x_ns<2>(g, ap, xa, s);
        case 3: return launch_x_ns<3>(g, ap, xa, s);
        case 4: return launch_x_ns<4>(g, ap, xa, s);
        case 5: return launch_x_ns<5>(g, ap, xa, s);
        case 6: return launch_x_ns<6>(g, ap, xa, s);
        case 7: return launch_x_ns<7>(g, ap, xa, s);
        case 8: return launch_x_ns<8>(g, ap, xa, s);
        default: return launch_x_ns<0>(g, ap, xa, s);
    }
}

}  // namespace osp
