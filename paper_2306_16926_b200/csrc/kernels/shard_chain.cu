// The sharded stage 1 as a reduction CHAIN over the ranks (single-exchange mode,
// SURVEY.md §8(e); one process per GPU, CUDA-IPC mappings).
//
// The reference aggregates every element in ascending worker order
// (protocol.cpp:9-30): sum = ((w0 x0 + w1 x1) + w2 x2) + ... in fp64. Rank r
// hosts workers [r*NL, (r+1)*NL), so the running fp64 sum after rank r's
// workers is an exact intermediate of that sequence: rank 0 starts it, every
// next rank continues it from the previous rank's prefix, and the last rank
// finishes it. Nothing but the 8-byte prefix crosses NVLink on the way there
// (the exchange form of shard_x.cu moves every peer worker's 4-byte row to the
// owner: 4*NL bytes), and the 4-byte aggregate comes back. At P = 2 with
// N = 8 that is 8 + 4 bytes per element instead of 10 + 10 each way.
//
// Item kinds (one per tile of the whole tile sequence; CTA c of C takes tiles
// c, c + C, ... so every rank's front moves through the tiles in order):
//   PRE    (ranks 0..P-2) bulk-copy the previous rank's prefix (over NVLink,
//          rank > 0), this rank's delta rows and, for a deferred layer, G;
//          continue the sum over the local workers and store the prefix in
//          local HBM; a deferred layer also gets its LGP local estimates here
//          (rows = G + x_w). Flag: the next rank's chain flag.
//   FIN    (rank P-1) the same from the last prefix, then agg = float(sum / W),
//          G' = G + agg: RS layers G = G', rows = G'; ICS layers the carry
//          C = G' and rows = G + x_w; the tile's PGP partial (importance.cpp
//          11-28) goes to every rank's partials. Flag: every other rank's tile
//          flag.
//   APPLY  (ranks 0..P-2) after the tile flag: bulk-copy agg and G; RS:
//          G = G + agg, rows = G'; ICS: C. By default the last rank has stored
//          agg into every rank's pull buffer (NVLink stores ahead of its
//          flag's fence); with xa.chain_pushagg = 0 it is pulled from the last
//          rank's HBM, and these ranks' resolve reads it there for its exact
//          fallback (osp_shard.cu).
// The running sums stay where they were written and the next rank pulls them
// with cp.async.bulk after acquiring a flag the writer pushed into its memory
// (the writer's system-scope fence then drains only local stores and tiny flag
// stores); the aggregate goes the other way as NVLink stores, so no read
// request shares the link that carries the running sums.
// Every CTA of a non-finishing rank takes both PRE and APPLY items of its
// tiles, PRE items leading (see next_item).
//
// Diagnostics (xa.solo): 1 = every rank's PRE / FIN items alone, no flags,
// no APPLY (throughput of each role without the chain; results meaningless);
// 3 = the APPLY items alone, no flags;
// 2 = flags released with a GPU-scope fence (timing of the fence only; not a
// valid ordering for a peer reader).
//
// Hazards across iterations: rank r overwrites its prefix at iteration i+1
// only after finishing iteration i, whose APPLY items waited for every FIN of
// iteration i, each of which consumed the prefixes of iteration i; likewise the
// last rank's agg of iteration i+1 follows rank 0's completion of iteration i.
// Flags carry the iteration number and are never reset; every wait is bounded.

#include <cstdlib>

#include "shard_common.cuh"

namespace osp {
namespace {

enum CItem { CI_PRE = 0, CI_FIN = 1, CI_APPLY = 2 };
constexpr int kCPQ = 16;  // publication queue entries per CTA
constexpr int kCCW = 8;   // consumer warps

struct CMeta {
    uint64_t s, e;  // element range
    int t;          // tile id, -1 = stop
    int kind;       // CItem
    int staged;     // rows in shared memory (else consumers read global memory)
    int ics;        // tile of a deferred layer
};

// The ring is an arena of xa.chain_arena floats cut into as many slots as the
// CTA's item kind needs (at most kCMaxSlots): the bytes in flight per SM, not
// the slot count, set an HBM-bound role's rate, so a PRE slot of rank 0 (rows
// and G only), an APPLY slot (agg and G) and a FIN slot (prefix, rows, G) each
// fill the same shared memory. Slot layout (floats): PRE / FIN: [0, 2X) the
// incoming prefix (X = T when the rank has a predecessor, else 0), then the NL
// local delta rows, then G; APPLY: row 0 = agg, row 1 = G.
constexpr int kCMaxSlots = 16;

template <int NL>
__global__ void __launch_bounds__((kCCW + 2) * 32) k_shard_chain(GroupView g, AggParams ap, XArgs xa) {
    constexpr int CW = kCCW;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int T = g.T, NT = g.NT, L = g.L;
    const int P = xa.world, R = xa.rank;

    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + xa.chain_arena);
    uint64_t* empty = full + kCMaxSlots;
    uint64_t* pdone = empty + kCMaxSlots;
    CMeta* meta = reinterpret_cast<CMeta*>(pdone + kCPQ);
    double* red = reinterpret_cast<double*>(meta + kCMaxSlots);  // [kCPQ][CW]
    int* pq_t = reinterpret_cast<int*>(red + kCPQ * CW);  // [kCPQ] tile id, -1 stop
    int* pq_k = pq_t + kCPQ;                              // [kCPQ] item kind
    int* pub_head = pq_k + kCPQ;
    unsigned char* tabmem = reinterpret_cast<unsigned char*>(pub_head + 4);
    uint64_t* t_off = reinterpret_cast<uint64_t*>(tabmem);
    uint64_t* t_cnt = t_off + L;
    int* t_tb = reinterpret_cast<int*>(t_cnt + L);
    uint8_t* t_flag = reinterpret_cast<uint8_t*>(t_tb + L + 1);

    for (int i = tid; i < L; i += blockDim.x) {
        t_off[i] = g.offsets[i];
        t_cnt[i] = g.counts[i];
        t_tb[i] = g.tile_base[i];
        t_flag[i] = g.flags[i];
    }
    if (tid == 0) t_tb[L] = g.tile_base[L];
    // this is the iteration's stage 1: block 0 snapshots the ICS lists the
    // carry broadcast of stage 2 walks (as k_stage_tma's stage 1 does)
    if (g.snap && blockIdx.x == 0) {
        const int used = g.meta[META_N_USED];
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
    // roles and this CTA's tiles: the last rank's CTAs take FIN items, every
    // other rank's CTAs both PRE and APPLY items of their tiles (splitting the
    // CTAs between the two kinds measured slower: 0.48-0.53 vs 0.45-0.47 ms)
    const bool fin = R == P - 1;
    const int C = static_cast<int>(gridDim.x);
    const int c = static_cast<int>(blockIdx.x);
    const int n_own = c < C && c < NT ? (NT - 1 - c) / C + 1 : 0;
    // slot size and count for this CTA's item kinds
    const int xoff = R > 0 ? 2 : 0;  // rows of the incoming prefix in a PRE / FIN slot
    // the running sums: pulled from the previous rank's buffer, ours kept in our
    // own (pushing them into the next rank with NVLink stores measured slower:
    // 0.57 vs 0.49 ms, profiles/r2_multi_gpu_notes.md)
    const double* pre_in = R == 0 ? nullptr : xa.pre[R - 1];
    double* pre_out = R == P - 1 ? nullptr : xa.pre[R];
    const int slot_pf = (xoff + NL + 1) * T, slot_ap = 2 * T;
    const int SF = fin ? slot_pf : max(slot_pf, slot_ap);
    const int KS = min(kCMaxSlots, xa.chain_arena / SF);
    OSP_DCHECK(KS >= 2, "chain: arena holds fewer than two slots");
    if (tid == 0) {
        for (int s = 0; s < KS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
        }
        for (int j = 0; j < kCPQ; ++j) mbar_init(&pdone[j], CW);
        *pub_head = 0;
        mbar_init_fence();
    }
    __syncthreads();

    // Next item (kind, tile) of this CTA; false when done. FIN CTAs have one
    // kind; the others choose by readiness: an
    // APPLY item whose flag has landed goes first once the PRE front is
    // xa.chain_lead items ahead, else a PRE item; so PRE items lead the chain
    // and the APPLY items follow the last rank without a tail of idle PRE CTAs.
    // Readiness comes from relaxed loads issued one iteration ahead (lane k:
    // the k-th next item's flag; their latency hides behind the copy issue),
    // and an item is issued only after an acquire: lanes 0..kProbe-1 acquire
    // the next kProbe flags at once and the ready prefix is cached (a flag only
    // goes from not-ready to ready within a launch). The acquiring lanes'
    // order reaches the copy-issuing lanes through __syncwarp.
    constexpr int kProbe = 8;
    int ip = 0, ia = 0;              // next PRE / APPLY index of this CTA's tiles
    int pre_upto = 0, app_upto = 0;  // items whose flags were acquired lie below these
    unsigned rp_pre = 0, rp_app = 0; // this lane's relaxed probe of item ip / ia + lane
    const bool do_pre = !fin && xa.solo != 3;
    const bool do_app = !fin && xa.solo != 1;
    const bool pre_flags = R > 0 && xa.solo != 1 && xa.solo != 3;  // PRE / FIN wait for a prefix
    const bool app_flags = xa.solo != 3;
    const int n_pf = (fin && xa.solo != 3) || do_pre ? n_own : 0;  // PRE or FIN items
    const unsigned* pflag = xa.tflag[R] + NT;  // chain flags (from rank R-1)
    const unsigned* aflag = xa.tflag[R];       // tile flags (from the last rank)
    auto issue_probes = [&]() {
        if (lane < kProbe) {
            if (pre_flags && ip + lane < n_pf) rp_pre = ld_relaxed_sys(pflag + c + (ip + lane) * C);
            if (do_app && app_flags && ia + lane < n_own) rp_app = ld_relaxed_sys(aflag + c + (ia + lane) * C);
        }
    };
    // ready prefix of items [from, from + kProbe), acquired
    auto acquire = [&](const unsigned* base, int from, int n) -> int {
        int ok = 0;
        if (lane < kProbe && from + lane < n)
            ok = static_cast<int>(ld_acquire_sys(base + c + (from + lane) * C) - xa.epoch) >= 0;
        const unsigned m = __ballot_sync(0xffffffffu, ok);
        return from + __ffs(~m) - 1;
    };
    auto next_item = [&](int& kind, int& t) -> bool {
        const bool pre_left = ip < n_pf, app_left = do_app && ia < n_own;
        if (!pre_left && !app_left) return false;
        // the relaxed probes of the head items (issued last iteration)
        const bool pr = pre_left && (!pre_flags || ip < pre_upto ||
                                     __shfl_sync(0xffffffffu, static_cast<int>(rp_pre - xa.epoch) >= 0, 0));
        const bool ar = app_left && (!app_flags || ia < app_upto ||
                                     __shfl_sync(0xffffffffu, static_cast<int>(rp_app - xa.epoch) >= 0, 0));
        const bool ahead = ip - ia >= xa.chain_lead;
        int choice;
        if (!pre_left) choice = CI_APPLY;
        else if (!app_left) choice = fin ? CI_FIN : CI_PRE;
        else if (ar && (ahead || !pr)) choice = CI_APPLY;
        else if (pr || !ahead) choice = CI_PRE;
        else choice = CI_APPLY;
        // acquire the chosen item's flag (and its successors') when it looked ready
        if (choice == CI_APPLY && app_flags && ia >= app_upto && ar) app_upto = acquire(aflag, ia, n_own);
        if (choice != CI_APPLY && pre_flags && ip >= pre_upto && pr) pre_upto = acquire(pflag, ip, n_pf);
        kind = choice;
        t = c + (choice == CI_APPLY ? ia++ : ip++) * C;
        return true;
    };
    // blocking wait for an item whose flag was not seen ready (lane 0)
    auto ensure = [&](int kind, int idx, int t, long long& t_flag, long long& n_block) {
        const bool flagged = kind == CI_APPLY ? app_flags : pre_flags;
        const int upto = kind == CI_APPLY ? app_upto : pre_upto;
        if (!flagged || idx < upto) return;
        const long long b0 = clock64();
        const unsigned* fl = kind == CI_APPLY ? xa.tflag[R] + t : xa.tflag[R] + NT + t;
        if (lane == 0) xspin(fl, xa.epoch, xa.error);
        __syncwarp();
        ++n_block;
        t_flag += clock64() - b0;
    };
    auto locate = [&](int t, int kind, CMeta& m) {
        int l, kk;
        xseq_lookup(t_tb, nullptr, L, t, l, kk);
        m.t = t;
        m.kind = kind;
        m.s = t_off[l] + static_cast<uint64_t>(kk) * T;
        const uint64_t le = t_off[l] + t_cnt[l];
        m.e = m.s + static_cast<uint64_t>(T) < le ? m.s + static_cast<uint64_t>(T) : le;
        m.ics = t_flag[l];
        OSP_DCHECK(l >= 0 && l < L && m.s < m.e && m.e - m.s <= static_cast<uint64_t>(T),
                   "chain: tile lookup");
        m.staged = xa.vec && (m.s % 4 == 0) && ((m.e - m.s) % 4 == 0);
    };

    if (warp == CW + 1) {
        // ================= publisher =================
        // FIN tiles: the partial into every rank's partials, then (batched under
        // one system-scope fence) the tile flag on every other rank; PRE tiles:
        // the chain flag on the next rank. The fence is cumulative over the
        // consumers' stores, acquired through the entry barrier.
        constexpr int kPubMax = 16;
        const int batch = xa.pub_batch < 1 ? 1 : (xa.pub_batch > kPubMax ? kPubMax : xa.pub_batch);
        int pend[kPubMax];
        int np = 0, nf = 0;  // pending flags, flushes so far (warp-uniform)
        long long t_fence = 0, n_flush = 0;
        auto flush = [&]() {
            if (np == 0) return;
            ++nf;
            if (lane == 0 && xa.solo != 1 && xa.solo != 3) {
                const long long f0 = clock64();
                if (xa.solo == 2) asm volatile("fence.acq_rel.gpu;" ::: "memory");  // diagnostics only
                else asm volatile("fence.acq_rel.sys;" ::: "memory");
                t_fence -= f0 - clock64();
                ++n_flush;
                const unsigned long long now = xa.trace ? now_ns() : 0;
                for (int j = 0; j < np; ++j) {
                    if (xa.trace) xa.trace[static_cast<size_t>(fin ? 4 : 2) * NT + pend[j]] = now;
                    if (fin) {
                        for (int r = 0; r < P; ++r)
                            if (r != R) *reinterpret_cast<volatile unsigned*>(xa.tflag[r] + pend[j]) = xa.epoch;
                    } else {
                        *reinterpret_cast<volatile unsigned*>(xa.tflag[R + 1] + NT + pend[j]) = xa.epoch;
                    }
                }
            }
            np = 0;
            __syncwarp();
        };
        for (int i = 0;; ++i) {
            const int j = i % kCPQ;
            const unsigned par = (i / kCPQ) & 1;
            if (!mbar_try(&pdone[j], par)) {
                if (np >= xa.pub_min) flush();
                const uint64_t w0 = now_ns();
                while (!mbar_try(&pdone[j], par)) {
                    const uint64_t dt = now_ns() - w0;
                    if (np > 0 && dt > 2000) flush();
                    if (dt > 20000000000ull) __trap();
                }
            }
            const int t = pq_t[j], kind = pq_k[j];
            double tot = 0.0;
            if (t >= 0 && kind == CI_FIN)
                for (int w = 0; w < CW; ++w) tot = __dadd_rn(tot, red[j * CW + w]);
            __syncwarp();
            if (lane == 0) st_release_cta_s32(pub_head, i + 1);
            if (t == -1) {
                flush();
                break;
            }
            if (kind == CI_APPLY) continue;
            if (kind == CI_FIN && lane == 0 && xa.solo != 1 && xa.solo != 3)
                for (int r = 0; r < P; ++r) xa.part[r][t] = tot;
            pend[np++] = t;
            // the first flushes carry 1, 2, 4, ... flags: the next rank's first
            // tiles are released at once, later ones in full batches
            if (np >= min(batch, 1 << min(nf, 4))) flush();
        }
        if (xa.dbg && lane == 0) {
            atomicAdd(xa.dbg + 3, static_cast<unsigned long long>(t_fence));
            atomicAdd(xa.dbg + 9, static_cast<unsigned long long>(n_flush));
        }
        return;
    }

    if (warp == CW) {
        // ================= producer (whole warp: probes; lane 0 issues the copies) =================
        long long t_flag = 0, t_empty = 0, n_block = 0, n_it[3] = {0, 0, 0}, t_next = 0, t_issue = 0;
        const long long t_start = clock64();
        const uint64_t ns0 = now_ns();
        issue_probes();
        for (int i = 0;; ++i) {
            const int s = i % KS;
            const int use = i / KS;
            if (use > 0) {
                const long long e0 = clock64();
                mbar_wait(&empty[s], (use - 1) & 1);
                t_empty += clock64() - e0;
            }
            int kind = 0, t = 0;
            const long long n0 = clock64();
            const bool more = next_item(kind, t);
            t_next += clock64() - n0;
            if (!more) {
                if (lane == 0) {
                    CMeta m{};
                    m.t = -1;
                    meta[s] = m;
                    mbar_arrive(&full[s]);
                }
                break;
            }
            const long long i0 = clock64();
            CMeta m{};
            locate(t, kind, m);
            const bool has_pre = kind != CI_APPLY && R > 0;
            ++n_it[kind];
            if (xa.trace && lane == 0 && kind == CI_PRE) xa.trace[t] = now_ns();
            ensure(kind, kind == CI_APPLY ? ia - 1 : ip - 1, t, t_flag, n_block);
            if (kind == CI_APPLY ? app_flags : pre_flags)
                fence_proxy_async();  // the acquired flags before this item's bulk reads
            issue_probes();       // readiness for the next choice, in flight meanwhile
            if (xa.trace && lane == 0 && (kind == CI_APPLY || has_pre))
                xa.trace[static_cast<size_t>(kind == CI_APPLY ? 5 : 3) * NT + t] = now_ns();
            const unsigned bytes = static_cast<unsigned>((m.e - m.s) * 4);
            const bool need_g = kind != CI_PRE || m.ics;
            unsigned total = 0;
            if (m.staged)
                total = kind == CI_APPLY ? 2 * bytes : (has_pre ? 2 * bytes : 0) + NL * bytes + (need_g ? bytes : 0);
            if (lane == 0) {
                meta[s] = m;
                if (m.staged) mbar_arrive_tx(&full[s], total);
                else mbar_arrive(&full[s]);
            }
            __syncwarp();
            if (m.staged && lane == 0) {  // one thread issues the item's copies (as k_stage_tma)
                float* dst = ring + s * SF;
                if (kind == CI_APPLY) {
                    bulk_g2s(dst, xa.agg[xa.chain_pushagg ? R : P - 1] + m.s, bytes, &full[s]);
                    bulk_g2s(dst + T, g.G + m.s, bytes, &full[s]);
                } else {
                    if (has_pre) bulk_g2s(dst, pre_in + m.s, 2 * bytes, &full[s]);
#pragma unroll
                    for (int w = 0; w < NL; ++w)
                        bulk_g2s(dst + static_cast<size_t>(xoff + w) * T, xa.xrow[R * NL + w] + m.s, bytes, &full[s]);
                    if (need_g) bulk_g2s(dst + static_cast<size_t>(xoff + NL) * T, g.G + m.s, bytes, &full[s]);
                }
            }
            t_issue += clock64() - i0;
        }
        if (xa.dbg && lane == 0) {
            atomicAdd(xa.dbg + 0, static_cast<unsigned long long>(t_flag));
            atomicAdd(xa.dbg + 1, static_cast<unsigned long long>(t_empty));
            atomicAdd(xa.dbg + 4, static_cast<unsigned long long>(clock64() - t_start));
            atomicAdd(xa.dbg + 5, static_cast<unsigned long long>(n_block));
            atomicAdd(xa.dbg + 6, static_cast<unsigned long long>(n_it[CI_PRE]));
            atomicAdd(xa.dbg + 7, static_cast<unsigned long long>(n_it[CI_APPLY]));
            atomicAdd(xa.dbg + 8, static_cast<unsigned long long>(n_it[CI_FIN]));
            atomicMax(xa.dbg + 10, static_cast<unsigned long long>(now_ns() - ns0));
            atomicAdd(xa.dbg + 11, static_cast<unsigned long long>(t_next));
            atomicAdd(xa.dbg + 12, static_cast<unsigned long long>(t_issue));
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
        const CMeta m = meta[s];
        const int j = i % kCPQ;
        if (m.t < 0) {
            if (lane == 0) {
                while (ld_acquire_cta_s32(pub_head) < i - kCPQ + 1) __nanosleep(32);
                if (warp == 0) pq_t[j] = -1;
                mbar_arrive(&pdone[j]);
            }
            break;
        }
        const float* buf = ring + s * SF;
        const bool has_pre = m.kind != CI_APPLY && R > 0;
        double acc = 0.0;
        if (m.staged) {
            const int nq = static_cast<int>((m.e - m.s) >> 2);
            for (int qd = ctid; qd < nq; qd += CW * 32) {
                const uint64_t f = m.s + 4ull * qd;
                if (m.kind == CI_APPLY) {
                    const float4 a = *reinterpret_cast<const float4*>(buf + 4 * qd);
                    const float4 go = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(T) + 4 * qd);
                    const float4 gn = add4x(go, a);
                    if (m.ics) {
                        st_stream4(g.C + f, gn);
                    } else {
                        *reinterpret_cast<float4*>(g.G + f) = gn;
#pragma unroll
                        for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
                    }
                    continue;
                }
                double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
                if (has_pre) {
                    const double2 p0 = *reinterpret_cast<const double2*>(buf + 8 * qd);
                    const double2 p1 = *reinterpret_cast<const double2*>(buf + 8 * qd + 4);
                    s0 = p0.x;
                    s1 = p0.y;
                    s2 = p1.x;
                    s3 = p1.y;
                }
                float4 v[NL];
#pragma unroll
                for (int w = 0; w < NL; ++w) {
                    v[w] = cvt4x(ap, *reinterpret_cast<const float4*>(buf + static_cast<size_t>(xoff + w) * T + 4 * qd));
                    const double wt = ap.w[R * NL + w];
                    s0 = agg_acc(s0, wt, v[w].x);
                    s1 = agg_acc(s1, wt, v[w].y);
                    s2 = agg_acc(s2, wt, v[w].z);
                    s3 = agg_acc(s3, wt, v[w].w);
                }
                const bool need_g = m.kind == CI_FIN || m.ics;
                const float4 go = need_g ? *reinterpret_cast<const float4*>(buf + static_cast<size_t>(xoff + NL) * T + 4 * qd)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
                if (m.kind == CI_PRE) {
                    double* pr = pre_out + f;
                    *reinterpret_cast<double2*>(pr) = make_double2(s0, s1);
                    *reinterpret_cast<double2*>(pr + 2) = make_double2(s2, s3);
                    if (m.ics) {
#pragma unroll
                        for (int w = 0; w < NL; ++w)
                            st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, add4x(go, v[w]));
                    }
                    continue;
                }
                const float4 a = make_float4(agg_finish(ap, s0), agg_finish(ap, s1), agg_finish(ap, s2),
                                             agg_finish(ap, s3));
                const float4 gn = add4x(go, a);
                *reinterpret_cast<float4*>(xa.agg[R] + f) = a;
                if (xa.chain_pushagg)  // every other rank's copy (NVLink stores), flagged below
                    for (int r = 0; r < P - 1; ++r) *reinterpret_cast<float4*>(xa.agg[r] + f) = a;
                if (m.ics) {
                    st_stream4(g.C + f, gn);
#pragma unroll
                    for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, add4x(go, v[w]));
                } else {
                    *reinterpret_cast<float4*>(g.G + f) = gn;
#pragma unroll
                    for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
                }
                acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
                acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
                acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
                acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
            }
        } else {
            // unstaged tile (unaligned layer): per element from global memory
            // (the previous prefix and the last rank's agg over NVLink)
            for (uint64_t f = m.s + ctid; f < m.e; f += CW * 32) {
                const float go = g.G[f];
                if (m.kind == CI_APPLY) {
                    const float a = __ldcg(xa.agg[xa.chain_pushagg ? R : P - 1] + f);
                    const float gn = __fadd_rn(go, a);
                    if (m.ics) {
                        g.C[f] = gn;
                    } else {
                        g.G[f] = gn;
                        for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
                    }
                    continue;
                }
                double sum = has_pre ? __ldcg(pre_in + f) : 0.0;
                float x[NL];
                for (int w = 0; w < NL; ++w) {
                    x[w] = xa.xrow[R * NL + w][f];
                    if (ap.sgd) x[w] = sgd_conv(ap.neg_lr, x[w]);
                    sum = agg_acc(sum, ap.w[R * NL + w], x[w]);
                }
                if (m.kind == CI_PRE) {
                    pre_out[f] = sum;
                    if (m.ics)
                        for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x[w]);
                    continue;
                }
                const float a = agg_finish(ap, sum);
                const float gn = __fadd_rn(go, a);
                xa.agg[R][f] = a;
                if (xa.chain_pushagg)
                    for (int r = 0; r < P - 1; ++r) xa.agg[r][f] = a;
                if (m.ics) {
                    g.C[f] = gn;
                    for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x[w]);
                } else {
                    g.G[f] = gn;
                    for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
                }
                acc = __dadd_rn(acc, pgp_term(a, gn));
            }
        }
        if (m.kind == CI_FIN) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
        }
        __syncwarp();
        if (xa.trace && warp == 0 && lane == 0 && m.kind == CI_APPLY) xa.trace[6ull * NT + m.t] = now_ns();
        if (lane == 0) {
            mbar_arrive(&empty[s]);
            while (ld_acquire_cta_s32(pub_head) < i - kCPQ + 1) __nanosleep(32);
            red[j * CW + warp] = acc;
            if (warp == 0) {
                pq_t[j] = m.t;
                pq_k[j] = m.kind;
            }
            mbar_arrive(&pdone[j]);
        }
    }
    if (xa.dbg && tid == 0) atomicAdd(xa.dbg + 2, static_cast<unsigned long long>(t_full));
}

size_t chain_ctl_bytes(int L) {
    const size_t ctl = 2 * kCMaxSlots * sizeof(uint64_t) + kCPQ * sizeof(uint64_t) +
                       kCMaxSlots * sizeof(CMeta) + kCPQ * kCCW * sizeof(double) + 2 * kCPQ * sizeof(int) + 16;
    const size_t tab = static_cast<size_t>(L) * 16 + (L + 1) * 4 + ((L + 15) & ~15) + 64;
    return ctl + tab;
}

// the ring arena in floats: OSP_SHARD_CHAIN_ARENA_KB (default 200), at least
// two FIN slots, and the whole CTA within 227 KB
// the ring arena in floats: OSP_SHARD_CHAIN_ARENA_KB (default 200: one CTA
// per SM, three FIN slots) on the last rank, OSP_SHARD_CHAIN_ARENA_KB0
// (default 100: two CTAs per SM, measured 0.455 vs 0.495 ms at P = 2 for
// ResNet-50, 1.96 vs 2.22 for VGG-16) on the others; at least two slots of
// the rank's largest item, the CTA within 227 KB
int chain_arena_floats(int n_loc, int T, int L, int rank, int world) {
    auto env_kb = [](const char* name, int dflt) {
        const char* e = std::getenv(name);
        const int v = e ? std::atoi(e) : dflt;
        return v >= 32 && v <= 224 ? v : dflt;
    };
    static const int kb_fin = env_kb("OSP_SHARD_CHAIN_ARENA_KB", 200);
    static const int kb_pre = env_kb("OSP_SHARD_CHAIN_ARENA_KB0", 100);
    const bool fin = rank == world - 1;
    const int rows = rank > 0 ? n_loc + 3 : n_loc + 1;  // (prefix) + rows + G
    const size_t cap = 227 * 1024 - chain_ctl_bytes(L);
    size_t bytes = std::min<size_t>(static_cast<size_t>(fin ? kb_fin : kb_pre) * 1024, cap);
    bytes = std::max<size_t>(bytes, 2ull * rows * T * sizeof(float));
    return static_cast<int>(bytes / sizeof(float)) & ~31;
}

template <int NL>
cudaError_t launch_chain_nl(const GroupView& g, const AggParams& ap, XArgs xa, cudaStream_t s) {
    auto kern = k_shard_chain<NL>;
    xa.chain_arena = chain_arena_floats(NL, g.T, g.L, xa.rank, xa.world);
    const size_t sm = static_cast<size_t>(xa.chain_arena) * sizeof(float) + chain_ctl_bytes(g.L);
    int per_sm = 0;
    cudaError_t e = tma_blocks_per_sm(reinterpret_cast<const void*>(kern), (kCCW + 2) * 32, sm, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const int grid = sm_count() * (per_sm > 2 ? 2 : per_sm);
    kern<<<grid, (kCCW + 2) * 32, sm, s>>>(g, ap, xa);
    return cudaGetLastError();
}

}  // namespace

bool shard_chain_supported(int n_loc, int T, int L) {
    if (n_loc < 1 || n_loc > kXMaxStagedWorkers || T < 512 || T > 4096) return false;
    return 2ull * (n_loc + 3) * T * sizeof(float) + chain_ctl_bytes(L) <= 227 * 1024;
}

cudaError_t launch_shard_chain(const GroupView& g, const AggParams& ap, const XArgs& xa, cudaStream_t s) {
    switch (xa.n_loc) {
        case 1: return launch_chain_nl<1>(g, ap, xa, s);
        case 2: return launch_chain_nl<2>(g, ap, xa, s);
        case 3: return launch_chain_nl<3>(g, ap, xa, s);
        case 4: return launch_chain_nl<4>(g, ap, xa, s);
        case 5: return launch_chain_nl<5>(g, ap, xa, s);
        case 6: return launch_chain_nl<6>(g, ap, xa, s);
        case 7: return launch_chain_nl<7>(g, ap, xa, s);
        case 8: return launch_chain_nl<8>(g, ap, xa, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace osp
