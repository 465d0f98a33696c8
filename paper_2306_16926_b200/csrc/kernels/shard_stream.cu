// Streaming sharded stage kernel: one launch per stage does the push
// (reduce-scatter), the aggregate, the pull (all-gather) and the local apply,
// with per-tile ready flags instead of grid-wide barriers.
//
// The stage's exchange tiles (RS layers in stage 1, ICS chunks [c0,c1) in
// stage 2) are dealt round-robin: sequence position u belongs to rank u % P.
// Per rank, three kinds of work item:
//   A  own exchange tile: bulk-copy (cp.async.bulk) every worker's delta rows
//      into shared memory — the local ones from HBM, the others straight out
//      of the peers' HBM over NVLink — plus the G slice; aggregate in the fixed
//      ascending worker order in fp64 (bit-exact), G' = G + agg; write G' to
//      local G and the local worker rows, and agg into every rank's pull
//      buffer (NVLink stores to the peers); publish the tile's PGP partial to
//      every rank, then the tile's ready flag (release, system scope) on every
//      peer.
//   C  (stage 1) local-estimate tile of an ICS layer: P_w = G + delta_w for the
//      local workers, no exchange.
//   B  a peer's exchange tile: wait for its flag, bulk-copy agg from the local
//      pull buffer (the owner wrote it) and the G slice, G' = G + agg, write G
//      and the local rows.
// Every rank thus ends the stage with the full aggregate in its pull buffer
// (agg_full), which the exact PGP fallback in resolve.cu reads.
//
// CTA = CW consumer warps + 1 producer warp + 1 publisher warp over a ring of
// shared-memory slots (as stage_tma.cu). The producer takes items from three
// dynamic counters in the order A, C, B (NVLink-bound exchange first, then the
// HBM-bound local work, which by then overlaps the peers' last exchange tiles,
// then the peers' tiles, mostly published by then); lane 0 prefetches the next
// grab while the current item is issued, and the bulk copies of an item are
// issued one row per lane. The publisher warp takes (tile, partial) entries
// from the consumers and does the system-scope publication off their path.
// Partial sums follow the stage_tma.cu tree (4 terms per thread, 5 shuffles,
// CW warps in order), inside resolve.cu's T/32+13 depth bound.
//
// Cross-rank ordering without a grid barrier:
//   * deltas-ready: at stage-1 start every producer stores xepoch into every
//     peer's slot; a producer waits for every peer's slot before its first A
//     item. A peer at iteration i has finished iteration i-1 (all reads of
//     the previous pull buffer / partials), so the pull buffer, partials and
//     flags need no double buffering.
//   * tile flags carry a strictly increasing epoch (2*iteration + stage - 2),
//     so they are never reset.
//   * publication: consumers' stores -> __syncwarp -> acq_rel CTA count -> queue
//     entry (release, CTA) -> publisher (acquire, CTA) -> st.release.sys flag.
// Every wait is bounded (20 s) and records pt.error instead of hanging.

#include <cstdlib>

#include "common.cuh"
#include "tma.cuh"

namespace osp {
namespace {

constexpr int kXReadyKind = 3;  // PeerTable flag slots: spare barrier kind
enum ItemKind { IT_A = 0, IT_B = 1, IT_C = 2 };

struct SMeta {
    uint64_t s, e;
    int t;       // global tile id, -1 = stop
    int kind;    // ItemKind
    int staged;  // data in shared memory (else consumers read global memory)
    int pad;
};

__device__ __forceinline__ void seq_lookup(const int* lp, const int* ll, int n, int u, int& l,
                                           int& k) {
    int a = 0, b = n - 1;
    while (a < b) {
        const int m = (a + b + 1) >> 1;
        if (lp[m] <= u) a = m;
        else b = m - 1;
    }
    l = ll[a];
    k = u - lp[a];
}

__device__ __forceinline__ void spin_until(const unsigned* p, unsigned want, unsigned* error) {
    if (static_cast<int>(ld_acquire_sys(p) - want) >= 0) return;
    const uint64_t t0 = now_ns();
    while (static_cast<int>(ld_acquire_sys(p) - want) < 0) {
        __nanosleep(64);
        if (now_ns() - t0 > 20000000000ull) {
            atomicExch(error, 1u);
            return;
        }
    }
}

template <int NS>
__device__ __forceinline__ float4 agg4(const AggParams& ap, const float4* xs, float4& a) {
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
    a = make_float4(agg_finish(ap, s0), agg_finish(ap, s1), agg_finish(ap, s2), agg_finish(ap, s3));
    return a;
}

constexpr int kMaxSt = 12;  // ring stages (control arrays are sized for this)
constexpr int kPubQ = 32;   // publication queue entries

struct PubEntry {
    double tot;
    int t;
    int seq;  // position + 1 once written
};

template <int NS, int CW>
__global__ void __launch_bounds__((CW + 2) * 32) k_shard_stream(GroupView g, AggParams ap,
                                                               PeerTable pt, StreamArgs sa) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int T = g.T;
    const int P = pt.world, R = pt.rank, NL = pt.n_loc;
    const int G = static_cast<int>(gridDim.x);
    const int rowG = NS;  // slot rows: deltas [0, NS), the G slice in row NS
    const size_t SF = static_cast<size_t>(NS + 1) * T;
    int nst = static_cast<int>(sa.ring_bytes / (SF * sizeof(float)));
    if (nst > kMaxSt) nst = kMaxSt;
    unsigned long long* dbg = sa.dbg;

    float* ring = reinterpret_cast<float*>(smem);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + sa.ring_bytes);
    uint64_t* empty = full + kMaxSt;
    SMeta* meta = reinterpret_cast<SMeta*>(empty + kMaxSt);
    double* red = reinterpret_cast<double*>(meta + kMaxSt);  // [kMaxSt][CW]
    int* cnt = reinterpret_cast<int*>(red + kMaxSt * CW);    // [kMaxSt]
    PubEntry* pq = reinterpret_cast<PubEntry*>(cnt + kMaxSt);  // [kPubQ]
    int* qctl = reinterpret_cast<int*>(pq + kPubQ);  // reserve, head, consumers done, pad
    unsigned char* tabmem = reinterpret_cast<unsigned char*>(qctl + 4);

    // ---- tables: layer geometry, exchange list, local-estimate list --------
    const int L = g.L;
    uint64_t* t_off = reinterpret_cast<uint64_t*>(tabmem);
    uint64_t* t_cnt = t_off + L;
    int* t_tb = reinterpret_cast<int*>(t_cnt + L);
    int* xl = t_tb + L + 1;
    int* xp = xl + L;
    int* cl = xp + L + 1;
    int* cp = cl + L;
    const int used = g.meta[META_N_USED];
    int xb = 0, xe = 0, cb = 0, ce = 0;
    const int* XL;
    const int* XP;
    if (sa.stage == 1) {
        XL = g.rs_layers;
        XP = g.rs_tile_prefix;
        xe = g.meta[META_N_RS];
        ce = used > 0 ? g.chunk_begin[used] : 0;
    } else {
        XL = g.ics_layers;
        XP = g.ics_tile_prefix;
        const int cc1 = sa.c1 > used ? used : sa.c1;
        if (sa.c0 < cc1) {
            xb = g.chunk_begin[sa.c0];
            xe = g.chunk_begin[cc1];
        }
    }
    const int nx = xe - xb, nc = ce - cb;
    for (int i = tid; i < L; i += blockDim.x) {
        t_off[i] = g.offsets[i];
        t_cnt[i] = g.counts[i];
        t_tb[i] = g.tile_base[i];
    }
    if (tid == 0) t_tb[L] = g.tile_base[L];
    for (int i = tid; i < nx; i += blockDim.x) xl[i] = XL[xb + i];
    for (int i = tid; nx > 0 && i <= nx; i += blockDim.x) xp[i] = XP[xb + i];
    for (int i = tid; i < nc; i += blockDim.x) cl[i] = g.ics_layers[cb + i];
    for (int i = tid; nc > 0 && i <= nc; i += blockDim.x) cp[i] = g.ics_tile_prefix[cb + i];
    for (int i = tid; i < kPubQ; i += blockDim.x) pq[i].seq = 0;
    if (tid == 0) {
        for (int s = 0; s < nst; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], CW);
            cnt[s] = 0;
        }
        qctl[0] = qctl[1] = qctl[2] = 0;
        mbar_init_fence();
    }
    __syncthreads();

    const int U0 = nx > 0 ? xp[0] : 0;
    const int U = nx > 0 ? xp[nx] - U0 : 0;
    const int nA = U > R ? (U - R + P - 1) / P : 0;
    const int nB = U - nA;
    const int V0 = nc > 0 ? cp[0] : 0;
    const int nC = nc > 0 ? cp[nc] - V0 : 0;

    auto locate = [&](int kind, int k, SMeta& m) {
        int l, kk;
        if (kind == IT_C) {
            seq_lookup(cp, cl, nc, V0 + k, l, kk);
        } else {
            int u;
            if (kind == IT_A) {
                u = U0 + k * P + R;
            } else {
                const int j = k % (P - 1);
                u = U0 + (k / (P - 1)) * P + (j < R ? j : j + 1);
            }
            seq_lookup(xp, xl, nx, u, l, kk);
        }
        m.t = t_tb[l] + kk;
        m.s = t_off[l] + static_cast<uint64_t>(kk) * T;
        const uint64_t le = t_off[l] + t_cnt[l];
        m.e = m.s + static_cast<uint64_t>(T) < le ? m.s + static_cast<uint64_t>(T) : le;
        m.kind = kind;
        m.staged = sa.vec && (m.s % 4 == 0) && ((m.e - m.s) % 4 == 0);
    };

    if (warp == CW + 1) {
        // ================= publisher =================
        if (lane == 0) {
            int head = 0;
            for (;;) {
                PubEntry* e = pq + (head % kPubQ);
                if (ld_acquire_cta_s32(&e->seq) == head + 1) {
                    const double tot = e->tot;
                    const int t = e->t;
                    for (int r = 0; r < P; ++r) sa.part[r][t] = tot;
                    for (int r = 0; r < P; ++r)
                        if (r != R) st_release_sys(sa.tflag[r] + t, sa.tepoch);
                    ++head;
                    st_release_cta_s32(&qctl[1], head);
                    continue;
                }
                if (ld_acquire_cta_s32(&qctl[2]) == CW && ld_acquire_cta_s32(&qctl[0]) == head) break;
                __nanosleep(32);
            }
        }
        return;
    }

    if (warp == CW) {
        // ================= producer (whole warp) =================
        if (sa.stage == 1 && lane == 0) {
            __threadfence_system();
            for (int q = 0; q < P; ++q)
                if (q != R) st_release_sys(pt.flags[q] + kXReadyKind * kMaxRanks + R, sa.xepoch);
        }
        int* ctr[3] = {g.sched + SCHED_SS_A, g.sched + SCHED_SS_B, g.sched + SCHED_SS_C};
        const int lim[3] = {nA, nB, nC};
        const int order[3] = {IT_A, IT_C, IT_B};
        int phase = 0;  // index into order
        int pending = 0;
        if (lane == 0) pending = atomicAdd(ctr[order[0]], 1);
        bool xok = false;
        long long w_empty = 0, w_b = 0, n_it[3] = {0, 0, 0};
        const long long p0 = clock64();
        for (int i = 0;; ++i) {
            const int s = i % nst;
            const int use = i / nst;
            const long long e0 = clock64();
            if (use > 0) mbar_wait(&empty[s], (use - 1) & 1);
            w_empty += clock64() - e0;
            // lane 0: resolve the pending grab (advancing phases), prefetch the next
            int kind = -1, k = 0;
            if (lane == 0) {
                while (phase < 3) {
                    const int kd = order[phase];
                    if (pending < lim[kd]) {
                        kind = kd;
                        k = pending;
                        pending = atomicAdd(ctr[kd], 1);  // prefetch, same phase
                        break;
                    }
                    ++phase;
                    if (phase < 3) pending = atomicAdd(ctr[order[phase]], 1);
                }
            }
            kind = __shfl_sync(0xffffffffu, kind, 0);
            k = __shfl_sync(0xffffffffu, k, 0);
            SMeta m{};
            if (kind < 0) {
                if (lane == 0) {
                    m.t = -1;
                    meta[s] = m;
                    mbar_arrive(&full[s]);
                }
                break;
            }
            locate(kind, k, m);  // every lane (cheap, shared-memory tables)
            ++n_it[kind];
            float* dst = ring + s * SF;
            const unsigned bytes = static_cast<unsigned>((m.e - m.s) * 4);
            if (kind == IT_A && !xok) {
                if (lane == 0)
                    for (int q = 0; q < P; ++q)
                        if (q != R)
                            spin_until(pt.flags[R] + kXReadyKind * kMaxRanks + q, sa.xepoch, pt.error);
                xok = true;
            }
            if (kind == IT_B && lane == 0) {
                const long long b0 = clock64();
                spin_until(sa.tflag[R] + m.t, sa.tepoch, pt.error);
                w_b += clock64() - b0;
                fence_proxy_async();
            }
            const int nrows = kind == IT_A ? NS : (kind == IT_C ? NL : 1);
            if (lane == 0) {
                meta[s] = m;
                if (m.staged) mbar_arrive_tx(&full[s], bytes * (nrows + 1));
            }
            __syncwarp();
            if (m.staged) {
                if (lane < nrows) {
                    const float* src = kind == IT_A ? pt.xrow[lane] + m.s
                                     : kind == IT_C ? pt.xrow[R * NL + lane] + m.s
                                                    : pt.agg[R] + m.s;
                    bulk_g2s(dst + static_cast<size_t>(lane) * T, src, bytes, &full[s]);
                } else if (lane == nrows) {
                    bulk_g2s(dst + static_cast<size_t>(rowG) * T, g.G + m.s, bytes, &full[s]);
                }
            } else if (lane == 0) {
                mbar_arrive(&full[s]);
            }
        }
        if (lane == 0) {
            if (atomicAdd(g.sched + SCHED_SS_DONE, 1) == G - 1) {
                for (int j = 0; j < 3; ++j) atomicExch(ctr[j], 0);
                atomicExch(g.sched + SCHED_SS_DONE, 0);
            }
            if (dbg) {
                atomicAdd(dbg + 0, static_cast<unsigned long long>(w_empty));
                atomicAdd(dbg + 1, static_cast<unsigned long long>(w_b));
                for (int j = 0; j < 3; ++j) atomicAdd(dbg + 3 + j, static_cast<unsigned long long>(n_it[j]));
                atomicAdd(dbg + 6, static_cast<unsigned long long>(clock64() - p0));
                atomicAdd(dbg + 12, 1ull);
                atomicMax(dbg + 13, static_cast<unsigned long long>(clock64() - p0));
            }
        }
        return;
    }

    // ================= consumers =================
    const int ctid = tid;
    long long cw_full = 0, cw_proc = 0;
    for (int i = 0;; ++i) {
        const int s = i % nst;
        const long long f0 = clock64();
        mbar_wait(&full[s], (i / nst) & 1);
        const long long f1 = clock64();
        cw_full += f1 - f0;
        const SMeta m = meta[s];
        if (m.t < 0) break;
        const float* buf = ring + s * SF;
        const float* bufG = buf + static_cast<size_t>(rowG) * T;
        double acc = 0.0;
        if (m.staged) {
            const int nq = static_cast<int>((m.e - m.s) >> 2);
            for (int q = ctid; q < nq; q += CW * 32) {
                const uint64_t f = m.s + 4ull * q;
                const float4 go = *reinterpret_cast<const float4*>(bufG + 4 * q);
                if (m.kind == IT_A) {
                    float4 xs[NS];
#pragma unroll
                    for (int w = 0; w < NS; ++w)
                        xs[w] = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(w) * T + 4 * q);
                    float4 a;
                    agg4<NS>(ap, xs, a);
                    const float4 gn = make_float4(__fadd_rn(go.x, a.x), __fadd_rn(go.y, a.y),
                                                  __fadd_rn(go.z, a.z), __fadd_rn(go.w, a.w));
                    *reinterpret_cast<float4*>(g.G + f) = gn;
                    for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
                    for (int r = 0; r < P; ++r) *reinterpret_cast<float4*>(pt.agg[r] + f) = a;
                    acc = __dadd_rn(acc, pgp_term(a.x, gn.x));
                    acc = __dadd_rn(acc, pgp_term(a.y, gn.y));
                    acc = __dadd_rn(acc, pgp_term(a.z, gn.z));
                    acc = __dadd_rn(acc, pgp_term(a.w, gn.w));
                } else if (m.kind == IT_B) {
                    const float4 a = *reinterpret_cast<const float4*>(buf + 4 * q);
                    const float4 gn = make_float4(__fadd_rn(go.x, a.x), __fadd_rn(go.y, a.y),
                                                  __fadd_rn(go.z, a.z), __fadd_rn(go.w, a.w));
                    *reinterpret_cast<float4*>(g.G + f) = gn;
                    for (int w = 0; w < NL; ++w) st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f, gn);
                } else {
                    for (int w = 0; w < NL; ++w) {
                        float4 v = *reinterpret_cast<const float4*>(buf + static_cast<size_t>(w) * T + 4 * q);
                        if (ap.sgd) {
                            v.x = sgd_conv(ap.neg_lr, v.x);
                            v.y = sgd_conv(ap.neg_lr, v.y);
                            v.z = sgd_conv(ap.neg_lr, v.z);
                            v.w = sgd_conv(ap.neg_lr, v.w);
                        }
                        st_stream4(g.P + static_cast<uint64_t>(w) * g.ldP + f,
                                   make_float4(__fadd_rn(go.x, v.x), __fadd_rn(go.y, v.y),
                                               __fadd_rn(go.z, v.z), __fadd_rn(go.w, v.w)));
                    }
                }
            }
        } else {
            for (uint64_t f = m.s + ctid; f < m.e; f += CW * 32) {
                if (m.kind == IT_A) {
                    double sum = 0.0;
                    for (int w = 0; w < NS; ++w) {
                        float x = pt.xrow[w][f];
                        if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                        sum = agg_acc(sum, ap.w[w], x);
                    }
                    const float a = agg_finish(ap, sum);
                    const float gn = __fadd_rn(g.G[f], a);
                    g.G[f] = gn;
                    for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
                    for (int r = 0; r < P; ++r) pt.agg[r][f] = a;
                    acc = __dadd_rn(acc, pgp_term(a, gn));
                } else if (m.kind == IT_B) {
                    const float gn = __fadd_rn(g.G[f], __ldcg(pt.agg[R] + f));
                    g.G[f] = gn;
                    for (int w = 0; w < NL; ++w) g.P[static_cast<uint64_t>(w) * g.ldP + f] = gn;
                } else {
                    const float go = g.G[f];
                    for (int w = 0; w < NL; ++w) {
                        float x = pt.xrow[R * NL + w][f];
                        if (ap.sgd) x = sgd_conv(ap.neg_lr, x);
                        g.P[static_cast<uint64_t>(w) * g.ldP + f] = __fadd_rn(go, x);
                    }
                }
            }
        }
        cw_proc += clock64() - f1;
        if (m.kind == IT_A) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc = __dadd_rn(acc, __shfl_down_sync(0xffffffffu, acc, o));
            __syncwarp();
            if (lane == 0) {
                red[s * CW + warp] = acc;
                // lanes' stores -> (syncwarp) -> acq_rel CTA count -> the last
                // warp hands (tile, partial) to the publisher warp
                if (atom_add_acqrel_cta(&cnt[s], 1) == CW - 1) {
                    const volatile double* rv = red + s * CW;
                    double tot = 0.0;
                    for (int w = 0; w < CW; ++w) tot = __dadd_rn(tot, rv[w]);
                    cnt[s] = 0;
                    const int pos = atom_add_acqrel_cta(&qctl[0], 1);
                    while (pos - ld_acquire_cta_s32(&qctl[1]) >= kPubQ) __nanosleep(32);
                    PubEntry* e = pq + (pos % kPubQ);
                    e->tot = tot;
                    e->t = m.t;
                    st_release_cta_s32(&e->seq, pos + 1);
                }
                mbar_arrive(&empty[s]);
            }
        } else if (lane == 0) {
            mbar_arrive(&empty[s]);
        }
        __syncwarp();
    }
    if (lane == 0) atom_add_acqrel_cta(&qctl[2], 1);  // this consumer warp is done
    if (dbg && warp == 0 && lane == 0) {
        atomicAdd(dbg + 8, static_cast<unsigned long long>(cw_full));
        atomicAdd(dbg + 9, static_cast<unsigned long long>(cw_proc));
    }
}

constexpr int kStreamCW = 8;

size_t stream_smem_bytes(size_t ring_bytes, int L) {
    const size_t ctl = kMaxSt * (2 * sizeof(uint64_t) + sizeof(SMeta) + kStreamCW * sizeof(double) +
                                 sizeof(int)) +
                       kPubQ * sizeof(PubEntry) + 4 * sizeof(int);
    const size_t tab = static_cast<size_t>(L) * 16 + static_cast<size_t>(L + 1) * 4 * 3 +
                       static_cast<size_t>(L) * 4 * 2 + 64;
    return ring_bytes + ctl + tab;
}

// default ring: 2 exchange-tile slots
size_t stream_ring_bytes(int NS, int T) {
    static const int ks_env = [] {
        const char* v = std::getenv("OSP_SS_KS");
        return v && *v ? std::atoi(v) : 0;
    }();
    const int ks = ks_env >= 1 && ks_env <= 8 ? ks_env : 2;
    return static_cast<size_t>(ks) * (NS + 1) * T * sizeof(float);
}

template <int NS>
cudaError_t launch_ns(const GroupView& g, const AggParams& ap, const PeerTable& pt,
                      const StreamArgs& sa_in, cudaStream_t s) {
    auto kern = k_shard_stream<NS, kStreamCW>;
    StreamArgs sa = sa_in;
    sa.ring_bytes = stream_ring_bytes(NS, g.T);
    const size_t sm = stream_smem_bytes(sa.ring_bytes, g.L);
    cudaError_t e = cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sm));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, (kStreamCW + 2) * 32, sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    kern<<<sm_count() * per_sm, (kStreamCW + 2) * 32, sm, s>>>(g, ap, pt, sa);
    return cudaGetLastError();
}

}  // namespace

bool shard_stream_supported(int n_workers, int T, int L) {
    if (!(n_workers == 1 || n_workers == 2 || n_workers == 4 || n_workers == 8)) return false;
    if (T != 1024 && T != 2048) return false;
    return stream_smem_bytes(stream_ring_bytes(n_workers, T), L) <= 220 * 1024;
}

cudaError_t launch_shard_stream(const GroupView& g, const AggParams& ap, const PeerTable& pt,
                                const StreamArgs& sa, cudaStream_t s) {
    switch (ap.n) {
        case 1: return launch_ns<1>(g, ap, pt, sa, s);
        case 2: return launch_ns<2>(g, ap, pt, sa, s);
        case 4: return launch_ns<4>(g, ap, pt, sa, s);
        case 8: return launch_ns<8>(g, ap, pt, sa, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace osp
