// C-ABI of the sharded multi-GPU path (include/osp_c.h, "Shard" section).
//
// One process per GPU. Rank r hosts workers [r*N/P, (r+1)*N/P), a full replica
// of the global vector, and the PS shard of every stage's tile sequence. The
// push (reduce-scatter), fixed-order aggregation, pull (all-gather) and local
// apply of a stage run in ONE kernel (kernels/shard_x.cu) over CUDA-IPC peer
// mappings of the other ranks' delta rows, pull buffers, partials and flags;
// the cross-GPU ordering is per tile inside that kernel. The local state
// (G replica, worker rows, carry, PGP partials, GIB lists) is an osp_group with
// the rank's workers, so the stage-2 broadcast, the resolve and every read-back
// reuse the group code.

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "handles.h"

using namespace osp;

namespace {

constexpr uint32_t kMagic = 0x0700b200u;

// default sync form of the single-exchange stage 1 by world size: the chain
// at 2 ranks (ResNet-50 0.45-0.49 vs 0.54 ms, VGG-16 2.09-2.18 vs 2.47 ms with
// per-tile flags); at 4 ranks the last rank's 3-way aggregate fan-out makes it
// slower than the barrier form (0.73 vs 0.55 ms; profiles/r2_multi_gpu_notes.md)
int kChainDefault(int world) { return world == 2 ? 1 : 0; }

struct ShardHandle {
    uint32_t magic;
    int32_t rank, world, n_loc, deferred, chain;
    uint64_t M, L, NT, ldX, buf_stride;
    cudaIpcMemHandle_t hx, hagg, hpart, htflag, hready, hpre;
};
static_assert(sizeof(ShardHandle) <= OSP_SHARD_HANDLE_BYTES, "handle too large");

}  // namespace

struct osp_shard {
    osp_group* grp = nullptr;  // local state: rank's workers
    const osp_partition* part = nullptr;
    int world = 1, rank = 0, n_loc = 1, N = 1, n_chunks = 1;
    bool deferred = false;     // OSP_SHARD_DEFER_ICS (or no carry buffer): stage 2 exchanges
    AggParams ap_all{};        // every worker, global weights (aggregation)
    float* X = nullptr;        // [2][n_loc][ldX] local delta rows, IPC-exported
    uint64_t ldX = 0, buf_stride = 0;
    float* agg = nullptr;      // [ldX] pull buffer, IPC-exported (the group's agg_full)
    unsigned* tflag = nullptr; // [2][NT] per-tile ready flags (tile, chain), IPC-exported
    double* pre = nullptr;     // [ldX] chain form: this rank's fp64 running sums, IPC-exported
    unsigned* ready = nullptr; // [kMaxRanks] deltas-ready slots, IPC-exported
    unsigned* error = nullptr; // [1] local
    XArgs xa[2]{};             // per delta buffer
    std::vector<void*> opened; // peer mappings to close
    bool connected = false;
    unsigned iter = 0;         // iterations started (stage-1 launches) = tile-flag epoch
    bool s1_open = false;      // stage 1 issued, iteration not yet resolved
    // exchange-kernel shape (profiles/r2_multi_gpu_notes.md, 2 B200, ResNet-50):
    // role-split CTAs, flags published 4..8 per fence, B items 10 A items behind
    int lag = 10;              // OSP_SHARD_LAG: B items' due-time lag (A items)
    int pub_batch = 8, pub_min = 4;  // OSP_SHARD_PUB="max,min": flags per fence
    int split = 1;             // OSP_SHARD_SPLIT=0: every CTA takes every item kind
    int barrier = -1;          // OSP_SHARD_SYNC=tile|barrier|chain; -1: by world size
    bool chain = false;        // single-exchange stage 1 as a reduction chain (shard_chain.cu)
    bool chain_fence_gpu = false;  // OSP_SHARD_CHAIN_FENCE=gpu: diagnostics only (not a valid order)
    unsigned* ticket = nullptr;  // [1] local, phase-1 last-CTA counter
    unsigned done_epoch = 0;     // barrier-form launches so far (a stage-2 chunk is one)
    unsigned long long* dbg = nullptr;  // OSP_SHARD_DEBUG=1: kernel counters [16]
    uint64_t n_trace = 0;               // OSP_SHARD_DEBUG=2: chain timeline entries after them
};

extern "C" {

osp_status osp_shard_create(const osp_partition* part, const osp_shard_config* cfg,
                            const float* init_params, void* stream, osp_shard** out) {
    if (!out || !part || !cfg || !cfg->weights) return fail(OSP_ERR_INVALID, "null argument");
    *out = nullptr;
    if (cfg->world < 1 || cfg->world > kMaxRanks)
        return fail(OSP_ERR_INVALID, "world size must be in [1, " + std::to_string(kMaxRanks) + "]");
    if (cfg->rank < 0 || cfg->rank >= cfg->world) return fail(OSP_ERR_INVALID, "rank out of range");
    if (cfg->n_workers < 1 || cfg->n_workers > OSP_MAX_WORKERS)
        return fail(OSP_ERR_CONFIG, "worker count out of range");
    if (cfg->n_workers % cfg->world != 0)
        return fail(OSP_ERR_CONFIG, "workers must split evenly across ranks");
    if (cfg->flags & ~OSP_SHARD_DEFER_ICS) return fail(OSP_ERR_INVALID, "unknown osp_shard_config flags");
    for (int w = 0; w < cfg->n_workers; ++w)
        if (cfg->weights[w] <= 0) return fail(OSP_ERR_CONFIG, "subset weight must be positive");
    double tw = 0.0;
    for (int w = 0; w < cfg->n_workers; ++w) tw += cfg->weights[w];
    if (!(tw > 0.0)) return fail(OSP_ERR_PROTOCOL, "aggregation weights must sum > 0");
    // default 2048-element tiles (fewer per-tile flags for the same bytes,
    // measured), smaller when the ring and the layer tables would not fit
    uint32_t T = cfg->tile_elems;
    if (!T) {
        T = 2048u;
        while (T > 512u && !shard_x_supported(cfg->n_workers, static_cast<int>(T),
                                               static_cast<int>(part->counts.size())))
            T /= 2;
    }
    if (T < 512 || T > 4096 || (T & (T - 1)))
        return fail(OSP_ERR_INVALID, "shard tile_elems must be a power of two in [512, 4096]");
    if (!shard_x_supported(cfg->n_workers, static_cast<int>(T), static_cast<int>(part->counts.size())))
        return fail(OSP_ERR_INVALID, "shard exchange ring and layer tables exceed shared memory");

    auto* s = new osp_shard();
    s->part = part;
    s->world = cfg->world;
    s->rank = cfg->rank;
    s->N = cfg->n_workers;
    s->n_loc = cfg->n_workers / cfg->world;
    s->n_chunks = cfg->n_chunks;
    s->ap_all = make_agg_params(s->N, cfg->weights, cfg->sgd_lr);
    if (const char* lg = std::getenv("OSP_SHARD_LAG")) s->lag = std::max(0, std::atoi(lg));
    if (const char* pb = std::getenv("OSP_SHARD_PUB")) {
        int a = 0, b = 0;
        if (std::sscanf(pb, "%d,%d", &a, &b) == 2 && a >= 1 && b >= 1 && b <= a) {
            s->pub_batch = a;
            s->pub_min = b;
        }
    }
    if (const char* sp = std::getenv("OSP_SHARD_SPLIT")) s->split = std::atoi(sp) == 0 ? 0 : 1;
    int want_chain = -1;
    if (const char* sy = std::getenv("OSP_SHARD_SYNC")) {
        s->barrier = std::strcmp(sy, "barrier") == 0 ? 1 : std::strcmp(sy, "tile") == 0 ? 0 : -1;
        want_chain = std::strcmp(sy, "chain") == 0 ? 1 : s->barrier >= 0 ? 0 : -1;
    }
    // measured: per-tile flags win at 2 ranks, own-tiles-then-barrier at 4
    if (s->barrier < 0) s->barrier = cfg->world >= 4 ? 1 : 0;
    // the local group: default (TMA-staged, carry) so the stage-2 broadcast and
    // the overlapped resolve are the single-GPU kernels; no single-launch step
    osp_group_config gc{s->n_loc, cfg->weights + s->rank * s->n_loc, cfg->n_chunks, T, cfg->sgd_lr,
                        OSP_GROUP_NO_SMALL};
    osp_status st = osp_group_create(part, &gc, init_params, stream, &s->grp);
    if (st != OSP_OK) {
        delete s;
        return st;
    }
    s->deferred = (cfg->flags & OSP_SHARD_DEFER_ICS) || s->grp->v.C == nullptr;
    // the chain form runs the single-exchange stage 1 (the deferred-ICS stages
    // keep the exchange forms); default by world size (measured,
    // profiles/r2_multi_gpu_notes.md)
    if (want_chain < 0) want_chain = kChainDefault(cfg->world);
    if (const char* cf = std::getenv("OSP_SHARD_CHAIN_FENCE")) s->chain_fence_gpu = std::strcmp(cf, "gpu") == 0;
    s->chain = want_chain == 1 && !s->deferred && cfg->world >= 2 &&
               shard_chain_supported(s->n_loc, static_cast<int>(T), static_cast<int>(part->counts.size()));
    const uint64_t M = part->total;
    s->ldX = (M + 3) & ~uint64_t(3);
    s->buf_stride = s->ldX * s->n_loc;
    const uint64_t NT = static_cast<uint64_t>(s->grp->v.NT);
    cudaError_t e = cudaMalloc(&s->X, 2 * s->buf_stride * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&s->agg, s->ldX * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&s->tflag, 2 * std::max<uint64_t>(NT, 1) * sizeof(unsigned));
    if (e == cudaSuccess && s->chain) e = cudaMalloc(&s->pre, s->ldX * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&s->ready, 2 * kMaxRanks * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&s->ticket, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(s->ticket, 0, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&s->error, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(s->X, 0, 2 * s->buf_stride * sizeof(float));
    if (e == cudaSuccess) e = cudaMemset(s->agg, 0, s->ldX * sizeof(float));
    if (e == cudaSuccess) e = cudaMemset(s->tflag, 0, 2 * std::max<uint64_t>(NT, 1) * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(s->ready, 0, 2 * kMaxRanks * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(s->error, 0, sizeof(unsigned));
    if (const char* d = std::getenv("OSP_SHARD_DEBUG"); d && (d[0] == '1' || d[0] == '2')) {
        // '2' adds the chain form's per-tile timeline [8][NT] after the counters
        s->n_trace = d[0] == '2' ? 8 * NT : 0;
        const size_t n = 16 + s->n_trace;
        if (e == cudaSuccess) e = cudaMalloc(&s->dbg, n * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMemset(s->dbg, 0, n * sizeof(unsigned long long));
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        osp_shard_destroy(s);
        return cuda_fail(e, "shard buffers");
    }
    s->grp->v.agg_full = s->agg;  // the resolve's exact fallback reads the applied aggregate
    *out = s;
    return OSP_OK;
}

void osp_shard_destroy(osp_shard* s) {
    if (!s) return;
    cudaDeviceSynchronize();
    for (void* p : s->opened) cudaIpcCloseMemHandle(p);
    if (s->X) cudaFree(s->X);
    if (s->agg) cudaFree(s->agg);
    if (s->tflag) cudaFree(s->tflag);
    if (s->pre) cudaFree(s->pre);
    if (s->ready) cudaFree(s->ready);
    if (s->error) cudaFree(s->error);
    if (s->dbg) cudaFree(s->dbg);
    if (s->ticket) cudaFree(s->ticket);
    if (s->grp) osp_group_destroy(s->grp);
    delete s;
}

uint64_t osp_shard_handle_size(void) { return OSP_SHARD_HANDLE_BYTES; }

osp_status osp_shard_export(osp_shard* s, uint8_t* handle) {
    if (!s || !handle) return fail(OSP_ERR_INVALID, "null argument");
    ShardHandle h{};
    h.magic = kMagic;
    h.rank = s->rank;
    h.world = s->world;
    h.n_loc = s->n_loc;
    h.deferred = s->deferred ? 1 : 0;
    h.chain = s->chain ? 1 : 0;
    h.M = s->part->total;
    h.L = s->part->counts.size();
    h.NT = static_cast<uint64_t>(s->grp->v.NT);
    h.ldX = s->ldX;
    h.buf_stride = s->buf_stride;
    OSP_CUDA(cudaIpcGetMemHandle(&h.hx, s->X));
    OSP_CUDA(cudaIpcGetMemHandle(&h.hagg, s->agg));
    OSP_CUDA(cudaIpcGetMemHandle(&h.hpart, s->grp->v.partials));
    OSP_CUDA(cudaIpcGetMemHandle(&h.htflag, s->tflag));
    OSP_CUDA(cudaIpcGetMemHandle(&h.hready, s->ready));
    if (s->chain) OSP_CUDA(cudaIpcGetMemHandle(&h.hpre, s->pre));
    std::memset(handle, 0, OSP_SHARD_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof h);
    return OSP_OK;
}

osp_status osp_shard_connect(osp_shard* s, const uint8_t* handles) {
    if (!s || !handles) return fail(OSP_ERR_INVALID, "null argument");
    if (s->connected) return fail(OSP_ERR_PROTOCOL, "shard already connected");
    std::vector<const float*> xbase(s->world);
    XArgs base{};
    for (int q = 0; q < s->world; ++q) {
        ShardHandle h;
        std::memcpy(&h, handles + static_cast<size_t>(q) * OSP_SHARD_HANDLE_BYTES, sizeof h);
        if (h.magic != kMagic || h.rank != q || h.world != s->world || h.n_loc != s->n_loc ||
            h.M != s->part->total || h.L != s->part->counts.size() ||
            h.NT != static_cast<uint64_t>(s->grp->v.NT) || h.ldX != s->ldX ||
            h.buf_stride != s->buf_stride || h.deferred != (s->deferred ? 1 : 0) ||
            h.chain != (s->chain ? 1 : 0))
            return fail(OSP_ERR_CONFIG, "rank " + std::to_string(q) +
                                            " exported an incompatible shard (partition, tiles, "
                                            "worker split, mode, sync form or world size differ)");
        if (q == s->rank) {
            xbase[q] = s->X;
            base.agg[q] = s->agg;
            base.part[q] = s->grp->v.partials;
            base.tflag[q] = s->tflag;
            base.ready[q] = s->ready;
            base.pre[q] = s->pre;
            continue;
        }
        void* p[6] = {};
        const cudaIpcMemHandle_t* hs[6] = {&h.hx, &h.hagg, &h.hpart, &h.htflag, &h.hready, &h.hpre};
        for (int k = 0; k < (s->chain ? 6 : 5); ++k) {
            OSP_CUDA(cudaIpcOpenMemHandle(&p[k], *hs[k], cudaIpcMemLazyEnablePeerAccess));
            s->opened.push_back(p[k]);
        }
        xbase[q] = static_cast<const float*>(p[0]);
        base.agg[q] = static_cast<float*>(p[1]);
        base.part[q] = static_cast<double*>(p[2]);
        base.tflag[q] = static_cast<unsigned*>(p[3]);
        base.ready[q] = static_cast<unsigned*>(p[4]);
        base.pre[q] = static_cast<double*>(p[5]);
    }
    base.error = s->error;
    base.world = s->world;
    base.rank = s->rank;
    base.n_loc = s->n_loc;
    base.slot_rows = x_slot_rows(s->N);
    base.lag = s->lag;
    base.pub_batch = s->pub_batch;
    base.pub_min = s->pub_min;
    base.split = s->split;
    base.chain_lead = 4;
    if (const char* cl = std::getenv("OSP_SHARD_CHAIN_LEAD")) base.chain_lead = std::max(0, std::atoi(cl));
    // the last rank stores the aggregate into every rank's pull buffer (NVLink
    // stores, 1 -> 0) instead of the others pulling it: its read requests no
    // longer share the link carrying the running sums (0.433 vs 0.441 ms,
    // VGG-16 1.90 vs 1.95; OSP_SHARD_CHAIN_PUSHAGG=0 pulls)
    base.chain_pushagg = 1;
    if (const char* pa = std::getenv("OSP_SHARD_CHAIN_PUSHAGG")) base.chain_pushagg = std::atoi(pa) ? 1 : 0;
    base.ticket = s->ticket;
    base.dbg = s->dbg;
    base.trace = s->n_trace ? s->dbg + 16 : nullptr;
    for (int b = 0; b < 2; ++b) {
        XArgs& xa = s->xa[b];
        xa = base;
        bool vec = (s->ldX % 4 == 0) && (s->grp->v.ldP % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(s->grp->v.G) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(s->grp->v.P) % 16 == 0) &&
                   (!s->grp->v.C || reinterpret_cast<uintptr_t>(s->grp->v.C) % 16 == 0);
        for (int w = 0; w < s->N; ++w) {
            const int q = w / s->n_loc, i = w % s->n_loc;
            xa.xrow[w] = xbase[q] + b * s->buf_stride + static_cast<uint64_t>(i) * s->ldX;
            vec = vec && (reinterpret_cast<uintptr_t>(xa.xrow[w]) % 16 == 0);
        }
        for (int q = 0; q < s->world; ++q)
            vec = vec && (reinterpret_cast<uintptr_t>(xa.agg[q]) % 16 == 0) &&
                  (reinterpret_cast<uintptr_t>(xa.pre[q]) % 32 == 0);
        xa.vec = vec ? 1 : 0;
    }
    // chain form pulling the aggregate: it lives on the last rank only (the
    // others' APPLY items read it there), so their resolve's exact fallback
    // reads it there; pushed, every rank holds it
    if (s->chain && s->rank != s->world - 1 && !base.chain_pushagg)
        s->grp->v.agg_full = base.agg[s->world - 1];
    s->connected = true;
    return OSP_OK;
}

float* osp_shard_deltas(osp_shard* s, int buf, uint64_t* ld) {
    if (!s || buf < 0 || buf > 1) return nullptr;
    if (ld) *ld = s->ldX;
    return s->X + buf * s->buf_stride;
}

osp_group* osp_shard_group(osp_shard* s) { return s ? s->grp : nullptr; }

int osp_shard_deferred_ics(const osp_shard* s) { return s && s->deferred ? 1 : 0; }

int osp_shard_sync_form(const osp_shard* s) {
    if (!s) return -1;
    return s->chain ? 2 : s->barrier ? 1 : 0;
}

static osp_status check_ready(osp_shard* s, int buf) {
    if (!s) return fail(OSP_ERR_INVALID, "null shard");
    if (!s->connected) return fail(OSP_ERR_PROTOCOL, "shard not connected to its peers");
    if (buf < 0 || buf > 1) return fail(OSP_ERR_INVALID, "delta buffer index must be 0 or 1");
    return OSP_OK;
}

// diagnostics: OSP_SHARD_SOLO=apply makes osp_shard_solo_agg time the chain
// form's APPLY items alone (else its PRE / FIN items alone)
static bool stage1_solo_apply() {
    const char* e = std::getenv("OSP_SHARD_SOLO");
    return e && std::strcmp(e, "apply") == 0;
}

static cudaError_t launch_x(osp_shard* s, int buf, int mode, int c0, int c1, int solo,
                            cudaStream_t st) {
    XArgs xa = s->xa[buf];
    xa.epoch = s->iter;
    xa.mode = mode;
    xa.c0 = c0;
    xa.c1 = c1;
    xa.solo = solo;
    if (s->chain && mode == XM_SINGLE) {
        if (!solo && s->chain_fence_gpu) xa.solo = 2;
        if (solo && stage1_solo_apply()) xa.solo = 3;
        return launch_shard_chain(s->grp->v, s->ap_all, xa, st);
    }
    if (solo || !s->barrier) {
        xa.phase = 0;
        return launch_shard_x(s->grp->v, s->ap_all, xa, st);
    }
    // barrier form: own tiles (then a cross-GPU signal), then the peers' tiles;
    // every CTA takes both kinds (no role split)
    xa.split = 0;
    xa.done_epoch = ++s->done_epoch;
    xa.phase = 1;
    cudaError_t e = launch_shard_x(s->grp->v, s->ap_all, xa, st);
    if (e != cudaSuccess) return e;
    xa.phase = 2;
    return launch_shard_peer_apply(s->grp->v, s->ap_all, xa, st);
}

// stage 1: SINGLE mode exchanges every tile (the carry keeps the deferred
// layers' aggregate), deferred-ICS mode the barrier layers (local estimates for
// the rest)
static cudaError_t stage1_kernels(osp_shard* s, int buf, cudaStream_t st) {
    s->iter += 1;
    return launch_x(s, buf, s->deferred ? XM_RS : XM_SINGLE, 0, 0, 0, st);
}

static cudaError_t stage2_kernels(osp_shard* s, int buf, int c0, int c1, cudaStream_t st) {
    osp_group* g = s->grp;
    if (s->deferred) return launch_x(s, buf, XM_ICS, c0, c1, 0, st);
    return launch_stage2_tma(g->v, g->ap, s->X + buf * s->buf_stride, s->ldX, c0, c1, st, 0);
}

osp_status osp_shard_stage1(osp_shard* s, int buf, void* stream) {
    OSP_RANGE("osp_shard_stage1");
    OSP_TRY(check_ready(s, buf));
    OSP_CUDA(stage1_kernels(s, buf, as_stream(stream)));
    s->s1_open = true;
    return OSP_OK;
}

osp_status osp_shard_stage2(osp_shard* s, int c0, int c1, int buf, void* stream) {
    OSP_RANGE("osp_shard_stage2");
    OSP_TRY(check_ready(s, buf));
    if (c0 < 0 || c1 > s->n_chunks || c0 > c1) return fail(OSP_ERR_INVALID, "chunk range");
    if (!s->s1_open) return fail(OSP_ERR_PROTOCOL, "stage 2 before stage 1 of this iteration");
    OSP_CUDA(stage2_kernels(s, buf, c0, c1, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_shard_resolve(osp_shard* s, int buf, void* stream) {
    OSP_RANGE("osp_shard_resolve");
    OSP_TRY(check_ready(s, buf));
    osp_group* g = s->grp;
    OSP_CUDA(launch_resolve(g->v, g->ap, s->X + buf * s->buf_stride, s->ldX, as_stream(stream)));
    s->s1_open = false;
    return OSP_OK;
}

// Whole iteration: stage 1, then (SINGLE) the resolve with the local stage-2
// broadcast beside it (joined on the device, as osp_group_stage2_resolve), or
// (deferred ICS) the stage-2 exchange of every chunk and the resolve.
osp_status osp_shard_step(osp_shard* s, int buf, void* stream) {
    OSP_RANGE("osp_shard_step");
    OSP_TRY(check_ready(s, buf));
    cudaStream_t st = as_stream(stream);
    osp_group* g = s->grp;
    float* Xb = s->X + buf * s->buf_stride;
    OSP_CUDA(stage1_kernels(s, buf, st));
    if (s->deferred) {
        OSP_CUDA(launch_x(s, buf, XM_ICS, 0, s->n_chunks, 0, st));
        OSP_CUDA(launch_resolve(g->v, g->ap, Xb, s->ldX, st));
    } else {
        OSP_CUDA(launch_resolve(g->v, g->ap, Xb, s->ldX, st));
        OSP_CUDA(launch_stage2_tma(g->v, g->ap, Xb, s->ldX, 0, s->n_chunks, st, 1));
    }
    s->s1_open = false;
    return OSP_OK;
}

osp_status osp_shard_solo_agg(osp_shard* s, int stage, int buf, void* stream) {
    OSP_TRY(check_ready(s, buf));
    if (stage != 1 && stage != 2) return fail(OSP_ERR_INVALID, "stage must be 1 or 2");
    if (stage == 2 && !s->deferred)
        return fail(OSP_ERR_PROTOCOL, "stage 2 exchanges nothing in single-exchange mode");
    const int mode = stage == 2 ? XM_ICS : (s->deferred ? XM_RS : XM_SINGLE);
    OSP_CUDA(launch_x(s, buf, mode, 0, s->n_chunks, 1, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_shard_profile(osp_shard* s, int buf, float* ms, void* stream) {
    OSP_TRY(check_ready(s, buf));
    if (!ms) return fail(OSP_ERR_INVALID, "null output");
    cudaStream_t st = as_stream(stream);
    osp_group* g = s->grp;
    float* Xb = s->X + buf * s->buf_stride;
    cudaEvent_t ev[4];
    for (auto& e : ev) OSP_CUDA(cudaEventCreate(&e));
    auto run = [&]() -> cudaError_t {
        cudaError_t e;
        for (int i = 0; i < 8; ++i) ms[i] = 0.f;
        if ((e = cudaEventRecord(ev[0], st)) != cudaSuccess) return e;
        if ((e = stage1_kernels(s, buf, st)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ev[1], st)) != cudaSuccess) return e;
        if ((e = stage2_kernels(s, buf, 0, s->n_chunks, st)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ev[2], st)) != cudaSuccess) return e;
        if ((e = launch_resolve(g->v, g->ap, Xb, s->ldX, st)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ev[3], st)) != cudaSuccess) return e;
        if ((e = cudaEventSynchronize(ev[3])) != cudaSuccess) return e;
        for (int i = 0; i < 3; ++i)
            if ((e = cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1])) != cudaSuccess) return e;
        return cudaSuccess;
    };
    cudaError_t e = run();
    s->s1_open = false;
    for (auto& x : ev) cudaEventDestroy(x);
    if (e != cudaSuccess) return cuda_fail(e, "shard profile");
    return OSP_OK;
}

osp_status osp_synth_deltas_range(uint64_t seed, int worker0, int n_workers, uint64_t iteration,
                                  uint64_t n, float* out, uint64_t ld, void* stream) {
    if (worker0 < 0 || n_workers < 0 || n_workers > 65535)
        return fail(OSP_ERR_INVALID, "bad worker range");
    if (ld < n) return fail(OSP_ERR_SHAPE, "ld smaller than the vector length");
    OSP_CUDA(launch_synth(seed, n_workers, iteration, 0, n, out, ld,
                          static_cast<uint64_t>(worker0), as_stream(stream)));
    return OSP_OK;
}

int osp_shard_debug_counters(osp_shard* s, unsigned long long* out16) {
    if (!s || !s->dbg || !out16) return 0;
    if (cudaMemcpy(out16, s->dbg, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) !=
        cudaSuccess)
        return 0;
    cudaMemset(s->dbg, 0, 16 * sizeof(unsigned long long));
    return 1;
}

uint64_t osp_shard_debug_trace(osp_shard* s, unsigned long long* out, uint64_t n) {
    if (!s || !s->n_trace) return 0;
    if (!out) return s->n_trace;
    const uint64_t k = std::min(n, s->n_trace);
    if (cudaMemcpy(out, s->dbg + 16, k * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    return k;
}

osp_status osp_shard_check(osp_shard* s, void* stream) {
    if (!s) return fail(OSP_ERR_INVALID, "null shard");
    unsigned err = 0;
    cudaStream_t st = as_stream(stream);
    OSP_CUDA(cudaMemcpyAsync(&err, s->error, sizeof err, cudaMemcpyDeviceToHost, st));
    OSP_CUDA(cudaStreamSynchronize(st));
    if (err) return fail(OSP_ERR_PROTOCOL, "cross-GPU wait timed out (a peer did not arrive)");
    return OSP_OK;
}

}  // extern "C"
