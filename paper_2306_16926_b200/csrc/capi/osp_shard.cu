// C-ABI of the sharded multi-GPU path (include/osp_c.h, "Shard" section).
//
// One process per GPU. Rank r hosts workers [r*N/P, (r+1)*N/P), a full replica
// of the global vector, and the PS shard of every stage's tile sequence. The
// push (reduce-scatter) and the pull (all-gather) are fused into k_shard_agg
// over CUDA-IPC peer mappings of the other ranks' delta rows and agg buffers;
// cross-GPU ordering uses epoch flags on peer-mapped slots that the kernels
// signal and wait on themselves (XSync in stage.cu). The local state
// (G replica, worker rows, PGP partials, GIB lists) is an osp_group with the
// rank's workers, so resolve and every read-back reuse the group code.

#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "handles.h"

using namespace osp;

namespace {

constexpr uint32_t kMagic = 0x0500b200u;

struct ShardHandle {
    uint32_t magic;
    int32_t rank, world, n_loc;
    uint64_t M, L, ldX, buf_stride;
    cudaIpcMemHandle_t hx, hagg, hflags;
    int32_t stream;      // streaming kernel in use
    uint64_t NT;         // tiles (streaming mode)
    cudaIpcMemHandle_t htf, hpart;
};
static_assert(sizeof(ShardHandle) <= OSP_SHARD_HANDLE_BYTES, "handle too large");

}  // namespace

struct osp_shard {
    osp_group* grp = nullptr;  // local state: rank's workers
    const osp_partition* part = nullptr;
    int world = 1, rank = 0, n_loc = 1, N = 1, n_chunks = 1;
    AggParams ap_all{};        // every worker, global weights (aggregation)
    AggParams ap_loc{};        // local workers (sgd conversion on the local estimate)
    float* X = nullptr;        // [2][n_loc][ldX] local delta rows, IPC-exported
    uint64_t ldX = 0, buf_stride = 0;
    float* agg = nullptr;      // [ldX] agg_full, IPC-exported
    unsigned* flags = nullptr; // [kBarKinds][kMaxRanks], IPC-exported
    unsigned* error = nullptr; // [1] local
    PeerTable pt[2]{};         // per delta buffer
    std::vector<void*> opened; // peer mappings to close
    bool connected = false;
    // streaming mode (kernels/shard_stream.cu)
    bool stream = false;
    uint64_t NT = 0;
    unsigned* tflag = nullptr; // [NT] per-tile ready flags, IPC-exported
    double* pbuf = nullptr;    // [NT] per-tile PGP partials (the group's), IPC-exported
    StreamArgs sa{};           // peer tables of tflag/pbuf
    int vec[2]{};              // per delta buffer: 16-byte aligned rows
    unsigned iter = 0;         // iterations started (stage-1 launches)
    unsigned xep[4] = {0, 0, 0, 0};  // barrier mode: epochs of the in-kernel cross-GPU syncs
                                     // (kinds 0, 1, 2 and 4)
    bool pipe = false;               // pipelined step (OSP_SHARD_PIPE, barrier mode)
    unsigned long long* dbg = nullptr;  // [2 stages][3 roles][16] diagnostics counters (OSP_SS_DEBUG=1)
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
    for (int w = 0; w < cfg->n_workers; ++w)
        if (cfg->weights[w] <= 0) return fail(OSP_ERR_CONFIG, "subset weight must be positive");
    double tw = 0.0;
    for (int w = 0; w < cfg->n_workers; ++w) tw += cfg->weights[w];
    if (!(tw > 0.0)) return fail(OSP_ERR_PROTOCOL, "aggregation weights must sum > 0");

    auto* s = new osp_shard();
    s->part = part;
    s->world = cfg->world;
    s->rank = cfg->rank;
    s->N = cfg->n_workers;
    s->n_loc = cfg->n_workers / cfg->world;
    s->n_chunks = cfg->n_chunks;
    s->ap_all = make_agg_params(s->N, cfg->weights, cfg->sgd_lr);
    s->ap_loc = make_agg_params(s->n_loc, cfg->weights + s->rank * s->n_loc, cfg->sgd_lr);
    // streaming kernel (opt-in: OSP_SHARD_STREAM=1) when the shape supports it;
    // barrier mode is the default (faster on the measured configurations, see
    // DESIGN.md "Multi-GPU")
    const char* se = std::getenv("OSP_SHARD_STREAM");
    const uint32_t Ts = cfg->tile_elems ? cfg->tile_elems : 2048u;
    s->stream = (se && se[0] == '1') &&
                shard_stream_supported(s->N, static_cast<int>(Ts), static_cast<int>(part->counts.size()));
    const char* pe = std::getenv("OSP_SHARD_PIPE");
    s->pipe = !s->stream && pe && pe[0] == '1';
    osp_group_config gc{s->n_loc, cfg->weights + s->rank * s->n_loc, cfg->n_chunks,
                        s->stream ? Ts : cfg->tile_elems, cfg->sgd_lr, OSP_GROUP_REGISTER};
    osp_status st = osp_group_create(part, &gc, init_params, stream, &s->grp);
    if (st != OSP_OK) {
        delete s;
        return st;
    }
    const uint64_t M = part->total;
    s->ldX = (M + 3) & ~uint64_t(3);
    s->buf_stride = s->ldX * s->n_loc;
    cudaError_t e = cudaMalloc(&s->X, 2 * s->buf_stride * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&s->agg, s->ldX * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&s->flags, kBarKinds * kMaxRanks * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMalloc(&s->error, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(s->X, 0, 2 * s->buf_stride * sizeof(float));
    if (e == cudaSuccess) e = cudaMemset(s->agg, 0, s->ldX * sizeof(float));
    if (e == cudaSuccess) e = cudaMemset(s->flags, 0, kBarKinds * kMaxRanks * sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(s->error, 0, sizeof(unsigned));
    if (s->stream) {
        const char* de = std::getenv("OSP_SS_DEBUG");
        if (de && de[0] == '1') {
            if (e == cudaSuccess) e = cudaMalloc(&s->dbg, 96 * sizeof(unsigned long long));
            if (e == cudaSuccess) e = cudaMemset(s->dbg, 0, 96 * sizeof(unsigned long long));
        }
        s->NT = static_cast<uint64_t>(s->grp->v.NT);
        const uint64_t nt = s->NT ? s->NT : 1;
        if (e == cudaSuccess) e = cudaMalloc(&s->tflag, nt * sizeof(unsigned));
        if (e == cudaSuccess) e = cudaMalloc(&s->pbuf, nt * sizeof(double));
        if (e == cudaSuccess) e = cudaMemset(s->tflag, 0, nt * sizeof(unsigned));
        if (e == cudaSuccess) e = cudaMemset(s->pbuf, 0, nt * sizeof(double));
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        osp_shard_destroy(s);
        return cuda_fail(e, "shard buffers");
    }
    s->grp->v.agg_full = s->agg;
    if (s->stream) s->grp->v.partials = s->pbuf;  // resolve reads the exchanged partials
    *out = s;
    return OSP_OK;
}

void osp_shard_destroy(osp_shard* s) {
    if (!s) return;
    cudaDeviceSynchronize();
    for (void* p : s->opened) cudaIpcCloseMemHandle(p);
    if (s->X) cudaFree(s->X);
    if (s->agg) cudaFree(s->agg);
    if (s->flags) cudaFree(s->flags);
    if (s->error) cudaFree(s->error);
    if (s->tflag) cudaFree(s->tflag);
    if (s->dbg) cudaFree(s->dbg);
    if (s->pbuf) cudaFree(s->pbuf);
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
    h.M = s->part->total;
    h.L = s->part->counts.size();
    h.ldX = s->ldX;
    h.buf_stride = s->buf_stride;
    OSP_CUDA(cudaIpcGetMemHandle(&h.hx, s->X));
    OSP_CUDA(cudaIpcGetMemHandle(&h.hagg, s->agg));
    OSP_CUDA(cudaIpcGetMemHandle(&h.hflags, s->flags));
    h.stream = s->stream ? 1 : 0;
    h.NT = s->NT;
    if (s->stream) {
        OSP_CUDA(cudaIpcGetMemHandle(&h.htf, s->tflag));
        OSP_CUDA(cudaIpcGetMemHandle(&h.hpart, s->pbuf));
    }
    std::memset(handle, 0, OSP_SHARD_HANDLE_BYTES);
    std::memcpy(handle, &h, sizeof h);
    return OSP_OK;
}

osp_status osp_shard_connect(osp_shard* s, const uint8_t* handles) {
    if (!s || !handles) return fail(OSP_ERR_INVALID, "null argument");
    if (s->connected) return fail(OSP_ERR_PROTOCOL, "shard already connected");
    std::vector<const float*> xbase(s->world);
    std::vector<float*> aggs(s->world);
    std::vector<unsigned*> flags(s->world);
    for (int q = 0; q < s->world; ++q) {
        ShardHandle h;
        std::memcpy(&h, handles + static_cast<size_t>(q) * OSP_SHARD_HANDLE_BYTES, sizeof h);
        if (h.magic != kMagic || h.rank != q || h.world != s->world || h.n_loc != s->n_loc ||
            h.M != s->part->total || h.L != s->part->counts.size() || h.ldX != s->ldX ||
            h.buf_stride != s->buf_stride || h.stream != (s->stream ? 1 : 0) || h.NT != s->NT)
            return fail(OSP_ERR_CONFIG, "rank " + std::to_string(q) +
                                            " exported an incompatible shard (partition, worker "
                                            "split or world size differ)");
        if (q == s->rank) {
            xbase[q] = s->X;
            aggs[q] = s->agg;
            flags[q] = s->flags;
            s->sa.tflag[q] = s->tflag;
            s->sa.part[q] = s->pbuf;
            continue;
        }
        if (s->stream) {
            void *pt = nullptr, *pp = nullptr;
            OSP_CUDA(cudaIpcOpenMemHandle(&pt, h.htf, cudaIpcMemLazyEnablePeerAccess));
            s->opened.push_back(pt);
            OSP_CUDA(cudaIpcOpenMemHandle(&pp, h.hpart, cudaIpcMemLazyEnablePeerAccess));
            s->opened.push_back(pp);
            s->sa.tflag[q] = static_cast<unsigned*>(pt);
            s->sa.part[q] = static_cast<double*>(pp);
        }
        void *px = nullptr, *pa = nullptr, *pf = nullptr;
        OSP_CUDA(cudaIpcOpenMemHandle(&px, h.hx, cudaIpcMemLazyEnablePeerAccess));
        s->opened.push_back(px);
        OSP_CUDA(cudaIpcOpenMemHandle(&pa, h.hagg, cudaIpcMemLazyEnablePeerAccess));
        s->opened.push_back(pa);
        OSP_CUDA(cudaIpcOpenMemHandle(&pf, h.hflags, cudaIpcMemLazyEnablePeerAccess));
        s->opened.push_back(pf);
        xbase[q] = static_cast<const float*>(px);
        aggs[q] = static_cast<float*>(pa);
        flags[q] = static_cast<unsigned*>(pf);
    }
    for (int b = 0; b < 2; ++b) {
        PeerTable& pt = s->pt[b];
        pt = PeerTable{};
        pt.world = s->world;
        pt.rank = s->rank;
        pt.n_loc = s->n_loc;
        const char* lm = std::getenv("OSP_PEER_LOAD");
        pt.ldmode = lm ? std::atoi(lm) : 2;  // default-cached peer loads measured fastest
        for (int w = 0; w < s->N; ++w) {
            const int q = w / s->n_loc, i = w % s->n_loc;
            pt.xrow[w] = xbase[q] + b * s->buf_stride + static_cast<uint64_t>(i) * s->ldX;
        }
        for (int q = 0; q < s->world; ++q) {
            pt.agg[q] = aggs[q];
            pt.flags[q] = flags[q];
        }
        pt.error = s->error;
        bool vec = (s->ldX % 4 == 0) && (s->grp->v.ldP % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(s->grp->v.G) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(s->grp->v.P) % 16 == 0);
        for (int w = 0; w < s->N; ++w) vec = vec && (reinterpret_cast<uintptr_t>(pt.xrow[w]) % 16 == 0);
        for (int q = 0; q < s->world; ++q) vec = vec && (reinterpret_cast<uintptr_t>(pt.agg[q]) % 16 == 0);
        s->vec[b] = vec ? 1 : 0;
    }
    s->connected = true;
    return OSP_OK;
}

float* osp_shard_deltas(osp_shard* s, int buf, uint64_t* ld) {
    if (!s || buf < 0 || buf > 1) return nullptr;
    if (ld) *ld = s->ldX;
    return s->X + buf * s->buf_stride;
}

osp_group* osp_shard_group(osp_shard* s) { return s ? s->grp : nullptr; }

static osp_status check_ready(osp_shard* s, int buf) {
    if (!s) return fail(OSP_ERR_INVALID, "null shard");
    if (!s->connected) return fail(OSP_ERR_PROTOCOL, "shard not connected to its peers");
    if (buf < 0 || buf > 1) return fail(OSP_ERR_INVALID, "delta buffer index must be 0 or 1");
    return OSP_OK;
}

static cudaError_t stream_stage(osp_shard* s, int buf, int stage, int c0, int c1, cudaStream_t st) {
    StreamArgs a = s->sa;
    a.stage = stage;
    a.c0 = c0;
    a.c1 = c1;
    a.tepoch = 2u * s->iter + static_cast<unsigned>(stage) - 2u;
    a.xepoch = s->iter;
    a.vec = s->vec[buf];
    a.dbg = s->dbg ? s->dbg + (stage - 1) * 48 : nullptr;
    return launch_shard_stream(s->grp->v, s->ap_all, s->pt[buf], a, st);
}

static XSync sync_wait(int kind, unsigned ep) {
    XSync y;
    y.wait = kind;
    y.ep_wait = ep;
    return y;
}

static XSync sync_signal_end(int kind, unsigned ep) {
    XSync y;
    y.signal_end = kind;
    y.ep_end = ep;
    return y;
}

// agg1: announce "deltas ready, previous iteration done" and wait for every
// peer's announcement before touching peer memory; signal kind 1 at the end
static XSync sync_agg1(const osp_shard* s) {
    XSync y;
    y.signal_start = 0;
    y.ep_start = s->xep[0];
    y.wait = 0;
    y.ep_wait = s->xep[0];
    y.signal_end = 1;
    y.ep_end = s->xep[1];
    return y;
}

// Barrier-mode kernels of one step (no resolve); ev (optional) gets 4 records:
// before agg1, before the fused launch, before apply2, after apply2.
static cudaError_t barrier_step_kernels(osp_shard* s, int buf, cudaStream_t st,
                                        cudaEvent_t* ev = nullptr) {
    osp_group* g = s->grp;
    float* Xb = s->X + buf * s->buf_stride;
    ++s->xep[0];
    ++s->xep[1];
    ++s->xep[2];
    cudaError_t e;
    if (s->pipe) {
        // agg1 (first half of the RS exchange) -> [apply: RS first half + local
        // estimates || agg: RS second half] -> [apply: RS second half || agg:
        // ICS] -> apply2; cross-GPU kinds 1, 4, 2 in that order
        ++s->xep[3];
        if (ev && (e = cudaEventRecord(ev[0], st)) != cudaSuccess) return e;
        if ((e = launch_shard_agg(g->v, s->ap_all, s->pt[buf], 1, 0, 0, g->grid, sync_agg1(s), st,
                                  1)) != cudaSuccess)
            return e;
        if (ev && (e = cudaEventRecord(ev[1], st)) != cudaSuccess) return e;
        XSync ya = sync_wait(1, s->xep[1]);
        ya.signal_end = 4;
        ya.ep_end = s->xep[3];
        FusedLists la;
        la.apply_mode = 1;
        la.agg_stage = 1;
        la.agg_part = 2;
        if ((e = launch_shard_fused(g->v, s->ap_all, s->ap_loc, s->pt[buf], Xb, s->ldX, 0, 0, g->grid,
                                    ya, st, la)) != cudaSuccess)
            return e;
        XSync yb = sync_wait(4, s->xep[3]);
        yb.signal_end = 2;
        yb.ep_end = s->xep[2];
        FusedLists lb;
        lb.apply_mode = 2;
        lb.agg_stage = 2;
        if ((e = launch_shard_fused(g->v, s->ap_all, s->ap_loc, s->pt[buf], Xb, s->ldX, 0,
                                    s->n_chunks, g->grid, yb, st, lb)) != cudaSuccess)
            return e;
        if (ev && (e = cudaEventRecord(ev[2], st)) != cudaSuccess) return e;
        if ((e = launch_shard_apply(g->v, s->ap_loc, s->pt[buf], Xb, s->ldX, 2, 0, s->n_chunks,
                                    g->grid, sync_wait(2, s->xep[2]), st)) != cudaSuccess)
            return e;
        if (ev && (e = cudaEventRecord(ev[3], st)) != cudaSuccess) return e;
        return cudaSuccess;
    }
    if (ev && (e = cudaEventRecord(ev[0], st)) != cudaSuccess) return e;
    if ((e = launch_shard_agg(g->v, s->ap_all, s->pt[buf], 1, 0, 0, g->grid, sync_agg1(s), st)) !=
        cudaSuccess)
        return e;
    if (ev && (e = cudaEventRecord(ev[1], st)) != cudaSuccess) return e;
    XSync yf = sync_wait(1, s->xep[1]);
    yf.signal_end = 2;
    yf.ep_end = s->xep[2];
    if ((e = launch_shard_fused(g->v, s->ap_all, s->ap_loc, s->pt[buf], Xb, s->ldX, 0, s->n_chunks,
                                g->grid, yf, st)) != cudaSuccess)
        return e;
    if (ev && (e = cudaEventRecord(ev[2], st)) != cudaSuccess) return e;
    if ((e = launch_shard_apply(g->v, s->ap_loc, s->pt[buf], Xb, s->ldX, 2, 0, s->n_chunks, g->grid,
                                sync_wait(2, s->xep[2]), st)) != cudaSuccess)
        return e;
    if (ev && (e = cudaEventRecord(ev[3], st)) != cudaSuccess) return e;
    return cudaSuccess;
}

osp_status osp_shard_stage1(osp_shard* s, int buf, void* stream) {
    OSP_TRY(check_ready(s, buf));
    cudaStream_t st = as_stream(stream);
    osp_group* g = s->grp;
    if (s->stream) {
        s->iter += 1;
        OSP_CUDA(stream_stage(s, buf, 1, 0, 0, st));
        return OSP_OK;
    }
    // kind 0: deltas ready / previous iteration's reads done (agg1 entry);
    // kind 1: every shard's stage-1 aggregate landed here (apply1 entry)
    ++s->xep[0];
    ++s->xep[1];
    OSP_CUDA(launch_shard_agg(g->v, s->ap_all, s->pt[buf], 1, 0, 0, g->grid, sync_agg1(s), st));
    OSP_CUDA(launch_shard_apply(g->v, s->ap_loc, s->pt[buf], s->X + buf * s->buf_stride, s->ldX, 1,
                                0, 0, g->grid, sync_wait(1, s->xep[1]), st));
    return OSP_OK;
}

osp_status osp_shard_stage2(osp_shard* s, int c0, int c1, int buf, void* stream) {
    OSP_TRY(check_ready(s, buf));
    if (c0 < 0 || c1 > s->n_chunks || c0 > c1) return fail(OSP_ERR_INVALID, "chunk range");
    cudaStream_t st = as_stream(stream);
    osp_group* g = s->grp;
    if (s->stream) {
        if (s->iter == 0) return fail(OSP_ERR_PROTOCOL, "stage 2 before any stage 1");
        OSP_CUDA(stream_stage(s, buf, 2, c0, c1, st));
        return OSP_OK;
    }
    ++s->xep[2];  // kind 2: every shard's aggregate of these chunks landed here
    OSP_CUDA(launch_shard_agg(g->v, s->ap_all, s->pt[buf], 2, c0, c1, g->grid,
                              sync_signal_end(2, s->xep[2]), st));
    OSP_CUDA(launch_shard_apply(g->v, s->ap_loc, s->pt[buf], s->X + buf * s->buf_stride, s->ldX, 2,
                                c0, c1, g->grid, sync_wait(2, s->xep[2]), st));
    return OSP_OK;
}

osp_status osp_shard_resolve(osp_shard* s, int buf, void* stream) {
    OSP_TRY(check_ready(s, buf));
    return osp_group_resolve(s->grp, s->X + buf * s->buf_stride, s->ldX, stream);
}

// Whole iteration with stage 2's push/pull running inside the stage-1 apply
// launch (k_shard_fused): agg1, apply1 || agg2, apply2, resolve — four
// launches, the cross-GPU ordering inside them (XSync). Same results as
// stage1 + stage2 + resolve.
osp_status osp_shard_step(osp_shard* s, int buf, void* stream) {
    OSP_TRY(check_ready(s, buf));
    cudaStream_t st = as_stream(stream);
    if (s->stream) {
        s->iter += 1;
        OSP_CUDA(stream_stage(s, buf, 1, 0, 0, st));
        OSP_CUDA(stream_stage(s, buf, 2, 0, s->n_chunks, st));
        return osp_shard_resolve(s, buf, stream);
    }
    OSP_CUDA(barrier_step_kernels(s, buf, st));
    return osp_shard_resolve(s, buf, stream);
}

osp_status osp_shard_solo_agg(osp_shard* s, int stage, int buf, void* stream) {
    OSP_TRY(check_ready(s, buf));
    if (stage != 1 && stage != 2) return fail(OSP_ERR_INVALID, "stage must be 1 or 2");
    osp_group* g = s->grp;
    OSP_CUDA(launch_shard_agg(g->v, s->ap_all, s->pt[buf], stage, 0, s->n_chunks, g->grid, XSync{},
                              as_stream(stream)));
    return OSP_OK;
}

osp_status osp_shard_profile(osp_shard* s, int buf, float* ms, void* stream) {
    OSP_TRY(check_ready(s, buf));
    if (!ms) return fail(OSP_ERR_INVALID, "null output");
    cudaStream_t st = as_stream(stream);
    osp_group* g = s->grp;
    cudaEvent_t ev[9];
    for (auto& e : ev) OSP_CUDA(cudaEventCreate(&e));
    osp_status rc = OSP_OK;
    auto step = [&]() -> cudaError_t {
        cudaError_t e;
        float* Xb = s->X + buf * s->buf_stride;
        if (s->stream) {
            s->iter += 1;
            for (int i = 0; i < 8; ++i) ms[i] = 0.f;
            if ((e = cudaEventRecord(ev[0], st)) != cudaSuccess) return e;
            if ((e = stream_stage(s, buf, 1, 0, 0, st)) != cudaSuccess) return e;
            if ((e = cudaEventRecord(ev[1], st)) != cudaSuccess) return e;
            if ((e = stream_stage(s, buf, 2, 0, s->n_chunks, st)) != cudaSuccess) return e;
            if ((e = cudaEventRecord(ev[2], st)) != cudaSuccess) return e;
            if ((e = launch_resolve(g->v, g->ap, Xb, s->ldX, st)) != cudaSuccess) return e;
            if ((e = cudaEventRecord(ev[3], st)) != cudaSuccess) return e;
            if ((e = cudaEventSynchronize(ev[3])) != cudaSuccess) return e;
            for (int i = 0; i < 3; ++i)
                if ((e = cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1])) != cudaSuccess) return e;
            return cudaSuccess;
        }
        for (int i = 0; i < 8; ++i) ms[i] = 0.f;
        if ((e = barrier_step_kernels(s, buf, st, ev)) != cudaSuccess) return e;
        if ((e = launch_resolve(g->v, g->ap, Xb, s->ldX, st)) != cudaSuccess) return e;
        if ((e = cudaEventRecord(ev[4], st)) != cudaSuccess) return e;
        if ((e = cudaEventSynchronize(ev[4])) != cudaSuccess) return e;
        for (int i = 0; i < 4; ++i)
            if ((e = cudaEventElapsedTime(&ms[i], ev[i], ev[i + 1])) != cudaSuccess) return e;
        return cudaSuccess;
    };
    cudaError_t e = step();
    if (e != cudaSuccess) rc = cuda_fail(e, "shard profile");
    for (auto& x : ev) cudaEventDestroy(x);
    return rc;
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

int osp_shard_streaming(const osp_shard* s) { return s && s->stream ? 1 : 0; }

// Diagnostics of the streaming kernel (OSP_SS_DEBUG=1 at create): 96 counters
// accumulated since create, [stage 1 | stage 2][48]: producer empty-wait
// cycles, peer-flag wait cycles, 0, A/B/C items, producer cycles, 0, consumer
// warp-0 full-wait cycles, consumer warp-0 processing cycles, 0, 0, producers,
// max producer cycles (atomicMax, never reset), 0... Returns 0 when disabled.
int osp_shard_debug_counters(osp_shard* s, unsigned long long* out96) {
    if (!s || !s->dbg || !out96) return 0;
    if (cudaMemcpy(out96, s->dbg, 96 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    return 1;
}

osp_status osp_shard_check(osp_shard* s, void* stream) {
    if (!s) return fail(OSP_ERR_INVALID, "null shard");
    unsigned err = 0;
    cudaStream_t st = as_stream(stream);
    OSP_CUDA(cudaMemcpyAsync(&err, s->error, sizeof err, cudaMemcpyDeviceToHost, st));
    OSP_CUDA(cudaStreamSynchronize(st));
    if (err) return fail(OSP_ERR_PROTOCOL, "cross-GPU barrier timed out (a peer did not arrive)");
    return OSP_OK;
}

}  // extern "C"
