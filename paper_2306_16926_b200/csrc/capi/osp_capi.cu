// C-ABI implementation (include/osp_c.h): handles, validation with the
// reference's error classes, and the launch sequences. No exception crosses
// this boundary; every failure sets a thread-local message and returns a status.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "handles.h"

namespace osp {

namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

osp_status fail(osp_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}

osp_status cuda_fail(cudaError_t e, const char* what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return OSP_ERR_CUDA;
}

int sm_count() {
    static int cached = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            cached = 148;
    });
    return cached;
}

unsigned long long current_ctx_id() {
    using GetCurrent = int (*)(void**);
    using GetId = int (*)(void*, unsigned long long*);
    static GetCurrent get_current = nullptr;
    static GetId get_id = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuCtxGetCurrent", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_current = reinterpret_cast<GetCurrent>(f);
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuCtxGetId", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            get_id = reinterpret_cast<GetId>(f);
    });
    void* ctx = nullptr;
    unsigned long long id = 0;
    if (get_current && get_current(&ctx) == 0 && ctx) {
        if (get_id && get_id(ctx, &id) == 0) return id;
        return reinterpret_cast<unsigned long long>(ctx);
    }
    int dev = 0;
    cudaGetDevice(&dev);
    return 0xffff000000000000ull | static_cast<unsigned>(dev);
}

AggParams make_agg_params(int n, const double* weights, double sgd_lr) {
    AggParams ap{};
    ap.n = n;
    double total = 0.0;
    for (int w = 0; w < n; ++w) {
        ap.w[w] = weights[w];
        total += weights[w];  // protocol.cpp:14-15, ascending
    }
    ap.total = total;
    ap.divide = total == 1.0 ? 0 : 1;
    ap.sgd = sgd_lr > 0 ? 1 : 0;
    ap.neg_lr = -sgd_lr;
    return ap;
}

}  // namespace osp

using namespace osp;

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------

namespace {

template <typename T>
osp_status dalloc(osp_group* g, T** out, size_t count) {
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
    g->owned.push_back(p);
    *out = static_cast<T*>(p);
    return OSP_OK;
}

osp_status check_weights(int n, const double* weights) {
    if (n < 1) return fail(OSP_ERR_PROTOCOL, "aggregation needs one contribution per worker");
    if (n > OSP_MAX_WORKERS)
        return fail(OSP_ERR_INVALID, "more than OSP_MAX_WORKERS (" +
                                         std::to_string(OSP_MAX_WORKERS) + ") workers");
    if (!weights) return fail(OSP_ERR_INVALID, "null weights");
    double tw = 0.0;
    for (int w = 0; w < n; ++w) tw += weights[w];
    if (!(tw > 0.0)) return fail(OSP_ERR_PROTOCOL, "aggregation weights must sum > 0");
    return OSP_OK;
}

// Device segment table from host (offset, count[, flag]) lists; freed stream-ordered.
struct SegTable {
    uint64_t* off = nullptr;
    uint64_t* cnt = nullptr;
    uint8_t* flag = nullptr;
    cudaStream_t s = nullptr;
    ~SegTable() {
        if (off) cudaFreeAsync(off, s);
        if (cnt) cudaFreeAsync(cnt, s);
        if (flag) cudaFreeAsync(flag, s);
    }
};

osp_status upload_segments(SegTable& t, const std::vector<uint64_t>& off,
                           const std::vector<uint64_t>& cnt, const std::vector<uint8_t>* flag,
                           cudaStream_t s) {
    t.s = s;
    const size_t n = std::max<size_t>(off.size(), 1);
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&t.off), n * 8, s));
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&t.cnt), n * 8, s));
    if (!off.empty()) {
        OSP_CUDA(cudaMemcpyAsync(t.off, off.data(), off.size() * 8, cudaMemcpyHostToDevice, s));
        OSP_CUDA(cudaMemcpyAsync(t.cnt, cnt.data(), cnt.size() * 8, cudaMemcpyHostToDevice, s));
    }
    if (flag) {
        OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&t.flag), n, s));
        if (!flag->empty())
            OSP_CUDA(cudaMemcpyAsync(t.flag, flag->data(), flag->size(), cudaMemcpyHostToDevice, s));
    }
    return OSP_OK;
}

void put_u32le(uint8_t* p, uint32_t v) {
    p[0] = v & 0xff;
    p[1] = (v >> 8) & 0xff;
    p[2] = (v >> 16) & 0xff;
    p[3] = (v >> 24) & 0xff;
}

uint32_t get_u32le(const uint8_t* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

}  // namespace

extern "C" {

const char* osp_last_error(void) { return g_last_error.c_str(); }

const char* osp_status_name(osp_status s) {
    switch (s) {
        case OSP_OK: return "OK";
        case OSP_ERR_PARTITION: return "PartitionError";
        case OSP_ERR_SHAPE: return "ShapeError";
        case OSP_ERR_LAYER: return "LayerError";
        case OSP_ERR_PARSE: return "ParseError";
        case OSP_ERR_CONFIG: return "ConfigError";
        case OSP_ERR_FORMAT: return "FormatError";
        case OSP_ERR_PROTOCOL: return "ProtocolError";
        case OSP_ERR_NUMERIC: return "NumericError";
        case OSP_ERR_CUDA: return "CudaError";
        case OSP_ERR_INVALID: return "InvalidArgument";
    }
    return "Unknown";
}

int osp_abi_version(void) { return OSP_ABI_VERSION; }

osp_status osp_device_info(int* device, int* sms, int* major, int* minor) {
    int dev = 0;
    OSP_CUDA(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    OSP_CUDA(cudaGetDeviceProperties(&prop, dev));
    if (device) *device = dev;
    if (sms) *sms = prop.multiProcessorCount;
    if (major) *major = prop.major;
    if (minor) *minor = prop.minor;
    return OSP_OK;
}

// ---- partition --------------------------------------------------------------

osp_status osp_partition_create(const uint64_t* layer_counts, uint64_t n_layers,
                                uint32_t bytes_per_element, osp_partition** out) {
    if (!out) return fail(OSP_ERR_INVALID, "null output handle");
    *out = nullptr;
    if (n_layers == 0) return fail(OSP_ERR_PARTITION, "partition needs at least one layer");
    if (bytes_per_element == 0) return fail(OSP_ERR_PARTITION, "bytes_per_element must be positive");
    if (!layer_counts) return fail(OSP_ERR_INVALID, "null layer_counts");
    auto* p = new (std::nothrow) osp_partition();
    if (!p) return fail(OSP_ERR_INVALID, "out of host memory");
    p->bpe = bytes_per_element;
    p->counts.assign(layer_counts, layer_counts + n_layers);
    p->offsets.resize(n_layers);
    uint64_t off = 0;
    for (uint64_t i = 0; i < n_layers; ++i) {
        if (layer_counts[i] == 0) {
            delete p;
            return fail(OSP_ERR_PARTITION, "layer " + std::to_string(i) + " has zero elements");
        }
        p->offsets[i] = off;
        off += layer_counts[i];
    }
    p->total = off;
    cudaError_t e = cudaMalloc(&p->d_offsets, n_layers * 8);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_counts, n_layers * 8);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_offsets, p->offsets.data(), n_layers * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_counts, p->counts.data(), n_layers * 8, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        osp_partition_destroy(p);
        return cuda_fail(e, "partition device mirror");
    }
    *out = p;
    return OSP_OK;
}

void osp_partition_destroy(osp_partition* p) {
    if (!p) return;
    if (p->scratch) osp_group_destroy(p->scratch);
    if (p->d_offsets) cudaFree(p->d_offsets);
    if (p->d_counts) cudaFree(p->d_counts);
    delete p;
}

uint64_t osp_partition_layer_count(const osp_partition* p) { return p ? p->counts.size() : 0; }
uint64_t osp_partition_total_count(const osp_partition* p) { return p ? p->total : 0; }
uint64_t osp_partition_total_bytes(const osp_partition* p) { return p ? p->total * p->bpe : 0; }
uint32_t osp_partition_bytes_per_element(const osp_partition* p) { return p ? p->bpe : 0; }

osp_status osp_partition_layer(const osp_partition* p, int64_t id, uint64_t* offset,
                               uint64_t* count) {
    if (!p) return fail(OSP_ERR_INVALID, "null partition");
    if (id < 0 || static_cast<uint64_t>(id) >= p->counts.size())
        return fail(OSP_ERR_LAYER, "layer id " + std::to_string(id) + " out of range (have " +
                                       std::to_string(p->counts.size()) + " layers)");
    if (offset) *offset = p->offsets[id];
    if (count) *count = p->counts[id];
    return OSP_OK;
}

// ---- buffers ----------------------------------------------------------------

osp_status osp_device_alloc(uint64_t bytes, void** out) {
    if (!out) return fail(OSP_ERR_INVALID, "null output");
    OSP_CUDA(cudaMalloc(out, std::max<uint64_t>(bytes, 4)));
    return OSP_OK;
}
osp_status osp_device_free(void* ptr) {
    if (ptr) OSP_CUDA(cudaFree(ptr));
    return OSP_OK;
}
osp_status osp_memcpy_h2d(void* dst, const void* src, uint64_t bytes, void* stream) {
    if (bytes) OSP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
    return OSP_OK;
}
osp_status osp_memcpy_d2h(void* dst, const void* src, uint64_t bytes, void* stream) {
    if (bytes) {
        OSP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
        OSP_CUDA(cudaStreamSynchronize(as_stream(stream)));
    }
    return OSP_OK;
}
osp_status osp_memcpy_d2d(void* dst, const void* src, uint64_t bytes, void* stream) {
    if (bytes) OSP_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
    return OSP_OK;
}
osp_status osp_memset(void* dst, int value, uint64_t bytes, void* stream) {
    if (bytes) OSP_CUDA(cudaMemsetAsync(dst, value, bytes, as_stream(stream)));
    return OSP_OK;
}
osp_status osp_stream_sync(void* stream) {
    OSP_CUDA(cudaStreamSynchronize(as_stream(stream)));
    return OSP_OK;
}

// ---- element-wise primitives ------------------------------------------------

osp_status osp_aggregate_layer(const float* const* contribs, int n_workers,
                               const double* weights, uint64_t n, float* out, void* stream) {
    OSP_TRY(check_weights(n_workers, weights));
    if (!contribs || !out) return fail(OSP_ERR_INVALID, "null pointer");
    for (int w = 0; w < n_workers; ++w)
        if (!contribs[w] && n) return fail(OSP_ERR_INVALID, "null contribution");
    AggParams ap = make_agg_params(n_workers, weights, 0.0);
    OSP_CUDA(launch_aggregate_layer(contribs, ap, n, out, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_aggregate_apply_layers(const osp_partition* part, const float* const* contribs,
                                      int n_workers, const double* weights,
                                      const int32_t* layer_ids, int64_t n_ids, float* global,
                                      float* agg_out, void* stream) {
    if (!part) return fail(OSP_ERR_INVALID, "null partition");
    OSP_TRY(check_weights(n_workers, weights));
    if (n_ids > 65535) return fail(OSP_ERR_INVALID, "too many layers in one call");
    std::vector<uint64_t> off, cnt;
    for (int64_t i = 0; i < n_ids; ++i) {
        uint64_t o = 0, c = 0;
        OSP_TRY(osp_partition_layer(part, layer_ids[i], &o, &c));
        off.push_back(o);
        cnt.push_back(c);
    }
    if (off.empty()) return OSP_OK;
    cudaStream_t s = as_stream(stream);
    SegTable t;
    OSP_TRY(upload_segments(t, off, cnt, nullptr, s));
    AggParams ap = make_agg_params(n_workers, weights, 0.0);
    OSP_CUDA(launch_aggregate_apply_segments(contribs, ap, t.off, t.cnt, static_cast<int>(off.size()),
                                             global, agg_out, s));
    return OSP_OK;
}

osp_status osp_apply_delta(float* p, const float* d, uint64_t n, float scale, void* stream) {
    OSP_CUDA(launch_apply_delta(p, d, n, scale, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_sgd_delta(const float* grad, uint64_t n, double lr, float* out, void* stream) {
    if (lr <= 0) return fail(OSP_ERR_CONFIG, "learning rate must be positive");
    OSP_CUDA(launch_sgd_delta(grad, n, lr, out, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_synth_delta(uint64_t seed, uint64_t worker, uint64_t iteration, uint64_t first,
                           uint64_t n, float* out, void* stream) {
    OSP_CUDA(launch_synth(seed, 1, iteration, first, n, out, n, worker, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_synth_deltas(uint64_t seed, int n_workers, uint64_t iteration, uint64_t n,
                            float* out, uint64_t ld, void* stream) {
    if (n_workers < 0 || n_workers > 65535) return fail(OSP_ERR_INVALID, "bad worker count");
    if (ld < n) return fail(OSP_ERR_SHAPE, "ld smaller than the vector length");
    OSP_CUDA(launch_synth(seed, n_workers, iteration, 0, n, out, ld, 0, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_lgp_partial(const osp_partition* part, float* params, const float* global_delta,
                           const float* local_delta, const uint8_t* ics_flags, float* base,
                           void* stream) {
    if (!part || !ics_flags) return fail(OSP_ERR_INVALID, "null argument");
    const size_t L = part->counts.size();
    std::vector<uint64_t> off, cnt;
    std::vector<uint8_t> loc;
    for (size_t l = 0; l < L; ++l) {
        if (ics_flags[l] > 1) continue;  // 2: in neither payload, left untouched
        off.push_back(part->offsets[l]);
        cnt.push_back(part->counts[l]);
        loc.push_back(ics_flags[l]);
    }
    if (off.empty()) return OSP_OK;
    if (off.size() > 65535) return fail(OSP_ERR_INVALID, "too many layers in one call");
    cudaStream_t s = as_stream(stream);
    SegTable t;
    OSP_TRY(upload_segments(t, off, cnt, &loc, s));
    OSP_CUDA(launch_lgp_partial_segments(params, global_delta, local_delta, base, t.off, t.cnt, t.flag,
                                         static_cast<int>(off.size()), s));
    return OSP_OK;
}

osp_status osp_lgp_correct(const osp_partition* part, float* params, const float* base,
                           const float* global_delta, const int32_t* layer_ids, int64_t n_ids,
                           void* stream) {
    if (!part) return fail(OSP_ERR_INVALID, "null partition");
    std::vector<uint64_t> off, cnt;
    for (int64_t i = 0; i < n_ids; ++i) {
        uint64_t o = 0, c = 0;
        OSP_TRY(osp_partition_layer(part, layer_ids[i], &o, &c));
        off.push_back(o);
        cnt.push_back(c);
    }
    if (off.empty()) return OSP_OK;
    if (off.size() > 65535) return fail(OSP_ERR_INVALID, "too many layers in one call");
    cudaStream_t s = as_stream(stream);
    SegTable t;
    OSP_TRY(upload_segments(t, off, cnt, nullptr, s));
    OSP_CUDA(launch_lgp_correct_segments(params, base, global_delta, t.off, t.cnt,
                                         static_cast<int>(off.size()), s));
    return OSP_OK;
}

osp_status osp_pgp_layer_importance(const osp_partition* part, const float* params,
                                    const float* grads, double* scores_host, void* stream) {
    if (!part || !scores_host) return fail(OSP_ERR_INVALID, "null argument");
    const int L = static_cast<int>(part->counts.size());
    cudaStream_t s = as_stream(stream);
    double* d = nullptr;
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), L * sizeof(double), s));
    cudaError_t e = launch_pgp_exact(params, grads, part->d_offsets, part->d_counts, L, d, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(scores_host, d, L * sizeof(double), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "pgp_layer_importance");
    return OSP_OK;
}

osp_status osp_rank_and_gib(const osp_partition* part, const double* scores_host,
                            uint64_t budget_bytes, int32_t* order_host, uint8_t* flags_host,
                            void* stream) {
    if (!part || !scores_host) return fail(OSP_ERR_INVALID, "null argument");
    const int L = static_cast<int>(part->counts.size());
    if (L > kMaxLayers)
        return fail(OSP_ERR_INVALID, "more than " + std::to_string(kMaxLayers) + " layers");
    cudaStream_t s = as_stream(stream);
    double* ds = nullptr;
    int* dord = nullptr;
    uint8_t* dfl = nullptr;
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ds), L * sizeof(double), s));
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dord), L * sizeof(int), s));
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dfl), L, s));
    cudaError_t e = cudaMemcpyAsync(ds, scores_host, L * sizeof(double), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
        e = launch_rank_gib(ds, part->d_counts, part->bpe, L, budget_bytes, dord, dfl, s);
    if (e == cudaSuccess && order_host)
        e = cudaMemcpyAsync(order_host, dord, L * sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess && flags_host)
        e = cudaMemcpyAsync(flags_host, dfl, L, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(ds, s);
    cudaFreeAsync(dord, s);
    cudaFreeAsync(dfl, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "rank_and_gib");
    return OSP_OK;
}

osp_status osp_pgp_rank_gib(const osp_partition* part, const float* params, const float* grads,
                            uint64_t budget_bytes, double* scores_host, int32_t* ics_order_host,
                            int64_t* n_ics, uint8_t* ics_flags_host, void* stream) {
    if (!part || !params || !grads) return fail(OSP_ERR_INVALID, "null argument");
    const int L = static_cast<int>(part->counts.size());
    if (L > kMaxLayers)
        return fail(OSP_ERR_INVALID, "more than " + std::to_string(kMaxLayers) + " layers");
    cudaStream_t s = as_stream(stream);
    auto* mp = const_cast<osp_partition*>(part);
    if (!mp->scratch) {
        const double w1 = 1.0;
        osp_group_config gc{1, &w1, 1, 0, 0.0, OSP_GROUP_REGISTER};
        OSP_TRY(osp_group_create(part, &gc, nullptr, stream, &mp->scratch));
    }
    // the group's resolve over the caller's vectors: tile partials of
    // |grads * params|, tree sums, certificate, exact sequential fallback on
    // touching intervals (reading agg_full = grads, G = params), rank, prefix rule
    GroupView v = mp->scratch->v;
    v.G = const_cast<float*>(params);
    v.agg_full = grads;
    v.C = nullptr;
    OSP_CUDA(launch_pgp_tiles(v, params, grads, s));
    OSP_CUDA(launch_set_budget(v, budget_bytes, s));
    OSP_CUDA(launch_resolve(v, mp->scratch->ap, grads, part->total, s));
    int meta[8];
    std::vector<double> sc(L), ex(L);
    std::vector<uint8_t> mk(L);
    OSP_CUDA(cudaMemcpyAsync(meta, v.meta, sizeof meta, cudaMemcpyDeviceToHost, s));
    if (scores_host) {
        OSP_CUDA(cudaMemcpyAsync(sc.data(), v.scores, L * sizeof(double), cudaMemcpyDeviceToHost, s));
        OSP_CUDA(cudaMemcpyAsync(ex.data(), v.exact, L * sizeof(double), cudaMemcpyDeviceToHost, s));
        OSP_CUDA(cudaMemcpyAsync(mk.data(), v.marked, L, cudaMemcpyDeviceToHost, s));
    }
    if (ics_flags_host) OSP_CUDA(cudaMemcpyAsync(ics_flags_host, v.flags, L, cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> ord(L);
    if (ics_order_host)
        OSP_CUDA(cudaMemcpyAsync(ord.data(), v.ics_layers, L * 4, cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaStreamSynchronize(s));
    const int k = meta[META_N_ICS];
    if (n_ics) *n_ics = k;
    if (ics_order_host) std::copy(ord.begin(), ord.begin() + k, ics_order_host);
    if (scores_host)
        for (int l = 0; l < L; ++l) scores_host[l] = mk[l] ? ex[l] : sc[l];
    return OSP_OK;
}

osp_status osp_split_for_sync(const osp_partition* part, const uint8_t* ics_flags,
                              const int32_t* ics_order, int64_t n_order, int n_chunks,
                              int32_t* rs_ids, int64_t* n_rs, int32_t* chunk_of, int* n_used) {
    if (!part || !ics_flags) return fail(OSP_ERR_INVALID, "null argument");
    if (n_chunks < 1) return fail(OSP_ERR_CONFIG, "need at least one chunk slot");
    const int L = static_cast<int>(part->counts.size());
    if (L > kMaxLayers)
        return fail(OSP_ERR_INVALID, "more than " + std::to_string(kMaxLayers) + " layers");
    // Scratch group view with one tile per layer; the device list builder
    // (k_install -> finalize_lists, resolve.cu) does the index math.
    std::vector<int> tb(L + 1);
    for (int l = 0; l <= L; ++l) tb[l] = l;
    std::vector<uint8_t> f(L);
    for (int l = 0; l < L; ++l) f[l] = ics_flags[l] ? 1 : 0;
    GroupView v{};
    v.L = L;
    v.T = 1 << 30;
    v.NT = L;
    v.n_chunks = n_chunks;
    v.bpe = part->bpe;
    v.offsets = part->d_offsets;
    v.counts = part->d_counts;
    std::vector<void*> tmp;
    auto al = [&](auto** p, size_t bytes) -> cudaError_t {
        cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(bytes, 8));
        if (e == cudaSuccess) tmp.push_back(*p);
        return e;
    };
    int* d_tb = nullptr;
    int* d_order = nullptr;
    cudaError_t e = al(&d_tb, (L + 1) * sizeof(int));
    if (e == cudaSuccess) e = al(&d_order, std::max<int64_t>(n_order, 1) * sizeof(int));
    if (e == cudaSuccess) e = al(&v.flags, L);
    if (e == cudaSuccess) e = al(&v.ics_layers, L * sizeof(int));
    if (e == cudaSuccess) e = al(&v.chunk_begin, (n_chunks + 1) * sizeof(int));
    if (e == cudaSuccess) e = al(&v.ics_tile_prefix, (L + 1) * sizeof(int));
    if (e == cudaSuccess) e = al(&v.meta, 8 * sizeof(int));
    if (e == cudaSuccess) e = al(&v.meta64, 8 * sizeof(uint64_t));
    if (e == cudaSuccess) e = al(&v.chunk_of, L * sizeof(int));
    if (e == cudaSuccess) e = al(&v.gib_bytes, osp_gib_wire_size(L, L));
    if (e == cudaSuccess && L > kSmemResolveLayers) e = al(&v.rscratch, resolve_scratch_bytes(L));
    v.tile_base = d_tb;
    if (e == cudaSuccess) e = cudaMemcpy(d_tb, tb.data(), (L + 1) * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(v.flags, f.data(), L, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && n_order > 0)
        e = cudaMemcpy(d_order, ics_order, n_order * sizeof(int), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = launch_install_gib(v, d_order, static_cast<int>(n_order), 0, nullptr);
    int meta[8] = {0};
    std::vector<int32_t> co(L);
    if (e == cudaSuccess) e = cudaMemcpy(meta, v.meta, sizeof meta, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(co.data(), v.chunk_of, L * 4, cudaMemcpyDeviceToHost);
    for (void* p : tmp) cudaFree(p);
    if (e != cudaSuccess) return cuda_fail(e, "split_for_sync");
    int64_t nr = 0;
    for (int l = 0; l < L; ++l) {
        if (!f[l] && rs_ids) rs_ids[nr] = l;
        if (!f[l]) ++nr;
    }
    if (n_rs) *n_rs = nr;
    if (chunk_of) std::copy(co.begin(), co.end(), chunk_of);
    if (n_used) *n_used = meta[META_N_USED];
    return OSP_OK;
}

// ---- GIB wire format --------------------------------------------------------

uint64_t osp_gib_encoded_size(uint64_t n_layers) { return 8 + (n_layers + 7) / 8; }

osp_status osp_gib_encode(uint32_t tag, uint64_t n_layers, const uint8_t* ics_flags, uint8_t* out,
                          uint64_t out_len) {
    const uint64_t need = osp_gib_encoded_size(n_layers);
    if (!out || out_len < need) return fail(OSP_ERR_INVALID, "gib output buffer too small");
    std::memset(out, 0, need);
    put_u32le(out, tag);
    put_u32le(out + 4, static_cast<uint32_t>(n_layers));
    for (uint64_t k = 0; k < n_layers; ++k)
        if (ics_flags[k]) out[8 + k / 8] |= static_cast<uint8_t>(1u << (k % 8));
    return OSP_OK;
}

osp_status osp_gib_decode(const uint8_t* buf, uint64_t len, uint32_t* tag, uint32_t* n_layers,
                          uint8_t* ics_flags, uint64_t flags_cap) {
    if (len < 8)
        return fail(OSP_ERR_FORMAT, "gib buffer truncated: " + std::to_string(len) + " bytes");
    const uint32_t t = get_u32le(buf), L = get_u32le(buf + 4);
    if (len < osp_gib_encoded_size(L))
        return fail(OSP_ERR_FORMAT, "gib bitmap truncated: need " +
                                        std::to_string(osp_gib_encoded_size(L)) + " bytes, have " +
                                        std::to_string(len));
    if (tag) *tag = t;
    if (n_layers) *n_layers = L;
    if (ics_flags) {
        if (L > flags_cap) return fail(OSP_ERR_INVALID, "flags buffer too small");
        for (uint64_t k = 0; k < L; ++k) ics_flags[k] = (buf[8 + k / 8] >> (k % 8)) & 1u;
    }
    return OSP_OK;
}

uint64_t osp_gib_wire_size(uint64_t n_layers, uint64_t n_order) {
    return osp_gib_encoded_size(n_layers) + 4 + 4 * n_order;
}

osp_status osp_gib_wire_encode(uint32_t tag, uint64_t n_layers, const uint8_t* ics_flags,
                               const int32_t* order, uint64_t n_order, uint8_t* out,
                               uint64_t cap, uint64_t* len) {
    if (!ics_flags && n_layers > 0) return fail(OSP_ERR_INVALID, "null flags");
    if (n_order > 0 && !order) return fail(OSP_ERR_INVALID, "null rank order");
    if (n_layers > 0xffffffffull || n_order > n_layers)
        return fail(OSP_ERR_INVALID, "rank order longer than the layer count");
    std::vector<uint8_t> seen(n_layers, 0);
    for (uint64_t r = 0; r < n_order; ++r) {
        const int32_t id = order[r];
        if (id < 0 || static_cast<uint64_t>(id) >= n_layers)
            return fail(OSP_ERR_LAYER, "rank order names layer " + std::to_string(id) +
                                           " beyond the partition");
        if (!ics_flags[id])
            return fail(OSP_ERR_PROTOCOL, "rank order names layer " + std::to_string(id) +
                                              " that the bitmap does not defer");
        if (seen[id]++) return fail(OSP_ERR_PROTOCOL, "rank order repeats layer " + std::to_string(id));
    }
    const uint64_t need = osp_gib_wire_size(n_layers, n_order);
    if (len) *len = need;
    if (!out) return OSP_OK;
    if (cap < need) return fail(OSP_ERR_INVALID, "gib wire buffer too small");
    OSP_TRY(osp_gib_encode(tag, n_layers, ics_flags, out, cap));
    uint8_t* p = out + osp_gib_encoded_size(n_layers);
    put_u32le(p, static_cast<uint32_t>(n_order));
    for (uint64_t r = 0; r < n_order; ++r) put_u32le(p + 4 + 4 * r, static_cast<uint32_t>(order[r]));
    return OSP_OK;
}

osp_status osp_gib_wire_decode(const uint8_t* buf, uint64_t len, uint32_t* tag, uint32_t* n_layers,
                               uint8_t* ics_flags, uint64_t flags_cap, int32_t* order,
                               uint64_t order_cap, int64_t* n_order) {
    if (!buf && len > 0) return fail(OSP_ERR_INVALID, "null buffer");
    uint32_t t = 0, L = 0;
    OSP_TRY(osp_gib_decode(buf, len, &t, &L, nullptr, 0));
    const uint64_t base = osp_gib_encoded_size(L);
    int64_t n = -1;  // -1: bitmap only (no side channel)
    if (len > base) {
        if (len < base + 4)
            return fail(OSP_ERR_FORMAT, "gib rank order truncated: " + std::to_string(len) + " bytes");
        const uint32_t k = get_u32le(buf + base);
        if (k > L) return fail(OSP_ERR_FORMAT, "gib rank order longer than the layer count");
        if (len != osp_gib_wire_size(L, k))
            return fail(OSP_ERR_FORMAT, "gib rank order of " + std::to_string(k) + " ids needs " +
                                            std::to_string(osp_gib_wire_size(L, k)) + " bytes, have " +
                                            std::to_string(len));
        n = k;
    }
    std::vector<uint8_t> f(L);
    for (uint64_t l = 0; l < L; ++l) f[l] = (buf[8 + l / 8] >> (l % 8)) & 1u;
    std::vector<uint8_t> seen(L, 0);
    for (int64_t r = 0; r < n; ++r) {
        const uint32_t id = get_u32le(buf + base + 4 + 4 * r);
        if (id >= L || !f[id] || seen[id]++)
            return fail(OSP_ERR_FORMAT, "gib rank order entry " + std::to_string(r) +
                                            " is not a distinct deferred layer");
    }
    if (ics_flags && L > flags_cap) return fail(OSP_ERR_INVALID, "flags buffer too small");
    if (order && n > 0 && static_cast<uint64_t>(n) > order_cap)
        return fail(OSP_ERR_INVALID, "rank order buffer too small");
    if (tag) *tag = t;
    if (n_layers) *n_layers = L;
    if (n_order) *n_order = n;
    if (ics_flags) std::copy(f.begin(), f.end(), ics_flags);
    if (order)
        for (int64_t r = 0; r < n; ++r) order[r] = static_cast<int32_t>(get_u32le(buf + base + 4 + 4 * r));
    return OSP_OK;
}

// ---- tuning (host scalar logic, tuning.cpp:8-48) ----------------------------

osp_status osp_compute_umax(double bw, double latency_s, double loss_rate, double t_c,
                            int n_workers, uint64_t model_bytes, int eq5_literal, uint64_t* out) {
    if (bw <= 0) return fail(OSP_ERR_CONFIG, "bandwidth must be positive");
    if (latency_s < 0) return fail(OSP_ERR_CONFIG, "latency must be non-negative");
    if (loss_rate < 0 || loss_rate >= 1) return fail(OSP_ERR_CONFIG, "loss_rate must be in [0, 1)");
    if (t_c < 0) return fail(OSP_ERR_CONFIG, "t_c must be non-negative");
    if (n_workers < 1) return fail(OSP_ERR_CONFIG, "n_workers must be at least 1");
    double raw = eq5_literal ? bw * (1.0 + loss_rate) * t_c / n_workers
                             : bw * t_c / (n_workers * (1.0 + loss_rate));
    double cap = 0.8 * static_cast<double>(model_bytes);
    *out = static_cast<uint64_t>(std::floor(std::min(raw, cap)));
    return OSP_OK;
}

osp_status osp_tune_sgu(osp_sgu_schedule* sched, uint64_t epoch_index, double epoch_loss,
                        uint64_t* budget_out) {
    if (!sched) return fail(OSP_ERR_INVALID, "null schedule");
    if (epoch_index < 1) return fail(OSP_ERR_CONFIG, "epoch index is 1-based");
    if (epoch_loss < 0) return fail(OSP_ERR_NUMERIC, "epoch loss must be non-negative");
    sched->epoch = epoch_index;
    if (epoch_index == 1) {
        sched->initial_loss = epoch_loss;
        sched->has_initial_loss = 1;
        sched->current_budget = 0;
        if (budget_out) *budget_out = 0;
        return OSP_OK;
    }
    if (!sched->has_initial_loss)
        return fail(OSP_ERR_PROTOCOL, "tune_sgu called for epoch " + std::to_string(epoch_index) +
                                          " before epoch 1 recorded the reference loss");
    const double ref = sched->initial_loss;
    const double factor = ref <= 0.0 ? 1.0 : std::clamp(1.0 - epoch_loss / ref, 0.0, 1.0);
    sched->current_budget =
        static_cast<uint64_t>(std::floor(factor * static_cast<double>(sched->u_max)));
    if (budget_out) *budget_out = sched->current_budget;
    return OSP_OK;
}

// ---- group ------------------------------------------------------------------

osp_status osp_group_create(const osp_partition* part, const osp_group_config* cfg,
                            const float* init_params, void* stream, osp_group** out) {
    if (!out || !part || !cfg) return fail(OSP_ERR_INVALID, "null argument");
    *out = nullptr;
    const int N = cfg->n_workers;
    if (N < 1) return fail(OSP_ERR_CONFIG, "server needs worker weights");
    if (N > OSP_MAX_WORKERS)
        return fail(OSP_ERR_INVALID, "more than OSP_MAX_WORKERS workers per group");
    if (!cfg->weights) return fail(OSP_ERR_INVALID, "null weights");
    for (int w = 0; w < N; ++w)
        if (cfg->weights[w] <= 0) return fail(OSP_ERR_CONFIG, "subset weight must be positive");
    if (cfg->n_chunks < 1) return fail(OSP_ERR_CONFIG, "need at least one chunk slot");
    if (cfg->sgd_lr < 0) return fail(OSP_ERR_CONFIG, "learning rate must be positive");
    const uint64_t L = part->counts.size();
    if (L > static_cast<uint64_t>(kMaxLayers))
        return fail(OSP_ERR_INVALID, "more than " + std::to_string(kMaxLayers) + " layers");
    // Stage kernels: TMA-staged unless OSP_GROUP_REGISTER (or unsupported shape
    // without an explicit OSP_GROUP_TMA request); default tiles 1024 / 512.
    const bool want_tma = (cfg->flags & OSP_GROUP_TMA) != 0;
    const bool force_reg = (cfg->flags & OSP_GROUP_REGISTER) != 0;
    if (want_tma && force_reg)
        return fail(OSP_ERR_INVALID, "OSP_GROUP_TMA and OSP_GROUP_REGISTER are exclusive");
    if (cfg->flags & ~(OSP_GROUP_TMA | OSP_GROUP_REGISTER | OSP_GROUP_NO_CARRY | OSP_GROUP_NO_SMALL))
        return fail(OSP_ERR_INVALID, "unknown osp_group_config flags");
    bool use_tma = false;
    if (!force_reg) {
        const uint32_t Tt = cfg->tile_elems ? cfg->tile_elems : kDefaultTmaTile;
        use_tma = tma_supported(N, static_cast<int>(Tt), static_cast<int>(L));
        if (want_tma && !use_tma)
            return fail(OSP_ERR_INVALID, "OSP_GROUP_TMA needs N in 1..8, tile_elems in "
                                         "[512, 4096] and the ring + layer tables within "
                                         "shared memory");
    }
    uint32_t T = cfg->tile_elems ? cfg->tile_elems : (use_tma ? kDefaultTmaTile : kDefaultTile);
    if (T < 256 || T > 65536 || (T & (T - 1)))
        return fail(OSP_ERR_INVALID, "tile_elems must be a power of two in [256, 65536]");

    auto* g = new (std::nothrow) osp_group();
    if (!g) return fail(OSP_ERR_INVALID, "out of host memory");
    auto cleanup = [&](osp_status s) {
        osp_group_destroy(g);
        return s;
    };
    g->part = part;
    g->N = N;
    g->n_chunks = cfg->n_chunks;
    g->sgd_lr = cfg->sgd_lr;
    g->weights.assign(cfg->weights, cfg->weights + N);
    g->ap = make_agg_params(N, cfg->weights, cfg->sgd_lr);

    // tile tables
    std::vector<int> tile_base(L + 1), tile_layer;
    uint64_t nt_total = 0;
    for (uint64_t l = 0; l < L; ++l) {
        tile_base[l] = static_cast<int>(nt_total);
        const uint64_t nt = (part->counts[l] + T - 1) / T;
        for (uint64_t k = 0; k < nt; ++k) tile_layer.push_back(static_cast<int>(l));
        nt_total += nt;
        if (nt_total > 0x7fffffffull) return cleanup(fail(OSP_ERR_INVALID, "too many tiles"));
    }
    tile_base[L] = static_cast<int>(nt_total);

    GroupView& v = g->v;
    v.L = static_cast<int>(L);
    v.T = static_cast<int>(T);
    v.NT = static_cast<int>(nt_total);
    v.n_chunks = cfg->n_chunks;
    v.bpe = part->bpe;
    v.offsets = part->d_offsets;
    v.counts = part->d_counts;
    const uint64_t M = part->total;
    v.ldP = (M + 3) & ~uint64_t(3);
    int *d_tb = nullptr, *d_tl = nullptr;
    osp_status st;
    if ((st = dalloc(g, &d_tb, L + 1)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &d_tl, nt_total)) != OSP_OK) return cleanup(st);
    v.tile_base = d_tb;
    v.tile_layer = d_tl;
    if ((st = dalloc(g, &v.G, M)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.P, v.ldP * N)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.partials, nt_total)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.flags, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.ics_layers, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.chunk_begin, cfg->n_chunks + 1)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.ics_tile_prefix, L + 1)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.meta, 8)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.meta64, 8)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.scores, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.exact, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.marked, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.chunk_of, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.gib_bytes, osp_gib_wire_size(L, L))) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &g->d_order_tmp, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.hist, kHist)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.sched, 16)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.lscore, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.rs_layers, L)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.rs_tile_prefix, L + 1)) != OSP_OK) return cleanup(st);
    if (L > static_cast<uint64_t>(kSmemResolveLayers) &&
        (st = dalloc(g, &v.rscratch, resolve_scratch_bytes(static_cast<int>(L)))) != OSP_OK)
        return cleanup(st);
    // resolve sum items: each layer's tiles in chunks of <= kSumChunk
    std::vector<int> items, layer_items(L + 1);
    for (uint64_t l = 0; l < L; ++l) {
        layer_items[l] = static_cast<int>(items.size() / 3);
        for (int t = tile_base[l]; t < tile_base[l + 1]; t += kSumChunk) {
            items.push_back(static_cast<int>(l));
            items.push_back(t);
            items.push_back(std::min(t + kSumChunk, tile_base[l + 1]));
        }
    }
    layer_items[L] = static_cast<int>(items.size() / 3);
    int *d_items = nullptr, *d_litems = nullptr;
    if ((st = dalloc(g, &d_items, std::max<size_t>(items.size(), 3))) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &d_litems, L + 1)) != OSP_OK) return cleanup(st);
    if ((st = dalloc(g, &v.item_sums, std::max<size_t>(items.size() / 3, 1))) != OSP_OK)
        return cleanup(st);
    v.sum_items = d_items;
    v.layer_items = d_litems;
    v.n_sum_items = static_cast<int>(items.size() / 3);

    cudaStream_t s = as_stream(stream);
    auto cu = [&](cudaError_t e, const char* what) -> osp_status {
        return e == cudaSuccess ? OSP_OK : cuda_fail(e, what);
    };
    if ((st = cu(cudaMemcpyAsync(d_tb, tile_base.data(), (L + 1) * sizeof(int),
                                 cudaMemcpyHostToDevice, s), "tile_base")) != OSP_OK)
        return cleanup(st);
    if ((st = cu(cudaMemcpyAsync(d_tl, tile_layer.data(), nt_total * sizeof(int),
                                 cudaMemcpyHostToDevice, s), "tile_layer")) != OSP_OK)
        return cleanup(st);
    if (!items.empty() &&
        (st = cu(cudaMemcpyAsync(d_items, items.data(), items.size() * sizeof(int),
                                 cudaMemcpyHostToDevice, s), "sum items")) != OSP_OK)
        return cleanup(st);
    if ((st = cu(cudaMemcpyAsync(d_litems, layer_items.data(), (L + 1) * sizeof(int),
                                 cudaMemcpyHostToDevice, s), "layer items")) != OSP_OK)
        return cleanup(st);
    if (init_params) {
        st = cu(cudaMemcpyAsync(v.G, init_params, M * 4, cudaMemcpyDeviceToDevice, s), "init G");
        for (int w = 0; w < N && st == OSP_OK; ++w)
            st = cu(cudaMemcpyAsync(v.P + static_cast<uint64_t>(w) * v.ldP, init_params, M * 4,
                                    cudaMemcpyDeviceToDevice, s), "init P");
    } else {
        st = cu(cudaMemsetAsync(v.G, 0, M * 4, s), "zero G");
        if (st == OSP_OK) st = cu(cudaMemsetAsync(v.P, 0, v.ldP * N * 4, s), "zero P");
    }
    if (st != OSP_OK) return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.partials, 0, nt_total * 8, s), "partials")) != OSP_OK)
        return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.flags, 0, L, s), "flags")) != OSP_OK) return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.marked, 0, L, s), "marked")) != OSP_OK) return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.sched, 0, 16 * sizeof(int), s), "sched")) != OSP_OK)
        return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.lscore, 0, L * sizeof(double), s), "lscore")) != OSP_OK)
        return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.hist, 0, kHist * 8, s), "hist")) != OSP_OK) return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.meta, 0, 8 * sizeof(int), s), "meta")) != OSP_OK)
        return cleanup(st);
    if ((st = cu(cudaMemsetAsync(v.meta64, 0, 8 * sizeof(uint64_t), s), "meta64")) != OSP_OK)
        return cleanup(st);
    // bootstrap GIB: nothing deferred, tag 0 (first_iteration_bootstrap, protocol.cpp:58-63)
    if ((st = cu(launch_install_gib(v, g->d_order_tmp, 0, 0, s), "install bootstrap gib")) != OSP_OK)
        return cleanup(st);
    if (use_tma && !(cfg->flags & OSP_GROUP_NO_CARRY)) {
        if ((st = dalloc(g, &v.C, M)) != OSP_OK) return cleanup(st);
        const int ns = snap_ints(static_cast<int>(L), cfg->n_chunks);
        if ((st = dalloc(g, &v.snap, ns)) != OSP_OK) return cleanup(st);
        if ((st = cu(cudaMemsetAsync(v.snap, 0, ns * sizeof(int), s), "snap")) != OSP_OK)
            return cleanup(st);
    }
    g->small = v.C != nullptr && small_step_supported(N, static_cast<int>(L), M) &&
               !(cfg->flags & OSP_GROUP_NO_SMALL);
    g->blocks_per_sm = stage_blocks_per_sm(N, static_cast<int>(L));
    g->tma = use_tma;
    g->grid = sm_count() * g->blocks_per_sm;
    if ((st = cu(cudaStreamSynchronize(s), "group create")) != OSP_OK) return cleanup(st);
    *out = g;
    return OSP_OK;
}

void osp_group_destroy(osp_group* g) {
    if (!g) return;
    cudaDeviceSynchronize();
    for (void* p : g->owned) cudaFree(p);
    if (g->d_staging) cudaFree(g->d_staging);
    for (int b = 0; b < 2; ++b) {
        if (g->d_stage2[b]) cudaFree(g->d_stage2[b]);
        if (g->ev_h2d[b]) cudaEventDestroy(g->ev_h2d[b]);
        if (g->ev_used[b]) cudaEventDestroy(g->ev_used[b]);
    }
    if (g->ev_d2h) cudaEventDestroy(g->ev_d2h);
    if (g->s_h2d) cudaStreamDestroy(g->s_h2d);
    if (g->s_d2h) cudaStreamDestroy(g->s_d2h);
    delete g;
}

osp_status osp_group_set_budget(osp_group* g, uint64_t budget, void* stream) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    OSP_CUDA(launch_set_budget(g->v, budget, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_group_set_gib(osp_group* g, const uint8_t* flags, const int32_t* order,
                             int64_t n_order, uint32_t tag, void* stream) {
    if (!g || !flags) return fail(OSP_ERR_INVALID, "null argument");
    if (g->s1_open)
        return fail(OSP_ERR_PROTOCOL, "GIB install between stage 1 and the resolve of an iteration");
    if (n_order < 0 || n_order > g->v.L)
        return fail(OSP_ERR_INVALID, "rank order longer than the layer count");
    cudaStream_t s = as_stream(stream);
    std::vector<uint8_t> f(flags, flags + g->v.L);
    for (auto& x : f) x = x ? 1 : 0;
    OSP_CUDA(cudaMemcpyAsync(g->v.flags, f.data(), g->v.L, cudaMemcpyHostToDevice, s));
    if (n_order > 0)
        OSP_CUDA(cudaMemcpyAsync(g->d_order_tmp, order, n_order * sizeof(int32_t),
                                 cudaMemcpyHostToDevice, s));
    OSP_CUDA(launch_install_gib(g->v, g->d_order_tmp, static_cast<int>(n_order), tag, s));
    OSP_CUDA(cudaStreamSynchronize(s));  // host vectors are released on return
    return OSP_OK;
}

osp_status osp_group_stage1(osp_group* g, const float* deltas, uint64_t ld, void* stream) {
    OSP_RANGE("osp_group_stage1 (barrier: RS + LGP partial)");
    if (!g || !deltas) return fail(OSP_ERR_INVALID, "null argument");
    if (ld < g->part->total) return fail(OSP_ERR_SHAPE, "delta rows shorter than the partition");
    if (g->tma) OSP_CUDA(launch_stage1_tma(g->v, g->ap, deltas, ld, as_stream(stream)));
    else OSP_CUDA(launch_stage1(g->v, g->ap, deltas, ld, g->grid, as_stream(stream)));
    g->s1_open = true;
    return OSP_OK;
}

static osp_status need_stage1(const osp_group* g) {
    if (!g->s1_open)
        return fail(OSP_ERR_PROTOCOL, "stage 2 before stage 1 of this iteration");
    return OSP_OK;
}

osp_status osp_group_stage2_chunk(osp_group* g, int chunk, const float* deltas, uint64_t ld,
                                  void* stream) {
    OSP_RANGE("osp_group_stage2_chunk (ICS)");
    if (!g || !deltas) return fail(OSP_ERR_INVALID, "null argument");
    if (chunk < 0 || chunk >= g->n_chunks) return fail(OSP_ERR_INVALID, "chunk out of range");
    if (ld < g->part->total) return fail(OSP_ERR_SHAPE, "delta rows shorter than the partition");
    OSP_TRY(need_stage1(g));
    if (g->v.V) deltas = g->v.V, ld = g->v.ldP;  // momentum: stage 1 left v' there
    if (g->tma) OSP_CUDA(launch_stage2_tma(g->v, g->ap, deltas, ld, chunk, chunk + 1, as_stream(stream)));
    else OSP_CUDA(launch_stage2(g->v, g->ap, deltas, ld, chunk, chunk + 1, g->grid, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_group_stage2_all(osp_group* g, const float* deltas, uint64_t ld, void* stream) {
    OSP_RANGE("osp_group_stage2_all (ICS)");
    if (!g || !deltas) return fail(OSP_ERR_INVALID, "null argument");
    if (ld < g->part->total) return fail(OSP_ERR_SHAPE, "delta rows shorter than the partition");
    OSP_TRY(need_stage1(g));
    if (g->v.V) deltas = g->v.V, ld = g->v.ldP;
    if (g->tma) OSP_CUDA(launch_stage2_tma(g->v, g->ap, deltas, ld, 0, g->n_chunks, as_stream(stream)));
    else OSP_CUDA(launch_stage2(g->v, g->ap, deltas, ld, 0, g->n_chunks, g->grid, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_group_resolve(osp_group* g, const float* deltas, uint64_t ld, void* stream) {
    OSP_RANGE("osp_group_resolve (PGP -> GIB)");
    if (!g || !deltas) return fail(OSP_ERR_INVALID, "null argument");
    if (g->v.V) deltas = g->v.V, ld = g->v.ldP;  // the exact fallback re-aggregates v'
    OSP_CUDA(launch_resolve(g->v, g->ap, deltas, ld, as_stream(stream)));
    g->s1_open = false;
    return OSP_OK;
}

osp_status osp_group_set_momentum(osp_group* g, double mu, void* stream) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    if (!(mu >= 0.0 && mu < 1.0)) return fail(OSP_ERR_CONFIG, "momentum must be in [0, 1)");
    cudaStream_t s = as_stream(stream);
    if (mu == 0.0) {  // plain sgd_delta (bit-identical to a group that never had momentum)
        if (g->v.V) {
            OSP_CUDA(cudaStreamSynchronize(s));
            auto it = std::find(g->owned.begin(), g->owned.end(), static_cast<void*>(g->v.V));
            if (it != g->owned.end()) g->owned.erase(it);
            cudaFree(g->v.V);
        }
        g->v.V = nullptr;
        g->v.mu = 0.0f;
        return OSP_OK;
    }
    if (!(g->sgd_lr > 0)) return fail(OSP_ERR_CONFIG, "momentum needs gradient inputs (sgd_lr > 0)");
    if (!g->tma) return fail(OSP_ERR_INVALID, "momentum needs the TMA-staged stage kernels");
    if (!tma_momentum_supported(g->N, g->v.T, g->v.L))
        return fail(OSP_ERR_INVALID, "momentum: the velocity rows do not fit the shared-memory "
                                     "ring at this tile size (tile_elems <= 1024 for 8 workers)");
    if (!g->v.V) {
        osp_status st = dalloc(g, &g->v.V, g->v.ldP * g->N);
        if (st != OSP_OK) return st;
        OSP_CUDA(cudaMemsetAsync(g->v.V, 0, g->v.ldP * g->N * 4, s));
    }
    g->v.mu = static_cast<float>(mu);
    return OSP_OK;
}

osp_status osp_group_stages(osp_group* g, const float* deltas, uint64_t ld, void* stream) {
    OSP_TRY(osp_group_stage1(g, deltas, ld, stream));
    return osp_group_stage2_all(g, deltas, ld, stream);
}

osp_status osp_group_stage2_resolve(osp_group* g, const float* deltas, uint64_t ld, void* stream) {
    OSP_RANGE("osp_group_stage2_resolve");
    if (!g || !deltas) return fail(OSP_ERR_INVALID, "null argument");
    if (ld < g->part->total) return fail(OSP_ERR_SHAPE, "delta rows shorter than the partition");
    OSP_TRY(need_stage1(g));
    if (!g->v.C) {
        OSP_TRY(osp_group_stage2_all(g, deltas, ld, stream));
        return osp_group_resolve(g, deltas, ld, stream);
    }
    // carry: every tile partial is known after stage 1, so the resolve goes
    // first and the stage-2 broadcast runs beside it (joined before it retires)
    cudaStream_t s = as_stream(stream);
    if (g->v.V) deltas = g->v.V, ld = g->v.ldP;
    OSP_CUDA(launch_resolve(g->v, g->ap, deltas, ld, s));
    OSP_CUDA(launch_stage2_tma(g->v, g->ap, deltas, ld, 0, g->n_chunks, s, 1));
    g->s1_open = false;
    return OSP_OK;
}

osp_status osp_group_step(osp_group* g, const float* deltas, uint64_t ld, void* stream) {
    OSP_RANGE("osp_group_step");
    if (g && deltas && g->small && !g->v.V && !g->s1_open) {
        if (ld < g->part->total) return fail(OSP_ERR_SHAPE, "delta rows shorter than the partition");
        OSP_CUDA(launch_step_small(g->v, g->ap, deltas, ld, as_stream(stream)));
        return OSP_OK;
    }
    OSP_TRY(osp_group_stage1(g, deltas, ld, stream));
    return osp_group_stage2_resolve(g, deltas, ld, stream);
}

osp_status osp_group_step_host(osp_group* g, const float* host_deltas, uint64_t host_ld,
                               uint8_t* gib_out, float* params_out, void* stream) {
    OSP_RANGE("osp_group_step_host");
    if (!g || !host_deltas) return fail(OSP_ERR_INVALID, "null argument");
    const uint64_t M = g->part->total;
    if (host_ld < M) return fail(OSP_ERR_SHAPE, "delta rows shorter than the partition");
    cudaStream_t s = as_stream(stream);
    if (!g->d_staging) OSP_CUDA(cudaMalloc(&g->d_staging, g->v.ldP * g->N * 4));
    OSP_CUDA(cudaMemcpy2DAsync(g->d_staging, g->v.ldP * 4, host_deltas, host_ld * 4, M * 4, g->N,
                               cudaMemcpyHostToDevice, s));
    OSP_TRY(osp_group_step(g, g->d_staging, g->v.ldP, stream));
    if (gib_out)
        OSP_CUDA(cudaMemcpyAsync(gib_out, g->v.gib_bytes, osp_gib_encoded_size(g->v.L),
                                 cudaMemcpyDeviceToHost, s));
    if (params_out)
        OSP_CUDA(cudaMemcpyAsync(params_out, g->v.G, M * 4, cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaStreamSynchronize(s));
    return OSP_OK;
}

// Pipelined host step: call k's H2D (copy stream, staging buffer k % 2) runs
// beside call k-1's step and D2H; the step waits for its rows and for the
// previous D2H of the global vector (which it is about to update); the D2H of
// its GIB and global vector runs on a third stream.
osp_status osp_group_step_host_async(osp_group* g, const float* host_deltas, uint64_t host_ld,
                                     uint8_t* gib_out, float* params_out, void* stream) {
    OSP_RANGE("osp_group_step_host_async");
    if (!g || !host_deltas) return fail(OSP_ERR_INVALID, "null argument");
    const uint64_t M = g->part->total;
    if (host_ld < M) return fail(OSP_ERR_SHAPE, "delta rows shorter than the partition");
    cudaStream_t s = as_stream(stream);
    if (!g->s_h2d) {
        OSP_CUDA(cudaStreamCreateWithFlags(&g->s_h2d, cudaStreamNonBlocking));
        OSP_CUDA(cudaStreamCreateWithFlags(&g->s_d2h, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            OSP_CUDA(cudaMalloc(&g->d_stage2[b], g->v.ldP * g->N * 4));
            OSP_CUDA(cudaEventCreateWithFlags(&g->ev_h2d[b], cudaEventDisableTiming));
            OSP_CUDA(cudaEventCreateWithFlags(&g->ev_used[b], cudaEventDisableTiming));
        }
        OSP_CUDA(cudaEventCreateWithFlags(&g->ev_d2h, cudaEventDisableTiming));
    }
    const int b = static_cast<int>(g->n_async & 1);
    if (g->n_async >= 2) OSP_CUDA(cudaStreamWaitEvent(g->s_h2d, g->ev_used[b], 0));  // step k-2 read it
    OSP_CUDA(cudaMemcpy2DAsync(g->d_stage2[b], g->v.ldP * 4, host_deltas, host_ld * 4, M * 4, g->N,
                               cudaMemcpyHostToDevice, g->s_h2d));
    OSP_CUDA(cudaEventRecord(g->ev_h2d[b], g->s_h2d));
    OSP_CUDA(cudaStreamWaitEvent(s, g->ev_h2d[b], 0));
    if (g->n_async >= 1) OSP_CUDA(cudaStreamWaitEvent(s, g->ev_d2h, 0));
    OSP_TRY(osp_group_step(g, g->d_stage2[b], g->v.ldP, stream));
    OSP_CUDA(cudaEventRecord(g->ev_used[b], s));
    OSP_CUDA(cudaStreamWaitEvent(g->s_d2h, g->ev_used[b], 0));
    if (gib_out)
        OSP_CUDA(cudaMemcpyAsync(gib_out, g->v.gib_bytes, osp_gib_encoded_size(g->v.L),
                                 cudaMemcpyDeviceToHost, g->s_d2h));
    if (params_out)
        OSP_CUDA(cudaMemcpyAsync(params_out, g->v.G, M * 4, cudaMemcpyDeviceToHost, g->s_d2h));
    OSP_CUDA(cudaEventRecord(g->ev_d2h, g->s_d2h));
    g->n_async += 1;
    return OSP_OK;
}

osp_status osp_group_host_wait(osp_group* g) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    if (g->s_d2h) OSP_CUDA(cudaStreamSynchronize(g->s_d2h));
    if (g->s_h2d) OSP_CUDA(cudaStreamSynchronize(g->s_h2d));
    return OSP_OK;
}

float* osp_group_global(osp_group* g) { return g ? g->v.G : nullptr; }
float* osp_group_worker_params(osp_group* g, uint64_t* ld) {
    if (!g) return nullptr;
    if (ld) *ld = g->v.ldP;
    return g->v.P;
}
double* osp_group_scores(osp_group* g) { return g ? g->v.scores : nullptr; }

osp_status osp_group_read_gib(osp_group* g, uint8_t* flags, int32_t* order, int64_t* n_order,
                              int32_t* chunk_of, int* n_used, uint32_t* tag, uint64_t* deferred,
                              void* stream) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    cudaStream_t s = as_stream(stream);
    int meta[8];
    uint64_t meta64[8];
    OSP_CUDA(cudaMemcpyAsync(meta, g->v.meta, sizeof meta, cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaMemcpyAsync(meta64, g->v.meta64, sizeof meta64, cudaMemcpyDeviceToHost, s));
    if (flags) OSP_CUDA(cudaMemcpyAsync(flags, g->v.flags, g->v.L, cudaMemcpyDeviceToHost, s));
    if (chunk_of)
        OSP_CUDA(cudaMemcpyAsync(chunk_of, g->v.chunk_of, g->v.L * 4, cudaMemcpyDeviceToHost, s));
    std::vector<int32_t> ord(g->v.L);
    if (order) OSP_CUDA(cudaMemcpyAsync(ord.data(), g->v.ics_layers, g->v.L * 4,
                                        cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaStreamSynchronize(s));
    const int k = meta[META_N_ICS];
    if (order) std::copy(ord.begin(), ord.begin() + k, order);
    if (n_order) *n_order = k;
    if (n_used) *n_used = meta[META_N_USED];
    if (tag) *tag = static_cast<uint32_t>(meta64[META64_TAG]);
    if (deferred) *deferred = meta64[META64_DEFERRED];
    return OSP_OK;
}

osp_status osp_group_gib_wire(osp_group* g, uint8_t* out, uint64_t cap, uint64_t* len,
                              void* stream) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    cudaStream_t s = as_stream(stream);
    const uint64_t L = static_cast<uint64_t>(g->v.L);
    std::vector<uint8_t> w(osp_gib_wire_size(L, L));
    OSP_CUDA(cudaMemcpyAsync(w.data(), g->v.gib_bytes, w.size(), cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaStreamSynchronize(s));
    const uint64_t k = get_u32le(w.data() + osp_gib_encoded_size(L));
    const uint64_t need = osp_gib_wire_size(L, k);
    if (len) *len = need;
    if (!out) return OSP_OK;
    if (cap < need) return fail(OSP_ERR_INVALID, "gib wire buffer too small");
    std::memcpy(out, w.data(), need);
    return OSP_OK;
}

const uint8_t* osp_group_gib_wire_device(const osp_group* g, uint64_t* max_len) {
    if (!g) return nullptr;
    if (max_len) *max_len = osp_gib_wire_size(g->v.L, g->v.L);
    return g->v.gib_bytes;
}

osp_status osp_group_set_gib_wire(osp_group* g, const uint8_t* buf, uint64_t len, void* stream) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    uint32_t tag = 0, L = 0;
    int64_t n = 0;
    OSP_TRY(osp_gib_wire_decode(buf, len, &tag, &L, nullptr, 0, nullptr, 0, &n));
    if (static_cast<int>(L) != g->v.L)
        return fail(OSP_ERR_SHAPE, "gib covers " + std::to_string(L) + " layers, the group " +
                                       std::to_string(g->v.L));
    std::vector<uint8_t> f(L);
    std::vector<int32_t> ord(L);
    OSP_TRY(osp_gib_wire_decode(buf, len, nullptr, nullptr, f.data(), L, ord.data(), L, &n));
    // bitmap-only wire: the reference's convention for a missing order (ascending
    // ids, split_for_sync's "missing ids appended ascending", protocol.cpp:122-166)
    return osp_group_set_gib(g, f.data(), ord.data(), n < 0 ? 0 : n, tag, stream);
}

osp_status osp_group_stats(osp_group* g, uint64_t* resolved, uint64_t* fb_layers,
                           uint64_t* fb_resolves, void* stream) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    uint64_t meta64[8];
    cudaStream_t s = as_stream(stream);
    OSP_CUDA(cudaMemcpyAsync(meta64, g->v.meta64, sizeof meta64, cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaStreamSynchronize(s));
    if (resolved) *resolved = meta64[META64_RESOLVED];
    if (fb_layers) *fb_layers = meta64[META64_FB_LAYERS];
    if (fb_resolves) *fb_resolves = meta64[META64_FB_RESOLVES];
    return OSP_OK;
}

osp_status osp_group_deferred_history(osp_group* g, uint32_t first_tag, int n, uint64_t* out,
                                      void* stream) {
    if (!g || !out) return fail(OSP_ERR_INVALID, "null argument");
    if (n < 0 || n > kHist) return fail(OSP_ERR_INVALID, "history window out of range");
    std::vector<uint64_t> h(kHist);
    cudaStream_t s = as_stream(stream);
    OSP_CUDA(cudaMemcpyAsync(h.data(), g->v.hist, kHist * 8, cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaStreamSynchronize(s));
    for (int i = 0; i < n; ++i) out[i] = h[(first_tag + i) % kHist];
    return OSP_OK;
}

uint32_t osp_group_flags(const osp_group* g) {
    if (!g) return 0;
    return (g->tma ? OSP_GROUP_TMA : OSP_GROUP_REGISTER) | (g->v.C ? 0u : OSP_GROUP_NO_CARRY) |
           (g->small && !g->v.V ? OSP_GROUP_SMALL : 0u);
}

osp_status osp_group_geometry(osp_group* g, uint32_t* tile_elems, uint64_t* n_tiles,
                              int* grid_blocks, int* block_threads) {
    if (!g) return fail(OSP_ERR_INVALID, "null group");
    if (tile_elems) *tile_elems = static_cast<uint32_t>(g->v.T);
    if (n_tiles) *n_tiles = static_cast<uint64_t>(g->v.NT);
    if (grid_blocks) *grid_blocks = g->grid;
    if (block_threads) *block_threads = kStageThreads;
    return OSP_OK;
}

}  // extern "C"
