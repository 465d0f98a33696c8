// C-ABI of the device payload codec (kernels/codec.cu; reference message.cpp:53-99).

#include <cuda_runtime.h>

#include <cstring>
#include <string>
#include <vector>

#include "handles.h"

using namespace osp;

extern "C" {

uint64_t osp_payload_encoded_size(const osp_partition* part, const int32_t* layer_ids,
                                  int64_t n_ids) {
    if (!part) return 0;
    uint64_t n = 7;
    for (int64_t i = 0; i < n_ids; ++i) {
        const int32_t id = layer_ids[i];
        if (id < 0 || static_cast<size_t>(id) >= part->counts.size()) return 0;
        n += 8 + 4 * part->counts[id];
    }
    return n;
}

osp_status osp_encode_payload(const osp_partition* part, const float* values,
                              const int32_t* layer_ids, int64_t n_ids, uint8_t kind,
                              uint32_t iteration, uint8_t* out, uint64_t out_cap,
                              uint64_t* out_len, void* stream) {
    if (!part || !out) return fail(OSP_ERR_INVALID, "null argument");
    if (n_ids > 0xffff) return fail(OSP_ERR_FORMAT, "payload has too many layers for the wire format");
    std::vector<CodecSeg> segs;
    uint64_t at = 7, max_count = 0;
    for (int64_t i = 0; i < n_ids; ++i) {
        uint64_t off = 0, cnt = 0;
        OSP_TRY(osp_partition_layer(part, layer_ids[i], &off, &cnt));
        if (i > 0 && layer_ids[i] <= layer_ids[i - 1])
            return fail(OSP_ERR_INVALID, "layer ids must be strictly ascending (std::map order)");
        segs.push_back(CodecSeg{at, off, static_cast<uint32_t>(layer_ids[i]), static_cast<uint32_t>(cnt)});
        at += 8 + 4 * cnt;
        if (cnt > max_count) max_count = cnt;
    }
    if (at > out_cap) return fail(OSP_ERR_INVALID, "output buffer too small");
    cudaStream_t s = as_stream(stream);
    uint8_t hdr[7];
    hdr[0] = kind;
    for (int b = 0; b < 4; ++b) hdr[1 + b] = (iteration >> (8 * b)) & 0xff;
    hdr[5] = n_ids & 0xff;
    hdr[6] = (n_ids >> 8) & 0xff;
    OSP_CUDA(cudaMemcpyAsync(out, hdr, 7, cudaMemcpyHostToDevice, s));
    if (!segs.empty()) {
        CodecSeg* d = nullptr;
        OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), segs.size() * sizeof(CodecSeg), s));
        cudaError_t e = cudaMemcpyAsync(d, segs.data(), segs.size() * sizeof(CodecSeg),
                                        cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = launch_encode(values, d, static_cast<int>(segs.size()), max_count, out, s);
        cudaFreeAsync(d, s);
        if (e != cudaSuccess) return cuda_fail(e, "encode_payload");
    }
    OSP_CUDA(cudaStreamSynchronize(s));  // header staging is a stack buffer
    if (out_len) *out_len = at;
    return OSP_OK;
}

osp_status osp_decode_payload(const osp_partition* part, const uint8_t* buf, uint64_t len,
                              float* values, uint8_t* kind, uint32_t* iteration, int32_t* layer_ids,
                              int64_t ids_cap, int64_t* n_ids, void* stream) {
    if (!part || !buf) return fail(OSP_ERR_INVALID, "null argument");
    cudaStream_t s = as_stream(stream);
    uint64_t* idx = nullptr;
    int* status = nullptr;
    uint32_t* hdr = nullptr;
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&idx), 3 * 65536 * sizeof(uint64_t), s));
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&status), sizeof(int), s));
    OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&hdr), 4 * sizeof(uint32_t), s));
    int st_h = 0;
    uint32_t hdr_h[4] = {0, 0, 0, 0};
    cudaError_t e = cudaMemsetAsync(status, 0, sizeof(int), s);
    if (e == cudaSuccess) e = launch_decode_index(buf, len, idx, status, hdr, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&st_h, status, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hdr_h, hdr, sizeof hdr_h, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    std::vector<uint64_t> idx_h;
    if (e == cudaSuccess && st_h == 0 && hdr_h[2] > 0) {
        idx_h.resize(3 * hdr_h[2]);
        e = cudaMemcpy(idx_h.data(), idx, idx_h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost);
    }
    cudaFreeAsync(idx, s);
    cudaFreeAsync(status, s);
    cudaFreeAsync(hdr, s);
    if (e != cudaSuccess) return cuda_fail(e, "decode_payload");
    static const char* why[] = {"", "message header truncated", "layer entry header truncated",
                                "layer values truncated", "trailing bytes after message payload"};
    if (st_h != 0) return fail(OSP_ERR_FORMAT, why[st_h]);
    const uint32_t entries = hdr_h[2];
    if (static_cast<int64_t>(entries) > ids_cap) return fail(OSP_ERR_INVALID, "layer id buffer too small");
    std::vector<CodecSeg> segs;
    std::vector<uint8_t> seen(part->counts.size(), 0);
    uint64_t max_count = 0;
    int64_t kept = 0;
    for (uint32_t i = 0; i < entries; ++i) {
        const int64_t id = static_cast<int64_t>(idx_h[3 * i]);
        const uint64_t cnt = idx_h[3 * i + 1];
        uint64_t off = 0, lcnt = 0;
        OSP_TRY(osp_partition_layer(part, id, &off, &lcnt));
        if (cnt != lcnt)
            return fail(OSP_ERR_SHAPE, "payload layer " + std::to_string(id) + " has " +
                                           std::to_string(cnt) + " values, expected " +
                                           std::to_string(lcnt));
        if (seen[id]) continue;  // std::map::emplace keeps the first entry of an id
        seen[id] = 1;
        if (layer_ids) layer_ids[kept] = static_cast<int32_t>(id);
        ++kept;
        segs.push_back(CodecSeg{idx_h[3 * i + 2], off, static_cast<uint32_t>(id),
                                static_cast<uint32_t>(cnt)});
        if (cnt > max_count) max_count = cnt;
    }
    if (kind) *kind = static_cast<uint8_t>(hdr_h[0]);
    if (iteration) *iteration = hdr_h[1];
    if (n_ids) *n_ids = kept;
    if (!segs.empty() && values) {
        CodecSeg* d = nullptr;
        OSP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), segs.size() * sizeof(CodecSeg), s));
        e = cudaMemcpyAsync(d, segs.data(), segs.size() * sizeof(CodecSeg), cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = launch_decode_scatter(buf, d, static_cast<int>(segs.size()), max_count, values, s);
        cudaFreeAsync(d, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) return cuda_fail(e, "decode_payload");
    }
    return OSP_OK;
}

}  // extern "C"
