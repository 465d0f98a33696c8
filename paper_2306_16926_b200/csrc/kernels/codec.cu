// Payload wire codec on the device: the reference's
// encode_payload_message / decode_payload_message (message.cpp:53-99) for
// layer payloads that live in device memory, so a byte transport can send
// straight from HBM. Layout: kind u8 | iteration u32 LE | entries u16 LE |
// per layer: id u32 LE, count u32 LE, count x fp32 LE. Value regions start at
// odd byte offsets, so values are written/read bytewise (coalesced per warp).

#include "common.cuh"

namespace osp {
namespace {

__device__ __forceinline__ void put32(uint8_t* p, uint32_t v) {
    p[0] = v & 0xff;
    p[1] = (v >> 8) & 0xff;
    p[2] = (v >> 16) & 0xff;
    p[3] = (v >> 24) & 0xff;
}

__device__ __forceinline__ uint32_t get32(const uint8_t* p) {
    return uint32_t(p[0]) | (uint32_t(p[1]) << 8) | (uint32_t(p[2]) << 16) | (uint32_t(p[3]) << 24);
}

// The 7-byte message header is written by the host (osp_encode_payload).
__global__ void k_encode(const float* __restrict__ values, const CodecSeg* __restrict__ segs,
                         uint8_t* __restrict__ out) {
    const CodecSeg sg = segs[blockIdx.y];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        put32(out + sg.hdr, sg.id);
        put32(out + sg.hdr + 4, sg.count);
    }
    uint8_t* dst = out + sg.hdr + 8;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < sg.count;
         i += uint64_t(gridDim.x) * blockDim.x)
        put32(dst + 4 * i, __float_as_uint(values[sg.src + i]));
}

// Single thread walks the entry headers: idx[e] = (id, count, value byte offset);
// status: 0 ok, 1 header truncated, 2 entry header truncated, 3 values truncated,
// 4 trailing bytes.
__global__ void k_decode_index(const uint8_t* __restrict__ buf, uint64_t len, uint64_t* idx,
                               int* status, uint32_t* hdr) {
    if (len < 7) {
        *status = 1;
        return;
    }
    hdr[0] = buf[0];
    hdr[1] = get32(buf + 1);
    const uint32_t entries = buf[5] | (buf[6] << 8);
    hdr[2] = entries;
    uint64_t at = 7;
    for (uint32_t e = 0; e < entries; ++e) {
        if (len < at + 8) {
            *status = 2;
            return;
        }
        const uint32_t id = get32(buf + at), count = get32(buf + at + 4);
        at += 8;
        if (len < at + uint64_t(count) * 4) {
            *status = 3;
            return;
        }
        idx[3 * e] = id;
        idx[3 * e + 1] = count;
        idx[3 * e + 2] = at;
        at += uint64_t(count) * 4;
    }
    *status = at != len ? 4 : 0;
}

__global__ void k_decode_scatter(const uint8_t* __restrict__ buf, const CodecSeg* __restrict__ segs,
                                 float* __restrict__ values) {
    const CodecSeg sg = segs[blockIdx.y];
    const uint8_t* src = buf + sg.hdr;  // value region offset (decode reuses `hdr`)
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < sg.count;
         i += uint64_t(gridDim.x) * blockDim.x)
        values[sg.src + i] = __uint_as_float(get32(src + 4 * i));
}

}  // namespace

cudaError_t launch_encode(const float* values, const CodecSeg* segs_dev, int n_seg,
                          uint64_t max_count, uint8_t* out, cudaStream_t s) {
    if (n_seg == 0) return cudaSuccess;
    uint64_t bx = (max_count + 255) / 256;
    bx = bx < 1 ? 1 : (bx > 256 ? 256 : bx);
    k_encode<<<dim3(static_cast<unsigned>(bx), n_seg), 256, 0, s>>>(values, segs_dev, out);
    return cudaGetLastError();
}

cudaError_t launch_decode_index(const uint8_t* buf, uint64_t len, uint64_t* idx, int* status,
                                uint32_t* hdr, cudaStream_t s) {
    k_decode_index<<<1, 1, 0, s>>>(buf, len, idx, status, hdr);
    return cudaGetLastError();
}

cudaError_t launch_decode_scatter(const uint8_t* buf, const CodecSeg* segs_dev, int n_seg,
                                  uint64_t max_count, float* values, cudaStream_t s) {
    if (n_seg == 0) return cudaSuccess;
    uint64_t bx = (max_count + 255) / 256;
    bx = bx < 1 ? 1 : (bx > 256 ? 256 : bx);
    k_decode_scatter<<<dim3(static_cast<unsigned>(bx), n_seg), 256, 0, s>>>(buf, segs_dev, values);
    return cudaGetLastError();
}

}  // namespace osp
