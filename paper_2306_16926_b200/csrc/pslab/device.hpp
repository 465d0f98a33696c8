// Internal helpers of the pslab façade: status -> exception mapping and a small
// RAII device buffer over the C-ABI (no CUDA headers needed here).
#pragma once

#include <algorithm>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "osp_c.h"
#include "pslab/errors.hpp"

namespace pslab_b200 {

[[noreturn]] void throw_status(osp_status s);

inline void check(osp_status s) {
    if (s != OSP_OK) throw_status(s);
}

// Caching device allocator for the façade's buffers (device.cpp). The reference
// API creates and drops per-iteration state (an OspServer round holds N
// contribution vectors of the whole model); cudaMalloc / cudaFree per round
// cost milliseconds and cudaFree synchronises the device. Freed blocks are
// kept per size class and handed out again. Safe because all façade work is
// ordered on the legacy default stream: a block's next owner can only enqueue
// work after everything its previous owner enqueued.
void* pool_alloc(size_t bytes, size_t* cls);
void pool_free(void* p, size_t cls);

// Device float buffer. All façade work runs on the legacy default stream, so a
// download is ordered after every kernel that produced the data.
class DevBuf {
public:
    DevBuf() = default;
    explicit DevBuf(size_t n) { reset(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept
        : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)), cls_(std::exchange(o.cls_, 0)) {}
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p_ = std::exchange(o.p_, nullptr);
            n_ = std::exchange(o.n_, 0);
            cls_ = std::exchange(o.cls_, 0);
        }
        return *this;
    }
    ~DevBuf() { release(); }

    void reset(size_t n) {
        release();
        p_ = static_cast<float*>(pool_alloc(std::max<size_t>(n, 1) * sizeof(float), &cls_));
        n_ = n;
    }
    void zero() { check(osp_memset(p_, 0, std::max<size_t>(n_, 1) * sizeof(float), nullptr)); }
    float* data() const { return p_; }
    size_t size() const { return n_; }
    void upload(const float* src, size_t n, size_t at = 0) {
        if (n) check(osp_memcpy_h2d(p_ + at, src, n * sizeof(float), nullptr));
    }
    void upload(const std::vector<float>& v, size_t at = 0) { upload(v.data(), v.size(), at); }
    void download(float* dst, size_t n, size_t at = 0) const {
        if (n) check(osp_memcpy_d2h(dst, p_ + at, n * sizeof(float), nullptr));
    }
    std::vector<float> slice(size_t at, size_t n) const {
        std::vector<float> out(n);
        download(out.data(), n, at);
        return out;
    }

private:
    void release() {
        if (p_) pool_free(p_, cls_);
        p_ = nullptr;
        n_ = 0;
    }
    float* p_ = nullptr;
    size_t n_ = 0;
    size_t cls_ = 0;
};

}  // namespace pslab_b200
