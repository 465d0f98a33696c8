// Handle layouts shared by the C-ABI translation units (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <vector>

#include "../osp_internal.h"

struct osp_partition {
    std::vector<uint64_t> counts;
    std::vector<uint64_t> offsets;
    uint64_t total = 0;
    uint32_t bpe = 4;
    uint64_t* d_offsets = nullptr;
    uint64_t* d_counts = nullptr;
    // lazily created one-worker group whose tile tables, lists and resolve
    // buffers serve osp_pgp_rank_gib (the certified resolve of given vectors)
    struct osp_group* scratch = nullptr;
};

struct osp_group {
    const osp_partition* part = nullptr;
    int N = 0;
    int n_chunks = 1;
    double sgd_lr = 0.0;
    std::vector<double> weights;
    osp::AggParams ap{};
    osp::GroupView v{};
    int grid = 1;
    int blocks_per_sm = 1;
    bool tma = false;  // OSP_GROUP_TMA
    // stage 1 issued and the iteration not yet resolved: stage 2 needs it (the
    // carry and its list snapshot are written by stage 1), a GIB install must
    // not land between the two (the overlapped stage 2 joins on the snapshot)
    bool s1_open = false;
    bool small = false;  // osp_group_step runs as one launch (kernels/step_small.cu)
    // owned device buffers
    std::vector<void*> owned;
    int* d_order_tmp = nullptr;
    float* d_staging = nullptr;
    // osp_group_step_host_async: two staging buffers, copy streams, events
    float* d_stage2[2] = {nullptr, nullptr};
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr}, ev_used[2] = {nullptr, nullptr}, ev_d2h = nullptr;
    unsigned long long n_async = 0;
};

// NVTX range over a C-ABI call (header-only NVTX3: a no-op unless a tool such as
// nsys or ncu --nvtx is attached), so a host profile shows the sync path's
// phases by their reference names.
struct OspRange {
    explicit OspRange(const char* name) { nvtxRangePushA(name); }
    ~OspRange() { nvtxRangePop(); }
    OspRange(const OspRange&) = delete;
    OspRange& operator=(const OspRange&) = delete;
};
#define OSP_RANGE(name) OspRange osp_range_guard_(name)

#define OSP_TRY(expr)                \
    do {                             \
        osp_status s_ = (expr);      \
        if (s_ != OSP_OK) return s_; \
    } while (0)
