// Copy-engine NVLink probe (diagnostic, P GPUs in one process): can the copy
// engines move the sharded step's rows faster than SM-issued peer loads when
// every GPU pulls from every other at once (the sharded step's pattern)?
//   A  every GPU pulls its shard's peer rows (n_loc rows, 2-D copy, pitch ldX)
//      from every peer, one copy per peer, all at once
//   B  the same in S segments (one 2-D copy per segment per peer)
//   C  B while every GPU streams an HBM copy kernel (the aggregation's traffic)
//   D  B plus the return push of the aggregate (1-D copy into every peer)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/ce_probe.cu -o gpurun_out/ce_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                       \
    do {                                                                            \
        cudaError_t e_ = (x);                                                       \
        if (e_ != cudaSuccess) {                                                    \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) b[i] = a[i];
}

int main(int argc, char** argv) {
    int P = 0;
    CK(cudaGetDeviceCount(&P));
    if (P < 2) {
        std::printf("need 2 GPUs\n");
        return 0;
    }
    const size_t M = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 25557032ull;  // ResNet-50
    const int N = 8, n_loc = N / P;
    const size_t shard = (M + P - 1) / P;
    const size_t ldX = (M + 63) / 64 * 64;
    std::printf("P=%d M=%zu n_loc=%d shard=%zu\n", P, M, n_loc, shard);
    std::vector<float*> X(P), stage(P), aggb(P), pull(P), h_a(P), h_b(P);
    std::vector<cudaStream_t> st(P * P);
    std::vector<cudaEvent_t> e0(P), e1(P);
    const size_t hbm_n4 = size_t(600) << 20 >> 4;  // 600 MB moved per GPU in C
    for (int d = 0; d < P; ++d) {
        CK(cudaSetDevice(d));
        for (int q = 0; q < P; ++q)
            if (q != d) CK(cudaDeviceEnablePeerAccess(q, 0));
        CK(cudaMalloc(&X[d], ldX * n_loc * 4));
        CK(cudaMalloc(&stage[d], shard * N * 4));
        CK(cudaMalloc(&aggb[d], shard * 4));
        CK(cudaMalloc(&pull[d], shard * P * 4));
        CK(cudaMalloc(&h_a[d], hbm_n4 * 16 / 2));
        CK(cudaMalloc(&h_b[d], hbm_n4 * 16 / 2));
        CK(cudaMemset(X[d], 0, ldX * n_loc * 4));
        for (int q = 0; q < P; ++q) CK(cudaStreamCreateWithFlags(&st[d * P + q], cudaStreamNonBlocking));
        CK(cudaEventCreate(&e0[d]));
        CK(cudaEventCreate(&e1[d]));
    }
    // the peer rows of owner d's shard from peer q: q's n_loc rows, columns [d*shard, ...)
    auto pull_seg = [&](int d, int q, size_t c0, size_t c1) {
        const size_t w = (c1 - c0) * 4;
        CK(cudaMemcpy2DAsync(stage[d] + size_t(q) * n_loc * shard + c0, shard * 4,
                             X[q] + size_t(d) * shard + c0, ldX * 4, w, n_loc,
                             cudaMemcpyDefault, st[d * P + q]));
    };
    auto push_seg = [&](int d, int q, size_t c0, size_t c1) {
        CK(cudaMemcpyAsync(pull[q] + size_t(d) * shard + c0, aggb[d] + c0, (c1 - c0) * 4,
                           cudaMemcpyDefault, st[d * P + q]));
    };
    auto run = [&](const char* name, int S, bool hbm, bool push, int reps) {
        float best = 1e30f, sum = 0.f;
        for (int r = 0; r < reps + 1; ++r) {
            for (int d = 0; d < P; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaDeviceSynchronize());
            }
            for (int d = 0; d < P; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventRecord(e0[d], st[d * P + d]));
                for (int q = 0; q < P; ++q)
                    if (q != d) CK(cudaStreamWaitEvent(st[d * P + q], e0[d], 0));
            }
            for (int d = 0; d < P; ++d) {
                CK(cudaSetDevice(d));
                if (hbm) k_copy<<<148 * 4, 512, 0, st[d * P + d]>>>(reinterpret_cast<float4*>(h_a[d]),
                                                                  reinterpret_cast<float4*>(h_b[d]),
                                                                  hbm_n4 / 2);
                for (int s = 0; s < S; ++s) {
                    const size_t c0 = shard * s / S, c1 = shard * (s + 1) / S;
                    for (int q = 0; q < P; ++q) {
                        if (q == d) continue;
                        pull_seg(d, q, c0, c1);
                        if (push) push_seg(d, q, c0, c1);
                    }
                }
            }
            for (int d = 0; d < P; ++d) {
                CK(cudaSetDevice(d));
                for (int q = 0; q < P; ++q)
                    if (q != d) {
                        cudaEvent_t e;
                        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                        CK(cudaEventRecord(e, st[d * P + q]));
                        CK(cudaStreamWaitEvent(st[d * P + d], e, 0));
                        CK(cudaEventDestroy(e));
                    }
                CK(cudaEventRecord(e1[d], st[d * P + d]));
            }
            float mx = 0.f;
            for (int d = 0; d < P; ++d) {
                CK(cudaSetDevice(d));
                CK(cudaEventSynchronize(e1[d]));
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
                mx = ms > mx ? ms : mx;
            }
            if (r > 0) {
                sum += mx;
                best = mx < best ? mx : best;
            }
        }
        const double in_bytes = double(shard) * 4 * n_loc * (P - 1);
        const double out_bytes = push ? double(shard) * 4 * (P - 1) : 0.0;
        std::printf("%-46s S=%-3d %.3f ms (best %.3f)  in %.1f GB/s/GPU, in+out %.1f GB/s/GPU\n", name, S,
                    sum / reps, best, in_bytes / (best * 1e-3) / 1e9,
                    (in_bytes + out_bytes) / (best * 1e-3) / 1e9);
    };
    run("A pull peer rows, all GPUs at once", 1, false, false, 5);
    for (int S : {4, 8, 16, 32}) run("B segmented pull", S, false, false, 5);
    for (int S : {8, 16}) run("C segmented pull + HBM copy kernel", S, true, false, 5);
    for (int S : {1, 8, 16}) run("D segmented pull + aggregate push", S, false, true, 5);
    for (int S : {8, 16}) run("E pull + push + HBM copy kernel", S, true, true, 5);
    // the HBM kernel alone
    {
        CK(cudaSetDevice(0));
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, st[0]));
        k_copy<<<148 * 4, 512, 0, st[0]>>>(reinterpret_cast<float4*>(h_a[0]), reinterpret_cast<float4*>(h_b[0]),
                                          hbm_n4 / 2);
        CK(cudaEventRecord(b, st[0]));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("HBM copy kernel alone (600 MB moved): %.3f ms\n", ms);
    }
    std::printf("done\n");
    return 0;
}
