// NVLink peer-memory probe (diagnostic, 2 GPUs in one process): read bandwidth
// of LDG.128 vs cp.async.bulk (UBLKCP) from a peer buffer, remote-store
// bandwidth of STG.128 into a peer buffer, and cudaMemcpyPeerAsync, each alone
// and while the local GPU streams HBM. Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/nvlink_probe.cu -o gpurun_out/nvlink_probe
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            std::printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
            std::exit(1);                                                             \
        }                                                                             \
    } while (0)

__global__ void k_ldg(const float4* __restrict__ src, size_t n4, float* sink) {
    float acc = 0.f;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < n4; i += 4 * stride) {
        float4 a = src[i], b = src[i + stride], c = src[i + 2 * stride], d = src[i + 3 * stride];
        acc += a.x + b.y + c.z + d.w;
    }
    for (; i < n4; i += stride) acc += src[i].x;
    if (acc == 12345.f) *sink = acc;
}

__global__ void k_stg(float4* dst, size_t n4) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride)
        dst[i] = make_float4(1.f, 2.f, 3.f, float(i));
}

__device__ __forceinline__ unsigned sa(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// each CTA: ring of S stages of B bytes, one thread issues bulk copies
template <int S>
__global__ void k_bulk(const char* src, size_t bytes, int B, float* sink) {
    extern __shared__ __align__(128) char sm[];
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(sm + size_t(S) * B);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const size_t nchunks = bytes / B;
    int it = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const int s = it % S;
        if (it >= S) {
            const unsigned par = ((it / S) - 1) & 1;
            unsigned ok = 0;
            while (!ok)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 "
                    "%0, 1, 0, p; }"
                    : "=r"(ok)
                    : "r"(sa(&bar[s])), "r"(par)
                    : "memory");
        }
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[s])),
                     "r"(B)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                sa(sm + size_t(s) * B)),
            "l"(src + c * B), "r"(B), "r"(sa(&bar[s]))
            : "memory");
    }
    // drain
    for (int k = it - S < 0 ? 0 : it - S; k < it; ++k) {
        const int s = k % S;
        const unsigned par = (k / S) & 1;
        unsigned ok = 0;
        while (!ok)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, "
                "1, 0, p; }"
                : "=r"(ok)
                : "r"(sa(&bar[s])), "r"(par)
                : "memory");
    }
    if (reinterpret_cast<float*>(sm)[0] == 12345.f) *sink = 1.f;
}

// local HBM copy (background load)
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n4) {
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += stride) b[i] = a[i];
}

int main() {
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n < 2) {
        std::printf("need 2 GPUs\n");
        return 0;
    }
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t bytes = size_t(1) << 30;  // 1 GiB
    float *src1, *dst1, *loc_a, *loc_b, *sink;
    CK(cudaSetDevice(1));
    CK(cudaMalloc(&src1, bytes));
    CK(cudaMalloc(&dst1, bytes));
    CK(cudaMemset(src1, 0, bytes));
    CK(cudaSetDevice(0));
    CK(cudaDeviceEnablePeerAccess(1, 0));
    CK(cudaMalloc(&loc_a, bytes));
    CK(cudaMalloc(&loc_b, bytes));
    CK(cudaMalloc(&sink, 4));
    CK(cudaMemset(loc_a, 0, bytes));
    cudaStream_t s0, s1;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const size_t n4 = bytes / 16;
    auto time = [&](auto fn, const char* name, double moved) {
        fn();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(a, s0));
        for (int r = 0; r < 5; ++r) fn();
        CK(cudaEventRecord(b, s0));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("%-44s %8.1f GB/s  (%.3f ms)\n", name, moved * 5 / (ms * 1e-3) / 1e9, ms / 5);
    };
    for (int per_sm : {1, 2, 4, 8}) {
        char nm[64];
        std::snprintf(nm, sizeof nm, "peer LDG.128 read, %d CTA/SM x 256", per_sm);
        time([&] { k_ldg<<<sms * per_sm, 256, 0, s0>>>((const float4*)src1, n4, sink); }, nm,
             double(bytes));
    }
    for (int B : {4096, 16384}) {
        for (int per_sm : {1, 2, 4}) {
            const int S = 4;
            const size_t smem = size_t(S) * B + 64;
            CK(cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            char nm[80];
            std::snprintf(nm, sizeof nm, "peer bulk read %dB x4 stages, %d CTA/SM", B, per_sm);
            time([&] { k_bulk<4><<<sms * per_sm, 32, smem, s0>>>((const char*)src1, bytes, B, sink); },
                 nm, double(bytes));
        }
    }
    for (int per_sm : {1, 2, 4}) {
        char nm[64];
        std::snprintf(nm, sizeof nm, "peer STG.128 write, %d CTA/SM x 256", per_sm);
        time([&] { k_stg<<<sms * per_sm, 256, 0, s0>>>((float4*)dst1, n4); }, nm, double(bytes));
    }
    time([&] { CK(cudaMemcpyPeerAsync(loc_b, 0, src1, 1, bytes, s0)); }, "cudaMemcpyPeerAsync 1->0 (pull)",
         double(bytes));
    time([&] { CK(cudaMemcpyPeerAsync(dst1, 1, loc_a, 0, bytes, s0)); }, "cudaMemcpyPeerAsync 0->1 (push)",
         double(bytes));
    time([&] { k_copy<<<sms * 4, 256, 0, s0>>>((const float4*)loc_a, (float4*)loc_b, n4); },
         "local HBM copy (read+write bytes)", 2.0 * bytes);
    // concurrency: peer bulk read on s0 with a local HBM copy on s1
    {
        const int B = 16384, S = 4;
        const size_t smem = size_t(S) * B + 64;
        CK(cudaEventRecord(a, s0));
        for (int r = 0; r < 5; ++r) {
            k_bulk<4><<<sms, 32, smem, s0>>>((const char*)src1, bytes, B, sink);
            k_copy<<<sms * 2, 256, 0, s1>>>((const float4*)loc_a, (float4*)loc_b, n4);
        }
        cudaEvent_t c;
        CK(cudaEventCreate(&c));
        CK(cudaEventRecord(c, s1));
        CK(cudaStreamWaitEvent(s0, c));
        CK(cudaEventRecord(b, s0));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        std::printf("concurrent: peer bulk 1 GiB + local copy 1 GiB  %.3f ms per pair\n", ms / 5);
    }
    // bidirectional: GPU0 reads GPU1 while GPU1 reads GPU0 (bulk 16 KB x4, 1 CTA/SM)
    {
        float *src0 = nullptr;
        CK(cudaSetDevice(1));
        CK(cudaDeviceEnablePeerAccess(0, 0));
        cudaStream_t t1;
        CK(cudaStreamCreateWithFlags(&t1, cudaStreamNonBlocking));
        float* sink1;
        CK(cudaMalloc(&sink1, 4));
        const int B = 16384, S = 4;
        const size_t smem = size_t(S) * B + 64;
        CK(cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        CK(cudaSetDevice(0));
        src0 = loc_a;
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaDeviceSynchronize());
            CK(cudaSetDevice(1));
            CK(cudaDeviceSynchronize());
            CK(cudaSetDevice(0));
            cudaEvent_t a0, b0;
            CK(cudaEventCreate(&a0));
            CK(cudaEventCreate(&b0));
            CK(cudaEventRecord(a0, s0));
            for (int r = 0; r < 5; ++r) {
                CK(cudaSetDevice(0));
                k_bulk<4><<<sms, 32, smem, s0>>>((const char*)src1, bytes, B, sink);
                CK(cudaSetDevice(1));
                k_bulk<4><<<sms, 32, smem, t1>>>((const char*)src0, bytes, B, sink1);
            }
            CK(cudaSetDevice(0));
            CK(cudaEventRecord(b0, s0));
            CK(cudaEventSynchronize(b0));
            CK(cudaSetDevice(1));
            CK(cudaStreamSynchronize(t1));
            CK(cudaSetDevice(0));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, a0, b0));
            std::printf("bidirectional bulk reads (both GPUs)            %8.1f GB/s per direction (GPU0 view)\n",
                        double(bytes) * 5 / (ms * 1e-3) / 1e9);
        }
        // GPU0 reads GPU1 (LDG) while GPU1 also reads GPU0 (LDG)
        CK(cudaDeviceSynchronize());
        cudaEvent_t a0, b0;
        CK(cudaEventCreate(&a0));
        CK(cudaEventCreate(&b0));
        CK(cudaEventRecord(a0, s0));
        for (int r = 0; r < 5; ++r) {
            CK(cudaSetDevice(0));
            k_ldg<<<sms * 2, 256, 0, s0>>>((const float4*)src1, n4, sink);
            CK(cudaSetDevice(1));
            k_ldg<<<sms * 2, 256, 0, t1>>>((const float4*)src0, n4, sink1);
        }
        CK(cudaSetDevice(0));
        CK(cudaEventRecord(b0, s0));
        CK(cudaEventSynchronize(b0));
        CK(cudaSetDevice(1));
        CK(cudaStreamSynchronize(t1));
        CK(cudaSetDevice(0));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a0, b0));
        std::printf("bidirectional LDG reads (both GPUs)             %8.1f GB/s per direction (GPU0 view)\n",
                    double(bytes) * 5 / (ms * 1e-3) / 1e9);
        // GPU0 reads GPU1 while GPU0 also writes GPU1 (read + write same link)
        CK(cudaEventRecord(a0, s0));
        cudaStream_t s2;
        CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        for (int r = 0; r < 5; ++r) {
            k_bulk<4><<<sms, 32, smem, s0>>>((const char*)src1, bytes, B, sink);
            k_stg<<<sms, 256, 0, s2>>>((float4*)dst1, n4 / 4);
        }
        cudaEvent_t c2;
        CK(cudaEventCreate(&c2));
        CK(cudaEventRecord(c2, s2));
        CK(cudaStreamWaitEvent(s0, c2));
        CK(cudaEventRecord(b0, s0));
        CK(cudaEventSynchronize(b0));
        CK(cudaEventElapsedTime(&ms, a0, b0));
        std::printf("GPU0 bulk-reads 1 GiB from GPU1 + writes 256 MiB to GPU1: %.3f ms per pair\n", ms / 5);
    }
    std::printf("done\n");
    return 0;
}
