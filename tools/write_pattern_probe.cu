// Write-pattern probe: does a broadcast of one source row into R destination
// rows (the stage-2 broadcast: G + N worker rows) reach the write-only HBM rate,
// and does the per-CTA chunk size (consecutive tiles per CTA) matter?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/wpp tools/write_pattern_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fill(float4* p, size_t n4) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_float4(1.f, 2.f, 3.f, 4.f);
}

// src row of n floats broadcast into R rows (stride ld floats); work unit = chunk
// floats; units dealt to CTAs round-robin (grid-stride over units)
__global__ void k_bcast(const float* __restrict__ src, float* dst, size_t ld, int R, size_t n,
                        size_t chunk) {
    const size_t units = (n + chunk - 1) / chunk;
    for (size_t u = blockIdx.x; u < units; u += gridDim.x) {
        const size_t s = u * chunk, e = s + chunk < n ? s + chunk : n;
        for (size_t f = s + 4 * threadIdx.x; f < e; f += 4 * blockDim.x) {
            const float4 v = *reinterpret_cast<const float4*>(src + f);
            for (int r = 0; r < R; ++r) *reinterpret_cast<float4*>(dst + r * ld + f) = v;
        }
    }
}

int main() {
    const size_t n = 12u << 20;  // 12 M floats per row (~ ResNet-50's deferred part)
    const int R = 9;
    float *src, *dst;
    cudaMalloc(&src, n * 4);
    cudaMalloc(&dst, n * 4 * R);
    cudaMemset(src, 0, n * 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms;
    for (int it = 0; it < 2; ++it) k_fill<<<sms * 8, 256>>>((float4*)dst, n * R / 4);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) k_fill<<<sms * 8, 256>>>((float4*)dst, n * R / 4);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("fill (1 stream, %zu MB): %.1f GB/s\n", n * R * 4 >> 20, n * R * 4 * 10 / (ms * 1e6));
    size_t chunks[] = {1024, 4096, 16384, 65536};
    int blocks[] = {4, 8, 16};
    for (size_t c : chunks)
        for (int bpsm : blocks) {
            for (int it = 0; it < 2; ++it) k_bcast<<<sms * bpsm, 256>>>(src, dst, n, R, n, c);
            cudaEventRecord(a);
            for (int it = 0; it < 10; ++it) k_bcast<<<sms * bpsm, 256>>>(src, dst, n, R, n, c);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("bcast 1->%d rows, chunk %6zu floats, %2d CTA/SM: %.1f GB/s (r+w)\n", R, c, bpsm,
                   (double)n * 4 * (R + 1) * 10 / (ms * 1e6));
        }
    return 0;
}
