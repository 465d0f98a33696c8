// The gradient producer on the other side of the sync path:
// the reference learner's MLP forward/backward (learner.cpp:299-367) for every
// worker at once, one CTA per worker, reading that worker's parameter row
// (OspWorker::params(), the group's P row) and writing its float gradient row
// straight into the delta rows the OSP step consumes (with the group's fused
// sgd_delta, the step applies float(-lr * g), learner.cpp:391-398).
//
// Arithmetic follows the reference operation by operation in fp64 with explicit
// _rn intrinsics (no FMA): z = b + sum_i w[o][i] * a[i] in ascending i
// (learner.cpp:316-322); softmax cross-entropy or MSE per sample (:231-260);
// the input-side delta sum_o dz[o] * w[o][i] in ascending o, then times the
// activation derivative (:337-351); every gradient accumulator sums its
// per-sample terms in batch order (:338-346), then g * (1 / B) rounded to
// float (:356-364); the loss sums the samples in batch order. relu and MSE are
// exact, so the relu+MSE gradients are bit-identical to the reference; tanh,
// exp and log come from CUDA's libdevice instead of the host libm (both within
// an ulp or two of the true value), so those gradients agree to a tolerance
// (tests/test_gpu_learner.py).
//
// Shared memory per CTA: pre-activations and activations of every sample and
// layer, two delta buffers (B x max width) and the worker's parameters, all
// fp64.

#include "common.cuh"

namespace osp {
namespace {

constexpr int kLearnThreads = 512;

__device__ __forceinline__ double act_fwd(int act, double z) {
    return act == 0 ? (z > 0.0 ? z : 0.0) : tanh(z);
}

__device__ __forceinline__ double act_bwd(int act, double z, double a) {
    return act == 0 ? (z > 0.0 ? 1.0 : 0.0) : __dsub_rn(1.0, __dmul_rn(a, a));
}

template <bool SW>  // SW: the worker's parameters staged in shared memory as doubles
__global__ void __launch_bounds__(kLearnThreads) k_mlp_grad(MlpArgs a) {
    extern __shared__ __align__(16) double lsm[];
    // programmatic dependent launch: the parameter rows are the previous step's
    // output (wait for it), and the step consuming these gradients may get
    // resident meanwhile (it waits for this grid before reading them)
    pdl_wait();
    pdl_trigger();
    const int w = blockIdx.x;
    const int tid = threadIdx.x;
    const int B = a.B, depth = a.depth;
    // layout: act/pre [B][S] with S = sum of widths (layer l at column off[l]),
    // dz0/dz1 [B][maxw], sample losses [B]
    int off[kMlpMaxDepth + 2];
    off[0] = 0;
    for (int l = 0; l <= depth; ++l) off[l + 1] = off[l] + a.widths[l];
    // rows of an odd number of doubles: a warp walking samples (one row each)
    // touches 16 distinct 8-byte banks per half-warp
    const int S = off[depth + 1] | 1;
    double* act = lsm;
    double* pre = act + static_cast<size_t>(B) * S;
    double* dzA = pre + static_cast<size_t>(B) * S;
    double* dzB = dzA + static_cast<size_t>(B) * a.maxw;
    double* sloss = dzB + static_cast<size_t>(B) * a.maxw;
    // this worker's parameters as doubles in shared memory (every forward and
    // backward inner loop reads them; exact conversion)
    double* Pd = sloss + B;
    const float* Pg = a.P + static_cast<uint64_t>(w) * a.ldP;
    if (SW)
        for (uint64_t k = tid; k < a.n_params; k += blockDim.x) Pd[k] = static_cast<double>(Pg[k]);
    auto wv = [&](uint64_t k) -> double { return SW ? Pd[k] : static_cast<double>(Pg[k]); };
    const int* batch = a.batch + static_cast<size_t>(w) * B;
    float* out = a.out + static_cast<uint64_t>(w) * a.ldo;

    // inputs: the batch rows as doubles (learner.cpp:314)
    const int d = a.widths[0];
    for (int k = tid; k < B * d; k += blockDim.x) {
        const int s = k / d, i = k % d;
        int r = batch[s];
        if (r < 0 || static_cast<uint64_t>(r) >= a.n_rows) {  // check_batch (learner.cpp:262-267)
            atomicExch(a.error, 2u);
            r = 0;
        }
        act[static_cast<size_t>(s) * S + i] = static_cast<double>(a.feats[static_cast<uint64_t>(r) * d + i]);
    }
    __syncthreads();

    // forward (learner.cpp:315-326): one (sample, unit) per thread
    uint64_t at = 0;  // parameter offset of layer l (W then b)
    for (int l = 0; l < depth; ++l) {
        const int in = a.widths[l], outw = a.widths[l + 1];
        const uint64_t bias = at + static_cast<uint64_t>(in) * outw;
        for (int k = tid; k < B * outw; k += blockDim.x) {
            const int s = k % B, o = k / B;  // lanes walk samples: the W row is a broadcast
            const double* ain = act + static_cast<size_t>(s) * S + off[l];
            double z = wv(bias + o);
            const uint64_t wr = at + static_cast<uint64_t>(o) * in;
            for (int i = 0; i < in; ++i) z = __dadd_rn(z, __dmul_rn(wv(wr + i), ain[i]));
            pre[static_cast<size_t>(s) * S + off[l + 1] + o] = z;
            act[static_cast<size_t>(s) * S + off[l + 1] + o] = l + 1 < depth ? act_fwd(a.act, z) : z;
        }
        at += static_cast<uint64_t>(in) * outw + outw;
        __syncthreads();
    }

    // loss and dloss/dz per sample (learner.cpp:231-260)
    const int kout = a.widths[depth];
    for (int s = tid; s < B; s += blockDim.x) {
        const double* z = act + static_cast<size_t>(s) * S + off[depth];
        double* dz = dzA + static_cast<size_t>(s) * a.maxw;
        const int r = batch[s];
        const int y = r >= 0 && static_cast<uint64_t>(r) < a.n_rows ? a.labels[r] : 0;
        double loss = 0.0;
        if (a.loss == 0) {  // softmax cross-entropy
            double zmax = z[0];
            for (int c = 1; c < kout; ++c) zmax = z[c] > zmax ? z[c] : zmax;
            double sum = 0.0;
            for (int c = 0; c < kout; ++c) sum = __dadd_rn(sum, exp(__dsub_rn(z[c], zmax)));
            const double logsum = __dadd_rn(log(sum), zmax);
            if (y < 0 || y >= kout) atomicExch(a.error, 2u);  // label exceeds output width
            loss = __dsub_rn(logsum, z[y < 0 || y >= kout ? 0 : y]);
            for (int c = 0; c < kout; ++c)
                dz[c] = __dsub_rn(exp(__dsub_rn(z[c], logsum)), c == y ? 1.0 : 0.0);
        } else {  // MSE: one-hot targets, or the label itself for a 1-wide output
            for (int c = 0; c < kout; ++c) {
                const double target = kout == 1 ? static_cast<double>(y) : (y == c ? 1.0 : 0.0);
                const double diff = __dsub_rn(z[c], target);
                loss = __dadd_rn(loss, __dmul_rn(diff, diff));
                dz[c] = __dmul_rn(2.0, diff);
            }
        }
        sloss[s] = loss;
    }
    __syncthreads();
    if (tid == 0) {  // total in batch order, then the mean (learner.cpp:329, 357)
        double tot = 0.0;
        for (int s = 0; s < B; ++s) tot = __dadd_rn(tot, sloss[s]);
        const double mean = __ddiv_rn(tot, static_cast<double>(B));
        if (a.loss_out) a.loss_out[w] = mean;
        if (!isfinite(mean)) atomicExch(a.error, 1u);
    }

    // backward (learner.cpp:331-353), top layer first
    const double inv = __ddiv_rn(1.0, static_cast<double>(B));
    double* dz = dzA;
    double* dn = dzB;
    for (int l = depth - 1; l >= 0; --l) {
        const int in = a.widths[l], outw = a.widths[l + 1];
        at -= static_cast<uint64_t>(in) * outw + outw;
        // weight and bias gradients: per-sample terms summed in batch order
        for (int k = tid; k < in * outw + outw; k += blockDim.x) {
            double acc = 0.0;
            if (k < in * outw) {
                const int o = k / in, i = k % in;
                for (int s = 0; s < B; ++s)
                    acc = __dadd_rn(acc, __dmul_rn(dz[static_cast<size_t>(s) * a.maxw + o],
                                                   act[static_cast<size_t>(s) * S + off[l] + i]));
            } else {
                const int o = k - in * outw;
                for (int s = 0; s < B; ++s) acc = __dadd_rn(acc, dz[static_cast<size_t>(s) * a.maxw + o]);
            }
            const double g = __dmul_rn(acc, inv);
            if (!isfinite(g)) atomicExch(a.error, 1u);
            out[at + k] = __double2float_rn(g);
        }
        if (l > 0) {  // the input side's delta, times the activation derivative
            for (int k = tid; k < B * in; k += blockDim.x) {
                const int s = k / in, i = k % in;
                double v = 0.0;
                for (int o = 0; o < outw; ++o)
                    v = __dadd_rn(v, __dmul_rn(dz[static_cast<size_t>(s) * a.maxw + o],
                                               wv(at + static_cast<uint64_t>(o) * in + i)));
                const size_t q = static_cast<size_t>(s) * S + off[l] + i;
                dn[static_cast<size_t>(s) * a.maxw + i] = __dmul_rn(v, act_bwd(a.act, pre[q], act[q]));
            }
        }
        __syncthreads();
        double* t = dz;
        dz = dn;
        dn = t;
    }
}

}  // namespace

size_t mlp_smem_bytes(const MlpArgs& a, bool stage_w) {
    int S = 0;
    for (int l = 0; l <= a.depth; ++l) S += a.widths[l];
    S |= 1;
    return (2ull * a.B * S + 2ull * a.B * a.maxw + a.B + (stage_w ? a.n_params : 0)) * sizeof(double);
}

// parameters staged in shared memory when the whole CTA still fits
bool mlp_stage_w(const MlpArgs& a) { return mlp_smem_bytes(a, true) <= 200 * 1024; }

size_t mlp_grad_smem(const MlpArgs& a) { return mlp_smem_bytes(a, mlp_stage_w(a)); }

cudaError_t launch_mlp_grad(const MlpArgs& a, int n_workers, cudaStream_t s) {
    const bool sw = mlp_stage_w(a);
    const size_t sm = mlp_smem_bytes(a, sw);
    void (*kern)(MlpArgs) = sw ? k_mlp_grad<true> : k_mlp_grad<false>;
    int per_sm = 0;  // opts the kernel into `sm` bytes (cached per context)
    cudaError_t e = tma_blocks_per_sm(reinterpret_cast<const void*>(kern), kLearnThreads, sm, &per_sm);
    if (e != cudaSuccess) return e;
    return launch_pdl(kern, dim3(n_workers), dim3(kLearnThreads), sm, s, a);
}

}  // namespace osp
