// C-ABI of the gradient producer (include/osp_c.h, "Learner" section): the
// reference learner's forward_backward (learner.hpp:63-64, learner.cpp:299-367)
// for N workers in one launch over a device-resident dataset.

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "handles.h"

using namespace osp;

struct osp_mlp {
    MlpArgs base{};          // spec, dataset and error flag; per call: params, batch, outputs
    unsigned* error = nullptr;
    uint64_t n_params = 0;   // mlp_partition total (learner.hpp:51-53)
};

extern "C" {

osp_status osp_mlp_create(const int32_t* widths, int n_widths, int activation, int loss,
                          const float* features, const int32_t* labels, uint64_t n_rows,
                          osp_mlp** out) {
    if (!out || !widths || !features || !labels) return fail(OSP_ERR_INVALID, "null argument");
    *out = nullptr;
    // MlpSpec::validate (learner.cpp:15-20)
    if (n_widths < 2) return fail(OSP_ERR_CONFIG, "mlp needs at least input and output widths");
    for (int l = 0; l < n_widths; ++l)
        if (widths[l] <= 0) return fail(OSP_ERR_CONFIG, "mlp widths must be positive");
    if (n_widths - 1 > kMlpMaxDepth)
        return fail(OSP_ERR_INVALID, "at most " + std::to_string(kMlpMaxDepth) + " linear layers");
    if (activation != OSP_ACT_RELU && activation != OSP_ACT_TANH) return fail(OSP_ERR_CONFIG, "unknown activation");
    if (loss != OSP_LOSS_CE && loss != OSP_LOSS_MSE) return fail(OSP_ERR_CONFIG, "unknown loss");
    if (n_rows == 0) return fail(OSP_ERR_CONFIG, "dataset is empty");
    auto* m = new osp_mlp();
    MlpArgs& a = m->base;
    a.depth = n_widths - 1;
    a.maxw = 0;
    for (int l = 0; l < n_widths; ++l) {
        a.widths[l] = widths[l];
        a.maxw = std::max(a.maxw, static_cast<int>(widths[l]));
        if (l + 1 < n_widths)
            m->n_params += static_cast<uint64_t>(widths[l]) * widths[l + 1] + widths[l + 1];
    }
    a.act = activation == OSP_ACT_TANH ? 1 : 0;
    a.loss = loss == OSP_LOSS_MSE ? 1 : 0;
    a.n_params = m->n_params;
    a.feats = features;
    a.labels = labels;
    a.n_rows = n_rows;
    cudaError_t e = cudaMalloc(&m->error, sizeof(unsigned));
    if (e == cudaSuccess) e = cudaMemset(m->error, 0, sizeof(unsigned));
    if (e != cudaSuccess) {
        delete m;
        return cuda_fail(e, "mlp error flag");
    }
    a.error = m->error;
    *out = m;
    return OSP_OK;
}

void osp_mlp_destroy(osp_mlp* m) {
    if (!m) return;
    if (m->error) cudaFree(m->error);
    delete m;
}

uint64_t osp_mlp_num_params(const osp_mlp* m) { return m ? m->n_params : 0; }

osp_status osp_mlp_grad(osp_mlp* m, const float* params, uint64_t ld_params, int n_workers,
                        const int32_t* batch, int batch_size, float* grad_out, uint64_t ld_out,
                        double* loss_out, void* stream) {
    OSP_RANGE("osp_mlp_grad");
    if (!m || !params || !batch || !grad_out) return fail(OSP_ERR_INVALID, "null argument");
    if (n_workers < 1 || n_workers > 65535) return fail(OSP_ERR_INVALID, "worker count out of range");
    if (batch_size < 1) return fail(OSP_ERR_SHAPE, "batch is empty");  // check_batch
    if (ld_params < m->n_params || ld_out < m->n_params)
        return fail(OSP_ERR_SHAPE, "params do not match the mlp partition");
    MlpArgs a = m->base;
    a.P = params;
    a.ldP = ld_params;
    a.batch = batch;
    a.B = batch_size;
    a.out = grad_out;
    a.ldo = ld_out;
    a.loss_out = loss_out;
    if (mlp_grad_smem(a) > 220 * 1024)
        return fail(OSP_ERR_INVALID, "batch x widths exceed the kernel's shared memory");
    OSP_CUDA(launch_mlp_grad(a, n_workers, as_stream(stream)));
    return OSP_OK;
}

osp_status osp_mlp_check(osp_mlp* m, void* stream) {
    if (!m) return fail(OSP_ERR_INVALID, "null learner");
    unsigned err = 0;
    cudaStream_t s = as_stream(stream);
    OSP_CUDA(cudaMemcpyAsync(&err, m->error, sizeof err, cudaMemcpyDeviceToHost, s));
    OSP_CUDA(cudaStreamSynchronize(s));
    if (err) OSP_CUDA(cudaMemsetAsync(m->error, 0, sizeof(unsigned), s));
    if (err == 1) return fail(OSP_ERR_NUMERIC, "loss or gradient is not finite");
    if (err == 2) return fail(OSP_ERR_SHAPE, "batch row index or label out of range");
    return OSP_OK;
}

}  // extern "C"
