/*
 * osp_oracle.h — CPU restatement of the reference OSP sync path (TEST
 * INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 kernels. Only tests/, the smoke()
 * entry and bench.py's cpu_baseline leg may load it. The product
 * (paper_2306_16926_b200/) never links, imports or calls it.
 *
 * Every function restates one reference function (file:line into
 * /root/reference/proj) on flat arrays. Parity pinning: tests/test_oracle.py
 * checks it against (1) the hand vectors of the reference unit tests and
 * (2) golden dumps produced by the unmodified reference engine
 * (oracle/_ref/ref_driver, committed as tests/golden/ (npz) by
 * oracle/gen_golden.py).
 */
#ifndef OSP_ORACLE_H
#define OSP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* rng.hpp:16-36 */
uint64_t oo_splitmix64(uint64_t* state);
uint64_t oo_derive_seed(uint64_t root, uint64_t tag, uint64_t a, uint64_t b);

/* runner.cpp:312-321 with rng.hpp:50-61: float(uniform(-1e-3, 1e-3)) from
 * Rng(derive_seed(seed, 6, worker, iteration)), elements [first, first+n). */
void oo_synth_delta(uint64_t seed, uint64_t worker, uint64_t iteration, uint64_t first,
                    uint64_t n, float* out);

/* learner.cpp:391-398 */
void oo_sgd_delta(const float* grad, uint64_t n, double lr, float* out);
/* learner.cpp:400-403 */
double oo_lr_at_epoch(double initial_lr, uint64_t epoch);

/* protocol.cpp:9-30. Returns 0, or -1 on a ProtocolError condition. */
int oo_aggregate_layer(int n_workers, const float* const* contribs, const double* weights,
                       uint64_t n, float* out);

/* importance.cpp:11-28 — scores[l] = sequential sum_j |(double)g_j * (double)p_j| */
void oo_pgp_accum(uint64_t n, const float* params, const float* grads, double* acc);
void oo_pgp(int64_t n_layers, const uint64_t* counts, const float* params, const float* grads,
            double* scores);
/* importance.cpp:30-40 — stable ascending, ties by id */
void oo_rank(int64_t n_layers, const double* scores, int32_t* order);
/* importance.cpp:42-59 — prefix rule, stop at first misfit */
void oo_build_gib(int64_t n_layers, const double* scores, const uint64_t* counts, uint32_t bpe,
                  uint64_t budget, uint8_t* ics_flags);
/* importance.cpp:61-117 */
uint64_t oo_gib_encoded_size(uint64_t n_layers);
void oo_gib_encode(uint32_t tag, uint64_t n_layers, const uint8_t* ics_flags, uint8_t* out);
/* returns 0, or -1 for a FormatError (truncation); flags_cap bounds the output */
int oo_gib_decode(const uint8_t* buf, uint64_t len, uint32_t* tag, uint32_t* n_layers,
                  uint8_t* flags, uint64_t flags_cap);

/* protocol.cpp:122-166. Outputs:
 *   rs_ids[n_rs]        RS layer ids ascending
 *   chunk_of[L]         compacted chunk index per ICS layer, -1 otherwise
 * returns the number of non-empty chunks, or -1 for n_chunks < 1. */
int oo_split(int64_t n_layers, const uint64_t* counts, uint32_t bpe, const uint8_t* ics_flags,
             const int32_t* ics_order, int64_t n_order, int n_chunks, int32_t* rs_ids,
             int64_t* n_rs, int32_t* chunk_of);

/* tuning.cpp:8-21 */
uint64_t oo_compute_umax(double bandwidth_bps, double loss_rate, double t_c_seconds,
                         int n_workers, uint64_t model_bytes, int eq5_literal);
/* tuning.cpp:23-48. (*initial_loss, *has_initial) is SguSchedule::initial_loss.
 * returns budget, or -1 (ConfigError) / -2 (NumericError) / -3 (ProtocolError). */
int64_t oo_tune_sgu(double* initial_loss, int* has_initial, uint64_t u_max,
                    uint64_t epoch_index, double epoch_loss);

/* message.cpp:53-78: kind u8 | iteration u32 | entries u16 | per layer id u32,
 * count u32, fp32 values; ids ascending. Returns bytes written. */
uint64_t oo_encode_payload(uint8_t kind, uint32_t iteration, int64_t n_layers,
                           const uint64_t* counts, const float* values, const int32_t* ids,
                           int64_t n_ids, uint8_t* out);

/* One synchronous OSP iteration for N co-resident workers, restated from the
 * OspWorker/OspServer message flow (protocol.cpp:172-447) in the order of
 * oracle/ref_driver.cpp. Worker parameters are read (not assumed equal to the
 * global vector) and per-layer base copies are kept, as lgp_partial does.
 *
 *   deltas [N*M], G [M] in/out, P [N*M] in/out
 *   ics_flags_in [L], order_in [n_order_in]: the GIB the workers split with
 *   p_stage1 [N*M] (may be NULL): worker params right after the pull
 *   agg [M]: aggregated delta per element (all layers)
 *   scores [L], ics_flags_out [L], order_out [<=L] (+n_order_out): next GIB
 *   chunk_of [L] (may be NULL): chunk of each layer for THIS iteration
 * returns the number of ICS chunks used this iteration, or <0 on error. */
int oo_step(int64_t n_layers, const uint64_t* counts, uint32_t bpe, int n_workers,
            const double* weights, const float* deltas, float* G, float* P,
            const uint8_t* ics_flags_in, const int32_t* order_in, int64_t n_order_in,
            int n_chunks, uint64_t budget, float* p_stage1, float* agg, double* scores,
            uint8_t* ics_flags_out, int32_t* order_out, int64_t* n_order_out, int32_t* chunk_of);

#ifdef __cplusplus
}
#endif

#endif
