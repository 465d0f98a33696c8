/*
 * osp_engine.h — C-ABI of the message-level OSP engines (drop-in boundary for
 * non-C++ hosts). The reference's engines are C++ classes driven one message
 * at a time (protocol.hpp:65-254); this header exposes the same worker/server
 * state machines over opaque handles, with messages as opaque handles that
 * encode to the reference's wire formats. Implemented in libpslab_b200.so on
 * top of the C++ façade (include/pslab), whose engine state lives on the GPU
 * and whose arithmetic runs in the sm_100a kernels of include/osp_c.h.
 *
 * Vectors are HOST float arrays of the partition's total element count (the
 * reference's wire type is std::vector<float>). Status codes are osp_status
 * (include/osp_c.h), 1:1 with the pslab::Error classes; the message of the last
 * failure on this thread is osp_engine_last_error(). No exceptions cross.
 */
#ifndef OSP_ENGINE_H
#define OSP_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#include "osp_c.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* osp_engine_last_error(void);

/* make_partition (param.hpp:43-46): dense ids, contiguous offsets. */
typedef struct osp_engine_partition osp_engine_partition;
osp_status osp_engine_partition_create(const uint64_t* layer_counts, uint64_t n_layers,
                                       uint32_t bytes_per_element, osp_engine_partition** out);
void osp_engine_partition_destroy(osp_engine_partition* p);
uint64_t osp_engine_partition_total_count(const osp_engine_partition* p);

/* ---- messages (message.hpp:13-42) ---------------------------------------- */
typedef struct osp_msg osp_msg;
/* MsgKind values: 0 PushImportant, 1 PushIcsChunk, 2 PullImportant,
 * 3 IcsGlobalChunk, 4 GibUpdate, 5 LossReport, 6 PushFull, 7 PullFull. */
int osp_msg_kind(const osp_msg* m);
uint32_t osp_msg_iteration(const osp_msg* m);
int osp_msg_from(const osp_msg* m);         /* worker id, -1 = server */
double osp_msg_scalar(const osp_msg* m);    /* LossReport value */
int osp_msg_layer_count(const osp_msg* m);  /* payload entries */
/* message_size_bytes (message.cpp:21-30): payload bytes, encoded GIB size or 8. */
uint64_t osp_msg_size_bytes(const osp_msg* m, const osp_engine_partition* part);
/* Payload wire format (message.cpp:53-99): kind u8 | iteration u32 | entries
 * u16 | per layer id u32, count u32, fp32 values (LE). *len = bytes needed;
 * OSP_ERR_INVALID if cap is too small (out may be NULL to query). */
osp_status osp_msg_encode(const osp_msg* m, uint8_t* out, uint64_t cap, uint64_t* len);
/* FormatError on malformed input; from_worker is carried, not encoded. */
osp_status osp_msg_decode(const uint8_t* buf, uint64_t len, int from_worker, osp_msg** out);
/* GibUpdate: encoded GIB (gib_encode wire, importance.cpp:61-117) and the ICS
 * rank order side channel (least important first). */
osp_status osp_msg_gib(const osp_msg* m, uint8_t* out, uint64_t cap, uint64_t* len);
osp_status osp_msg_rank_order(const osp_msg* m, int32_t* out, uint64_t cap, uint64_t* n);
void osp_msg_destroy(osp_msg* m);

/* ---- worker: OspWorker (protocol.hpp:71-109) ------------------------------- */
typedef struct osp_worker osp_worker;
osp_status osp_worker_create(const osp_engine_partition* part, int worker_id,
                             const float* init_params /*host, may be NULL = zeros*/,
                             double subset_weight, osp_worker** out);
void osp_worker_destroy(osp_worker* w);
/* on_compute_done (protocol.cpp:180-210): split with the current GIB. Returns
 * the RS push, the loss report and up to max_chunks ICS chunk messages
 * (*n_chunks = how many; OSP_ERR_INVALID if more than max_chunks). */
osp_status osp_worker_compute_done(osp_worker* w, uint64_t iteration, const float* delta,
                                   double loss, int n_chunks, osp_msg** rs_push,
                                   osp_msg** loss_report, osp_msg** ics_chunks, int max_chunks,
                                   int* n_ics_chunks);
/* on_pull_important (protocol.cpp:212-241): *applied = 0 if stashed. */
osp_status osp_worker_on_pull_important(osp_worker* w, const osp_msg* pull, int* applied);
osp_status osp_worker_on_ics_global_chunk(osp_worker* w, const osp_msg* chunk);
int osp_worker_stashed_pull_ready(const osp_worker* w);
osp_status osp_worker_apply_stashed_pull(osp_worker* w);
osp_status osp_worker_on_gib_update(osp_worker* w, const osp_msg* gib_update);
uint64_t osp_worker_iteration(const osp_worker* w);
int osp_worker_pending_empty(const osp_worker* w);
/* Worker parameters (host copy, total_count floats). */
osp_status osp_worker_params(const osp_worker* w, float* out);

/* ---- server: OspServer (protocol.hpp:113-180) ------------------------------ */
typedef struct osp_server osp_server;
typedef struct osp_server_config {
    int n_workers;
    const double* weights;          /* host, n_workers subset weights */
    uint64_t u_max;                 /* SguSchedule::u_max */
    uint64_t iterations_per_epoch;  /* OspServerOptions */
    int has_fixed_budget;           /* OspServerOptions::fixed_budget_bytes set */
    uint64_t fixed_budget_bytes;
} osp_server_config;
osp_status osp_server_create(const osp_engine_partition* part, const float* init_global /*host or NULL*/,
                             const osp_server_config* cfg, osp_server** out);
void osp_server_destroy(osp_server* s);
/* on_push_important / on_push_ics_chunk (protocol.cpp:309-353): each output
 * is set to a new message or NULL. */
osp_status osp_server_on_push_important(osp_server* s, const osp_msg* msg, osp_msg** pull_important,
                                        osp_msg** ics_broadcast, osp_msg** gib_update);
osp_status osp_server_on_push_ics_chunk(osp_server* s, const osp_msg* msg, osp_msg** pull_important,
                                        osp_msg** ics_broadcast, osp_msg** gib_update);
osp_status osp_server_on_loss_report(osp_server* s, const osp_msg* msg);
osp_status osp_server_set_umax(osp_server* s, uint64_t u_max);
osp_status osp_server_global_params(const osp_server* s, float* out);
uint64_t osp_server_resolved_count(const osp_server* s);
uint64_t osp_server_dropped_stale(const osp_server* s);
uint64_t osp_server_budget_for_epoch(const osp_server* s, uint64_t epoch);
uint64_t osp_server_epoch_of_iteration(const osp_server* s, uint64_t iteration);

#ifdef __cplusplus
}
#endif

#endif /* OSP_ENGINE_H */
