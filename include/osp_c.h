/*
 * osp_c.h — C-ABI of the B200-native OSP sync path (drop-in boundary).
 *
 * Plain C: opaque handles, plain pointers and sizes, status codes. No
 * exceptions and no torch types cross this boundary. Vectors are DEVICE
 * pointers (fp32, flat over a layer partition) unless a parameter says host.
 * Every device operation is stream-ordered on the `stream` argument
 * (a cudaStream_t passed as void*; NULL = legacy default stream).
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/proj, file:line). The reference has no FFI: its boundary is
 * the C++ library API in include/pslab/{param,importance,protocol,tuning}.hpp
 * and learner.hpp:77. The C++ façade in include/pslab/ (this repo) re-exposes
 * that API on top of these functions, rethrowing the matching pslab::Error
 * subclass from the status code.
 */
#ifndef OSP_C_H
#define OSP_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OSP_ABI_VERSION 2
/* Workers per aggregation call / group (kernel-parameter weights table; the
 * kernels' parameter blocks use the > 4 KB parameter space of CUDA 12.1+). */
#define OSP_MAX_WORKERS 256

/* Status codes, 1:1 with the pslab::Error hierarchy (errors.hpp:11-69). */
typedef enum osp_status {
    OSP_OK = 0,
    OSP_ERR_PARTITION = 1, /* PartitionError */
    OSP_ERR_SHAPE = 2,     /* ShapeError */
    OSP_ERR_LAYER = 3,     /* LayerError */
    OSP_ERR_PARSE = 4,     /* ParseError */
    OSP_ERR_CONFIG = 5,    /* ConfigError */
    OSP_ERR_FORMAT = 6,    /* FormatError */
    OSP_ERR_PROTOCOL = 7,  /* ProtocolError */
    OSP_ERR_NUMERIC = 8,   /* NumericError */
    OSP_ERR_CUDA = 20,     /* CUDA runtime / launch failure (no reference analogue) */
    OSP_ERR_INVALID = 21   /* null handle or pointer, unsupported size */
} osp_status;

/* Thread-local message of the last failing call on this thread. */
const char* osp_last_error(void);
const char* osp_status_name(osp_status s);
int osp_abi_version(void);
/* Device the library runs on (cudaGetDevice) and its SM count. */
osp_status osp_device_info(int* device, int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------------------
 * Partition — LayerPartition::make / make_partition (param.hpp:19-46,
 * param.cpp:8-42). Layer ids dense from 0, offsets contiguous in id order.
 * A device mirror of offsets/counts is kept for the kernels.
 * ---------------------------------------------------------------------- */
typedef struct osp_partition osp_partition;

osp_status osp_partition_create(const uint64_t* layer_counts /*host*/, uint64_t n_layers,
                                uint32_t bytes_per_element, osp_partition** out);
void osp_partition_destroy(osp_partition* p);
uint64_t osp_partition_layer_count(const osp_partition* p);
uint64_t osp_partition_total_count(const osp_partition* p);
uint64_t osp_partition_total_bytes(const osp_partition* p);
uint32_t osp_partition_bytes_per_element(const osp_partition* p);
/* LayerPartition::layer (param.cpp:31-37): LayerError when out of range. */
osp_status osp_partition_layer(const osp_partition* p, int64_t id, uint64_t* offset,
                               uint64_t* count);

/* ------------------------------------------------------------------------
 * Device buffers (the façade's storage; the Python side uses torch).
 * ---------------------------------------------------------------------- */
osp_status osp_device_alloc(uint64_t bytes, void** out);
osp_status osp_device_free(void* ptr);
osp_status osp_memcpy_h2d(void* dst, const void* src, uint64_t bytes, void* stream);
osp_status osp_memcpy_d2h(void* dst, const void* src, uint64_t bytes, void* stream);
osp_status osp_memcpy_d2d(void* dst, const void* src, uint64_t bytes, void* stream);
osp_status osp_memset(void* dst, int value, uint64_t bytes, void* stream);
osp_status osp_stream_sync(void* stream);

/* ------------------------------------------------------------------------
 * Element-wise primitives (one kernel each).
 * ---------------------------------------------------------------------- */

/* aggregate_layer (protocol.cpp:9-30): out[e] = float(sum_w w_k*(double)x_k[e] / sum w),
 * fp64 mul then add in ascending worker order, no FMA. contribs is a HOST array
 * of n_workers device pointers; weights is a host array. ProtocolError if
 * n_workers < 1 or the weights do not sum > 0. */
osp_status osp_aggregate_layer(const float* const* contribs, int n_workers,
                               const double* weights, uint64_t n, float* out, void* stream);

/* OspServer::finish_layer (protocol.cpp:292-307) for a set of layers in one
 * launch: agg = aggregate(contribs), global += agg. contribs are HOST arrays of
 * n_workers device pointers, each to a FLAT vector over the partition; layer_ids
 * (host) selects the layers. agg_out (flat, may be NULL) receives the aggregate. */
osp_status osp_aggregate_apply_layers(const osp_partition* part, const float* const* contribs,
                                      int n_workers, const double* weights,
                                      const int32_t* layer_ids, int64_t n_ids, float* global,
                                      float* agg_out, void* stream);

/* apply_delta (param.cpp:127-150): p[i] = p[i] + scale*d[i] (fp32 mul, then add). */
osp_status osp_apply_delta(float* p, const float* d, uint64_t n, float scale, void* stream);

/* sgd_delta (learner.cpp:391-398): out = float(-lr * (double)g). ConfigError if lr <= 0. */
osp_status osp_sgd_delta(const float* grad, uint64_t n, double lr, float* out, void* stream);

/* Synthetic delta source (runner.cpp:312-321, rng.hpp:16-61): elements
 * [first, first+n) of float(uniform(-1e-3, 1e-3)) drawn from
 * Rng(derive_seed(seed, kSynthGrad=6, worker, iteration)). */
osp_status osp_synth_delta(uint64_t seed, uint64_t worker, uint64_t iteration, uint64_t first,
                           uint64_t n, float* out, void* stream);
/* Same stream, n_workers rows of a [n_workers][ld] block in one launch. */
osp_status osp_synth_deltas(uint64_t seed, int n_workers, uint64_t iteration, uint64_t n,
                            float* out, uint64_t ld, void* stream);

/* lgp_partial (protocol.cpp:69-97) on flat vectors. ics_flags (HOST, one byte per
 * layer): 0 = the layer takes the global delta (p += 1.0f*global_delta),
 * 1 = local estimate (base = p; p += local_delta), 2 = in neither payload
 * (untouched). base is written on local layers only. */
osp_status osp_lgp_partial(const osp_partition* part, float* params, const float* global_delta,
                           const float* local_delta, const uint8_t* ics_flags, float* base,
                           void* stream);

/* lgp_correct (protocol.cpp:99-116): p = base + global_delta on the listed
 * layers (HOST ids). */
osp_status osp_lgp_correct(const osp_partition* part, float* params, const float* base,
                           const float* global_delta, const int32_t* layer_ids, int64_t n_ids,
                           void* stream);

/* pgp_layer_importance (importance.cpp:11-28), reference-exact: scores (HOST,
 * n_layers doubles) bit-identical to the sequential double sum. One CTA per
 * layer, summed in ascending element order. */
osp_status osp_pgp_layer_importance(const osp_partition* part, const float* params,
                                    const float* grads, double* scores_host, void* stream);

/* rank_layers (importance.cpp:30-40) + build_gib (:42-59) on HOST scores, run as
 * the single-CTA device kernel of the group path. order_host: all layer ids
 * ascending by (score, id); ics_flags_host: prefix rule under budget_bytes. */
osp_status osp_rank_and_gib(const osp_partition* part, const double* scores_host,
                            uint64_t budget_bytes, int32_t* order_host, uint8_t* ics_flags_host,
                            void* stream);

/* The resolution's importance -> GIB step (OspServer::check_resolution,
 * protocol.cpp:407-419: pgp_layer_importance + rank_layers + build_gib) on
 * DEVICE vectors, the way the group path does it: per-tile tree sums of
 * |grads * params|, a per-layer interval certificate against the reference's
 * sequential sum, the exact sequential sum only for layers whose intervals
 * touch, then the stable (score, id) rank and the prefix rule under
 * budget_bytes. The deferred set and its rank order equal the reference's
 * bit for bit. HOST outputs (any may be NULL): scores [L] (the tree sums, exact
 * where recomputed), the deferred ids in rank order (*n_ics of them, capacity
 * L), flags [L]. Synchronises `stream`. */
osp_status osp_pgp_rank_gib(const osp_partition* part, const float* params, const float* grads,
                            uint64_t budget_bytes, double* scores_host, int32_t* ics_order_host,
                            int64_t* n_ics, uint8_t* ics_flags_host, void* stream);

/* split_for_sync (protocol.cpp:122-166) index lists (payload copies are not
 * made: the device path works on segment lists). HOST in/out. rs_ids gets the
 * RS layer ids ascending; chunk_of[l] the compacted chunk of each deferred layer
 * (-1 for RS); *n_used the number of non-empty chunks. ConfigError if
 * n_chunks < 1, ShapeError if ics_flags does not cover the partition. */
osp_status osp_split_for_sync(const osp_partition* part, const uint8_t* ics_flags,
                              const int32_t* ics_order, int64_t n_order, int n_chunks,
                              int32_t* rs_ids, int64_t* n_rs, int32_t* chunk_of, int* n_used);

/* GIB wire format (importance.cpp:61-117): tag u32 LE, L u32 LE, ceil(L/8)
 * bitmap bytes, bit k%8 of byte k/8 marks layer k deferred. HOST buffers. */
uint64_t osp_gib_encoded_size(uint64_t n_layers);
osp_status osp_gib_encode(uint32_t tag, uint64_t n_layers, const uint8_t* ics_flags,
                          uint8_t* out, uint64_t out_len);
/* FormatError on truncation. flags_cap bounds the decoded bitmap. */
osp_status osp_gib_decode(const uint8_t* buf, uint64_t len, uint32_t* tag, uint32_t* n_layers,
                          uint8_t* ics_flags, uint64_t flags_cap);

/* GIB wire with the rank-order side channel (the gap named
 * in the reference README.md:207-210 — the bitmap alone does not carry the
 * chunk emission order). Layout: the gib_encode bytes above, then n u32 LE and
 * n layer ids u32 LE, the deferred layers least important first
 * (Message::ics_rank_order, message.hpp:33-36). The reference's gib_decode
 * reads only the bitmap prefix (it accepts longer buffers, importance.cpp:99-
 * 117), so a wire is still a valid reference GIB message.
 * encode: every order id must be a distinct deferred layer (LayerError beyond
 *   L, ProtocolError otherwise); *len = bytes (out may be NULL to query).
 * decode: FormatError on truncation, a bad length or a bad id; *n_order = -1
 *   for a bitmap-only buffer (no side channel). Any output may be NULL. */
uint64_t osp_gib_wire_size(uint64_t n_layers, uint64_t n_order);
osp_status osp_gib_wire_encode(uint32_t tag, uint64_t n_layers, const uint8_t* ics_flags,
                               const int32_t* order, uint64_t n_order, uint8_t* out,
                               uint64_t cap, uint64_t* len);
osp_status osp_gib_wire_decode(const uint8_t* buf, uint64_t len, uint32_t* tag, uint32_t* n_layers,
                               uint8_t* ics_flags, uint64_t flags_cap, int32_t* order,
                               uint64_t order_cap, int64_t* n_order);

/* Payload wire codec on the device: encode_payload_message /
 * decode_payload_message (message.cpp:53-99) for payloads resident in HBM, so a
 * byte transport can send straight from the device. Layout: kind u8 |
 * iteration u32 LE | entries u16 LE | per layer: id u32 LE, count u32 LE,
 * count fp32 LE.
 * encode: the listed layers (HOST ids, strictly ascending = std::map order) of
 *   the flat DEVICE vector `values` into DEVICE `out`; FormatError above 65535
 *   layers. osp_payload_encoded_size gives the byte count (0 on a bad id).
 * decode: DEVICE buffer -> values scattered into the flat DEVICE vector at the
 *   layers' offsets; ids (HOST, first occurrence kept like std::map::emplace),
 *   kind and iteration returned; FormatError on truncation or trailing bytes,
 *   LayerError / ShapeError if an entry does not fit the partition. */
uint64_t osp_payload_encoded_size(const osp_partition* part, const int32_t* layer_ids,
                                  int64_t n_ids);
osp_status osp_encode_payload(const osp_partition* part, const float* values,
                              const int32_t* layer_ids, int64_t n_ids, uint8_t kind,
                              uint32_t iteration, uint8_t* out, uint64_t out_cap,
                              uint64_t* out_len, void* stream);
osp_status osp_decode_payload(const osp_partition* part, const uint8_t* buf, uint64_t len,
                              float* values, uint8_t* kind, uint32_t* iteration, int32_t* layer_ids,
                              int64_t ids_cap, int64_t* n_ids, void* stream);

/* compute_umax / tune_sgu (tuning.cpp:8-48), host scalar logic. */
osp_status osp_compute_umax(double bandwidth_bps, double latency_s, double loss_rate,
                            double t_c_seconds, int n_workers, uint64_t model_bytes,
                            int eq5_literal, uint64_t* out);
typedef struct osp_sgu_schedule {
    uint64_t u_max;
    int has_initial_loss;
    double initial_loss;
    uint64_t current_budget;
    uint64_t epoch;
} osp_sgu_schedule;
osp_status osp_tune_sgu(osp_sgu_schedule* sched, uint64_t epoch_index, double epoch_loss,
                        uint64_t* budget_out);

/* ------------------------------------------------------------------------
 * Group: the batched fast path for N co-resident logical workers + the PS on
 * one GPU (OspWorker x N + OspServer in the synchronous fresh-GIB regime,
 * protocol.cpp:172-447). Device state: global vector G [M], worker params
 * P [N][ldP], per-tile PGP partials, current GIB, ICS order and chunk lists.
 *
 * Iteration i:  stage1 (barrier: RS aggregate/apply/pull + LGP partial on ICS)
 *               stage2_chunk(c) for c < n_chunks (ICS aggregate/apply/correct)
 *               resolve (PGP -> certified rank -> GIB tag i+1 -> next lists)
 * Deltas are [N][ld] fp32 on the device (ld >= M). With sgd_lr > 0 they are raw
 * gradients and delta = float(-lr*(double)g) is fused into the load.
 * ---------------------------------------------------------------------- */
typedef struct osp_group osp_group;

typedef struct osp_group_config {
    int n_workers;            /* N, 1..OSP_MAX_WORKERS */
    const double* weights;    /* HOST, N subset weights (OspServer weights) */
    int n_chunks;             /* ICS chunk slots per iteration (>= 1) */
    uint32_t tile_elems;      /* elements per warp tile; 0 = default 512 (power of two, 256..65536) */
    double sgd_lr;            /* 0 = inputs are deltas; > 0 fuse sgd_delta */
    uint32_t flags;           /* OSP_GROUP_* bits */
} osp_group_config;

/* Stage-kernel family. Default (flags 0): the TMA-staged kernels (tiles moved
 * global->shared by cp.async.bulk into an mbarrier ring, tile_elems default 1024)
 * when the shape allows them (N in 1..8, tile_elems in [512, 4096]), else
 * the register-staged kernels (tile_elems default 512). OSP_GROUP_TMA requires
 * the TMA family (OSP_ERR_INVALID if unsupported); OSP_GROUP_REGISTER forces the
 * register-staged one. Both produce identical results. */
#define OSP_GROUP_TMA 1u
#define OSP_GROUP_REGISTER 2u
/* ICS carry (TMA family, on by default): stage 1 also aggregates the ICS
 * elements from the delta rows it already holds in shared memory and keeps
 * G_old + agg in an extra [M] device buffer, so stage 2 only writes G and the
 * worker rows from it (reads 1 row instead of N + 1). The ICS payload is the
 * one split at stage-1 time, as in the reference (split_for_sync copies it,
 * protocol.cpp:122-166): stage 2 ignores its `deltas` argument then.
 * OSP_GROUP_NO_CARRY keeps the re-reading stage 2 (identical results). */
#define OSP_GROUP_NO_CARRY 4u
/* Launch-bound layouts (L <= 32 layers, M <= 32768 parameters, with the carry
 * and without momentum): osp_group_step runs the whole iteration — stage 1,
 * the carry broadcast and a single-warp resolve — as ONE launch of ONE CTA
 * (identical results). OSP_GROUP_NO_SMALL keeps the three-launch step;
 * osp_group_flags reports OSP_GROUP_SMALL when the single-launch step is used. */
#define OSP_GROUP_NO_SMALL 8u
#define OSP_GROUP_SMALL 16u

/* init_params: DEVICE pointer to M floats (P0), or NULL for zeros. Every worker
 * and the server start from it (runner.cpp:214-231). */
osp_status osp_group_create(const osp_partition* part, const osp_group_config* cfg,
                            const float* init_params, void* stream, osp_group** out);
void osp_group_destroy(osp_group* g);

/* Deferred-byte budget used by the NEXT resolve (budget_for_epoch(epoch(i+1)),
 * protocol.cpp:396-405, 446-451). Stream-ordered. */
osp_status osp_group_set_budget(osp_group* g, uint64_t budget_bytes, void* stream);
/* Overwrite the current GIB (flags HOST [L], rank-ordered ICS ids HOST).
 * Mirrors OspWorker::on_gib_update (protocol.cpp:252-256). */
osp_status osp_group_set_gib(osp_group* g, const uint8_t* ics_flags, const int32_t* ics_order,
                             int64_t n_order, uint32_t tag, void* stream);

osp_status osp_group_stage1(osp_group* g, const float* deltas, uint64_t ld, void* stream);
osp_status osp_group_stage2_chunk(osp_group* g, int chunk, const float* deltas, uint64_t ld,
                                  void* stream);
/* Every ICS chunk of the iteration in ONE launch (identical results to calling
 * stage2_chunk for c = 0..n_chunks-1 in order: chunks touch disjoint layers).
 * The single-GPU step uses it; per-chunk launches remain for overlap with
 * transfers (multi-GPU) and for the reference's message-by-message flow. */
osp_status osp_group_stage2_all(osp_group* g, const float* deltas, uint64_t ld, void* stream);
osp_status osp_group_resolve(osp_group* g, const float* deltas, uint64_t ld, void* stream);
/* stage1 + stage2_all (two launches; a single-launch variant with per-tile
 * dependency flags measured slower, profiles/r1_ncu_summary.md). */
osp_status osp_group_stages(osp_group* g, const float* deltas, uint64_t ld, void* stream);
/* Heavy-ball momentum on gradient inputs (extension beyond the reference, whose
 * learner is plain SGD, learner.cpp:391-403; parity of mu > 0 is pinned to the
 * oracle fed with deltas from the same rule, not to a reference run): per worker
 * v <- fl(fl(mu*v) + g), delta = sgd_delta(v) = float(-lr*(double)v), fused into
 * stage 1 (the velocity rows [N][M] are read and written once per step).
 * mu = 0 returns to plain sgd_delta (bit-identical). Needs sgd_lr > 0
 * (ConfigError) and the TMA family (OSP_ERR_INVALID); velocities start at 0. */
osp_status osp_group_set_momentum(osp_group* g, double mu, void* stream);
/* stage2_all + resolve, same results (on_push_ics_chunk + check_resolution,
 * protocol.cpp:326-353, 384-439). With the ICS carry the resolve needs
 * nothing from stage 2 (every PGP partial is published by stage 1), so it is
 * launched first and the stage-2 broadcast runs beside it, reading a stage-1
 * snapshot of the ICS lists the resolve rewrites; the stage-2 grid retires only
 * after the resolve has published (device-side join), so the next launch on
 * `stream` sees both. */
osp_status osp_group_stage2_resolve(osp_group* g, const float* deltas, uint64_t ld, void* stream);
/* stage1 + stage2_resolve. */
osp_status osp_group_step(osp_group* g, const float* deltas, uint64_t ld, void* stream);
/* End-to-end step from HOST (pinned or pageable) deltas: H2D copy of the N rows
 * into the group's staging buffer, the step, a D2H read of the encoded next GIB
 * into gib_out (osp_gib_encoded_size(L) bytes, may be NULL) and of the updated
 * global vector into params_out (HOST, M floats, may be NULL) — at the iteration
 * boundary every worker's parameters equal it bit for bit, so it is the
 * step's result as OspServer::global_params() / OspWorker::params() return it
 * (protocol.hpp). Synchronous. */
osp_status osp_group_step_host(osp_group* g, const float* host_deltas, uint64_t host_ld,
                               uint8_t* gib_out, float* params_out, void* stream);
/* Pipelined osp_group_step_host: returns once issued. Call k's H2D (its own
 * copy stream, one of two staging buffers) overlaps call k-1's step and D2H;
 * the step runs on `stream`. gib_out / params_out are written when
 * osp_group_host_wait returns (or when a later call's step has started); host
 * buffers should be pinned, and host_deltas must stay unchanged until the
 * next-but-one call or the wait. Do not issue other steps or GIB installs on
 * the group between the first asynchronous call and osp_group_host_wait (the
 * read-back of the global vector runs on its own stream). */
osp_status osp_group_step_host_async(osp_group* g, const float* host_deltas, uint64_t host_ld,
                                     uint8_t* gib_out, float* params_out, void* stream);
osp_status osp_group_host_wait(osp_group* g);

/* Device pointers into the group state (valid until destroy). */
float* osp_group_global(osp_group* g);
float* osp_group_worker_params(osp_group* g, uint64_t* ld);
double* osp_group_scores(osp_group* g);
/* HOST snapshot of the current GIB / rank order / chunk map (synchronises
 * `stream`). Any pointer may be NULL. chunk_of: [L], -1 for RS layers. */
osp_status osp_group_read_gib(osp_group* g, uint8_t* ics_flags, int32_t* ics_order,
                              int64_t* n_order, int32_t* chunk_of, int* n_used_chunks,
                              uint32_t* tag, uint64_t* deferred_bytes, void* stream);
/* The current GIB as a wire (bitmap + rank order), written on the device by
 * every resolve and install: HOST copy (synchronises `stream`; *len = bytes,
 * out may be NULL to query), the DEVICE buffer itself for a transport that
 * sends from HBM (valid until destroy; its length is in the header: bitmap
 * size, then n), and install from a wire (a bitmap-only wire installs the
 * ascending deferred ids, the reference's convention for a missing order). */
osp_status osp_group_gib_wire(osp_group* g, uint8_t* out, uint64_t cap, uint64_t* len,
                              void* stream);
const uint8_t* osp_group_gib_wire_device(const osp_group* g, uint64_t* max_len);
osp_status osp_group_set_gib_wire(osp_group* g, const uint8_t* buf, uint64_t len, void* stream);
/* Counters: iterations resolved, layers that needed the exact sequential PGP
 * fallback (certificate failures), and resolves that used it. */
osp_status osp_group_stats(osp_group* g, uint64_t* resolved, uint64_t* fallback_layers,
                           uint64_t* fallback_resolves, void* stream);
/* Deferred (ICS) bytes of the GIBs with tags first_tag .. first_tag+n-1 (a
 * device ring of the last 4096 resolutions): the u of each iteration for the
 * algorithmic-byte accounting, without a host sync inside a timed loop. */
osp_status osp_group_deferred_history(osp_group* g, uint32_t first_tag, int n, uint64_t* out,
                                      void* stream);
/* Tile geometry (for roofline accounting and tests). */
/* Effective flags of a group (OSP_GROUP_TMA or OSP_GROUP_REGISTER, plus
 * OSP_GROUP_NO_CARRY when stage 2 re-reads the deltas). */
uint32_t osp_group_flags(const osp_group* g);
osp_status osp_group_geometry(osp_group* g, uint32_t* tile_elems, uint64_t* n_tiles,
                              int* grid_blocks, int* block_threads);

/* ------------------------------------------------------------------------
 * Shard: the multi-GPU path, one process per GPU (PS sharded one shard per
 * GPU). Rank r hosts workers [r*N/P, (r+1)*N/P) and a full
 * replica of the global vector. A stage's exchanged tile sequence is cut into
 * P owner ranges; the owner of a tile reads every worker's delta rows (its own
 * from HBM, the peers' straight out of their HBM over NVLink, CUDA IPC),
 * aggregates them in the reference's fixed worker order in fp64 (push =
 * reduce-scatter, bit-exact), applies locally and stores the aggregate into
 * every rank's pull buffer (pull = all-gather), then raises the tile's flag on
 * every peer, which applies it as soon as it lands. Push, aggregate, pull and
 * apply are ONE kernel per stage (kernels/shard_x.cu); the cross-GPU ordering
 * is per tile inside it, and every rank resolves the identical next GIB.
 *
 * Modes. Default: ONE exchange per iteration — stage 1 moves every tile, the
 * deferred (ICS) layers' aggregate is kept in the carry (the payload split at
 * stage 1, as split_for_sync copies it, protocol.cpp:122-166) and the
 * worker rows get the LGP local estimate; stage 2 is then a local broadcast of
 * the carry (no NVLink traffic). OSP_SHARD_DEFER_ICS: stage 1 exchanges the
 * barrier (RS) layers only and stage 2 exchanges the deferred chunks — the
 * OSP schedule in which the ICS traffic runs beside the next iteration's
 * compute on a side stream. Both are bit-identical to the oracle.
 *
 * Setup: create on every rank, export a handle, exchange the handles (e.g.
 * torch.distributed all_gather), connect with all of them (rank order).
 * The caller writes its workers' deltas into osp_shard_deltas(buf) and steps
 * with that buffer index (two buffers, so the next iteration's compute can
 * fill one while stage 2 still reads the other).
 * ---------------------------------------------------------------------- */
#define OSP_SHARD_HANDLE_BYTES 512
#define OSP_SHARD_DEFER_ICS 1u
typedef struct osp_shard osp_shard;
typedef struct osp_shard_config {
    int world;              /* ranks (GPUs), <= 8 */
    int rank;
    int n_workers;          /* N total logical workers, N % world == 0 */
    const double* weights;  /* HOST, N weights (all workers) */
    int n_chunks;
    uint32_t tile_elems;    /* 0 = default 2048; power of two in [512, 4096] */
    double sgd_lr;          /* 0 = deltas; > 0 fused sgd_delta */
    uint32_t flags;         /* OSP_SHARD_* bits */
} osp_shard_config;

osp_status osp_shard_create(const osp_partition* part, const osp_shard_config* cfg,
                            const float* init_params, void* stream, osp_shard** out);
void osp_shard_destroy(osp_shard* s);
uint64_t osp_shard_handle_size(void);
osp_status osp_shard_export(osp_shard* s, uint8_t* handle);
/* handles: world consecutive OSP_SHARD_HANDLE_BYTES blocks in rank order. */
osp_status osp_shard_connect(osp_shard* s, const uint8_t* handles);
/* Local workers' delta rows of buffer buf (0/1): [N/P][ld] device floats. */
float* osp_shard_deltas(osp_shard* s, int buf, uint64_t* ld);
/* The rank-local state (global replica, worker rows, GIB, stats): use the
 * osp_group_* getters on it. Do not step it directly. */
osp_group* osp_shard_group(osp_shard* s);
/* 1 when stage 2 exchanges the deferred layers (OSP_SHARD_DEFER_ICS, or a
 * local group without the carry buffer), 0 for the single-exchange default. */
int osp_shard_deferred_ics(const osp_shard* s);
/* Synchronisation form of the exchange kernels: 0 per-tile flags, 1 own tiles
 * then a cross-GPU barrier, 2 the reduction chain of the single-exchange
 * stage 1 (rank r continues rank r-1's fp64 running sum; deferred-ICS stages
 * use form 0/1). Environment OSP_SHARD_SYNC=tile|barrier|chain at create. */
int osp_shard_sync_form(const osp_shard* s);
osp_status osp_shard_stage1(osp_shard* s, int buf, void* stream);
/* ProtocolError before stage 1 of the iteration. */
osp_status osp_shard_stage2(osp_shard* s, int c0, int c1, int buf, void* stream);
osp_status osp_shard_resolve(osp_shard* s, int buf, void* stream);
osp_status osp_shard_step(osp_shard* s, int buf, void* stream);
/* One step with CUDA events between the phases (synchronises `stream`):
 * ms[0] = stage 1 (exchange kernel), ms[1] = stage 2, ms[2] = resolve. */
osp_status osp_shard_profile(osp_shard* s, int buf, float* ms, void* stream);
/* Diagnostics: this rank's own tiles of a stage's exchange launched alone (no
 * cross-GPU waits, no flags), so a profiler that serialises kernels (ncu) can
 * replay it. The peers must be idle with their rows in place. */
osp_status osp_shard_solo_agg(osp_shard* s, int stage, int buf, void* stream);
/* ProtocolError if a cross-GPU wait timed out (synchronises `stream`). */
osp_status osp_shard_check(osp_shard* s, void* stream);
/* Diagnostics (OSP_SHARD_DEBUG=1 in the environment at create): the exchange
 * kernel's counters summed over CTAs since the last read, then reset —
 * [0] producer cycles blocked on a peer's tile flag, [1] producer cycles
 * waiting for a free ring slot, [2] consumer (warp 0) cycles waiting for data,
 * [3] publisher cycles in the system-scope fence + flag stores, [4] producer
 * cycles in total, [5] blocking B waits, [6..8] A / B / L items, [9] flag
 * batches. Returns 1 when filled, 0 when disabled. */
int osp_shard_debug_counters(osp_shard* s, unsigned long long* out16);
/* OSP_SHARD_DEBUG=2 (chain form): the last stage-1 launch's per-tile timeline,
 * [8][NT] globaltimer ns (0 PRE issued, 2 PRE flag published, 3 FIN flag
 * acquired, 4 FIN published, 5 APPLY flag acquired, 6 APPLY done). out null:
 * returns the entry count; else copies min(n, count) entries and returns it. */
uint64_t osp_shard_debug_trace(osp_shard* s, unsigned long long* out, uint64_t n);
/* Synthetic deltas of workers [worker0, worker0+n_workers) into [n_workers][ld]. */
osp_status osp_synth_deltas_range(uint64_t seed, int worker0, int n_workers, uint64_t iteration,
                                  uint64_t n, float* out, uint64_t ld, void* stream);

/* ------------------------------------------------------------------------
 * Learner: the gradient producer on the other side of the sync path — the
 * reference learner's MLP forward_backward (learner.hpp:63-64,
 * learner.cpp:299-367) for N workers at once over a device-resident dataset
 * (Dataset, learner.hpp:23-31: features [n][widths[0]] row-major, labels [n]).
 * Parameters are the partition-ordered vector W0, b0, W1, b1, ... of
 * mlp_partition (learner.hpp:51-53), one row per worker (e.g. the group's
 * worker rows); gradients come out as float rows, ready for an OSP group
 * created with sgd_lr > 0 (the step applies sgd_delta, learner.cpp:391-398).
 * fp64 arithmetic in the reference's order: relu+MSE is bit-exact; tanh and
 * the softmax's exp/log use CUDA's libm (tolerance, tests/test_gpu_learner.py).
 * ---------------------------------------------------------------------- */
typedef struct osp_mlp osp_mlp;
#define OSP_ACT_RELU 0
#define OSP_ACT_TANH 1
#define OSP_LOSS_CE 0  /* Loss::softmax_cross_entropy */
#define OSP_LOSS_MSE 1 /* Loss::mse */
/* ConfigError for the MlpSpec::validate cases (learner.cpp:15-20); the dataset
 * pointers are borrowed (device memory, must outlive the handle). */
osp_status osp_mlp_create(const int32_t* widths, int n_widths, int activation, int loss,
                          const float* features, const int32_t* labels, uint64_t n_rows,
                          osp_mlp** out);
void osp_mlp_destroy(osp_mlp* m);
uint64_t osp_mlp_num_params(const osp_mlp* m);
/* Asynchronous: batch is [n_workers][batch_size] device row indices; grad_out
 * [n_workers][ld_out] floats; loss_out (device, may be NULL) [n_workers] mean
 * batch losses. Row / label range and finiteness are flagged on the device and
 * reported by osp_mlp_check (ShapeError / NumericError, as the reference throws). */
osp_status osp_mlp_grad(osp_mlp* m, const float* params, uint64_t ld_params, int n_workers,
                        const int32_t* batch, int batch_size, float* grad_out, uint64_t ld_out,
                        double* loss_out, void* stream);
osp_status osp_mlp_check(osp_mlp* m, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* OSP_C_H */
