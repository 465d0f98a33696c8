// Internal declarations shared by the kernels and the C-ABI layer.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "osp_c.h"

namespace osp {

// ---- error plumbing (C-ABI never throws) -----------------------------------
void set_error(const std::string& msg);
osp_status fail(osp_status s, const std::string& msg);
osp_status cuda_fail(cudaError_t e, const char* what);

#define OSP_CUDA(call)                                            \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return ::osp::cuda_fail(e_, #call); \
    } while (0)

#define OSP_CHECK_LAUNCH(what)                                    \
    do {                                                          \
        cudaError_t e_ = cudaGetLastError();                      \
        if (e_ != cudaSuccess) return ::osp::cuda_fail(e_, what); \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();
// Identity of the calling thread's current CUDA context (cuCtxGetId through the
// runtime's driver entry point). Function attributes such as the dynamic
// shared-memory opt-in belong to a context, so launch-side caches key on this:
// a recreated primary context (cudaDeviceReset) gets a new id.
unsigned long long current_ctx_id();

// ---- aggregation parameters (kernel argument, by value) ---------------------
struct AggParams {
    int n;                       // workers
    int divide;                  // 0 when sum(weights) == 1.0 exactly (x / 1.0 == x)
    int sgd;                     // inputs are gradients: x = float(-lr * (double)g)
    double neg_lr;
    double total;                // sum of weights, ascending (protocol.cpp:14-15)
    double w[OSP_MAX_WORKERS];
};

AggParams make_agg_params(int n, const double* weights, double sgd_lr);

// ---- group device view (kernel argument, by value) ---------------------------
struct GroupView {
    int L;                       // layers
    int T;                       // tile elements (power of two)
    int NT;                      // total tiles
    int n_chunks;                // chunk slots
    uint32_t bpe;
    const uint64_t* offsets;     // [L]
    const uint64_t* counts;      // [L]
    const int* tile_base;        // [L+1] first global tile of each layer
    const int* tile_layer;       // [NT]
    float* G;                    // [M]
    float* P;                    // [N][ldP]
    uint64_t ldP;
    double* partials;            // [NT] per-tile PGP partial sums
    uint8_t* flags;              // [L] current GIB (1 = ICS)
    int* ics_layers;             // [L] ICS layers, rank order (valid prefix n_ics)
    int* chunk_begin;            // [n_chunks+1] into ics_layers, compacted chunks
    int* ics_tile_prefix;        // [L+1] exclusive tile prefix along ics_layers
    int* meta;                   // [8] n_ics, n_used_chunks, need_fallback, ...
    uint64_t* meta64;            // [8] budget, tag, deferred_bytes, resolved, fb_layers, fb_resolves
    double* scores;              // [L] approximate (tree) scores
    double* exact;               // [L] exact sequential scores (fallback layers)
    uint8_t* marked;             // [L] needs exact score
    int* chunk_of;               // [L] compacted chunk or -1
    uint8_t* gib_bytes;          // [8 + ceil(L/8) + 4 + 4L] current GIB wire: bitmap || n || rank order
    uint64_t* hist;              // [kHist] deferred bytes of the GIB with tag t at t % kHist
    int* sched;                  // [16] dynamic tile scheduler counters (SchedIdx)
    double* lscore;              // [L] per-layer tree sum of the tile partials
    int* rs_layers;              // [L] RS (barrier) layers, ascending id (valid prefix n_rs)
    int* rs_tile_prefix;         // [L+1] exclusive tile prefix along rs_layers
    const float* agg_full;       // [M] aggregated deltas (sharded path), or null
    // ICS carry (TMA family): stage 1 aggregates the ICS elements while it has
    // their delta rows in shared memory anyway and stores G_old + agg here; the
    // stage-2 kernels then only broadcast it into G and the worker rows. Null =
    // stage 2 re-reads the deltas and G (register-staged family, sharded path).
    float* C;                    // [M] or null
    // Stage-1 snapshot of the current ICS lists for the carry stage 2, so the
    // next GIB's resolve may rewrite the live lists while stage 2 still runs
    // (osp_group_step: resolve overlapped with stage 2). Layout: [0] n_used
    // chunks, [1] the resolve epoch stage 2 joins on, [4..] chunk_begin
    // [n_chunks+1], ics_layers [L], ics_tile_prefix [L+1]. Null without carry.
    int* snap;
    // Heavy-ball momentum on the gradient inputs (extension, TMA family, sgd only):
    // per worker v <- mu*v + g (fp32, no FMA) in stage 1, delta = sgd_delta(v).
    // V [N][ldP] holds the updated velocities after stage 1. Null = plain SGD.
    float* V;
    float mu;
    // resolve's per-layer sums are split into items of <= kSumChunk tiles so a
    // huge layer is summed by many blocks (fixed order: items ascending)
    const int* sum_items;        // [n_sum_items][3] layer, first tile, end tile
    int n_sum_items;
    const int* layer_items;      // [L+1] first item of each layer
    double* item_sums;           // [n_sum_items]
    // the single-CTA resolve's per-layer arrays when L > kSmemResolveLayers
    // (global memory; null: dynamic shared memory)
    char* rscratch;
};
constexpr int kSumChunk = 4096;  // tiles per resolve sum item

enum SchedIdx {
    SCHED_S1_NEXT = 0,
    SCHED_S1_DONE = 1,
    SCHED_S2_NEXT = 2,
    SCHED_S2_DONE = 3,
    SCHED_RESOLVE_DONE = 4
};
enum MetaIdx { META_N_ICS = 0, META_N_USED = 1, META_NEED_FB = 2, META_N_RS = 3 };
enum Meta64Idx {
    META64_BUDGET = 0,
    META64_TAG = 1,
    META64_DEFERRED = 2,
    META64_RESOLVED = 3,
    META64_FB_LAYERS = 4,
    META64_FB_RESOLVES = 5,
    META64_RESOLVE_DONE = 6  // == META64_RESOLVED once that resolve's lists are written
};
constexpr int kSnapHead = 4;
__host__ __device__ inline int snap_ints(int L, int n_chunks) { return kSnapHead + n_chunks + 1 + 2 * L + 1; }

constexpr int kHist = 4096;
// Layers per partition. The single-CTA resolve keeps ~60 B per layer in shared
// memory up to kSmemResolveLayers layers and in a global scratch buffer above.
constexpr int kMaxLayers = 65536;
constexpr int kSmemResolveLayers = 3072;
size_t resolve_scratch_bytes(int L);
constexpr int kStageThreads = 256;
constexpr uint32_t kDefaultTile = 512;  // elements per warp tile (sweep: profiles/)
constexpr uint32_t kDefaultTmaTile = 1024;  // TMA-staged kernels (tools/tma_sweep.sh)
constexpr int kResolveThreads = 1024;

// ---- sharded (multi-GPU) path (kernels/shard_x.cu) ---------------------------
constexpr int kMaxRanks = 8;           // one NVLink/NVSwitch node
constexpr int kXMaxStagedWorkers = 8;  // A items stage every worker's row in shared memory

// Exchange modes: SINGLE = every tile in one exchange (the ICS payload split at
// stage 1, kept in the carry, broadcast locally by stage 2); RS = the barrier
// layers only, local estimates for the deferred ones; ICS = the deferred layers
// of chunks [c0, c1) (stage 2 of the deferred-ICS mode).
enum XMode { XM_SINGLE = 0, XM_RS = 1, XM_ICS = 2 };

struct XArgs {
    const float* xrow[OSP_MAX_WORKERS];  // every worker's delta row (local HBM or peer)
    float* agg[kMaxRanks];               // every rank's pull buffer [ldX]
    double* part[kMaxRanks];             // every rank's per-tile PGP partials [NT]
    unsigned* tflag[kMaxRanks];          // every rank's per-tile ready flags [NT]
    unsigned* ready[kMaxRanks];          // every rank's slots [2][kMaxRanks]: deltas ready, own tiles done
    double* pre[kMaxRanks];              // chain form: every rank's fp64 running sums [ldX]
    int chain_lead;                      // chain form, mixed CTAs: PRE items kept ahead of APPLY
    int chain_arena;                     // chain form: ring arena in floats (set at launch)
    int chain_pushagg;                   // chain form: the last rank stores agg into every rank
    unsigned long long* trace;           // chain form diagnostics: [8][NT] globaltimer stamps or null
    unsigned* error;                     // local: set when a bounded wait timed out
    int world, rank, n_loc;
    unsigned epoch;                      // iteration number (1-based)
    int mode;                            // XMode
    int c0, c1;                          // XM_ICS chunk range
    int solo;                            // diagnostics: own tiles only, no waits or flags
    int vec;                             // every row and buffer 16-byte aligned
    int slot_rows;                       // shared-memory rows per ring slot
    int lag;                             // B items' due-time lag behind the A items
    int pub_batch;                       // flags published under one fence, at most
    int pub_min;                         // ... and at least, unless the stage ends
    int split;                           // CTA roles: even = own tiles, odd = peers' + local
    int phase;                           // 0 per-tile flags; 1 own tiles + signal; 2 peers' tiles
    unsigned* ticket;                    // local: last-CTA counter of phase 1
    unsigned done_epoch;                 // phase 1/2: count of barrier-form launches (all ranks alike)
    unsigned long long* dbg;             // diagnostics counters [16] or null
};
int x_slot_rows(int n_workers);
bool shard_x_supported(int n_workers, int T, int L);
cudaError_t launch_shard_x(const GroupView& g, const AggParams& ap, const XArgs& xa, cudaStream_t s);
// the barrier form's phase 2: the peers' tiles from the pull buffer (128-bit loads)
cudaError_t launch_shard_peer_apply(const GroupView& g, const AggParams& ap, const XArgs& xa,
                                    cudaStream_t s);

// The chain form of the single-exchange stage 1 (kernels/shard_chain.cu):
// rank r continues rank r-1's fp64 running sum over its own workers, the last
// rank finishes and the others pull the aggregate back; tflag holds [2][NT]
// (tile flags, chain flags).
bool shard_chain_supported(int n_loc, int T, int L);
cudaError_t launch_shard_chain(const GroupView& g, const AggParams& ap, const XArgs& xa, cudaStream_t s);

// ---- gradient producer: the reference learner's MLP forward/backward (kernels/learner.cu)
constexpr int kMlpMaxDepth = 8;  // linear layers
struct MlpArgs {
    int depth;                       // linear layers
    int widths[kMlpMaxDepth + 1];    // input, hidden..., output
    int act;                         // 0 relu, 1 tanh
    int loss;                        // 0 softmax cross-entropy, 1 MSE
    int maxw;                        // largest width
    int B;                           // batch rows per worker
    uint64_t n_params;               // mlp_partition total
    const float* P;                  // [N][ldP] worker parameter rows
    uint64_t ldP;
    const float* feats;              // [n][widths[0]] dataset rows
    uint64_t n_rows;                 // n
    const int* labels;               // [n]
    const int* batch;                // [N][B] row indices
    float* out;                      // [N][ldo] float gradients
    uint64_t ldo;
    double* loss_out;                // [N] mean batch loss, or null
    unsigned* error;                 // 1 non-finite (NumericError), 2 label out of range (ShapeError)
};
size_t mlp_grad_smem(const MlpArgs& a);
cudaError_t launch_mlp_grad(const MlpArgs& a, int n_workers, cudaStream_t s);

// Opt a kernel into `smem` bytes of dynamic shared memory and return its
// occupancy, cached per (context, kernel, bytes) (stage_tma.cu).
cudaError_t tma_blocks_per_sm(const void* kern, int threads, size_t smem, int* per_sm);

// ---- payload wire codec (kernels/codec.cu) -----------------------------------
struct CodecSeg {
    uint64_t hdr;    // encode: byte offset of the layer's (id, count) header; decode: value offset
    uint64_t src;    // element offset in the flat vector
    uint32_t id;
    uint32_t count;
};
cudaError_t launch_encode(const float* values, const CodecSeg* segs_dev, int n_seg,
                          uint64_t max_count, uint8_t* out, cudaStream_t s);
cudaError_t launch_decode_index(const uint8_t* buf, uint64_t len, uint64_t* idx, int* status,
                                uint32_t* hdr, cudaStream_t s);
cudaError_t launch_decode_scatter(const uint8_t* buf, const CodecSeg* segs_dev, int n_seg,
                                  uint64_t max_count, float* values, cudaStream_t s);

// ---- launchers (kernels/*.cu) ----------------------------------------------
cudaError_t launch_stage1(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int grid, cudaStream_t s);
// Chunks [c0, c1) of the current ICS list in one launch.
cudaError_t launch_stage2(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                          int c0, int c1, int grid, cudaStream_t s);
cudaError_t launch_resolve(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                           cudaStream_t s);
cudaError_t launch_set_budget(const GroupView& g, uint64_t budget, cudaStream_t s);
// Per-tile PGP partials |grads * params| in g's tile geometry (g.partials).
cudaError_t launch_pgp_tiles(const GroupView& g, const float* params, const float* grads,
                             cudaStream_t s);
// Rebuild device lists from g.flags + the given rank-ordered ICS ids (device).
cudaError_t launch_install_gib(const GroupView& g, const int* order, int n_order, uint32_t tag,
                               cudaStream_t s);
int stage_blocks_per_sm(int n_workers, int n_layers);
// Whole iteration (stage 1, carry broadcast, warp-level resolve) in one launch
// of one CTA for launch-bound layouts (kernels/step_small.cu). Needs the carry
// buffer C, no momentum, L <= kSmallMaxLayers and M within the tile table.
constexpr int kSmallMaxLayers = 32;
constexpr int kSmallMaxTiles = 1056;
bool small_step_supported(int n_workers, int L, uint64_t M);
cudaError_t launch_step_small(const GroupView& g, const AggParams& ap, const float* X,
                              uint64_t ldX, cudaStream_t s);
// TMA-staged stage kernels (stage_tma.cu)
bool tma_supported(int n_workers, int T, int L);
// momentum stages N velocity rows beside the N delta rows + G
bool tma_momentum_supported(int n_workers, int T, int L);
cudaError_t launch_stage1_tma(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                              cudaStream_t s);
// overlap = 1 (carry only): launched after the resolve of the same iteration,
// runs beside it and joins on its epoch before retiring (osp_group_step).
cudaError_t launch_stage2_tma(const GroupView& g, const AggParams& ap, const float* X, uint64_t ldX,
                              int c0, int c1, cudaStream_t s, int overlap = 0);

cudaError_t launch_aggregate_layer(const float* const* contribs, const AggParams& ap, uint64_t n,
                                   float* out, cudaStream_t s);
cudaError_t launch_aggregate_apply_segments(const float* const* contribs, const AggParams& ap,
                                            const uint64_t* seg_off, const uint64_t* seg_cnt,
                                            int n_seg, float* global, float* agg_out,
                                            cudaStream_t s);
cudaError_t launch_apply_delta(float* p, const float* d, uint64_t n, float scale, cudaStream_t s);
cudaError_t launch_sgd_delta(const float* g, uint64_t n, double lr, float* out, cudaStream_t s);
cudaError_t launch_synth(uint64_t seed, int n_workers, uint64_t iteration, uint64_t first,
                         uint64_t n, float* out, uint64_t ld, uint64_t worker0, cudaStream_t s);
cudaError_t launch_lgp_partial_segments(float* p, const float* global_delta,
                                        const float* local_delta, float* base,
                                        const uint64_t* seg_off, const uint64_t* seg_cnt,
                                        const uint8_t* seg_local, int n_seg, cudaStream_t s);
cudaError_t launch_lgp_correct_segments(float* p, const float* base, const float* global_delta,
                                        const uint64_t* seg_off, const uint64_t* seg_cnt,
                                        int n_seg, cudaStream_t s);
cudaError_t launch_pgp_exact(const float* params, const float* grads, const uint64_t* offsets,
                             const uint64_t* counts, int L, double* scores, cudaStream_t s);
cudaError_t launch_rank_gib(const double* scores, const uint64_t* counts, uint32_t bpe, int L,
                            uint64_t budget, int* order, uint8_t* flags, cudaStream_t s);

}  // namespace osp
