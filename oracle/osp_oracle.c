/*
 * osp_oracle.c — CPU restatement of the reference OSP sync path.
 *
 * TEST INFRASTRUCTURE ONLY: the parity checker for the B200 kernels. Loaded by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg; never by the
 * product. Built with -ffp-contract=off and no -march so every double/float
 * operation rounds exactly where the reference's does (hard part 3).
 *
 * Parity pinned against the reference unit-test hand vectors and against dumps
 * of the unmodified reference engine (tests/golden/, oracle/gen_golden.py).
 */
#include "osp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- rng.hpp:16-36 ------------------------------------------------------ */

#define OO_GAMMA 0x9e3779b97f4a7c15ULL

static uint64_t oo_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t oo_splitmix64(uint64_t* state) {
    *state += OO_GAMMA;
    return oo_mix(*state);
}

uint64_t oo_derive_seed(uint64_t root, uint64_t tag, uint64_t a, uint64_t b) {
    uint64_t s = root;
    oo_splitmix64(&s);
    s ^= 0x6a09e667f3bcc908ULL + tag;
    oo_splitmix64(&s);
    s ^= 0xbb67ae8584caa73bULL + a;
    oo_splitmix64(&s);
    s ^= 0x3c6ef372fe94f82bULL + b;
    return oo_splitmix64(&s);
}

/* Rng(seed) warms up with two draws (rng.hpp:50-54), so draw k reads the state
 * seed + (k + 3) * gamma. uniform(lo, hi) = lo + (hi - lo) * u53 (rng.hpp:59-61),
 * rounded to float by the caller (runner.cpp:318-320). */
void oo_synth_delta(uint64_t seed, uint64_t worker, uint64_t iteration, uint64_t first,
                    uint64_t n, float* out) {
    uint64_t s = oo_derive_seed(seed, 6, worker, iteration);
    volatile double lo = -1e-3, hi = 1e-3;
    double span = hi - lo;
    double l = lo;
    for (uint64_t k = 0; k < n; ++k) {
        uint64_t x = oo_mix(s + (first + k + 3) * OO_GAMMA);
        double u = (double)(x >> 11) * 0x1.0p-53;
        double prod = span * u;
        out[k] = (float)(l + prod);
    }
}

/* ---- learner.cpp:391-403 ------------------------------------------------ */

void oo_sgd_delta(const float* grad, uint64_t n, double lr, float* out) {
    for (uint64_t i = 0; i < n; ++i) out[i] = (float)(-lr * (double)grad[i]);
}

double oo_lr_at_epoch(double initial_lr, uint64_t epoch) {
    return ldexp(initial_lr, -(int)(epoch / 10));
}

/* ---- protocol.cpp:9-30 -------------------------------------------------- */

int oo_aggregate_layer(int n_workers, const float* const* contribs, const double* weights,
                       uint64_t n, float* out) {
    if (n_workers < 1) return -1;
    double tw = 0.0;
    for (int w = 0; w < n_workers; ++w) tw += weights[w];
    if (!(tw > 0.0)) return -1;
    for (uint64_t e = 0; e < n; ++e) {
        double sum = 0.0;
        for (int w = 0; w < n_workers; ++w) {
            double term = weights[w] * (double)contribs[w][e];
            sum += term;
        }
        out[e] = (float)(sum / tw);
    }
    return 0;
}

/* ---- importance.cpp ----------------------------------------------------- */

void oo_pgp(int64_t n_layers, const uint64_t* counts, const float* params, const float* grads,
            double* scores) {
    uint64_t off = 0;
    for (int64_t l = 0; l < n_layers; ++l) {
        double sum = 0.0;
        for (uint64_t j = off; j < off + counts[l]; ++j) {
            sum += fabs((double)grads[j] * (double)params[j]);
        }
        scores[l] = sum;
        off += counts[l];
    }
}

/* importance.cpp:20-25 continued over a stream: the same sequential sum of one
 * layer, fed in consecutive pieces (acc carries the running sum). Used by the
 * 1B-parameter parity test, whose layers do not fit the host in one piece. */
void oo_pgp_accum(uint64_t n, const float* params, const float* grads, double* acc) {
    double sum = *acc;
    for (uint64_t j = 0; j < n; ++j) sum += fabs((double)grads[j] * (double)params[j]);
    *acc = sum;
}

static const double* g_rank_scores;

static int rank_cmp(const void* a, const void* b) {
    int32_t ia = *(const int32_t*)a, ib = *(const int32_t*)b;
    double sa = g_rank_scores[ia], sb = g_rank_scores[ib];
    if (sa != sb) return sa < sb ? -1 : 1;
    return (ia > ib) - (ia < ib);
}

void oo_rank(int64_t n_layers, const double* scores, int32_t* order) {
    for (int64_t i = 0; i < n_layers; ++i) order[i] = (int32_t)i;
    g_rank_scores = scores;
    /* (score, id) keys are unique, so any correct sort equals stable_sort. */
    qsort(order, (size_t)n_layers, sizeof(int32_t), rank_cmp);
}

void oo_build_gib(int64_t n_layers, const double* scores, const uint64_t* counts, uint32_t bpe,
                  uint64_t budget, uint8_t* ics_flags) {
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_layers ? n_layers : 1));
    oo_rank(n_layers, scores, order);
    memset(ics_flags, 0, (size_t)n_layers);
    uint64_t used = 0;
    for (int64_t r = 0; r < n_layers; ++r) {
        int32_t id = order[r];
        uint64_t sz = counts[id] * (uint64_t)bpe;
        if (used + sz > budget) break;
        ics_flags[id] = 1;
        used += sz;
    }
    free(order);
}

uint64_t oo_gib_encoded_size(uint64_t n_layers) { return 8 + (n_layers + 7) / 8; }

static void put_u32le(uint8_t* p, uint32_t v) {
    p[0] = (uint8_t)(v & 0xff);
    p[1] = (uint8_t)((v >> 8) & 0xff);
    p[2] = (uint8_t)((v >> 16) & 0xff);
    p[3] = (uint8_t)((v >> 24) & 0xff);
}

static uint32_t get_u32le(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

void oo_gib_encode(uint32_t tag, uint64_t n_layers, const uint8_t* ics_flags, uint8_t* out) {
    uint64_t size = oo_gib_encoded_size(n_layers);
    memset(out, 0, (size_t)size);
    put_u32le(out, tag);
    put_u32le(out + 4, (uint32_t)n_layers);
    for (uint64_t k = 0; k < n_layers; ++k) {
        if (ics_flags[k]) out[8 + k / 8] |= (uint8_t)(1u << (k % 8));
    }
}

int oo_gib_decode(const uint8_t* buf, uint64_t len, uint32_t* tag, uint32_t* n_layers,
                  uint8_t* flags, uint64_t flags_cap) {
    if (len < 8) return -1;
    *tag = get_u32le(buf);
    *n_layers = get_u32le(buf + 4);
    if (len < oo_gib_encoded_size(*n_layers)) return -1;
    if (*n_layers > flags_cap) return -2;
    for (uint64_t k = 0; k < *n_layers; ++k) flags[k] = (buf[8 + k / 8] >> (k % 8)) & 1u;
    return 0;
}

/* ---- protocol.cpp:122-166 ----------------------------------------------- */

int oo_split(int64_t n_layers, const uint64_t* counts, uint32_t bpe, const uint8_t* ics_flags,
             const int32_t* ics_order, int64_t n_order, int n_chunks, int32_t* rs_ids,
             int64_t* n_rs, int32_t* chunk_of) {
    if (n_chunks < 1) return -1;
    int64_t nr = 0;
    for (int64_t l = 0; l < n_layers; ++l) {
        if (!ics_flags[l]) rs_ids[nr++] = (int32_t)l;
        chunk_of[l] = -1;
    }
    *n_rs = nr;
    /* deferred order: rank order filtered by the bitmap, then missing ids ascending */
    int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_layers + n_order + 1));
    uint8_t* seen = (uint8_t*)calloc(n_layers > 0 ? (size_t)n_layers : 1u, 1);
    int64_t no = 0;
    for (int64_t i = 0; i < n_order; ++i) {
        int32_t id = ics_order[i];
        if (id >= 0 && id < n_layers && ics_flags[id]) {
            order[no++] = id;
            seen[id] = 1;
        }
    }
    for (int64_t l = 0; l < n_layers; ++l) {
        if (ics_flags[l] && !seen[l]) order[no++] = (int32_t)l;
    }
    int used_chunks = 0;
    if (no > 0) {
        uint64_t total = 0;
        for (int64_t i = 0; i < no; ++i) total += counts[order[i]] * (uint64_t)bpe;
        int* raw = (int*)malloc(sizeof(int) * (size_t)no);
        uint64_t cum = 0;
        for (int64_t i = 0; i < no; ++i) {
            uint64_t idx = total == 0 ? 0 : (cum * (uint64_t)n_chunks) / total;
            if (idx > (uint64_t)(n_chunks - 1)) idx = (uint64_t)(n_chunks - 1);
            raw[i] = (int)idx;
            cum += counts[order[i]] * (uint64_t)bpe;
        }
        /* empty chunks are dropped: renumber the distinct raw indices in order */
        int* remap = (int*)malloc(sizeof(int) * (size_t)n_chunks);
        for (int c = 0; c < n_chunks; ++c) remap[c] = -1;
        for (int64_t i = 0; i < no; ++i) remap[raw[i]] = 0;
        for (int c = 0; c < n_chunks; ++c) {
            if (remap[c] == 0) remap[c] = used_chunks++;
        }
        for (int64_t i = 0; i < no; ++i) chunk_of[order[i]] = remap[raw[i]];
        free(remap);
        free(raw);
    }
    free(order);
    free(seen);
    return used_chunks;
}

/* ---- tuning.cpp --------------------------------------------------------- */

uint64_t oo_compute_umax(double bandwidth_bps, double loss_rate, double t_c_seconds,
                         int n_workers, uint64_t model_bytes, int eq5_literal) {
    double raw;
    if (eq5_literal) raw = bandwidth_bps * (1.0 + loss_rate) * t_c_seconds / n_workers;
    else raw = bandwidth_bps * t_c_seconds / (n_workers * (1.0 + loss_rate));
    double cap = 0.8 * (double)model_bytes;
    return (uint64_t)floor(raw < cap ? raw : cap);
}

int64_t oo_tune_sgu(double* initial_loss, int* has_initial, uint64_t u_max, uint64_t epoch_index,
                    double epoch_loss) {
    if (epoch_index < 1) return -1;
    if (epoch_loss < 0) return -2;
    if (epoch_index == 1) {
        *initial_loss = epoch_loss;
        *has_initial = 1;
        return 0;
    }
    if (!*has_initial) return -3;
    double factor;
    if (*initial_loss <= 0.0) {
        factor = 1.0;
    } else {
        factor = 1.0 - epoch_loss / *initial_loss;
        if (factor < 0.0) factor = 0.0;
        if (factor > 1.0) factor = 1.0;
    }
    return (int64_t)(uint64_t)floor(factor * (double)u_max);
}

/* ---- one synchronous iteration (protocol.cpp:172-447) ------------------- */

int oo_step(int64_t n_layers, const uint64_t* counts, uint32_t bpe, int n_workers,
            const double* weights, const float* deltas, float* G, float* P,
            const uint8_t* ics_flags_in, const int32_t* order_in, int64_t n_order_in,
            int n_chunks, uint64_t budget, float* p_stage1, float* agg, double* scores,
            uint8_t* ics_flags_out, int32_t* order_out, int64_t* n_order_out, int32_t* chunk_of) {
    uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n_layers + 1));
    offsets[0] = 0;
    for (int64_t l = 0; l < n_layers; ++l) offsets[l + 1] = offsets[l] + counts[l];
    uint64_t M = offsets[n_layers];
    int32_t* rs_ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_layers + 1));
    int32_t* chunks = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_layers + 1));
    int64_t n_rs = 0;
    int used = oo_split(n_layers, counts, bpe, ics_flags_in, order_in, n_order_in, n_chunks,
                        rs_ids, &n_rs, chunks);
    if (used < 0) {
        free(offsets);
        free(rs_ids);
        free(chunks);
        return -1;
    }
    const float** contribs = (const float**)malloc(sizeof(float*) * (size_t)n_workers);
    /* base copies: what lgp_partial records before applying the local estimate */
    float* base = (float*)malloc(sizeof(float) * (size_t)(M * (uint64_t)n_workers + 1));

    /* barrier: RS layers aggregate (ascending id), global += agg (protocol.cpp:292-307) */
    for (int64_t r = 0; r < n_rs; ++r) {
        int32_t id = rs_ids[r];
        for (int w = 0; w < n_workers; ++w) contribs[w] = deltas + (uint64_t)w * M + offsets[id];
        oo_aggregate_layer(n_workers, contribs, weights, counts[id], agg + offsets[id]);
        for (uint64_t e = offsets[id]; e < offsets[id + 1]; ++e) G[e] += agg[e];
    }
    /* pull: lgp_partial per worker (protocol.cpp:69-97, 212-228) */
    for (int w = 0; w < n_workers; ++w) {
        float* p = P + (uint64_t)w * M;
        const float* d = deltas + (uint64_t)w * M;
        for (int64_t l = 0; l < n_layers; ++l) {
            if (!ics_flags_in[l]) {
                for (uint64_t e = offsets[l]; e < offsets[l + 1]; ++e) p[e] += 1.0f * agg[e];
            }
        }
        for (int64_t l = 0; l < n_layers; ++l) {
            if (ics_flags_in[l]) {
                for (uint64_t e = offsets[l]; e < offsets[l + 1]; ++e) {
                    base[(uint64_t)w * M + e] = p[e];
                    p[e] += d[e];
                }
            }
        }
    }
    if (p_stage1) memcpy(p_stage1, P, sizeof(float) * (size_t)(M * (uint64_t)n_workers));
    /* ICS chunks in order: aggregate, apply, then workers correct = base + global */
    for (int c = 0; c < used; ++c) {
        for (int64_t l = 0; l < n_layers; ++l) {
            if (chunks[l] != c) continue;
            for (int w = 0; w < n_workers; ++w) contribs[w] = deltas + (uint64_t)w * M + offsets[l];
            oo_aggregate_layer(n_workers, contribs, weights, counts[l], agg + offsets[l]);
            for (uint64_t e = offsets[l]; e < offsets[l + 1]; ++e) G[e] += agg[e];
            for (int w = 0; w < n_workers; ++w) {
                float* p = P + (uint64_t)w * M;
                for (uint64_t e = offsets[l]; e < offsets[l + 1]; ++e)
                    p[e] = base[(uint64_t)w * M + e] + agg[e];
            }
        }
    }
    /* resolution: PGP on (aggregated deltas, post-update global), GIB, rank order
     * restricted to the bitmap (protocol.cpp:384-439) */
    oo_pgp(n_layers, counts, G, agg, scores);
    oo_build_gib(n_layers, scores, counts, bpe, budget, ics_flags_out);
    int32_t* rank = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n_layers + 1));
    oo_rank(n_layers, scores, rank);
    int64_t no = 0;
    for (int64_t r = 0; r < n_layers; ++r) {
        if (ics_flags_out[rank[r]]) order_out[no++] = rank[r];
    }
    *n_order_out = no;
    if (chunk_of) memcpy(chunk_of, chunks, sizeof(int32_t) * (size_t)n_layers);
    free(rank);
    free(base);
    free(contribs);
    free(offsets);
    free(rs_ids);
    free(chunks);
    return used;
}

/* ---- message.cpp:53-78 (payload wire encoding) -------------------------- */

uint64_t oo_encode_payload(uint8_t kind, uint32_t iteration, int64_t n_layers,
                           const uint64_t* counts, const float* values, const int32_t* ids,
                           int64_t n_ids, uint8_t* out) {
    uint64_t* offsets = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(n_layers + 1));
    offsets[0] = 0;
    for (int64_t l = 0; l < n_layers; ++l) offsets[l + 1] = offsets[l] + counts[l];
    uint64_t at = 0;
    out[at++] = kind;
    put_u32le(out + at, iteration);
    at += 4;
    out[at++] = (uint8_t)(n_ids & 0xff);
    out[at++] = (uint8_t)((n_ids >> 8) & 0xff);
    for (int64_t i = 0; i < n_ids; ++i) {
        const int32_t id = ids[i];
        put_u32le(out + at, (uint32_t)id);
        put_u32le(out + at + 4, (uint32_t)counts[id]);
        at += 8;
        for (uint64_t e = 0; e < counts[id]; ++e) {
            uint32_t bits;
            memcpy(&bits, &values[offsets[id] + e], 4);
            put_u32le(out + at, bits);
            at += 4;
        }
    }
    free(offsets);
    return at;
}
