// C-ABI of the message-level engines (include/osp_engine.h) over the C++
// façade classes. Every entry point converts exceptions to osp_status (the
// inverse of the façade's status -> pslab::Error mapping) and records the
// message for osp_engine_last_error().

#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "osp_engine.h"
#include "pslab/message.hpp"
#include "pslab/protocol.hpp"

namespace {

thread_local std::string g_last_error;

osp_status set_error(osp_status s, const char* what) {
    g_last_error = what ? what : "";
    return s;
}

template <typename F>
osp_status guarded(F&& f) {
    try {
        f();
        return OSP_OK;
    } catch (const pslab::PartitionError& e) {
        return set_error(OSP_ERR_PARTITION, e.what());
    } catch (const pslab::ShapeError& e) {
        return set_error(OSP_ERR_SHAPE, e.what());
    } catch (const pslab::LayerError& e) {
        return set_error(OSP_ERR_LAYER, e.what());
    } catch (const pslab::ParseError& e) {
        return set_error(OSP_ERR_PARSE, e.what());
    } catch (const pslab::ConfigError& e) {
        return set_error(OSP_ERR_CONFIG, e.what());
    } catch (const pslab::FormatError& e) {
        return set_error(OSP_ERR_FORMAT, e.what());
    } catch (const pslab::ProtocolError& e) {
        return set_error(OSP_ERR_PROTOCOL, e.what());
    } catch (const pslab::NumericError& e) {
        return set_error(OSP_ERR_NUMERIC, e.what());
    } catch (const pslab::DeviceError& e) {
        return set_error(OSP_ERR_CUDA, e.what());
    } catch (const std::exception& e) {
        return set_error(OSP_ERR_INVALID, e.what());
    }
}

osp_status null_arg() { return set_error(OSP_ERR_INVALID, "null argument"); }

}  // namespace

struct osp_engine_partition {
    pslab::PartitionPtr part;
};

struct osp_msg {
    pslab::Message m;
};

struct osp_worker {
    pslab::PartitionPtr part;
    pslab::OspWorker w;
};

struct osp_server {
    pslab::PartitionPtr part;
    pslab::OspServer s;
};

namespace {

std::vector<float> host_vector(const pslab::PartitionPtr& part, const float* v) {
    std::vector<float> out(part->total_count(), 0.0f);
    if (v) std::memcpy(out.data(), v, out.size() * sizeof(float));
    return out;
}

osp_msg* wrap(pslab::Message&& m) { return new osp_msg{std::move(m)}; }

template <typename Out>
void emit(Out& o, osp_msg** pull, osp_msg** ics, osp_msg** gib) {
    if (pull) *pull = o.pull_important ? wrap(std::move(*o.pull_important)) : nullptr;
    if (ics) *ics = o.ics_broadcast ? wrap(std::move(*o.ics_broadcast)) : nullptr;
    if (gib) *gib = o.gib_update ? wrap(std::move(*o.gib_update)) : nullptr;
}

}  // namespace

extern "C" {

const char* osp_engine_last_error(void) { return g_last_error.c_str(); }

osp_status osp_engine_partition_create(const uint64_t* layer_counts, uint64_t n_layers,
                                       uint32_t bytes_per_element, osp_engine_partition** out) {
    if (!out || (!layer_counts && n_layers)) return null_arg();
    *out = nullptr;
    return guarded([&] {
        std::vector<size_t> counts(layer_counts, layer_counts + n_layers);
        *out = new osp_engine_partition{pslab::make_partition(counts, bytes_per_element)};
    });
}

void osp_engine_partition_destroy(osp_engine_partition* p) { delete p; }

uint64_t osp_engine_partition_total_count(const osp_engine_partition* p) {
    return p ? p->part->total_count() : 0;
}

// ---- messages -------------------------------------------------------------------

int osp_msg_kind(const osp_msg* m) { return m ? static_cast<int>(m->m.kind) : -1; }
uint32_t osp_msg_iteration(const osp_msg* m) { return m ? m->m.iteration : 0; }
int osp_msg_from(const osp_msg* m) { return m ? m->m.from_worker : -1; }
double osp_msg_scalar(const osp_msg* m) { return m ? m->m.scalar : 0.0; }
int osp_msg_layer_count(const osp_msg* m) {
    return m ? static_cast<int>(m->m.payload.size()) : 0;
}

uint64_t osp_msg_size_bytes(const osp_msg* m, const osp_engine_partition* part) {
    if (!m || !part) return 0;
    uint64_t n = 0;
    if (guarded([&] { n = pslab::message_size_bytes(m->m, *part->part); }) != OSP_OK) return 0;
    return n;
}

osp_status osp_msg_encode(const osp_msg* m, uint8_t* out, uint64_t cap, uint64_t* len) {
    if (!m || !len) return null_arg();
    std::vector<uint8_t> buf;
    osp_status st = guarded([&] { buf = pslab::encode_payload_message(m->m); });
    if (st != OSP_OK) return st;
    *len = buf.size();
    if (!out) return OSP_OK;
    if (cap < buf.size()) return set_error(OSP_ERR_INVALID, "output buffer too small");
    std::memcpy(out, buf.data(), buf.size());
    return OSP_OK;
}

osp_status osp_msg_decode(const uint8_t* buf, uint64_t len, int from_worker, osp_msg** out) {
    if (!out || (!buf && len)) return null_arg();
    *out = nullptr;
    return guarded([&] {
        pslab::Message m = pslab::decode_payload_message(std::span<const uint8_t>(buf, len));
        m.from_worker = from_worker;
        *out = wrap(std::move(m));
    });
}

osp_status osp_msg_gib(const osp_msg* m, uint8_t* out, uint64_t cap, uint64_t* len) {
    if (!m || !len) return null_arg();
    if (!m->m.gib) return set_error(OSP_ERR_PROTOCOL, "message carries no GIB");
    std::vector<uint8_t> buf;
    osp_status st = guarded(
        [&] { buf = pslab::gib_encode(*m->m.gib, m->m.gib->ics_set.layer_count()); });
    if (st != OSP_OK) return st;
    *len = buf.size();
    if (!out) return OSP_OK;
    if (cap < buf.size()) return set_error(OSP_ERR_INVALID, "output buffer too small");
    std::memcpy(out, buf.data(), buf.size());
    return OSP_OK;
}

osp_status osp_msg_rank_order(const osp_msg* m, int32_t* out, uint64_t cap, uint64_t* n) {
    if (!m || !n) return null_arg();
    const auto& order = m->m.ics_rank_order;
    *n = order.size();
    if (!out) return OSP_OK;
    if (cap < order.size()) return set_error(OSP_ERR_INVALID, "output buffer too small");
    for (size_t i = 0; i < order.size(); ++i) out[i] = order[i];
    return OSP_OK;
}

void osp_msg_destroy(osp_msg* m) { delete m; }

// ---- worker ------------------------------------------------------------------------

osp_status osp_worker_create(const osp_engine_partition* part, int worker_id,
                             const float* init_params, double subset_weight, osp_worker** out) {
    if (!part || !out) return null_arg();
    *out = nullptr;
    return guarded([&] {
        pslab::ParamVector init{part->part, host_vector(part->part, init_params)};
        *out = new osp_worker{part->part, pslab::OspWorker(worker_id, std::move(init), subset_weight)};
    });
}

void osp_worker_destroy(osp_worker* w) { delete w; }

osp_status osp_worker_compute_done(osp_worker* w, uint64_t iteration, const float* delta,
                                   double loss, int n_chunks, osp_msg** rs_push,
                                   osp_msg** loss_report, osp_msg** ics_chunks, int max_chunks,
                                   int* n_ics_chunks) {
    if (!w || !delta || !rs_push || !loss_report || !n_ics_chunks) return null_arg();
    *rs_push = *loss_report = nullptr;
    *n_ics_chunks = 0;
    return guarded([&] {
        pslab::GradVector d{w->part, host_vector(w->part, delta)};
        auto o = w->w.on_compute_done(iteration, d, loss, n_chunks);
        if (static_cast<int>(o.ics_chunks.size()) > max_chunks || (!ics_chunks && !o.ics_chunks.empty()))
            throw pslab::Error("more ICS chunks than the output array holds");
        *rs_push = wrap(std::move(o.rs_push));
        *loss_report = wrap(std::move(o.loss_report));
        for (size_t j = 0; j < o.ics_chunks.size(); ++j) ics_chunks[j] = wrap(std::move(o.ics_chunks[j]));
        *n_ics_chunks = static_cast<int>(o.ics_chunks.size());
    });
}

osp_status osp_worker_on_pull_important(osp_worker* w, const osp_msg* pull, int* applied) {
    if (!w || !pull) return null_arg();
    return guarded([&] {
        const bool a = w->w.on_pull_important(pull->m);
        if (applied) *applied = a ? 1 : 0;
    });
}

osp_status osp_worker_on_ics_global_chunk(osp_worker* w, const osp_msg* chunk) {
    if (!w || !chunk) return null_arg();
    return guarded([&] { w->w.on_ics_global_chunk(chunk->m); });
}

int osp_worker_stashed_pull_ready(const osp_worker* w) {
    return w && w->w.stashed_pull_ready() ? 1 : 0;
}

osp_status osp_worker_apply_stashed_pull(osp_worker* w) {
    if (!w) return null_arg();
    return guarded([&] { w->w.apply_stashed_pull(); });
}

osp_status osp_worker_on_gib_update(osp_worker* w, const osp_msg* gib_update) {
    if (!w || !gib_update) return null_arg();
    return guarded([&] { w->w.on_gib_update(gib_update->m); });
}

uint64_t osp_worker_iteration(const osp_worker* w) { return w ? w->w.iteration() : 0; }
int osp_worker_pending_empty(const osp_worker* w) { return w && w->w.pending_empty() ? 1 : 0; }

osp_status osp_worker_params(const osp_worker* w, float* out) {
    if (!w || !out) return null_arg();
    return guarded([&] {
        const auto& v = w->w.params().values;
        std::memcpy(out, v.data(), v.size() * sizeof(float));
    });
}

// ---- server ------------------------------------------------------------------------

osp_status osp_server_create(const osp_engine_partition* part, const float* init_global,
                             const osp_server_config* cfg, osp_server** out) {
    if (!part || !cfg || !out || (!cfg->weights && cfg->n_workers > 0)) return null_arg();
    *out = nullptr;
    return guarded([&] {
        pslab::ParamVector init{part->part, host_vector(part->part, init_global)};
        std::vector<double> weights(cfg->weights, cfg->weights + cfg->n_workers);
        pslab::SguSchedule sched;
        sched.u_max = cfg->u_max;
        pslab::OspServerOptions opts;
        opts.iterations_per_epoch = cfg->iterations_per_epoch;
        if (cfg->has_fixed_budget) opts.fixed_budget_bytes = cfg->fixed_budget_bytes;
        *out = new osp_server{part->part,
                              pslab::OspServer(std::move(init), std::move(weights), sched, opts)};
    });
}

void osp_server_destroy(osp_server* s) { delete s; }

osp_status osp_server_on_push_important(osp_server* s, const osp_msg* msg, osp_msg** pull_important,
                                        osp_msg** ics_broadcast, osp_msg** gib_update) {
    if (!s || !msg) return null_arg();
    return guarded([&] {
        auto o = s->s.on_push_important(msg->m);
        emit(o, pull_important, ics_broadcast, gib_update);
    });
}

osp_status osp_server_on_push_ics_chunk(osp_server* s, const osp_msg* msg, osp_msg** pull_important,
                                        osp_msg** ics_broadcast, osp_msg** gib_update) {
    if (!s || !msg) return null_arg();
    return guarded([&] {
        auto o = s->s.on_push_ics_chunk(msg->m);
        emit(o, pull_important, ics_broadcast, gib_update);
    });
}

osp_status osp_server_on_loss_report(osp_server* s, const osp_msg* msg) {
    if (!s || !msg) return null_arg();
    return guarded([&] { s->s.on_loss_report(msg->m); });
}

osp_status osp_server_set_umax(osp_server* s, uint64_t u_max) {
    if (!s) return null_arg();
    s->s.set_umax(u_max);
    return OSP_OK;
}

osp_status osp_server_global_params(const osp_server* s, float* out) {
    if (!s || !out) return null_arg();
    return guarded([&] {
        const auto& v = s->s.global_params().values;
        std::memcpy(out, v.data(), v.size() * sizeof(float));
    });
}

uint64_t osp_server_resolved_count(const osp_server* s) { return s ? s->s.resolved_count() : 0; }
uint64_t osp_server_dropped_stale(const osp_server* s) { return s ? s->s.dropped_stale() : 0; }
uint64_t osp_server_budget_for_epoch(const osp_server* s, uint64_t epoch) {
    return s ? s->s.budget_for_epoch(epoch) : 0;
}
uint64_t osp_server_epoch_of_iteration(const osp_server* s, uint64_t iteration) {
    return s ? s->s.epoch_of_iteration(iteration) : 0;
}

}  // extern "C"
