// pslab façade: budget tuning (reference tuning.cpp:8-48, via the C-ABI), the
// message kinds / simulated sizes / payload codec (message.cpp:7-99) and the
// SGD step that feeds the sync path (learner.cpp:391-398, device kernel).
#include <cstring>
#include <string>

#include "device.hpp"
#include "pslab/message.hpp"
#include "pslab/tuning.hpp"

namespace pslab {

using pslab_b200::check;
using pslab_b200::DevBuf;

uint64_t compute_umax(const NetworkParams& net, double t_c_seconds, int n_workers,
                      uint64_t model_bytes, bool eq5_literal) {
    uint64_t out = 0;
    check(osp_compute_umax(net.bandwidth_bps, net.latency_s, net.loss_rate, t_c_seconds, n_workers,
                           model_bytes, eq5_literal ? 1 : 0, &out));
    return out;
}

uint64_t tune_sgu(SguSchedule& sched, uint64_t epoch_index, double epoch_loss) {
    osp_sgu_schedule s{};
    s.u_max = sched.u_max;
    s.has_initial_loss = sched.initial_loss.has_value() ? 1 : 0;
    s.initial_loss = sched.initial_loss.value_or(0.0);
    s.current_budget = sched.current_budget;
    s.epoch = sched.epoch;
    uint64_t budget = 0;
    check(osp_tune_sgu(&s, epoch_index, epoch_loss, &budget));
    sched.epoch = s.epoch;
    sched.current_budget = s.current_budget;
    if (s.has_initial_loss) sched.initial_loss = s.initial_loss;
    return budget;
}

const char* msg_kind_name(MsgKind k) {
    static const char* const names[] = {"PushImportant", "PushIcsChunk", "PullImportant",
                                        "IcsGlobalChunk", "GibUpdate",   "LossReport",
                                        "PushFull",      "PullFull"};
    const auto i = static_cast<unsigned>(k);
    return i < 8 ? names[i] : "?";
}

uint64_t message_size_bytes(const Message& msg, const LayerPartition& part) {
    if (msg.kind == MsgKind::GibUpdate) return gib_encoded_size(part.layer_count());
    if (msg.kind == MsgKind::LossReport) return 8;
    return payload_value_bytes(msg.payload, part);
}

namespace {

template <typename T>
void put_le(std::vector<uint8_t>& out, T v) {
    for (size_t i = 0; i < sizeof(T); ++i) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
}

uint32_t read_u32(std::span<const uint8_t> b, size_t at) {
    uint32_t v = 0;
    for (int i = 3; i >= 0; --i) v = (v << 8) | b[at + i];
    return v;
}

}  // namespace

std::vector<uint8_t> encode_payload_message(const Message& msg) {
    if (msg.payload.size() > 0xffff) throw FormatError("payload has too many layers for the wire format");
    std::vector<uint8_t> out;
    out.push_back(static_cast<uint8_t>(msg.kind));
    put_le<uint32_t>(out, msg.iteration);
    put_le<uint16_t>(out, static_cast<uint16_t>(msg.payload.size()));
    for (const auto& [id, vals] : msg.payload) {
        put_le<uint32_t>(out, static_cast<uint32_t>(id));
        put_le<uint32_t>(out, static_cast<uint32_t>(vals.size()));
        for (float f : vals) {
            uint32_t bits;
            std::memcpy(&bits, &f, 4);
            put_le<uint32_t>(out, bits);
        }
    }
    return out;
}

Message decode_payload_message(std::span<const uint8_t> buf) {
    if (buf.size() < 7) throw FormatError("message header truncated");
    Message m;
    m.kind = static_cast<MsgKind>(buf[0]);
    m.iteration = read_u32(buf, 1);
    const unsigned entries = buf[5] | (buf[6] << 8);
    size_t at = 7;
    for (unsigned e = 0; e < entries; ++e) {
        if (buf.size() < at + 8) throw FormatError("layer entry header truncated");
        const uint32_t id = read_u32(buf, at), count = read_u32(buf, at + 4);
        at += 8;
        if (buf.size() < at + static_cast<size_t>(count) * 4) throw FormatError("layer values truncated");
        std::vector<float> vals(count);
        for (uint32_t i = 0; i < count; ++i, at += 4) {
            const uint32_t bits = read_u32(buf, at);
            std::memcpy(&vals[i], &bits, 4);
        }
        m.payload.emplace(static_cast<int>(id), std::move(vals));
    }
    if (at != buf.size()) throw FormatError("trailing bytes after message payload");
    return m;
}

// learner.hpp:77 (the reference header is not part of this façade)
GradVector sgd_delta(const GradVector& grad, double learning_rate);

GradVector sgd_delta(const GradVector& grad, double learning_rate) {
    if (learning_rate <= 0) throw ConfigError("learning rate must be positive");
    GradVector out;
    out.part = grad.part;
    out.values.resize(grad.values.size());
    const size_t n = grad.values.size();
    if (n == 0) return out;
    DevBuf dg(n), dd(n);
    dg.upload(grad.values);
    check(osp_sgd_delta(dg.data(), n, learning_rate, dd.data(), nullptr));
    dd.download(out.values.data(), n);
    return out;
}

}  // namespace pslab
