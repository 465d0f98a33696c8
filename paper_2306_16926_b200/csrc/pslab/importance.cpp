// pslab façade: PGP / rank / GIB (reference importance.cpp:11-117 semantics)
// over the device kernels (osp_pgp_layer_importance, osp_rank_and_gib) and the
// C-ABI GIB codec.
#include "pslab/importance.hpp"

#include <map>
#include <mutex>
#include <string>

#include "device.hpp"

namespace pslab {

using pslab_b200::check;
using pslab_b200::DevBuf;

LayerImportance pgp_layer_importance(const ParamVector& params, const GradVector& grads) {
    check_same_shape(params, grads);
    if (params.part->layer_count() != grads.part->layer_count())
        throw ShapeError("param/grad partitions disagree on layer count");
    LayerImportance imp;
    imp.scores.assign(params.part->layer_count(), 0.0);
    const size_t n = params.values.size();
    DevBuf dp(n), dg(n);
    dp.upload(params.values);
    dg.upload(grads.values);
    check(osp_pgp_layer_importance(params.part->device(), dp.data(), dg.data(), imp.scores.data(),
                                   nullptr));
    return imp;
}

namespace {

// rank_layers has no partition argument: rank on a unit-count table of the
// same length (cached per layer count).
const osp_partition* unit_partition(size_t layers) {
    static std::mutex mu;
    static std::map<size_t, PartitionPtr> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(layers);
    if (it == cache.end())
        it = cache.emplace(layers, make_partition(std::vector<size_t>(layers, 1))).first;
    return it->second->device();
}

}  // namespace

std::vector<int> rank_layers(const LayerImportance& imp) {
    std::vector<int> order(imp.scores.size());
    if (order.empty()) return order;
    check(osp_rank_and_gib(unit_partition(imp.scores.size()), imp.scores.data(), 0, order.data(),
                           nullptr, nullptr));
    return order;
}

Gib build_gib(const LayerImportance& imp, const LayerPartition& part, uint64_t budget_bytes,
              uint32_t iteration_tag) {
    if (imp.scores.size() != part.layer_count())
        throw ShapeError("importance covers " + std::to_string(imp.scores.size()) +
                         " layers, partition has " + std::to_string(part.layer_count()));
    std::vector<uint8_t> flags(part.layer_count());
    check(osp_rank_and_gib(part.device(), imp.scores.data(), budget_bytes, nullptr, flags.data(),
                           nullptr));
    Gib g;
    g.iteration_tag = iteration_tag;
    g.ics_set = LayerSet::none(part.layer_count());
    for (size_t l = 0; l < flags.size(); ++l)
        if (flags[l]) g.ics_set.set(static_cast<int>(l));
    return g;
}

uint64_t gib_encoded_size(size_t layer_count) { return osp_gib_encoded_size(layer_count); }

std::vector<uint8_t> gib_encode(const Gib& g, size_t layer_count) {
    if (g.ics_set.layer_count() != layer_count)
        throw ShapeError("gib bitmap covers " + std::to_string(g.ics_set.layer_count()) +
                         " layers, expected " + std::to_string(layer_count));
    std::vector<uint8_t> flags(layer_count);
    for (size_t k = 0; k < layer_count; ++k) flags[k] = g.ics_set.test(static_cast<int>(k)) ? 1 : 0;
    std::vector<uint8_t> out(gib_encoded_size(layer_count));
    check(osp_gib_encode(g.iteration_tag, layer_count, flags.data(), out.data(), out.size()));
    return out;
}

Gib gib_decode(std::span<const uint8_t> buf) {
    uint32_t tag = 0, layers = 0;
    check(osp_gib_decode(buf.data(), buf.size(), &tag, &layers, nullptr, 0));
    std::vector<uint8_t> flags(layers);
    check(osp_gib_decode(buf.data(), buf.size(), &tag, &layers, flags.data(), flags.size()));
    Gib g;
    g.iteration_tag = tag;
    g.ics_set = LayerSet::none(layers);
    for (uint32_t k = 0; k < layers; ++k)
        if (flags[k]) g.ics_set.set(static_cast<int>(k));
    return g;
}

}  // namespace pslab
