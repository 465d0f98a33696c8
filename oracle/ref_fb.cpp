// Oracle driver: the UNMODIFIED reference learner (pslab::forward_backward,
// learner.cpp:299-367) on its own synthetic dataset and parameter init, dumped
// as raw little-endian files for tests/golden/learner/ (tests/golden/
// gen_learner_golden.py). Test infrastructure only; built by `make -C oracle
// ref` into oracle/_ref/ against the reference sources.
//
// Usage: ref_fb <out_dir>   |   ref_fb --bench <widths> <act> <loss> <batch> <workers> <reps>
// For every case: <out>/<name>.meta (text: widths, activation, loss, n, d,
// workers, batch) and <name>.{feat.f32, label.i32, param.f32, batch.i32,
// grad.f32, loss.f64}.

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>
#include <vector>

#include "pslab/learner.hpp"

using namespace pslab;

namespace {

template <typename T>
void dump(const std::string& path, const std::vector<T>& v) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(T)));
}

struct Case {
    const char* name;
    std::vector<int> widths;
    Activation act;
    Loss loss;
    size_t n, classes;
    double sep;
    int workers;
    size_t batch;
    uint64_t seed;
};

void run(const std::string& out, const Case& c) {
    MlpSpec spec;
    spec.widths = c.widths;
    spec.activation = c.act;
    spec.loss = c.loss;
    const size_t d = static_cast<size_t>(c.widths.front());
    Dataset ds = synth_dataset(c.seed, c.n, d, c.classes, c.sep);
    std::vector<float> params, grads;
    std::vector<int> batches;
    std::vector<double> losses;
    for (int w = 0; w < c.workers; ++w) {
        // every worker its own parameters and its own shuffled batch
        ParamVector p = init_params(spec, c.seed * 131 + static_cast<uint64_t>(w));
        if (w % 2 == 1)  // nonzero biases too (init_params zeroes them)
            for (size_t k = 0; k < p.values.size(); ++k) p.values[k] += 1e-2f * static_cast<float>(static_cast<int>(k % 7) - 3);
        std::vector<size_t> perm = shuffle_epoch(c.n, c.seed, 1, static_cast<uint64_t>(w));
        Batch b(perm.begin(), perm.begin() + static_cast<long>(c.batch));
        ForwardBackwardResult r = forward_backward(spec, p, ds, b);
        params.insert(params.end(), p.values.begin(), p.values.end());
        grads.insert(grads.end(), r.grad.values.begin(), r.grad.values.end());
        for (size_t i : b) batches.push_back(static_cast<int>(i));
        losses.push_back(r.loss);
    }
    const std::string base = out + "/" + c.name;
    {
        std::ofstream m(base + ".meta");
        for (size_t l = 0; l < c.widths.size(); ++l) m << (l ? "," : "") << c.widths[l];
        m << "\n" << (c.act == Activation::relu ? "relu" : "tanh") << "\n"
          << (c.loss == Loss::mse ? "mse" : "ce") << "\n"
          << c.n << "\n" << d << "\n" << c.workers << "\n" << c.batch << "\n";
    }
    dump(base + ".feat.f32", ds.features);
    dump(base + ".label.i32", ds.labels);
    dump(base + ".param.f32", params);
    dump(base + ".batch.i32", batches);
    dump(base + ".grad.f32", grads);
    dump(base + ".loss.f64", losses);
}

}  // namespace

// bench mode: the reference learner's cost per training iteration of config
// #1's shape: forward_backward of every worker's batch, one host thread
// (the reference harness runs the workers' learners one after the other).
int bench(int argc, char** argv) {
    // ref_fb --bench <w0,w1,...> <relu|tanh> <ce|mse> <batch> <workers> <reps>
    if (argc < 8) return 2;
    MlpSpec spec;
    for (const char* p = argv[2]; *p;) {
        spec.widths.push_back(std::atoi(p));
        while (*p && *p != ',') ++p;
        if (*p) ++p;
    }
    spec.activation = std::string(argv[3]) == "tanh" ? Activation::tanh : Activation::relu;
    spec.loss = std::string(argv[4]) == "mse" ? Loss::mse : Loss::softmax_cross_entropy;
    const size_t B = std::strtoul(argv[5], nullptr, 10);
    const int N = std::atoi(argv[6]), reps = std::atoi(argv[7]);
    Dataset ds = synth_dataset(7, 1024, static_cast<size_t>(spec.widths.front()),
                               static_cast<size_t>(spec.widths.back()), 6.0);
    std::vector<ParamVector> ps;
    std::vector<Batch> bs;
    for (int w = 0; w < N; ++w) {
        ps.push_back(init_params(spec, 100 + static_cast<uint64_t>(w)));
        std::vector<size_t> perm = shuffle_epoch(ds.n, 7, 1, static_cast<uint64_t>(w));
        bs.emplace_back(perm.begin(), perm.begin() + static_cast<long>(B));
    }
    double sink = 0.0;
    auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r)
        for (int w = 0; w < N; ++w) sink += forward_backward(spec, ps[w], ds, bs[w]).loss;
    auto t1 = std::chrono::steady_clock::now();
    const double us = std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
    std::printf("{\"us_per_iteration\": %.4f, \"workers\": %d, \"batch\": %zu, \"reps\": %d, "
                "\"sink\": %.3f}\n", us, N, B, reps, sink);
    return 0;
}

int main(int argc, char** argv) {
    if (argc >= 2 && std::string(argv[1]) == "--bench") return bench(argc, argv);
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_fb <out_dir> | ref_fb --bench ...\n");
        return 2;
    }
    const std::string out = argv[1];
    const std::vector<Case> cases = {
        // config #1's default MlpSpec (config.hpp:30-41): relu, softmax CE
        {"mlp_relu_ce", {8, 32, 4}, Activation::relu, Loss::softmax_cross_entropy, 1024, 4, 6.0, 4, 32, 7},
        {"mlp_relu_mse", {8, 32, 4}, Activation::relu, Loss::mse, 1024, 4, 6.0, 4, 32, 8},
        {"mlp_tanh_ce", {8, 32, 4}, Activation::tanh, Loss::softmax_cross_entropy, 512, 4, 3.0, 3, 48, 9},
        {"deep_tanh_mse", {16, 64, 64, 4}, Activation::tanh, Loss::mse, 512, 4, 3.0, 2, 64, 10},
        {"deep_relu_ce", {16, 64, 64, 4}, Activation::relu, Loss::softmax_cross_entropy, 512, 4, 3.0, 2, 40, 11},
        {"scalar_out_relu_mse", {8, 16, 1}, Activation::relu, Loss::mse, 256, 3, 2.0, 2, 17, 12},
    };
    for (const Case& c : cases) run(out, c);
    std::printf("wrote %zu cases to %s\n", cases.size(), out.c_str());
    return 0;
}
