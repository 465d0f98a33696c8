// Oracle driver: runs the UNMODIFIED reference pslab OSP engines (OspWorker /
// OspServer from /root/reference/proj/src/protocol.cpp) in the synchronous
// "fresh GIB" order that the B200 step reproduces, and either
//   golden  - dumps every per-iteration artefact as raw little-endian files
//             (used to pin oracle/osp_oracle.c and to build tests/golden/), or
//   bench   - times the engine step on the host (bench.py cpu_baseline /
//             --impl reference).
//
// Test infrastructure only (see oracle/README.md). Built by `make -C oracle ref`
// into oracle/_ref/ against the reference sources; never part of the product.
//
// Message order per iteration mirrors the reference Orchestrator
// (runner.cpp:358-409, 411-448, 519-604) with every flow delivered in worker
// order: loss reports, RS pushes, pull broadcast, ICS chunk j of every worker,
// ICS broadcasts, GIB update (gib_push_negligible = true, runner.cpp:427-433).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "pslab/importance.hpp"
#include "pslab/learner.hpp"
#include "pslab/protocol.hpp"
#include "pslab/rng.hpp"
#include "pslab/tuning.hpp"

using namespace pslab;

namespace {

struct Args {
    std::string mode;
    std::string out_dir = ".";
    std::vector<size_t> layers;
    int workers = 8;
    std::vector<double> weights;  // empty: 1/N
    uint64_t seed = 11;
    int64_t budget = -1;           // bytes; <0 with budget_frac<0: tuned
    double budget_frac = -1.0;     // fraction of model bytes
    int n_chunks = 4;
    int iters = 4;
    int warmup = 1;
    uint32_t bpe = 4;
    std::string p0 = "zeros";      // zeros | random:<seed>
    uint64_t ipe = 1000000;        // iterations per epoch (tuner)
    uint64_t umax = 0;             // u_max for the tuner
    int threads = 1;
    bool dump_deltas = true;
};

std::vector<size_t> parse_sizes(const std::string& s) {
    std::vector<size_t> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
        if (!tok.empty()) out.push_back(std::stoull(tok));
    }
    return out;
}

std::vector<double> parse_doubles(const std::string& s) {
    std::vector<double> out;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
        if (!tok.empty()) out.push_back(std::stod(tok));
    }
    return out;
}

std::vector<size_t> read_layers_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) {
        std::fprintf(stderr, "cannot read %s\n", path.c_str());
        std::exit(2);
    }
    std::vector<size_t> out;
    std::string tok;
    while (in >> tok) {
        for (auto v : parse_sizes(tok)) out.push_back(v);
    }
    return out;
}

Args parse(int argc, char** argv) {
    Args a;
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_driver golden|bench [--key value]...\n");
        std::exit(2);
    }
    a.mode = argv[1];
    for (int i = 2; i + 1 < argc; i += 2) {
        std::string k = argv[i], v = argv[i + 1];
        if (k == "--out") a.out_dir = v;
        else if (k == "--layers") a.layers = parse_sizes(v);
        else if (k == "--layers-file") a.layers = read_layers_file(v);
        else if (k == "--workers") a.workers = std::stoi(v);
        else if (k == "--weights") a.weights = parse_doubles(v);
        else if (k == "--seed") a.seed = std::stoull(v);
        else if (k == "--budget") a.budget = std::stoll(v);
        else if (k == "--budget-frac") a.budget_frac = std::stod(v);
        else if (k == "--chunks") a.n_chunks = std::stoi(v);
        else if (k == "--iters") a.iters = std::stoi(v);
        else if (k == "--warmup") a.warmup = std::stoi(v);
        else if (k == "--bpe") a.bpe = static_cast<uint32_t>(std::stoul(v));
        else if (k == "--p0") a.p0 = v;
        else if (k == "--ipe") a.ipe = std::stoull(v);
        else if (k == "--umax") a.umax = std::stoull(v);
        else if (k == "--threads") a.threads = std::stoi(v);
        else if (k == "--dump-deltas") a.dump_deltas = std::stoi(v) != 0;
        else {
            std::fprintf(stderr, "unknown flag %s\n", k.c_str());
            std::exit(2);
        }
    }
    if (a.layers.empty()) {
        std::fprintf(stderr, "need --layers or --layers-file\n");
        std::exit(2);
    }
    return a;
}

// Synthetic delta exactly as runner.cpp:312-321.
void synth_delta(GradVector& g, uint64_t seed, int worker, uint64_t iteration) {
    Rng rng(derive_seed(seed, seed_purpose::kSynthGrad, static_cast<uint64_t>(worker), iteration));
    for (float& v : g.values) v = static_cast<float>(rng.uniform(-1e-3, 1e-3));
}

template <typename T>
void write_raw(const std::string& path, const T* data, size_t n) {
    std::FILE* f = std::fopen(path.c_str(), "wb");
    if (!f) {
        std::fprintf(stderr, "cannot write %s\n", path.c_str());
        std::exit(3);
    }
    if (n) std::fwrite(data, sizeof(T), n, f);
    std::fclose(f);
}

std::vector<int32_t> flatten_chunks(const std::vector<Message>& chunks) {
    // [n_chunks, (count, ids...)...]
    std::vector<int32_t> out;
    out.push_back(static_cast<int32_t>(chunks.size()));
    for (const auto& c : chunks) {
        out.push_back(static_cast<int32_t>(c.payload.size()));
        for (const auto& [id, vals] : c.payload) {
            (void)vals;
            out.push_back(id);
        }
    }
    return out;
}

struct Engine {
    PartitionPtr part;
    std::vector<double> weights;
    std::unique_ptr<OspServer> server;
    std::vector<std::unique_ptr<OspWorker>> workers;
    std::vector<GradVector> deltas;
    int n_chunks;
    int threads;

    Engine(const Args& a) : n_chunks(a.n_chunks), threads(std::max(1, a.threads)) {
        part = make_partition(a.layers, a.bpe);
        int n = a.workers;
        weights = a.weights.empty() ? std::vector<double>(n, 1.0 / n) : a.weights;
        ParamVector init = zeros_params(part);
        if (a.p0.rfind("random:", 0) == 0) {
            Rng rng(std::stoull(a.p0.substr(7)));
            for (float& v : init.values) v = static_cast<float>(rng.uniform(-1.0, 1.0));
        }
        SguSchedule sched;
        sched.u_max = a.umax;
        OspServerOptions opts;
        opts.iterations_per_epoch = a.ipe;
        if (a.budget >= 0) opts.fixed_budget_bytes = static_cast<uint64_t>(a.budget);
        else if (a.budget_frac >= 0)
            opts.fixed_budget_bytes =
                static_cast<uint64_t>(std::floor(a.budget_frac * static_cast<double>(part->total_bytes())));
        server = std::make_unique<OspServer>(init, weights, sched, opts);
        for (int w = 0; w < n; ++w) workers.push_back(std::make_unique<OspWorker>(w, init, weights[w]));
        deltas.assign(static_cast<size_t>(n), zeros_grads(part));
    }

    template <typename F>
    void for_workers(F f) {
        int n = static_cast<int>(workers.size());
        if (threads <= 1) {
            for (int w = 0; w < n; ++w) f(w);
            return;
        }
        std::vector<std::thread> pool;
        int t = std::min(threads, n);
        for (int k = 0; k < t; ++k) {
            pool.emplace_back([&, k] {
                for (int w = k; w < n; w += t) f(w);
            });
        }
        for (auto& th : pool) th.join();
    }

    // One synchronous OSP iteration. Observers are optional.
    struct Trace {
        std::vector<Message> chunks_w0;
        LayerPayload pull_payload;
        std::vector<std::vector<float>> params_stage1;
        std::optional<Message> gib_update;
    };

    void step(uint64_t it, double loss, Trace* tr) {
        int n = static_cast<int>(workers.size());
        std::vector<OspWorker::ComputeOutput> outs(static_cast<size_t>(n));
        for_workers([&](int w) {
            outs[w] = workers[w]->on_compute_done(it, deltas[w], loss, n_chunks);
        });
        for (int w = 0; w < n; ++w) server->on_loss_report(outs[w].loss_report);
        std::optional<Message> pull, gib;
        for (int w = 0; w < n; ++w) {
            auto o = server->on_push_important(outs[w].rs_push);
            if (o.pull_important) pull = std::move(o.pull_important);
            if (o.gib_update) gib = std::move(o.gib_update);
            if (o.ics_broadcast) {
                std::fprintf(stderr, "unexpected ics broadcast at barrier\n");
                std::exit(4);
            }
        }
        if (!pull) {
            std::fprintf(stderr, "barrier did not close at iteration %llu\n",
                         static_cast<unsigned long long>(it));
            std::exit(4);
        }
        for_workers([&](int w) {
            if (!workers[w]->on_pull_important(*pull)) {
                std::fprintf(stderr, "pull stashed unexpectedly\n");
                std::exit(4);
            }
        });
        if (tr) {
            tr->pull_payload = pull->payload;
            tr->chunks_w0 = outs[0].ics_chunks;
            for (int w = 0; w < n; ++w) tr->params_stage1.push_back(workers[w]->params().values);
        }
        size_t nc = outs[0].ics_chunks.size();
        for (size_t j = 0; j < nc; ++j) {
            for (int w = 0; w < n; ++w) {
                auto o = server->on_push_ics_chunk(outs[w].ics_chunks[j]);
                if (o.ics_broadcast) {
                    const Message& bc = *o.ics_broadcast;
                    for_workers([&](int w2) { workers[w2]->on_ics_global_chunk(bc); });
                }
                if (o.gib_update) gib = std::move(o.gib_update);
                if (o.pull_important) {
                    std::fprintf(stderr, "unexpected pull during ics\n");
                    std::exit(4);
                }
            }
        }
        if (!gib || server->resolved_count() != it + 1) {
            std::fprintf(stderr, "iteration %llu did not resolve\n",
                         static_cast<unsigned long long>(it));
            std::exit(4);
        }
        for_workers([&](int w) { workers[w]->on_gib_update(*gib); });
        if (tr) tr->gib_update = gib;
    }
};

int run_golden(const Args& a) {
    Engine e(a);
    const std::string& d = a.out_dir;
    size_t L = e.part->layer_count();
    size_t M = e.part->total_count();
    int n = a.workers;
    {
        std::vector<uint64_t> counts(a.layers.begin(), a.layers.end());
        write_raw(d + "/layers.bin", counts.data(), counts.size());
        write_raw(d + "/weights.bin", e.weights.data(), e.weights.size());
        write_raw(d + "/p0.bin", e.server->global_params().values.data(), M);
    }
    for (int it = 0; it < a.iters; ++it) {
        char pre[64];
        std::snprintf(pre, sizeof pre, "/it%03d_", it);
        std::string p = d + pre;
        for (int w = 0; w < n; ++w) synth_delta(e.deltas[w], a.seed, w, static_cast<uint64_t>(it));
        if (a.dump_deltas) {
            std::vector<float> all;
            for (int w = 0; w < n; ++w)
                all.insert(all.end(), e.deltas[w].values.begin(), e.deltas[w].values.end());
            write_raw(p + "deltas.bin", all.data(), all.size());
        }
        const WorkerState& ws0 = e.workers[0]->state();
        auto gib_in = gib_encode(ws0.current_gib, L);
        write_raw(p + "gib_in.bin", gib_in.data(), gib_in.size());
        write_raw(p + "order_in.bin", ws0.current_ics_order.data(), ws0.current_ics_order.size());

        double loss = std::pow(0.7, static_cast<double>(e.server->epoch_of_iteration(it) - 1));
        Engine::Trace tr;
        e.step(static_cast<uint64_t>(it), loss, &tr);

        auto chunks = flatten_chunks(tr.chunks_w0);
        write_raw(p + "chunks.bin", chunks.data(), chunks.size());
        std::vector<int32_t> rs_ids;
        for (const auto& [id, vals] : tr.pull_payload) {
            (void)vals;
            rs_ids.push_back(id);
        }
        write_raw(p + "rs_ids.bin", rs_ids.data(), rs_ids.size());
        std::vector<float> st1;
        for (auto& v : tr.params_stage1) st1.insert(st1.end(), v.begin(), v.end());
        write_raw(p + "params_stage1.bin", st1.data(), st1.size());
        std::vector<float> fin;
        for (int w = 0; w < n; ++w) {
            const auto& v = e.workers[w]->params().values;
            fin.insert(fin.end(), v.begin(), v.end());
        }
        write_raw(p + "params_final.bin", fin.data(), fin.size());
        const ParamVector& g = e.server->global_params();
        write_raw(p + "global.bin", g.values.data(), M);
        auto delta = e.server->take_resolved_delta(static_cast<uint64_t>(it));
        GradVector agg = zeros_grads(e.part);
        merge_payload(agg, *delta);
        write_raw(p + "agg.bin", agg.values.data(), M);
        LayerImportance imp = pgp_layer_importance(g, agg);
        write_raw(p + "scores.bin", imp.scores.data(), L);
        auto gib_out = gib_encode(*tr.gib_update->gib, L);
        write_raw(p + "gib_out.bin", gib_out.data(), gib_out.size());
        write_raw(p + "order_out.bin", tr.gib_update->ics_rank_order.data(),
                  tr.gib_update->ics_rank_order.size());
        uint64_t budget = e.server->budget_for_epoch(e.server->epoch_of_iteration(it + 1));
        write_raw(p + "budget.bin", &budget, 1);
    }
    std::printf("{\"ok\": true, \"layers\": %zu, \"params\": %zu, \"iters\": %d}\n", L, M, a.iters);
    return 0;
}

int run_bench(const Args& a) {
    using clk = std::chrono::steady_clock;
    Engine e(a);
    size_t M = e.part->total_count();
    int n = a.workers;
    std::vector<double> ms;
    double gen_ms = 0.0;
    int total = a.warmup + a.iters;
    for (int it = 0; it < total; ++it) {
        auto g0 = clk::now();
        e.for_workers([&](int w) { synth_delta(e.deltas[w], a.seed, w, static_cast<uint64_t>(it)); });
        auto t0 = clk::now();
        gen_ms += std::chrono::duration<double, std::milli>(t0 - g0).count();
        double loss = std::pow(0.7, static_cast<double>(e.server->epoch_of_iteration(it) - 1));
        e.step(static_cast<uint64_t>(it), loss, nullptr);
        e.server->take_resolved_delta(static_cast<uint64_t>(it));
        auto t1 = clk::now();
        if (it >= a.warmup) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    std::vector<double> sorted = ms;
    std::sort(sorted.begin(), sorted.end());
    double med = sorted[sorted.size() / 2];
    double sum = 0;
    for (double v : ms) sum += v;
    std::printf(
        "{\"impl\": \"reference-engine\", \"params\": %zu, \"layers\": %zu, \"workers\": %d, "
        "\"threads\": %d, \"steps\": %zu, \"median_ms\": %.6f, \"mean_ms\": %.6f, "
        "\"total_ms\": %.6f, \"min_ms\": %.6f, \"params_per_s\": %.6e, "
        "\"synth_gen_ms_total\": %.3f}\n",
        M, e.part->layer_count(), n, e.threads, ms.size(), med, sum / ms.size(), sum,
        sorted.front(), static_cast<double>(M) / (med * 1e-3), gen_ms);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    Args a = parse(argc, argv);
    try {
        if (a.mode == "golden") return run_golden(a);
        if (a.mode == "bench") return run_bench(a);
    } catch (const std::exception& ex) {
        std::fprintf(stderr, "reference error: %s\n", ex.what());
        return 5;
    }
    std::fprintf(stderr, "unknown mode %s\n", a.mode.c_str());
    return 2;
}
