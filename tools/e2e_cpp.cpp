// e2e_cpp.cpp — end-to-end time of the C++ drop-in (include/modmetrics/gpu.hpp)
// as a user of the reference calls it: from the reference's own SystemModel +
// DependencyTable (built by its generate(), generate.hpp:94) to the ordered
// std::vector<MoveSuggestion>, every host <-> device copy included.
//
//   free functions (the reference's signatures, each call uploads the model as
//   the reference takes it by const& each time):
//     cm = gpu::parallel_class_metrics(model, deps, n)    (parallel.hpp:149)
//     t  = gpu::compute_thresholds(report)                (suggest.hpp:46)
//     s  = gpu::suggest_all(model, deps, report, t, {Cohesion, Coupling}, Union)
//   engine (one upload, the same calls on a resident gpu::Engine):
//     e.upload(model, deps); e.parallel_class_metrics(); e.compute_thresholds(); e.suggest_all(...)
//
// Prints one JSON line: per-step milliseconds (median over the timed steps,
// wall clock around complete calls — the results are host vectors), the
// candidate count and the list length. Built by tools/Makefile where the
// reference headers exist; the binary travels to the GPU box (tools/_build).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <modmetrics/generate.hpp>
#include <modmetrics/metrics.hpp>
#include <modmetrics/parallel.hpp>
#include <modmetrics/suggest.hpp>

#include "modmetrics/gpu.hpp"

using namespace modmetrics;
using Clock = std::chrono::steady_clock;

static double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v.empty() ? 0.0 : v[v.size() / 2];
}

int main(int argc, char** argv) {
    int steps = 10, warmup = 3;
    for (int i = 1; i + 1 < argc; ++i) {
        if (!std::strcmp(argv[i], "--steps")) steps = std::atoi(argv[++i]);
        else if (!std::strcmp(argv[i], "--warmup")) warmup = std::atoi(argv[++i]);
    }
    GeneratorConfig cfg;  // C4 (BASELINE.json configs[3], SURVEY.md §8d seeds)
    cfg.seed = 1;
    cfg.n_classes = 100000;
    cfg.n_methods = 1000000;
    cfg.n_attributes = 2000000;
    cfg.k_max_calls = 4;
    cfg.k_max_accesses = 4;
    cfg.intra_class_bias = 0.5;
    const GeneratedSystem gs = generate(cfg);
    const SystemModel& model = gs.model;
    const DependencyTable& deps = gs.deps;
    const std::vector<Criterion> crit = {Criterion::Cohesion, Criterion::Coupling};

    size_t n_sugg = 0;
    std::vector<double> t_free, t_eng;
    // (1) free functions
    for (int s = 0; s < warmup + steps; ++s) {
        const auto t0 = Clock::now();
        const ClassMetrics cm = gpu::parallel_class_metrics(model, deps, 1);
        MetricsReport report;
        report.lcom = cm.lcom;
        report.cbo = cm.cbo;
        const Thresholds t = gpu::compute_thresholds(report);
        const std::vector<MoveSuggestion> out = gpu::suggest_all(model, deps, report, t, crit, Combine::Union);
        const auto t1 = Clock::now();
        n_sugg = out.size();
        if (s >= warmup) t_free.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    // (2) one resident engine
    gpu::Engine e;
    for (int s = 0; s < warmup + steps; ++s) {
        const auto t0 = Clock::now();
        e.upload(model, deps);
        const ClassMetrics cm = e.parallel_class_metrics();
        MetricsReport report;
        report.lcom = cm.lcom;
        report.cbo = cm.cbo;
        const Thresholds t = e.compute_thresholds(report);
        const std::vector<MoveSuggestion> out = e.suggest_all(report, t, crit, Combine::Union);
        const auto t1 = Clock::now();
        if (out.size() != n_sugg) {
            std::printf("{\"error\": \"engine list length %zu != %zu\"}\n", out.size(), n_sugg);
            return 1;
        }
        if (s >= warmup) t_eng.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    }
    uint64_t cand = 0;
    for (MethodId p = 0; p < model.method_count(); ++p)
        cand += detail::used_classes(p, model.method_owner[p], model, deps).size();
    std::printf("{\"config\": \"c4\", \"steps\": %d, \"candidates\": %llu, \"suggestions\": %zu, "
                "\"free_functions_ms\": %.4f, \"engine_ms\": %.4f}\n",
                steps, (unsigned long long)cand, n_sugg, median(t_free), median(t_eng));
    return 0;
}
