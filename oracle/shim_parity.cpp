// shim_parity.cpp — the reference library and the GPU drop-in, side by side.
//
// TEST INFRASTRUCTURE. Built by oracle/Makefile from the UNMODIFIED reference
// headers (/root/reference/proj/include, compiled in place) plus
// include/modmetrics/gpu.hpp, linked against libmmgpu.so. Run on a GPU box by
// tests/test_cpp_shim.py. Every comparison uses the reference's own types
// and their defaulted operator== (bitwise doubles, exact vector order), and
// exception TYPES must match.
#include <atomic>
#include <cstdio>
#include <mutex>
#include <thread>
#include <exception>
#include <functional>
#include <stdexcept>
#include <string>
#include <typeinfo>
#include <vector>

#include <modmetrics/generate.hpp>
#include <modmetrics/metrics.hpp>
#include <modmetrics/parallel.hpp>
#include <modmetrics/suggest.hpp>
#include <modmetrics/gpu.hpp>

using namespace modmetrics;

static std::atomic<int> g_fail{0}, g_checks{0};
static std::mutex g_print;

static void expect(bool ok, const std::string& what) {
    ++g_checks;
    if (!ok) {
        ++g_fail;
        std::lock_guard<std::mutex> lk(g_print);
        std::printf("FAIL %s\n", what.c_str());
    }
}

// same exception type (or both succeed with equal results)
template <class A, class B>
static void same_outcome(A ref, B gpu, const std::string& what) {
    std::string et_ref = "none", et_gpu = "none";
    decltype(ref()) r{};
    decltype(gpu()) g{};
    try { r = ref(); } catch (const std::out_of_range&) { et_ref = "out_of_range"; } catch (const std::invalid_argument&) { et_ref = "invalid_argument"; }
    try { g = gpu(); } catch (const std::out_of_range&) { et_gpu = "out_of_range"; } catch (const std::invalid_argument&) { et_gpu = "invalid_argument"; }
    expect(et_ref == et_gpu && (et_ref != "none" || r == g), what + " (ref " + et_ref + ", gpu " + et_gpu + ")");
}

static MetricsReport report_without_similarity(const SystemModel& m, const DependencyTable& d) {
    MetricsReport r;
    r.fan_in = fan_in(m, d);
    r.fan_out = fan_out(m, d);
    r.lcom.resize(m.class_count());
    r.lcom_ck.resize(m.class_count());
    r.cbo.resize(m.class_count());
    for (ClassId c = 0; c < m.class_count(); ++c) {
        r.lcom[c] = lcom_normalized(c, m, d);
        r.lcom_ck[c] = lcom_ck(c, m, d);
        r.cbo[c] = cbo(c, m, d);
    }
    r.workload = estimate_workload(m, d);
    return r;
}

static void check_system(const std::string& name, const SystemModel& model, const DependencyTable& deps,
                         bool all_whatifs) {
    gpu::Engine e;
    e.upload(model, deps);
    for (unsigned w : {1u, 3u, 8u}) {
        expect(e.parallel_class_metrics(w) == parallel_class_metrics(model, deps, w), name + " class metrics");
        expect(e.parallel_lcom_ck(w) == parallel_lcom_ck(model, deps, w), name + " lcom_ck");
    }
    expect(gpu::parallel_class_metrics(model, deps, 2) == parallel_class_metrics(model, deps, 2),
           name + " free parallel_class_metrics");
    for (unsigned w : {1u, 4u})
        expect(e.parallel_fan_metrics(w) == parallel_fan_metrics(model, deps, w), name + " fan metrics");
    expect(gpu::fan_in(model, deps) == fan_in(model, deps), name + " fan_in");
    expect(gpu::estimate_workload(model, deps) == estimate_workload(model, deps), name + " estimate_workload");
    expect(e.report_without_similarity() == report_without_similarity(model, deps),
           name + " report without similarity");
    if (model.method_count() <= 3000) {  // the reference's tables are O(m^2)
        // every criterion, with the report's similarity table
        MetricsReport full = report_without_similarity(model, deps);
        full.similarity = all_similarities(model, deps);
        Thresholds ts = compute_thresholds(full);
        for (bool allc : {false, true}) {
            SuggestOptions o;
            o.all_candidates = allc;
            expect(e.suggest_by_similarity(full, ts, o) == suggest_by_similarity(model, deps, full, ts, o),
                   name + " suggest_by_similarity");
            for (Combine cb : {Combine::Union, Combine::Intersection})
                expect(e.suggest_all(full, ts, {Criterion::Similarity, Criterion::Cohesion, Criterion::Coupling}, cb,
                                     o) == suggest_all(model, deps, full, ts,
                                                       {Criterion::Similarity, Criterion::Cohesion,
                                                        Criterion::Coupling},
                                                       cb, o),
                       name + " suggest_all every criterion");
        }
        expect(e.full_report() == full_report(model, deps), name + " full_report");
        expect(gpu::parallel_full_report(model, deps, 3) == parallel_full_report(model, deps, 3),
               name + " parallel_full_report");
        expect(gpu::all_similarities(model, deps) == all_similarities(model, deps), name + " all_similarities");
    }
    expect(gpu::fan_out(model, deps) == fan_out(model, deps), name + " fan_out");
    same_outcome([&] { return parallel_fan_metrics(model, deps, 0); },
                 [&] { return gpu::parallel_fan_metrics(model, deps, 0); }, name + " fan zero workers");
    const ClassId C = static_cast<ClassId>(model.class_count());
    for (ClassId c = 0; c < C + 2; ++c) {
        same_outcome([&] { return lcom_normalized(c, model, deps); }, [&] { return e.lcom_normalized(c); },
                     name + " lcom_normalized " + std::to_string(c));
        same_outcome([&] { return cbo(c, model, deps); }, [&] { return e.cbo(c); }, name + " cbo");
        same_outcome([&] { return lcom_ck(c, model, deps); }, [&] { return e.lcom_ck(c); }, name + " lcom_ck");
    }
    if (all_whatifs) {
        for (MethodId u = 0; u < model.method_count() + 1; ++u)
            for (ClassId o = 0; o < C + 1; ++o)
                for (ClassId d = 0; d < C + 1; ++d) {
                    if (u < model.method_count() && o != model.method_owner[u] && (u + o + d) % 5) continue;
                    same_outcome([&] { return what_if_move(u, o, d, model, deps); },
                                 [&] { return e.what_if_move(u, o, d); },
                                 name + " what_if " + std::to_string(u) + "," + std::to_string(o) + "," +
                                     std::to_string(d));
                }
    }
    MetricsReport report = report_without_similarity(model, deps);
    const std::vector<Thresholds> thrs = {
        compute_thresholds(report),
        compute_thresholds(report, ThresholdOverrides{0.2, 0.4, 1.0}),
        compute_thresholds(report, ThresholdOverrides{std::nullopt, 0.0, 0.0}),
    };
    // compute_thresholds on the device (suggest.hpp:46-61), similarity table included when small
    {
        MetricsReport withsim = report;
        if (model.method_count() <= 3000) withsim.similarity = all_similarities(model, deps);
        for (const ThresholdOverrides& ov : {ThresholdOverrides{}, ThresholdOverrides{0.2, 0.4, 1.0},
                                             ThresholdOverrides{std::nullopt, 0.0, std::nullopt}})
            expect(gpu::compute_thresholds(withsim, ov) == compute_thresholds(withsim, ov),
                   name + " gpu::compute_thresholds");
    }
    // n_workers -> GPUs: the multi-GPU group (one GPU here) and parallel_suggest_all
    {
        gpu::Group grp(1);
        grp.upload(model, deps);
        const Thresholds t0 = thrs[0];
        for (Combine cb : {Combine::Union, Combine::Intersection})
            for (bool allc : {false, true}) {
                SuggestOptions o;
                o.all_candidates = allc;
                const auto want = suggest_all(model, deps, report, t0, {Criterion::Cohesion, Criterion::Coupling}, cb, o);
                expect(grp.suggest_all(report, t0, {Criterion::Cohesion, Criterion::Coupling}, cb, o) == want,
                       name + " gpu::Group suggest_all");
                expect(gpu::parallel_suggest_all(model, deps, report, t0, {Criterion::Cohesion, Criterion::Coupling},
                                                 cb, o, 4) == want,
                       name + " gpu::parallel_suggest_all");
            }
        same_outcome([&] { return parallel_lcom_ck(model, deps, 0).size(); },
                     [&] { return gpu::parallel_suggest_all(model, deps, report, t0, {Criterion::Cohesion}, Combine::Union,
                                                            SuggestOptions{}, 0).size(); },
                     name + " zero workers");
    }
    const std::vector<std::vector<Criterion>> crits = {
        {Criterion::Cohesion}, {Criterion::Coupling}, {Criterion::Cohesion, Criterion::Coupling},
        {Criterion::Coupling, Criterion::Cohesion, Criterion::Cohesion}};
    for (size_t ti = 0; ti < thrs.size(); ++ti)
        for (bool allc : {false, true}) {
            SuggestOptions o;
            o.all_candidates = allc;
            const std::string tag = name + " t" + std::to_string(ti) + (allc ? " all" : " best");
            expect(e.suggest_by_cohesion(report, thrs[ti], o) ==
                       suggest_by_cohesion(model, deps, report, thrs[ti], o),
                   tag + " suggest_by_cohesion (order included)");
            expect(e.suggest_by_coupling(report, thrs[ti], o) ==
                       suggest_by_coupling(model, deps, report, thrs[ti], o),
                   tag + " suggest_by_coupling (order included)");
            for (const auto& cr : crits)
                for (Combine cb : {Combine::Union, Combine::Intersection})
                    expect(e.suggest_all(report, thrs[ti], cr, cb, o) ==
                               suggest_all(model, deps, report, thrs[ti], cr, cb, o),
                           tag + " suggest_all");
        }
    // gates come from the caller's report, even when it is not this system's
    MetricsReport skew = report;
    for (size_t c = 0; c < skew.lcom.size(); ++c) {
        if (c % 3 == 0) skew.lcom[c] = 1.0;
        if (c % 4 == 1) skew.cbo[c] += 7;
    }
    const Thresholds t0 = compute_thresholds(report);
    expect(e.suggest_all(skew, t0, {Criterion::Cohesion, Criterion::Coupling}, Combine::Union) ==
               suggest_all(model, deps, skew, t0, {Criterion::Cohesion, Criterion::Coupling}, Combine::Union),
           name + " caller-report gates");
    same_outcome([&] { return suggest_all(model, deps, report, t0, {}, Combine::Union); },
                 [&] { return e.suggest_all(report, t0, {}, Combine::Union); }, name + " empty criteria");
}

int main() {
    // the reference's own fixtures (tests/test_suggest.cpp:17-40)
    {
        SystemModel m;
        DependencyTable d;
        auto build = [&](std::vector<std::pair<std::vector<AttributeId>, std::vector<MethodId>>> cls,
                         std::vector<std::vector<MethodId>> calls, std::vector<std::vector<AttributeId>> acc) {
            SystemModel model;
            size_t nm = 0, na = 0;
            for (auto& c : cls) { nm += c.second.size(); na += c.first.size(); }
            model.method_owner.resize(nm);
            model.attribute_owner.resize(na);
            model.method_names.resize(nm);
            model.attribute_names.resize(na);
            for (size_t i = 0; i < cls.size(); ++i) {
                ClassRecord r;
                r.id = static_cast<ClassId>(i);
                r.attribute_ids = cls[i].first;
                r.method_ids = cls[i].second;
                for (auto p : r.method_ids) model.method_owner[p] = r.id;
                for (auto a : r.attribute_ids) model.attribute_owner[a] = r.id;
                model.classes.push_back(r);
            }
            calls.resize(nm);
            acc.resize(nm);
            DependencyTable deps{calls, acc};
            return std::make_pair(model, deps);
        };
        auto envy = build({{{0, 1}, {0, 1}}, {{2, 3}, {2}}}, {{2}, {}, {}}, {{2, 3}, {0, 1}, {2}});
        check_system("envy", envy.first, envy.second, true);
        auto coh = build({{{0, 1}, {0, 1}}, {{2, 3}, {2}}}, {{}, {2}, {}}, {{0, 1}, {2, 3}, {2}});
        check_system("cohesion", coh.first, coh.second, true);
        auto coup = build({{{}, {0}}, {{}, {1}}, {{}, {2}}}, {{1, 2}, {2}, {}}, {});
        check_system("coupling", coup.first, coup.second, true);
        (void)m;
        (void)d;
    }
    // generated systems: small (every what-if) to acceptance-sized, checked
    // concurrently (one host thread and one engine per system: the reference
    // functions are pure and the drop-in's engines are per thread)
    std::vector<std::thread> pool;
    for (uint64_t seed = 0; seed < 12; ++seed) {
        SplitMix64 draw(seed * 0x9e3779b9ULL + 1);
        GeneratorConfig cfg;
        cfg.seed = seed;
        const bool small = seed < 6;
        cfg.n_methods = static_cast<uint32_t>(small ? 5 + draw.below(40) : 10 + draw.below(1991));
        cfg.n_classes = static_cast<uint32_t>(small ? 2 + draw.below(9) : 2 + draw.below(199));
        cfg.n_attributes = static_cast<uint32_t>(1 + draw.below(std::max<uint64_t>(1, cfg.n_methods / 2)));
        cfg.k_max_calls = static_cast<uint32_t>(draw.below(6));
        cfg.k_max_accesses = static_cast<uint32_t>(draw.below(6));
        cfg.intra_class_bias = draw.unit();
        pool.emplace_back([cfg, seed, small] {
            const GeneratedSystem g = generate(cfg);
            check_system("gen" + std::to_string(seed), g.model, g.deps, small);
        });
    }
    // dense classes (the CTA path) and C2
    pool.emplace_back([] {
        GeneratorConfig cfg{3, 6, 3000, 384, 4, 32, 0.9};
        const GeneratedSystem g = generate(cfg);
        check_system("dense", g.model, g.deps, false);
    });
    pool.emplace_back([] {
        GeneratorConfig c2{1, 1000, 10000, 20000, 4, 4, 0.5};
        const GeneratedSystem g2 = generate(c2);
        check_system("c2", g2.model, g2.deps, false);
    });
    for (std::thread& t : pool) t.join();
    std::printf("%s: %d checks, %d failures\n", g_fail ? "FAIL" : "PASS", g_checks.load(), g_fail.load());
    return g_fail ? 1 : 0;
}
