// modmetrics/gpu.hpp — drop-in B200 engine for the reference library's metric
// and move-method suggestion path.
//
// Include this next to the reference headers (proj/include/modmetrics/) and
// link libmmgpu.so. The functions below have the reference's names,
// signatures, argument meaning, result types and exceptions; results are
// bit-identical (every double, every integer, and the ORDER of the returned
// vectors). Everything computes on the GPU through the C ABI in mmgpu.h;
// there is no CPU fallback (no device -> std::runtime_error).
//
//   reference (namespace modmetrics)          here (namespace modmetrics::gpu)
//   parallel_class_metrics  parallel.hpp:149  parallel_class_metrics / Engine::
//   parallel_lcom_ck        parallel.hpp:164  parallel_lcom_ck / Engine::
//   fan_in / fan_out        metrics.hpp:79-93 fan_in / fan_out
//   parallel_fan_metrics    parallel.hpp:186  parallel_fan_metrics / Engine::
//   estimate_workload       metrics.hpp:228   estimate_workload / Engine::
//   all_similarities        metrics.hpp:67    all_similarities / Engine::similarities
//   parallel_similarities   parallel.hpp:71   parallel_similarities
//   full_report             metrics.hpp:249   full_report / Engine:: (every field on the GPU)
//   parallel_full_report    parallel.hpp:210  parallel_full_report
//   lcom_normalized/lcom_ck/cbo metrics.hpp:128,159,187   Engine::
//   compute_thresholds      suggest.hpp:46    compute_thresholds / Engine:: (device sequential-sum means)
//   what_if_move            suggest.hpp:87    what_if_move / Engine::
//   suggest_by_cohesion     suggest.hpp:239   suggest_by_cohesion / Engine::
//   suggest_by_coupling     suggest.hpp:266   suggest_by_coupling / Engine::
//   suggest_by_similarity   suggest.hpp:206   suggest_by_similarity / Engine::
//   suggest_all             suggest.hpp:303   suggest_all / Engine:: (every criterion)
//
// A persistent Engine keeps the system resident in HBM across calls; the
// free functions upload per call (like the reference, which takes the model
// by const& every time).
#pragma once

#include <algorithm>
#include <cstdint>
#include <exception>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <modmetrics/metrics.hpp>
#include <modmetrics/model.hpp>
#include <modmetrics/parallel.hpp>
#include <modmetrics/suggest.hpp>

#include "../mmgpu.h"

namespace modmetrics::gpu {

namespace detail {

// status -> the reference's exception types (no exception crosses the C ABI)
inline void check(mm_status st, const mm_ctx* ctx, const char* what) {
    if (st == MM_OK) return;
    const char* detail = ctx ? mm_last_error(ctx)
                       : st == MM_E_CUDA ? "no usable CUDA device (this engine has no CPU fallback)"
                       : st == MM_E_RANGE ? "device index out of range" : "failed";
    const std::string msg = std::string(what) + ": " + detail;
    switch (st) {
        case MM_E_RANGE: throw std::out_of_range(msg);
        case MM_E_ARG: throw std::invalid_argument(msg);
        case MM_E_OOM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

// SystemModel + DependencyTable -> CSR (mm_system points into this object)
// Pinned host memory (mm_pinned_alloc), grown on demand and reused: the
// flattened system is staged here so the upload copies at the link's full
// rate instead of through the driver's pageable bounce buffers.
class PinnedArena {
public:
    PinnedArena() = default;
    PinnedArena(const PinnedArena&) = delete;
    PinnedArena& operator=(const PinnedArena&) = delete;
    PinnedArena(PinnedArena&& o) noexcept : p_(o.p_), cap_(o.cap_) { o.p_ = nullptr; o.cap_ = 0; }
    PinnedArena& operator=(PinnedArena&& o) noexcept {
        if (this != &o) {
            if (p_) mm_pinned_free(p_);
            p_ = o.p_; cap_ = o.cap_;
            o.p_ = nullptr; o.cap_ = 0;
        }
        return *this;
    }
    ~PinnedArena() { if (p_) mm_pinned_free(p_); }
    // n u32 slots per array, each array 64-byte aligned inside one block
    uint32_t* reserve(const size_t* counts, size_t n_arrays, uint32_t** out) {
        size_t total = 0;
        for (size_t k = 0; k < n_arrays; ++k) total += (counts[k] + 15) & ~size_t(15);
        if (total * 4 > cap_) {
            if (p_) mm_pinned_free(p_);
            p_ = nullptr;
            cap_ = 0;
            void* q = nullptr;
            if (mm_pinned_alloc(total * 4 + (total * 4) / 8, &q) != MM_OK) throw std::bad_alloc();
            p_ = q;
            cap_ = total * 4 + (total * 4) / 8;
        }
        uint32_t* at = static_cast<uint32_t*>(p_);
        for (size_t k = 0; k < n_arrays; ++k) {
            out[k] = at;
            at += (counts[k] + 15) & ~size_t(15);
        }
        return static_cast<uint32_t*>(p_);
    }

private:
    void* p_ = nullptr;
    size_t cap_ = 0;
};

// for_each over [0, n) on up to 16 host threads (worker exceptions rethrown
// after every started thread joined)
template <class Fn>
inline void parallel_ranges(size_t n, Fn&& fn) {
    const unsigned hw = std::thread::hardware_concurrency();
    const size_t T = n >= (size_t(1) << 15) ? std::min<size_t>(16, hw ? hw : 1) : 1;
    if (T <= 1) { fn(size_t(0), n); return; }
    std::vector<std::exception_ptr> errs(T);
    std::vector<std::thread> th;
    th.reserve(T);
    std::exception_ptr spawn_err;
    for (size_t k = 0; k < T && !spawn_err; ++k) {
        try {
            th.emplace_back([&, k] {
                try { fn(n * k / T, n * (k + 1) / T); } catch (...) { errs[k] = std::current_exception(); }
            });
        } catch (...) {
            spawn_err = std::current_exception();
        }
    }
    for (std::thread& t : th) t.join();
    if (spawn_err) std::rethrow_exception(spawn_err);
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

// The reference's vector-of-vectors model flattened to the CSR mm_upload
// takes: exact sizes first, then every row copied in parallel straight into
// pinned staging (arena) — or into owned vectors when no arena is given.
struct Csr {
    std::vector<uint32_t> own;  // backing store without an arena
    mm_system sys{};

    Csr(const SystemModel& model, const DependencyTable& deps, PinnedArena* arena = nullptr) {
        const size_t C = model.classes.size(), m = model.method_count(), A = model.attribute_count();
        if (deps.calls.size() != m || deps.accesses.size() != m)
            throw std::invalid_argument("gpu: dependency table rows != method count");
        // offsets (sizes, then an exclusive scan)
        std::vector<uint32_t> cmo(C + 1), cao(C + 1), co(m + 1), ao(m + 1);
        parallel_ranges(C, [&](size_t b, size_t e) {
            for (size_t c = b; c < e; ++c) {
                cmo[c + 1] = static_cast<uint32_t>(model.classes[c].method_ids.size());
                cao[c + 1] = static_cast<uint32_t>(model.classes[c].attribute_ids.size());
            }
        });
        parallel_ranges(m, [&](size_t b, size_t e) {
            for (size_t p = b; p < e; ++p) {
                co[p + 1] = static_cast<uint32_t>(deps.calls[p].size());
                ao[p + 1] = static_cast<uint32_t>(deps.accesses[p].size());
            }
        });
        for (size_t c = 0; c < C; ++c) { cmo[c + 1] += cmo[c]; cao[c + 1] += cao[c]; }
        for (size_t p = 0; p < m; ++p) { co[p + 1] += co[p]; ao[p + 1] += ao[p]; }
        const size_t counts[10] = {C + 1, cmo[C], C + 1, cao[C], m + 1, co[m], m + 1, ao[m], m, A};
        uint32_t* a[10];
        if (arena) {
            arena->reserve(counts, 10, a);
        } else {
            size_t total = 0;
            for (size_t k = 0; k < 10; ++k) total += counts[k];
            own.resize(total ? total : 1);
            uint32_t* at = own.data();
            for (size_t k = 0; k < 10; ++k) { a[k] = at; at += counts[k]; }
        }
        std::copy(cmo.begin(), cmo.end(), a[0]);
        std::copy(cao.begin(), cao.end(), a[2]);
        std::copy(co.begin(), co.end(), a[4]);
        std::copy(ao.begin(), ao.end(), a[6]);
        parallel_ranges(C, [&](size_t b, size_t e) {
            for (size_t c = b; c < e; ++c) {
                const ClassRecord& r = model.classes[c];
                std::copy(r.method_ids.begin(), r.method_ids.end(), a[1] + cmo[c]);
                std::copy(r.attribute_ids.begin(), r.attribute_ids.end(), a[3] + cao[c]);
            }
        });
        parallel_ranges(m, [&](size_t b, size_t e) {
            for (size_t p = b; p < e; ++p) {
                std::copy(deps.calls[p].begin(), deps.calls[p].end(), a[5] + co[p]);
                std::copy(deps.accesses[p].begin(), deps.accesses[p].end(), a[7] + ao[p]);
            }
            std::copy(model.method_owner.begin() + b, model.method_owner.begin() + e, a[8] + b);
        });
        parallel_ranges(A, [&](size_t b, size_t e) {
            std::copy(model.attribute_owner.begin() + b, model.attribute_owner.begin() + e, a[9] + b);
        });
        sys.n_classes = static_cast<uint32_t>(C);
        sys.n_methods = static_cast<uint32_t>(m);
        sys.n_attributes = static_cast<uint32_t>(A);
        sys.class_method_off = a[0];
        sys.class_methods = a[1];
        sys.class_attr_off = a[2];
        sys.class_attrs = a[3];
        sys.call_off = a[4];
        sys.call_tgt = a[5];
        sys.acc_off = a[6];
        sys.acc_tgt = a[7];
        sys.method_owner = a[8];
        sys.attribute_owner = a[9];
    }
};

inline WhatIfMetrics to_whatif(const mm_suggestion& r) {
    WhatIfMetrics w;
    w.lcom_origin_before = r.lcom_origin_before;
    w.lcom_origin_after = r.lcom_origin_after;
    w.lcom_dest_before = r.lcom_dest_before;
    w.lcom_dest_after = r.lcom_dest_after;
    w.cbo_origin_before = r.cbo_origin_before;
    w.cbo_origin_after = r.cbo_origin_after;
    w.cbo_dest_before = r.cbo_dest_before;
    w.cbo_dest_after = r.cbo_dest_after;
    w.origin_degenerate_after = r.origin_degenerate_after != 0;
    w.dest_degenerate_after = r.dest_degenerate_after != 0;
    return w;
}

inline MoveSuggestion to_suggestion(const mm_suggestion& r) {
    MoveSuggestion s;
    s.method = r.method;
    s.origin = r.origin;
    s.destination = r.destination;
    for (Criterion c : {Criterion::Similarity, Criterion::Cohesion, Criterion::Coupling})
        if (r.criteria & (1u << static_cast<unsigned>(c))) s.criteria.push_back(c);
    s.impact = to_whatif(r);
    return s;
}

}  // namespace detail

class Engine {
public:
    explicit Engine(int device = 0) {
        mm_ctx* c = nullptr;
        detail::check(mm_ctx_create(device, &c), nullptr, "mm_ctx_create");
        ctx_.reset(c);
    }

    // Uploads (copies) the system into HBM; the model may be destroyed afterwards.
    void upload(const SystemModel& model, const DependencyTable& deps) {
        const detail::Csr csr(model, deps, &stage_);
        detail::check(mm_upload(ctx_.get(), &csr.sys), ctx_.get(), "mm_upload");
        n_classes_ = csr.sys.n_classes;
        n_methods_ = csr.sys.n_methods;
    }

    // Uploads a CSR system as-is (e.g. the direct view of gpu::Facts, gpu_facts.hpp).
    void upload(const mm_system& sys) {
        detail::check(mm_upload(ctx_.get(), &sys), ctx_.get(), "mm_upload");
        n_classes_ = sys.n_classes;
        n_methods_ = sys.n_methods;
    }

    WorkloadEstimate estimate_workload() {
        mm_workload w{};
        detail::check(mm_estimate_workload(ctx_.get(), &w), ctx_.get(), "estimate_workload");
        WorkloadEstimate e;
        e.m = w.m; e.c = w.c; e.k_m = w.k_m; e.k_a = w.k_a;
        e.n_fan = w.n_fan; e.n_sim = w.n_sim; e.n_lcom = w.n_lcom; e.n_cbo = w.n_cbo; e.n_total = w.n_total;
        return e;
    }

    // full_report (metrics.hpp:249-264) with every field but `similarity`
    // (left empty: the all-pairs table is outside this engine)
    MetricsReport report_without_similarity() {
        MetricsReport r;
        FanMetrics f = parallel_fan_metrics();
        r.fan_in = std::move(f.fan_in);
        r.fan_out = std::move(f.fan_out);
        r.lcom.resize(n_classes_);
        r.lcom_ck.resize(n_classes_);
        r.cbo.resize(n_classes_);
        detail::check(mm_class_metrics(ctx_.get(), r.lcom.data(), r.lcom_ck.data(), r.cbo.data()), ctx_.get(),
                      "report_without_similarity");
        r.workload = estimate_workload();
        return r;
    }

    std::vector<SimilarityEntry> similarities() {
        uint64_t n = 0;
        detail::check(mm_similarities(ctx_.get(), nullptr, 0, &n), ctx_.get(), "all_similarities");
        std::vector<mm_similarity> raw(n);
        if (n) detail::check(mm_similarities(ctx_.get(), raw.data(), n, &n), ctx_.get(), "all_similarities");
        std::vector<SimilarityEntry> out(n);
        for (uint64_t k = 0; k < n; ++k) out[k] = SimilarityEntry{raw[k].first, raw[k].second, raw[k].value};
        return out;
    }

    // full_report (metrics.hpp:249-264), every field computed on the device
    MetricsReport full_report() {
        MetricsReport r = report_without_similarity();
        r.similarity = similarities();
        return r;
    }

    FanMetrics parallel_fan_metrics(unsigned n_workers = 1) {
        if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");  // parallel.hpp:29
        FanMetrics out;
        out.fan_in.resize(n_methods_);
        out.fan_out.resize(n_methods_);
        detail::check(mm_fan_metrics(ctx_.get(), out.fan_in.data(), out.fan_out.data()), ctx_.get(),
                      "parallel_fan_metrics");
        return out;
    }

    ClassMetrics parallel_class_metrics(unsigned n_workers = 1) {
        if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");  // parallel.hpp:29
        ClassMetrics out;
        out.lcom.resize(n_classes_);
        out.cbo.resize(n_classes_);
        detail::check(mm_class_metrics(ctx_.get(), out.lcom.data(), nullptr, out.cbo.data()), ctx_.get(),
                      "parallel_class_metrics");
        return out;
    }

    std::vector<std::uint64_t> parallel_lcom_ck(unsigned n_workers = 1) {
        if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");
        std::vector<std::uint64_t> out(n_classes_);
        detail::check(mm_class_metrics(ctx_.get(), nullptr, out.data(), nullptr), ctx_.get(), "parallel_lcom_ck");
        return out;
    }

    // compute_thresholds (suggest.hpp:46-61) on the caller's report: the three
    // means on the device, bit-identical to the reference's sequential sums
    Thresholds compute_thresholds(const MetricsReport& report, const ThresholdOverrides& ov = {}) {
        std::vector<double> sim(report.similarity.size());
        for (size_t k = 0; k < sim.size(); ++k) sim[k] = report.similarity[k].value;
        mm_overrides o{};
        if (ov.similarity) { o.has_similarity = 1; o.similarity = *ov.similarity; }
        if (ov.lcom) { o.has_lcom = 1; o.lcom = *ov.lcom; }
        if (ov.cbo) { o.has_cbo = 1; o.cbo = *ov.cbo; }
        mm_thresholds t{};
        detail::check(mm_report_thresholds(ctx_.get(), report.lcom.data(), report.lcom.size(), report.cbo.data(),
                                           report.cbo.size(), sim.data(), sim.size(), &o, &t),
                      ctx_.get(), "compute_thresholds");
        Thresholds r;
        r.similarity = t.similarity;
        r.lcom = t.lcom;
        r.cbo = t.cbo;
        r.explicit_mode = t.explicit_mode != 0;
        return r;
    }

    double lcom_normalized(ClassId c) {
        double v = 0;
        detail::check(mm_lcom_normalized(ctx_.get(), c, &v), ctx_.get(), "lcom_normalized");
        return v;
    }
    std::uint64_t lcom_ck(ClassId c) {
        std::uint64_t v = 0;
        detail::check(mm_lcom_ck(ctx_.get(), c, &v), ctx_.get(), "lcom_ck");
        return v;
    }
    std::uint32_t cbo(ClassId c) {
        std::uint32_t v = 0;
        detail::check(mm_cbo(ctx_.get(), c, &v), ctx_.get(), "cbo");
        return v;
    }

    WhatIfMetrics what_if_move(MethodId method, ClassId origin, ClassId destination) {
        mm_whatif w;
        detail::check(mm_what_if(ctx_.get(), method, origin, destination, &w), ctx_.get(), "what_if_move");
        mm_suggestion r{};
        r.lcom_origin_before = w.lcom_origin_before;
        r.lcom_origin_after = w.lcom_origin_after;
        r.lcom_dest_before = w.lcom_dest_before;
        r.lcom_dest_after = w.lcom_dest_after;
        r.cbo_origin_before = w.cbo_origin_before;
        r.cbo_origin_after = w.cbo_origin_after;
        r.cbo_dest_before = w.cbo_dest_before;
        r.cbo_dest_after = w.cbo_dest_after;
        r.origin_degenerate_after = w.origin_degenerate_after;
        r.dest_degenerate_after = w.dest_degenerate_after;
        return detail::to_whatif(r);
    }

    // suggest_all, suggest.hpp:303. Gates use report.lcom / report.cbo (the
    // caller's report, exactly as the reference does).
    std::vector<MoveSuggestion> suggest_all(const MetricsReport& report, const Thresholds& thresholds,
                                            const std::vector<Criterion>& criteria, Combine combine,
                                            const SuggestOptions& opts = {}) {
        std::vector<Criterion> sel = criteria;
        std::sort(sel.begin(), sel.end());
        sel.erase(std::unique(sel.begin(), sel.end()), sel.end());
        if (sel.empty()) throw std::invalid_argument("suggest_all: no criteria selected");  // suggest.hpp:313
        uint32_t mask = 0;
        for (Criterion c : sel) mask |= 1u << static_cast<unsigned>(c);
        if (!(mask & MM_CRIT_SIMILARITY)) return run(report, thresholds, mask, combine == Combine::Intersection, opts);
        // similarity runs on its own; merged by (method, destination) with the
        // other criteria's records, tags unioned (suggest.hpp:315-341)
        const bool inter = combine == Combine::Intersection;
        std::vector<MoveSuggestion> parts = suggest_by_similarity(report, thresholds, opts);
        if (mask & ~MM_CRIT_SIMILARITY) {
            std::vector<MoveSuggestion> rest = run(report, thresholds, mask & ~MM_CRIT_SIMILARITY, inter, opts);
            parts.insert(parts.end(), rest.begin(), rest.end());
        }
        std::map<std::pair<MethodId, ClassId>, MoveSuggestion> merged;
        for (MoveSuggestion& m : parts) {
            auto [it, fresh] = merged.try_emplace(std::make_pair(m.method, m.destination), m);
            if (!fresh) it->second.criteria.insert(it->second.criteria.end(), m.criteria.begin(), m.criteria.end());
        }
        std::vector<MoveSuggestion> out;
        for (auto& [key, m] : merged) {
            std::sort(m.criteria.begin(), m.criteria.end());
            m.criteria.erase(std::unique(m.criteria.begin(), m.criteria.end()), m.criteria.end());
            if (inter && m.criteria.size() != sel.size()) continue;
            out.push_back(std::move(m));
        }
        std::sort(out.begin(), out.end(), [](const MoveSuggestion& a, const MoveSuggestion& b) {
            if (a.origin != b.origin) return a.origin < b.origin;
            if (a.method != b.method) return a.method < b.method;
            return a.destination < b.destination;
        });
        return out;
    }

    // suggest_by_similarity (suggest.hpp:206): pairs from report.similarity
    // (the caller's table, as the reference reads it), ordered by method,
    // then destination — the reference's map order.
    std::vector<MoveSuggestion> suggest_by_similarity(const MetricsReport& report, const Thresholds& thresholds,
                                                      const SuggestOptions& opts = {}) {
        std::vector<mm_similarity> tab(report.similarity.size());
        for (size_t k = 0; k < tab.size(); ++k)
            tab[k] = mm_similarity{report.similarity[k].first, report.similarity[k].second, report.similarity[k].value};
        uint64_t n = 0;
        const mm_status st = mm_suggest_similarity(ctx_.get(), tab.data(), tab.size(), thresholds.similarity,
                                                   opts.all_candidates ? 1u : 0u, nullptr, 0, &n);
        if (st != MM_OK && st != MM_E_CAPACITY) detail::check(st, ctx_.get(), "suggest_by_similarity");
        std::vector<mm_suggestion> raw(n);
        if (n)
            detail::check(mm_suggest_similarity(ctx_.get(), tab.data(), tab.size(), thresholds.similarity,
                                                opts.all_candidates ? 1u : 0u, raw.data(), n, &n),
                          ctx_.get(), "suggest_by_similarity");
        std::vector<MoveSuggestion> out;
        out.reserve(raw.size());
        out.resize(raw.size());
        detail::parallel_ranges(raw.size(), [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) out[i] = detail::to_suggestion(raw[i]);
        });
        return out;
    }

    // suggest_by_cohesion (suggest.hpp:239): same records, in the reference's
    // emission order (classes by id; methods by fan_out desc, then id).
    std::vector<MoveSuggestion> suggest_by_cohesion(const MetricsReport& report, const Thresholds& thresholds,
                                                    const SuggestOptions& opts = {}) {
        auto v = run(report, thresholds, MM_CRIT_COHESION, false, opts);
        order_like_reference(v, [&](MethodId m) { return std::uint64_t(report.fan_out[m]); });
        return v;
    }

    // suggest_by_coupling (suggest.hpp:266): methods by fan_in + fan_out desc, then id.
    std::vector<MoveSuggestion> suggest_by_coupling(const MetricsReport& report, const Thresholds& thresholds,
                                                    const SuggestOptions& opts = {}) {
        auto v = run(report, thresholds, MM_CRIT_COUPLING, false, opts);
        order_like_reference(v, [&](MethodId m) {
            return std::uint64_t(report.fan_in[m]) + std::uint64_t(report.fan_out[m]);
        });
        return v;
    }

    mm_ctx* handle() { return ctx_.get(); }

private:
    struct Del {
        void operator()(mm_ctx* c) const { mm_ctx_destroy(c); }
    };
    std::unique_ptr<mm_ctx, Del> ctx_;
    detail::PinnedArena stage_;  // pinned staging of the flattened system, reused across uploads
    uint32_t n_classes_ = 0;
    uint32_t n_methods_ = 0;

    std::vector<MoveSuggestion> run(const MetricsReport& report, const Thresholds& t, uint32_t mask, bool inter,
                                    const SuggestOptions& opts) {
        if (report.lcom.size() != n_classes_ || report.cbo.size() != n_classes_)
            throw std::invalid_argument("gpu: report does not match the uploaded system");
        detail::check(mm_set_gates(ctx_.get(), report.lcom.data(), report.cbo.data()), ctx_.get(), "mm_set_gates");
        mm_sweep_params p{};
        p.criteria = mask;
        p.combine = inter ? MM_COMBINE_INTERSECTION : MM_COMBINE_UNION;
        p.all_candidates = opts.all_candidates ? 1u : 0u;
        p.top_k = 1;
        p.thr_lcom = t.lcom;
        p.thr_cbo = t.cbo;
        p.threshold_source = MM_THR_EXPLICIT;
        uint64_t n = 0;
        detail::check(mm_sweep(ctx_.get(), &p, &n), ctx_.get(), "mm_sweep");
        std::vector<mm_suggestion> raw(n);
        if (n) detail::check(mm_copy_suggestions(ctx_.get(), raw.data(), n, &n), ctx_.get(), "mm_copy_suggestions");
        detail::check(mm_set_gates(ctx_.get(), nullptr, nullptr), ctx_.get(), "mm_set_gates");
        std::vector<MoveSuggestion> out;
        out.reserve(raw.size());
        out.resize(raw.size());
        detail::parallel_ranges(raw.size(), [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) out[i] = detail::to_suggestion(raw[i]);
        });
        return out;
    }

    // Within one origin class the GPU list is (method, destination) ordered;
    // the per-criterion reference vectors list methods by a busyness key,
    // descending, id ascending (destinations of one method stay ascending).
    template <class Key>
    static void order_like_reference(std::vector<MoveSuggestion>& v, Key key) {
        std::stable_sort(v.begin(), v.end(), [&](const MoveSuggestion& a, const MoveSuggestion& b) {
            if (a.origin != b.origin) return a.origin < b.origin;
            const auto ka = key(a.method), kb = key(b.method);
            if (ka != kb) return ka > kb;
            return a.method < b.method;
        });
    }
};

// ---- several GPUs: n_workers -> GPUs (mm_group, include/mmgpu.h) --------

// The sweep on n GPUs of one process: each GPU recomputes the metric pass
// (replicas) and sweeps a cost-balanced class range; the shard lists are
// exchanged over NCCL with exact counts and concatenated in rank order, which
// is suggest_all's ordered list. Criteria ⊆ {Cohesion, Coupling}.
class Group {
public:
    explicit Group(unsigned n_gpus) {
        if (n_gpus == 0) throw std::invalid_argument("plan_partition: zero workers");  // parallel.hpp:29
        mm_group* g = nullptr;
        const mm_status st = mm_group_create(nullptr, static_cast<int>(n_gpus), &g);
        if (st != MM_OK) detail::check(st, nullptr, "mm_group_create");
        g_.reset(g);
    }
    unsigned size() const { return static_cast<unsigned>(mm_group_size(g_.get())); }

    void upload(const SystemModel& model, const DependencyTable& deps) {
        const detail::Csr csr(model, deps);
        check(mm_group_upload(g_.get(), &csr.sys), "mm_group_upload");
        n_classes_ = csr.sys.n_classes;
    }

    std::vector<MoveSuggestion> suggest_all(const MetricsReport& report, const Thresholds& thresholds,
                                            const std::vector<Criterion>& criteria, Combine combine,
                                            const SuggestOptions& opts = {}) {
        uint32_t mask = 0;
        for (Criterion c : criteria) mask |= 1u << static_cast<unsigned>(c);
        if (!mask) throw std::invalid_argument("suggest_all: no criteria selected");  // suggest.hpp:313
        if (mask & MM_CRIT_SIMILARITY)
            throw std::invalid_argument("gpu::Group: the similarity criterion runs on one GPU (gpu::Engine)");
        if (report.lcom.size() != n_classes_ || report.cbo.size() != n_classes_)
            throw std::invalid_argument("gpu: report does not match the uploaded system");
        check(mm_group_set_gates(g_.get(), report.lcom.data(), report.cbo.data()), "mm_group_set_gates");
        mm_sweep_params p{};
        p.criteria = mask;
        p.combine = combine == Combine::Intersection ? MM_COMBINE_INTERSECTION : MM_COMBINE_UNION;
        p.all_candidates = opts.all_candidates ? 1u : 0u;
        p.top_k = 1;
        p.thr_lcom = thresholds.lcom;
        p.thr_cbo = thresholds.cbo;
        p.threshold_source = MM_THR_EXPLICIT;
        uint64_t n = 0;
        check(mm_group_run(g_.get(), &p, &n), "mm_group_run");
        std::vector<mm_suggestion> raw(n);
        if (n) check(mm_group_copy_suggestions(g_.get(), raw.data(), n, &n), "mm_group_copy_suggestions");
        std::vector<MoveSuggestion> out;
        out.reserve(raw.size());
        out.resize(raw.size());
        detail::parallel_ranges(raw.size(), [&](size_t b, size_t e) {
            for (size_t i = b; i < e; ++i) out[i] = detail::to_suggestion(raw[i]);
        });
        return out;
    }

    mm_group* handle() { return g_.get(); }

private:
    struct Del {
        void operator()(mm_group* g) const { mm_group_destroy(g); }
    };
    std::unique_ptr<mm_group, Del> g_;
    uint32_t n_classes_ = 0;

    void check(mm_status st, const char* what) {
        if (st == MM_OK) return;
        const std::string msg = std::string(what) + ": " + mm_group_last_error(g_.get());
        switch (st) {
            case MM_E_RANGE: throw std::out_of_range(msg);
            case MM_E_ARG: throw std::invalid_argument(msg);
            case MM_E_OOM: throw std::bad_alloc();
            default: throw std::runtime_error(msg);
        }
    }
};

namespace detail {
// The free functions keep one engine per host thread (a context, its streams
// and device buffers persist across calls; the system is uploaded per call,
// as the reference takes the model by const& each time).
inline Engine& thread_engine() {
    thread_local Engine e;
    return e;
}

inline unsigned visible_gpus() {
    const int n = mm_device_count();
    return n > 0 ? static_cast<unsigned>(n) : 0u;
}
}  // namespace detail

// ---- free functions with the reference signatures ------------------------

inline Thresholds compute_thresholds(const MetricsReport& report, const ThresholdOverrides& ov = {}) {
    return detail::thread_engine().compute_thresholds(report, ov);
}

// suggest_all on min(n_workers, visible GPUs) GPUs (an extension in the
// reference's parallel_* naming: the reference's suggest_all is sequential).
// One GPU, or the similarity criterion: the single-GPU engine.
inline std::vector<MoveSuggestion> parallel_suggest_all(const SystemModel& model, const DependencyTable& deps,
                                                        const MetricsReport& report, const Thresholds& thresholds,
                                                        const std::vector<Criterion>& criteria, Combine combine,
                                                        const SuggestOptions& opts, unsigned n_workers) {
    if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");
    const unsigned n = std::min(n_workers, detail::visible_gpus());
    bool sim = false;
    for (Criterion c : criteria) sim |= c == Criterion::Similarity;
    if (n <= 1 || sim) {
        Engine& e = detail::thread_engine();
        e.upload(model, deps);
        return e.suggest_all(report, thresholds, criteria, combine, opts);
    }
    Group g(n);
    g.upload(model, deps);
    return g.suggest_all(report, thresholds, criteria, combine, opts);
}

inline ClassMetrics parallel_class_metrics(const SystemModel& model, const DependencyTable& deps,
                                           unsigned n_workers) {
    if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.parallel_class_metrics(n_workers);
}

inline FanMetrics parallel_fan_metrics(const SystemModel& model, const DependencyTable& deps, unsigned n_workers) {
    if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.parallel_fan_metrics(n_workers);
}

inline std::vector<SimilarityEntry> all_similarities(const SystemModel& model, const DependencyTable& deps) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.similarities();
}

inline std::vector<SimilarityEntry> parallel_similarities(const SystemModel& model, const DependencyTable& deps,
                                                          unsigned n_workers) {
    if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");  // parallel.hpp:29
    return gpu::all_similarities(model, deps);
}

inline MetricsReport full_report(const SystemModel& model, const DependencyTable& deps) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.full_report();
}

inline MetricsReport parallel_full_report(const SystemModel& model, const DependencyTable& deps, unsigned n_workers) {
    if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");
    return gpu::full_report(model, deps);
}

inline WorkloadEstimate estimate_workload(const SystemModel& model, const DependencyTable& deps) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.estimate_workload();
}

inline std::vector<std::uint32_t> fan_in(const SystemModel& model, const DependencyTable& deps) {
    return gpu::parallel_fan_metrics(model, deps, 1u).fan_in;
}

inline std::vector<std::uint32_t> fan_out(const SystemModel& model, const DependencyTable& deps) {
    return gpu::parallel_fan_metrics(model, deps, 1u).fan_out;
}

inline std::vector<std::uint64_t> parallel_lcom_ck(const SystemModel& model, const DependencyTable& deps,
                                                   unsigned n_workers) {
    if (n_workers == 0) throw std::invalid_argument("plan_partition: zero workers");
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.parallel_lcom_ck(n_workers);
}

inline WhatIfMetrics what_if_move(MethodId method, ClassId origin, ClassId destination, const SystemModel& model,
                                  const DependencyTable& deps) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.what_if_move(method, origin, destination);
}

inline std::vector<MoveSuggestion> suggest_by_cohesion(const SystemModel& model, const DependencyTable& deps,
                                                       const MetricsReport& report, const Thresholds& thresholds,
                                                       const SuggestOptions& opts = {}) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.suggest_by_cohesion(report, thresholds, opts);
}

inline std::vector<MoveSuggestion> suggest_by_coupling(const SystemModel& model, const DependencyTable& deps,
                                                       const MetricsReport& report, const Thresholds& thresholds,
                                                       const SuggestOptions& opts = {}) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.suggest_by_coupling(report, thresholds, opts);
}

inline std::vector<MoveSuggestion> suggest_by_similarity(const SystemModel& model, const DependencyTable& deps,
                                                         const MetricsReport& report, const Thresholds& thresholds,
                                                         const SuggestOptions& opts = {}) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.suggest_by_similarity(report, thresholds, opts);
}

inline std::vector<MoveSuggestion> suggest_all(const SystemModel& model, const DependencyTable& deps,
                                               const MetricsReport& report, const Thresholds& thresholds,
                                               const std::vector<Criterion>& criteria, Combine combine,
                                               const SuggestOptions& opts = {}) {
    Engine& e = detail::thread_engine();
    e.upload(model, deps);
    return e.suggest_all(report, thresholds, criteria, combine, opts);
}

}  // namespace modmetrics::gpu
