// ref_shim.cpp — a C ABI around the UNMODIFIED reference headers.
//
// TEST / BASELINE INFRASTRUCTURE ONLY. Compiled by oracle/Makefile against
// /root/reference/proj/include in place (nothing copied) into
// oracle/_ref/libmmref.so. Used to (a) validate the oracle restatement and
// the native generator here, (b) generate tests/golden fixtures, and (c) time
// the reference CPU path for bench.py's cpu_baseline / --impl reference arm.
// The product never links it.
#include <atomic>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <stdexcept>
#include <vector>

#include <modmetrics/generate.hpp>
#include <modmetrics/metrics.hpp>
#include <modmetrics/parallel.hpp>
#include <modmetrics/suggest.hpp>

#include "../include/mmgpu.h"

using namespace modmetrics;

namespace {

struct RefModel {
    SystemModel model;
    DependencyTable deps;
    // CSR view for generate() round trips
    std::vector<uint32_t> mo, ao, cmo, cm, cao, ca, co, ct, ao2, at;
    mm_system view{};
    std::vector<mm_suggestion> last;  // ref_sweep's result (ref_sweep_copy)
};

void to_csr(RefModel& r) {
    const SystemModel& m = r.model;
    const DependencyTable& d = r.deps;
    r.mo = m.method_owner;
    r.ao = m.attribute_owner;
    r.cmo.assign(1, 0);
    r.cao.assign(1, 0);
    r.cm.clear();
    r.ca.clear();
    for (const ClassRecord& c : m.classes) {
        r.cm.insert(r.cm.end(), c.method_ids.begin(), c.method_ids.end());
        r.ca.insert(r.ca.end(), c.attribute_ids.begin(), c.attribute_ids.end());
        r.cmo.push_back(static_cast<uint32_t>(r.cm.size()));
        r.cao.push_back(static_cast<uint32_t>(r.ca.size()));
    }
    r.co.assign(1, 0);
    r.ao2.assign(1, 0);
    r.ct.clear();
    r.at.clear();
    for (size_t p = 0; p < d.calls.size(); ++p) {
        r.ct.insert(r.ct.end(), d.calls[p].begin(), d.calls[p].end());
        r.at.insert(r.at.end(), d.accesses[p].begin(), d.accesses[p].end());
        r.co.push_back(static_cast<uint32_t>(r.ct.size()));
        r.ao2.push_back(static_cast<uint32_t>(r.at.size()));
    }
    r.view.n_classes = static_cast<uint32_t>(m.classes.size());
    r.view.n_methods = static_cast<uint32_t>(m.method_owner.size());
    r.view.n_attributes = static_cast<uint32_t>(m.attribute_owner.size());
    r.view.method_owner = r.mo.data();
    r.view.attribute_owner = r.ao.data();
    r.view.class_method_off = r.cmo.data();
    r.view.class_methods = r.cm.data();
    r.view.class_attr_off = r.cao.data();
    r.view.class_attrs = r.ca.data();
    r.view.call_off = r.co.data();
    r.view.call_tgt = r.ct.data();
    r.view.acc_off = r.ao2.data();
    r.view.acc_tgt = r.at.data();
}

void from_csr(RefModel& r, const mm_system* s) {
    SystemModel& m = r.model;
    m.classes.resize(s->n_classes);
    for (uint32_t c = 0; c < s->n_classes; ++c) {
        ClassRecord& rec = m.classes[c];
        rec.id = c;
        rec.name = "C" + std::to_string(c);
        rec.method_ids.assign(s->class_methods + s->class_method_off[c],
                              s->class_methods + s->class_method_off[c + 1]);
        rec.attribute_ids.assign(s->class_attrs + s->class_attr_off[c],
                                 s->class_attrs + s->class_attr_off[c + 1]);
    }
    m.method_owner.assign(s->method_owner, s->method_owner + s->n_methods);
    m.attribute_owner.assign(s->attribute_owner, s->attribute_owner + s->n_attributes);
    m.method_names.resize(s->n_methods);
    m.attribute_names.resize(s->n_attributes);
    r.deps.calls.resize(s->n_methods);
    r.deps.accesses.resize(s->n_methods);
    for (uint32_t p = 0; p < s->n_methods; ++p) {
        r.deps.calls[p].assign(s->call_tgt + s->call_off[p], s->call_tgt + s->call_off[p + 1]);
        r.deps.accesses[p].assign(s->acc_tgt + s->acc_off[p], s->acc_tgt + s->acc_off[p + 1]);
    }
}

int status_of(const std::exception_ptr& e) {
    try {
        std::rethrow_exception(e);
    } catch (const std::out_of_range&) {
        return MM_E_RANGE;
    } catch (const std::invalid_argument&) {
        return MM_E_ARG;
    } catch (...) {
        return MM_E_STATE;
    }
}

void fill(mm_suggestion& o, const MoveSuggestion& s) {
    std::memset(&o, 0, sizeof o);
    o.method = s.method;
    o.origin = s.origin;
    o.destination = s.destination;
    for (Criterion c : s.criteria) o.criteria |= static_cast<uint8_t>(1u << static_cast<unsigned>(c));
    o.lcom_origin_before = s.impact.lcom_origin_before;
    o.lcom_origin_after = s.impact.lcom_origin_after;
    o.lcom_dest_before = s.impact.lcom_dest_before;
    o.lcom_dest_after = s.impact.lcom_dest_after;
    o.cbo_origin_before = s.impact.cbo_origin_before;
    o.cbo_origin_after = s.impact.cbo_origin_after;
    o.cbo_dest_before = s.impact.cbo_dest_before;
    o.cbo_dest_after = s.impact.cbo_dest_after;
    o.origin_degenerate_after = s.impact.origin_degenerate_after;
    o.dest_degenerate_after = s.impact.dest_degenerate_after;
}

std::vector<Criterion> criteria_of(uint32_t mask) {
    std::vector<Criterion> v;
    if (mask & MM_CRIT_SIMILARITY) v.push_back(Criterion::Similarity);
    if (mask & MM_CRIT_COHESION) v.push_back(Criterion::Cohesion);
    if (mask & MM_CRIT_COUPLING) v.push_back(Criterion::Coupling);
    return v;
}


// ---- config C3: Zipf class sizes -----------------------
// The reference has no skewed generator. Ownership is restated here from the
// C3 recipe (sizes ∝ 1/rank^s, min 1, ids shuffled by SplitMix64 seeded
// seed ^ 0x5a17f00dd15ea5e5); the dependencies are drawn by the reference's
// own SplitMix64 / detail::pick_excluding / detail::pick_foreign in
// generate()'s exact loop (generate.hpp:124-161). tests/test_abi_cpu.py pins
// the product's mm_generate(zipf_s) against this.
std::vector<uint32_t> zipf_sizes(uint32_t n, uint32_t c, double s) {
    std::vector<double> w(c);
    double W = 0.0;
    for (uint32_t r = 0; r < c; ++r) W += (w[r] = 1.0 / std::pow(double(r) + 1.0, s));
    std::vector<uint32_t> sz(c);
    uint64_t total = 0;
    const uint32_t lo = n >= c ? 1u : 0u;
    for (uint32_t r = 0; r < c; ++r) {
        sz[r] = std::max<uint32_t>(lo, static_cast<uint32_t>(std::floor(double(n) * w[r] / W)));
        total += sz[r];
    }
    for (uint32_t r = 0; total > n; r = (r + 1) % c)
        if (sz[r] > lo) { --sz[r]; --total; }
    for (uint32_t r = 0; total < n; r = (r + 1) % c) { ++sz[r]; ++total; }
    return sz;
}

std::vector<ClassId> zipf_owner(uint32_t n, uint32_t c, double s, SplitMix64& shuffle) {
    std::vector<uint32_t> perm(n);
    for (uint32_t i = 0; i < n; ++i) perm[i] = i;
    for (uint32_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[shuffle.below(i)]);
    const std::vector<uint32_t> sz = zipf_sizes(n, c, s);
    std::vector<ClassId> owner(n);
    uint32_t at = 0;
    for (uint32_t r = 0; r < c; ++r)
        for (uint32_t k = 0; k < sz[r]; ++k) owner[perm[at++]] = r;
    return owner;
}

void generate_zipf(RefModel& r, const GeneratorConfig& cfg, double zs) {
    if (cfg.n_classes == 0) throw std::invalid_argument("generate: n_classes must be positive");
    SystemModel& model = r.model;
    model.classes.resize(cfg.n_classes);
    for (ClassId c = 0; c < cfg.n_classes; ++c) {
        model.classes[c].id = c;
        model.classes[c].name = "C" + std::to_string(c);
    }
    SplitMix64 shuffle(cfg.seed ^ 0x5a17f00dd15ea5e5ULL);
    model.method_owner = zipf_owner(cfg.n_methods, cfg.n_classes, zs, shuffle);
    model.attribute_owner = zipf_owner(cfg.n_attributes, cfg.n_classes, zs, shuffle);
    model.method_names.resize(cfg.n_methods);
    model.attribute_names.resize(cfg.n_attributes);
    for (MethodId p = 0; p < cfg.n_methods; ++p) model.classes[model.method_owner[p]].method_ids.push_back(p);
    for (AttributeId a = 0; a < cfg.n_attributes; ++a)
        model.classes[model.attribute_owner[a]].attribute_ids.push_back(a);
    SplitMix64 rng(cfg.seed);
    DependencyTable& deps = r.deps;
    deps.calls.assign(cfg.n_methods, {});
    deps.accesses.assign(cfg.n_methods, {});
    for (MethodId p = 0; p < cfg.n_methods; ++p) {
        const ClassId home = model.method_owner[p];
        const std::uint64_t n_calls = cfg.k_max_calls ? rng.below(cfg.k_max_calls + 1ULL) : 0;
        for (std::uint64_t i = 0; i < n_calls; ++i) {
            const bool stay = rng.unit() < cfg.intra_class_bias;
            std::uint32_t target;
            if (stay ? detail::pick_excluding(rng, model.classes[home].method_ids, p, target)
                     : detail::pick_foreign(rng, model.method_owner, home, target))
                deps.calls[p].push_back(target);
        }
        const std::uint64_t n_acc = cfg.k_max_accesses ? rng.below(cfg.k_max_accesses + 1ULL) : 0;
        for (std::uint64_t i = 0; i < n_acc; ++i) {
            const bool stay = rng.unit() < cfg.intra_class_bias;
            std::uint32_t target;
            if (stay) {
                const auto& pool = model.classes[home].attribute_ids;
                if (pool.empty()) continue;
                target = pool[rng.below(pool.size())];
            } else if (!detail::pick_foreign(rng, model.attribute_owner, home, target)) {
                continue;
            }
            deps.accesses[p].push_back(target);
        }
        auto& cs = deps.calls[p];
        std::sort(cs.begin(), cs.end());
        cs.erase(std::unique(cs.begin(), cs.end()), cs.end());
        auto& as = deps.accesses[p];
        std::sort(as.begin(), as.end());
        as.erase(std::unique(as.begin(), as.end()), as.end());
    }
}

}  // namespace

extern "C" {

void* ref_model_create(const mm_system* s) {
    RefModel* r = new RefModel();
    from_csr(*r, s);
    return r;
}

void ref_model_free(void* h) { delete static_cast<RefModel*>(h); }

int ref_validate(void* h) {
    const RefModel* r = static_cast<RefModel*>(h);
    return static_cast<int>(validate(r->model, r->deps).violations.size());
}

// reference generate() -> handle (its CSR view via ref_model_view)
void* ref_generate(const mm_gen_config* cfg) {
    GeneratorConfig g;
    g.seed = cfg->seed;
    g.n_classes = cfg->n_classes;
    g.n_methods = cfg->n_methods;
    g.n_attributes = cfg->n_attributes;
    g.k_max_calls = cfg->k_max_calls;
    g.k_max_accesses = cfg->k_max_accesses;
    g.intra_class_bias = cfg->intra_class_bias;
    RefModel* r = new RefModel();
    if (cfg->zipf_s > 0.0) {
        generate_zipf(*r, g, cfg->zipf_s);
    } else {
        GeneratedSystem gs = generate(g);
        r->model = std::move(gs.model);
        r->deps = std::move(gs.deps);
    }
    to_csr(*r);
    return r;
}

const mm_system* ref_model_view(void* h) { return &static_cast<RefModel*>(h)->view; }

// n_workers == 0: all_similarities (metrics.hpp:67-77); otherwise
// parallel_similarities (parallel.hpp:71-121). Two-call size query.
int ref_similarities(void* h, unsigned n_workers, mm_similarity* out, uint64_t cap, uint64_t* n_out) {
    const RefModel* r = static_cast<RefModel*>(h);
    try {
        const std::vector<SimilarityEntry> v =
            n_workers == 0 ? all_similarities(r->model, r->deps) : parallel_similarities(r->model, r->deps, n_workers);
        *n_out = v.size();
        if (!out) return MM_OK;
        if (cap < v.size()) return MM_E_CAPACITY;
        for (size_t k = 0; k < v.size(); ++k) {
            out[k].first = v[k].first;
            out[k].second = v[k].second;
            out[k].value = v[k].value;
        }
    } catch (...) {
        return status_of(std::current_exception());
    }
    return MM_OK;
}

// n_workers == 0: fan_in / fan_out (metrics.hpp:79-93); otherwise
// parallel_fan_metrics (parallel.hpp:186-206).
int ref_fan_metrics(void* h, unsigned n_workers, uint32_t* fan_in_out, uint32_t* fan_out_out) {
    const RefModel* r = static_cast<RefModel*>(h);
    try {
        FanMetrics f;
        if (n_workers == 0) {
            f.fan_in = fan_in(r->model, r->deps);
            f.fan_out = fan_out(r->model, r->deps);
        } else {
            f = parallel_fan_metrics(r->model, r->deps, n_workers);
        }
        for (size_t p = 0; p < f.fan_in.size(); ++p) {
            if (fan_in_out) fan_in_out[p] = f.fan_in[p];
            if (fan_out_out) fan_out_out[p] = f.fan_out[p];
        }
    } catch (...) {
        return status_of(std::current_exception());
    }
    return MM_OK;
}

// n_workers == 0: sequential full_report class loop (metrics.hpp:253-261);
// otherwise parallel_class_metrics + parallel_lcom_ck (parallel.hpp:149,164).
int ref_class_metrics(void* h, unsigned n_workers, double* lcom, uint64_t* ck, uint32_t* cbo) {
    const RefModel* r = static_cast<RefModel*>(h);
    const size_t C = r->model.class_count();
    try {
        if (n_workers == 0) {
            for (ClassId c = 0; c < C; ++c) {
                if (lcom) lcom[c] = lcom_normalized(c, r->model, r->deps);
                if (ck) ck[c] = lcom_ck(c, r->model, r->deps);
                if (cbo) cbo[c] = modmetrics::cbo(c, r->model, r->deps);
            }
        } else {
            const ClassMetrics cm = parallel_class_metrics(r->model, r->deps, n_workers);
            const std::vector<uint64_t> k = parallel_lcom_ck(r->model, r->deps, n_workers);
            for (size_t c = 0; c < C; ++c) {
                if (lcom) lcom[c] = cm.lcom[c];
                if (cbo) cbo[c] = cm.cbo[c];
                if (ck) ck[c] = k[c];
            }
        }
    } catch (...) {
        return status_of(std::current_exception());
    }
    return MM_OK;
}

int ref_single_metric(void* h, int which, uint32_t cls, double* dv, uint64_t* uv) {
    const RefModel* r = static_cast<RefModel*>(h);
    try {
        if (which == 0) *dv = lcom_normalized(cls, r->model, r->deps);
        else if (which == 1) *uv = lcom_ck(cls, r->model, r->deps);
        else *uv = modmetrics::cbo(cls, r->model, r->deps);
    } catch (...) {
        return status_of(std::current_exception());
    }
    return MM_OK;
}

int ref_thresholds(const double* lcom, const uint32_t* cbo, uint64_t n, const double* sim,
                   uint64_t n_sim, const mm_overrides* ov, mm_thresholds* out) {
    MetricsReport rep;
    rep.lcom.assign(lcom, lcom + n);
    rep.cbo.assign(cbo, cbo + n);
    for (uint64_t i = 0; i < n_sim; ++i) rep.similarity.push_back({0, 1, sim[i]});
    ThresholdOverrides o;
    if (ov && ov->has_similarity) o.similarity = ov->similarity;
    if (ov && ov->has_lcom) o.lcom = ov->lcom;
    if (ov && ov->has_cbo) o.cbo = ov->cbo;
    const Thresholds t = compute_thresholds(rep, o);
    std::memset(out, 0, sizeof *out);
    out->similarity = t.similarity;
    out->lcom = t.lcom;
    out->cbo = t.cbo;
    out->explicit_mode = t.explicit_mode;
    return MM_OK;
}

int ref_what_if(void* h, uint32_t u, uint32_t o, uint32_t d, mm_whatif* out) {
    const RefModel* r = static_cast<RefModel*>(h);
    try {
        const WhatIfMetrics w = what_if_move(u, o, d, r->model, r->deps);
        std::memset(out, 0, sizeof *out);
        out->lcom_origin_before = w.lcom_origin_before;
        out->lcom_origin_after = w.lcom_origin_after;
        out->lcom_dest_before = w.lcom_dest_before;
        out->lcom_dest_after = w.lcom_dest_after;
        out->cbo_origin_before = w.cbo_origin_before;
        out->cbo_origin_after = w.cbo_origin_after;
        out->cbo_dest_before = w.cbo_dest_before;
        out->cbo_dest_after = w.cbo_dest_after;
        out->origin_degenerate_after = w.origin_degenerate_after;
        out->dest_degenerate_after = w.dest_degenerate_after;
    } catch (...) {
        return status_of(std::current_exception());
    }
    return MM_OK;
}

// suggest_all (suggest.hpp:303) with gates from the given per-class vectors
// and thresholds from params. Similarity is rejected (needs the O(m²) table).
// out == NULL or too small -> MM_E_CAPACITY with *n_out set.
int ref_suggest(void* h, const double* lcom_gate, const uint32_t* cbo_gate,
                const mm_sweep_params* p, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    const RefModel* r = static_cast<RefModel*>(h);
    if (p->criteria & MM_CRIT_SIMILARITY) return MM_E_UNSUPPORTED;
    MetricsReport rep;
    rep.fan_in = fan_in(r->model, r->deps);
    rep.fan_out = fan_out(r->model, r->deps);
    rep.lcom.assign(lcom_gate, lcom_gate + r->model.class_count());
    rep.cbo.assign(cbo_gate, cbo_gate + r->model.class_count());
    Thresholds t;
    t.lcom = p->thr_lcom;
    t.cbo = p->thr_cbo;
    SuggestOptions opts;
    opts.all_candidates = p->all_candidates != 0;
    std::vector<MoveSuggestion> s;
    try {
        s = suggest_all(r->model, r->deps, rep, t, criteria_of(p->criteria),
                        p->combine == MM_COMBINE_INTERSECTION ? Combine::Intersection : Combine::Union,
                        opts);
    } catch (...) {
        return status_of(std::current_exception());
    }
    *n_out = s.size();
    if (!out || cap < s.size()) return s.empty() ? MM_OK : MM_E_CAPACITY;
    for (size_t i = 0; i < s.size(); ++i) fill(out[i], s[i]);
    return MM_OK;
}

// suggest_all with the similarity criterion available: the report's
// similarity table is the reference's all_similarities (O(m^2): small systems),
// thresholds.similarity = thr_sim.
int ref_suggest_full(void* h, const double* lcom_gate, const uint32_t* cbo_gate, const mm_sweep_params* p,
                     double thr_sim, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    const RefModel* r = static_cast<RefModel*>(h);
    MetricsReport rep;
    rep.fan_in = fan_in(r->model, r->deps);
    rep.fan_out = fan_out(r->model, r->deps);
    rep.similarity = all_similarities(r->model, r->deps);
    rep.lcom.assign(lcom_gate, lcom_gate + r->model.class_count());
    rep.cbo.assign(cbo_gate, cbo_gate + r->model.class_count());
    Thresholds t;
    t.similarity = thr_sim;
    t.lcom = p->thr_lcom;
    t.cbo = p->thr_cbo;
    SuggestOptions opts;
    opts.all_candidates = p->all_candidates != 0;
    std::vector<MoveSuggestion> s;
    try {
        s = suggest_all(r->model, r->deps, rep, t, criteria_of(p->criteria),
                        p->combine == MM_COMBINE_INTERSECTION ? Combine::Intersection : Combine::Union, opts);
    } catch (...) {
        return status_of(std::current_exception());
    }
    *n_out = s.size();
    if (!out || cap < s.size()) return s.empty() ? MM_OK : MM_E_CAPACITY;
    for (size_t i = 0; i < s.size(); ++i) fill(out[i], s[i]);
    return MM_OK;
}

// One criterion alone, in the reference's own emission order
// (suggest_by_cohesion :239 / suggest_by_coupling :266).
int ref_suggest_by(void* h, uint32_t crit, const double* lcom_gate, const uint32_t* cbo_gate,
                   const mm_sweep_params* p, mm_suggestion* out, uint64_t cap, uint64_t* n_out) {
    const RefModel* r = static_cast<RefModel*>(h);
    MetricsReport rep;
    rep.fan_in = fan_in(r->model, r->deps);
    rep.fan_out = fan_out(r->model, r->deps);
    rep.lcom.assign(lcom_gate, lcom_gate + r->model.class_count());
    rep.cbo.assign(cbo_gate, cbo_gate + r->model.class_count());
    Thresholds t;
    t.lcom = p->thr_lcom;
    t.cbo = p->thr_cbo;
    SuggestOptions opts;
    opts.all_candidates = p->all_candidates != 0;
    std::vector<MoveSuggestion> s;
    if (crit == MM_CRIT_COHESION) s = suggest_by_cohesion(r->model, r->deps, rep, t, opts);
    else if (crit == MM_CRIT_COUPLING) s = suggest_by_coupling(r->model, r->deps, rep, t, opts);
    else return MM_E_UNSUPPORTED;
    *n_out = s.size();
    if (!out || cap < s.size()) return s.empty() ? MM_OK : MM_E_CAPACITY;
    for (size_t i = 0; i < s.size(); ++i) fill(out[i], s[i]);
    return MM_OK;
}

// CPU baseline: the reference's cohesion+coupling sweep for origins in
// [class_begin, class_end), "reference logic, harness threads"
// (SURVEY.md §8d item 4): detail::used_classes + detail::emit_for_method +
// what_if_move with the reference's own predicates, classes split by the
// reference's detail::run_partitioned over n_workers std::threads. Returns
// suggestions emitted (per criterion, before merge) and candidates
// (Σ |used_classes(u)| over ALL swept methods, ungated).
int ref_sweep_sample(void* h, const double* lcom_gate, const uint32_t* cbo_gate, double thr_lcom,
                     double thr_cbo, uint32_t class_begin, uint32_t class_end, unsigned n_workers,
                     uint64_t* n_suggestions, uint64_t* n_candidates) {
    const RefModel* r = static_cast<RefModel*>(h);
    const SystemModel& model = r->model;
    const DependencyTable& deps = r->deps;
    std::vector<uint64_t> sugg(n_workers ? n_workers : 1, 0), cand(n_workers ? n_workers : 1, 0);
    const SuggestOptions opts;
    auto body = [&](unsigned w, size_t b, size_t e) {
        std::vector<MoveSuggestion> out;
        for (size_t c = class_begin + b; c < class_begin + e; ++c) {
            const bool coh = lcom_gate[c] > thr_lcom;
            const bool coup = static_cast<double>(cbo_gate[c]) > thr_cbo;
            for (MethodId u : model.classes[c].method_ids) {
                const std::vector<ClassId> dests =
                    detail::used_classes(u, static_cast<ClassId>(c), model, deps);
                cand[w] += dests.size();
                if (coh)
                    detail::emit_for_method(u, static_cast<ClassId>(c), dests, Criterion::Cohesion,
                                            detail::lcom_improves, detail::lcom_key, opts, model,
                                            deps, out);
                if (coup)
                    detail::emit_for_method(
                        u, static_cast<ClassId>(c), dests, Criterion::Coupling,
                        [](const WhatIfMetrics& wm) {
                            return wm.cbo_origin_after < wm.cbo_origin_before &&
                                   wm.cbo_dest_after <= wm.cbo_dest_before;
                        },
                        [](const WhatIfMetrics& wm) { return static_cast<double>(wm.cbo_dest_after); },
                        opts, model, deps, out);
            }
        }
        sugg[w] += out.size();
    };
    try {
        detail::run_partitioned(class_end - class_begin, n_workers ? n_workers : 1, body);
    } catch (...) {
        return status_of(std::current_exception());
    }
    *n_suggestions = 0;
    *n_candidates = 0;
    for (size_t i = 0; i < sugg.size(); ++i) {
        *n_suggestions += sugg[i];
        *n_candidates += cand[i];
    }
    return MM_OK;
}

// The reference's cohesion/coupling sweep restricted to a method subset,
// records in suggest_all's order — "reference logic, harness threads"
// (SURVEY.md §8d item 4), for the parity tests at the BASELINE sizes and the
// CPU arm. Per method, exactly suggest_by_cohesion / suggest_by_coupling's
// body (suggest.hpp:239-294): class gate, detail::used_classes,
// detail::emit_for_method with detail::lcom_improves / lcom_key or the
// coupling pass/key, which run the reference's what_if_move. Then
// suggest_all's merge (suggest.hpp:315-348): keyed by (method, destination),
// the first criterion's record kept and later criteria appended, sort-unique
// of the tags, intersection filter, sort by (origin, method, destination).
// Per-method work is independent given the report and thresholds, so any
// subset and any thread split give suggest_all's list restricted to that
// subset. methods == NULL: every method. dynamic != 0: methods handed out in
// small chunks from an atomic counter (Zipf giants); else the reference's
// detail::run_partitioned contiguous ranges. *n_candidates = Σ
// |used_classes(u)| over the swept methods (ungated). Result kept in the
// model handle (ref_sweep_copy).
int ref_sweep(void* h, const double* lcom_gate, const uint32_t* cbo_gate, const mm_sweep_params* p,
              const uint32_t* methods, uint64_t n_methods, unsigned n_workers, int dynamic, uint64_t* n_records,
              uint64_t* n_candidates) {
    RefModel* r = static_cast<RefModel*>(h);
    const SystemModel& model = r->model;
    const DependencyTable& deps = r->deps;
    const uint64_t n = methods ? n_methods : model.method_owner.size();
    const unsigned W = n_workers ? n_workers : 1;
    const bool want_coh = p->criteria & MM_CRIT_COHESION, want_coup = p->criteria & MM_CRIT_COUPLING;
    if (!want_coh && !want_coup) return MM_E_ARG;
    if (p->criteria & MM_CRIT_SIMILARITY) return MM_E_UNSUPPORTED;
    SuggestOptions opts;
    opts.all_candidates = p->all_candidates != 0;
    struct Part {
        std::vector<MoveSuggestion> coh, coup;
        uint64_t cand = 0;
    };
    std::vector<Part> parts(W);
    auto one = [&](Part& pt, MethodId u) {
        const ClassId c = model.method_owner[u];
        const std::vector<ClassId> dests = detail::used_classes(u, c, model, deps);
        pt.cand += dests.size();
        if (want_coh && lcom_gate[c] > p->thr_lcom)
            detail::emit_for_method(u, c, dests, Criterion::Cohesion, detail::lcom_improves, detail::lcom_key, opts,
                                    model, deps, pt.coh);
        if (want_coup && static_cast<double>(cbo_gate[c]) > p->thr_cbo)
            detail::emit_for_method(
                u, c, dests, Criterion::Coupling,
                [](const WhatIfMetrics& wm) {
                    return wm.cbo_origin_after < wm.cbo_origin_before && wm.cbo_dest_after <= wm.cbo_dest_before;
                },
                [](const WhatIfMetrics& wm) { return static_cast<double>(wm.cbo_dest_after); }, opts, model, deps,
                pt.coup);
    };
    auto mid = [&](uint64_t i) -> MethodId { return methods ? methods[i] : static_cast<MethodId>(i); };
    try {
        if (dynamic) {
            std::atomic<uint64_t> next{0};
            const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(64, n / (16ull * W)));
            std::vector<std::thread> th;
            for (unsigned w = 0; w < W; ++w)
                th.emplace_back([&, w] {
                    for (;;) {
                        const uint64_t b = next.fetch_add(chunk);
                        if (b >= n) break;
                        for (uint64_t i = b; i < std::min<uint64_t>(n, b + chunk); ++i) one(parts[w], mid(i));
                    }
                });
            for (std::thread& t : th) t.join();
        } else {
            detail::run_partitioned(n, W, [&](unsigned w, size_t b, size_t e) {
                for (size_t i = b; i < e; ++i) one(parts[w], mid(i));
            });
        }
    } catch (...) {
        return status_of(std::current_exception());
    }
    // suggest_all's merge, criteria in ascending order (Cohesion < Coupling)
    std::map<std::pair<MethodId, ClassId>, MoveSuggestion> merged;
    uint64_t cand = 0;
    for (Part& pt : parts) cand += pt.cand;
    for (int pass = 0; pass < 2; ++pass)
        for (Part& pt : parts)
            for (MoveSuggestion& s : pass == 0 ? pt.coh : pt.coup) {
                const Criterion crit = s.criteria.front();
                const auto key = std::make_pair(s.method, s.destination);
                auto [it, inserted] = merged.try_emplace(key, std::move(s));
                if (!inserted) it->second.criteria.push_back(crit);
            }
    const size_t n_sel = (want_coh ? 1 : 0) + (want_coup ? 1 : 0);
    std::vector<MoveSuggestion> out;
    out.reserve(merged.size());
    for (auto& [key, s] : merged) {
        std::sort(s.criteria.begin(), s.criteria.end());
        s.criteria.erase(std::unique(s.criteria.begin(), s.criteria.end()), s.criteria.end());
        if (p->combine == MM_COMBINE_INTERSECTION && s.criteria.size() != n_sel) continue;
        out.push_back(std::move(s));
    }
    std::sort(out.begin(), out.end(), [](const MoveSuggestion& a, const MoveSuggestion& b) {
        if (a.origin != b.origin) return a.origin < b.origin;
        if (a.method != b.method) return a.method < b.method;
        return a.destination < b.destination;
    });
    r->last.resize(out.size());
    for (size_t i = 0; i < out.size(); ++i) fill(r->last[i], out[i]);
    *n_records = out.size();
    *n_candidates = cand;
    return MM_OK;
}

int ref_sweep_copy(void* h, mm_suggestion* out, uint64_t cap) {
    RefModel* r = static_cast<RefModel*>(h);
    if (cap < r->last.size()) return MM_E_CAPACITY;
    std::memcpy(out, r->last.data(), r->last.size() * sizeof(mm_suggestion));
    return MM_OK;
}

// N_cand = Σ_u |used_classes(u)| with the reference's own
// detail::used_classes.
uint64_t ref_candidates(void* h) {
    const RefModel* r = static_cast<RefModel*>(h);
    uint64_t n = 0;
    for (MethodId u = 0; u < r->model.method_owner.size(); ++u)
        n += detail::used_classes(u, r->model.method_owner[u], r->model, r->deps).size();
    return n;
}

}  // extern "C"
