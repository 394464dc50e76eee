// modmetrics/gpu_facts.hpp — facts ingest straight to the engine's CSR.
//
//   reference (namespace modmetrics)   here (namespace modmetrics::gpu)
//   parse_facts    facts.hpp:91        parse_facts  (same LoadResult, same exceptions + messages)
//   load_facts     facts.hpp:258       load_facts
//   facts_to_json  facts.hpp:270       Facts::to_json (canonical bytes from the CSR)
//
// gpu::Facts keeps the parse as CSR (mmfacts.h) and uploads it without ever
// building the reference's vector-of-vectors; parse_facts/load_facts build the
// reference's LoadResult from it for callers that want the reference types.
// Needs the reference's facts.hpp (and so nlohmann/json.hpp) on the include
// path only for the exception and LoadResult types.
#pragma once

#include <memory>
#include <string>
#include <string_view>
#include <exception>
#include <thread>
#include <utility>
#include <vector>

#include <modmetrics/facts.hpp>

#include "../mmfacts.h"
#include "gpu.hpp"

namespace modmetrics::gpu {

class Facts {
public:
    static Facts parse(std::string_view text) {
        mm_facts* f = nullptr;
        const mm_status st = mm_facts_parse(text.data(), text.size(), &f);
        return Facts(f, st);
    }
    static Facts load(const std::string& path) {
        mm_facts* f = nullptr;
        const mm_status st = mm_facts_load(path.c_str(), &f);
        return Facts(f, st);
    }

    const mm_system& system() const { return sys_; }

    std::vector<std::string> warnings() const {
        std::vector<std::string> w;
        const uint32_t n = mm_facts_warning_count(f_.get());
        w.reserve(n);
        for (uint32_t i = 0; i < n; ++i) w.emplace_back(mm_facts_warning(f_.get(), i));
        return w;
    }

    // The reference's LoadResult (facts.hpp:43-47), field for field.
    LoadResult to_load_result() const {
        LoadResult r;
        SystemModel& m = r.model;
        const mm_system& s = sys_;
        m.classes.resize(s.n_classes);
        for (uint32_t c = 0; c < s.n_classes; ++c) {
            ClassRecord& rec = m.classes[c];
            rec.id = c;
            size_t len = 0;
            const char* nm = mm_facts_class_name(f_.get(), c, &len);
            rec.name.assign(nm, len);
            rec.method_ids.assign(s.class_methods + s.class_method_off[c], s.class_methods + s.class_method_off[c + 1]);
            rec.attribute_ids.assign(s.class_attrs + s.class_attr_off[c], s.class_attrs + s.class_attr_off[c + 1]);
        }
        m.method_owner.assign(s.method_owner, s.method_owner + s.n_methods);
        m.attribute_owner.assign(s.attribute_owner, s.attribute_owner + s.n_attributes);
        m.method_names.resize(s.n_methods);
        m.attribute_names.resize(s.n_attributes);
        r.deps.calls.resize(s.n_methods);
        r.deps.accesses.resize(s.n_methods);
        // every index is written by one thread only
        for_ranges(s.n_methods, [&](uint32_t b, uint32_t e) {
            for (uint32_t p = b; p < e; ++p) {
                size_t len = 0;
                const char* nm = mm_facts_method_name(f_.get(), p, &len);
                m.method_names[p].assign(nm, len);
                r.deps.calls[p].assign(s.call_tgt + s.call_off[p], s.call_tgt + s.call_off[p + 1]);
                r.deps.accesses[p].assign(s.acc_tgt + s.acc_off[p], s.acc_tgt + s.acc_off[p + 1]);
            }
        });
        for_ranges(s.n_attributes, [&](uint32_t b, uint32_t e) {
            for (uint32_t a = b; a < e; ++a) {
                size_t len = 0;
                const char* nm = mm_facts_attribute_name(f_.get(), a, &len);
                m.attribute_names[a].assign(nm, len);
            }
        });
        r.warnings = warnings();
        return r;
    }

    std::string to_json() const {
        size_t n = 0;
        mm_facts_to_json(f_.get(), nullptr, 0, &n);
        std::string out(n, '\0');
        const mm_status st = mm_facts_to_json(f_.get(), out.data(), out.size(), &n);
        if (st != MM_OK) throw std::runtime_error("mm_facts_to_json failed");
        return out;
    }

private:
    template <class Fn>
    static void for_ranges(uint32_t n, Fn&& fn) {
        const unsigned hw = std::thread::hardware_concurrency();
        const uint32_t T = n >= (1u << 16) ? std::min(8u, hw ? hw : 1u) : 1u;
        if (T <= 1) { fn(0u, n); return; }
        // exceptions (e.g. bad_alloc from a worker's assign) are carried back
        // and rethrown after every started thread joined, as the reference's
        // single-threaded walk would throw them to the caller
        std::vector<std::exception_ptr> errs(T);
        std::vector<std::thread> th;
        th.reserve(T);
        std::exception_ptr spawn_err;
        for (uint32_t k = 0; k < T && !spawn_err; ++k) {
            try {
                th.emplace_back([&, k] {
                    try {
                        fn(uint32_t(uint64_t(n) * k / T), uint32_t(uint64_t(n) * (k + 1) / T));
                    } catch (...) {
                        errs[k] = std::current_exception();
                    }
                });
            } catch (...) {
                spawn_err = std::current_exception();
            }
        }
        for (std::thread& t : th) t.join();
        if (spawn_err) std::rethrow_exception(spawn_err);
        for (const std::exception_ptr& e : errs)
            if (e) std::rethrow_exception(e);
    }

    struct Del {
        void operator()(mm_facts* f) const { mm_facts_free(f); }
    };
    std::unique_ptr<mm_facts, Del> f_;
    mm_system sys_{};

    Facts(mm_facts* f, mm_status st) : f_(f) {
        if (st == MM_OK) {
            mm_facts_system(f, &sys_);
            return;
        }
        const std::string msg = f ? mm_facts_error(f) : "facts: invalid argument";
        switch (st) {
            case MM_E_PARSE: throw ParseError(msg);
            case MM_E_IO: throw IoError(msg);
            case MM_E_VALIDATION: {
                std::vector<Violation> v;
                const uint32_t n = mm_facts_violation_count(f);
                for (uint32_t i = 0; i < n; ++i) {
                    int kind = 0;
                    const char* m = nullptr;
                    mm_facts_violation(f, i, &kind, &m);
                    v.push_back({static_cast<ViolationKind>(kind), m});
                }
                throw ValidationError(msg, std::move(v));
            }
            case MM_E_RANGE:  // a float token that overflows a double (what nlohmann throws, unwrapped)
                throw nlohmann::json::out_of_range::create(406, msg, nullptr);
            case MM_E_OOM: throw std::bad_alloc();
            default: throw std::invalid_argument(msg);
        }
    }
};

inline LoadResult parse_facts(std::string_view text) { return Facts::parse(text).to_load_result(); }

inline LoadResult load_facts(const std::string& path) { return Facts::load(path).to_load_result(); }

}  // namespace modmetrics::gpu
