// mmgpu — the reference's command line front end with the B200 engine behind
// `--engine gpu`.
//
// Same subcommands, options, outputs and exit codes as the reference CLI
// (/root/reference/proj/tools/modmetrics.cpp:1-346) for the paths it shares:
// analyze, suggest, validate, generate (bench is the repo's bench.py). The
// reference's dispatch point is compute_report (modmetrics.cpp:82-86); here it
// gains a third engine:
//
//   --engine gpu        (default) facts -> CSR in one streaming pass
//                       (gpu_facts.hpp), uploaded as-is; full_report and
//                       suggest_all on the device (gpu.hpp)
//   --engine sequential the reference's full_report / suggest_all
//   --engine parallel   the reference's parallel_full_report
//
// Output bytes come from the reference's own renderers (report_io.hpp), so a
// gpu run and a sequential run print identical bytes (tests/test_cli.py).
// CLI11 is not available in this image, so options are parsed by hand with
// the same names, defaults and checks; a usage error exits 64.
//
// Build: tools/Makefile (needs the reference headers, like every user of the
// drop-in headers: the north star keeps proj/include as the API surface).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <fstream>
#include <iostream>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include <modmetrics/modmetrics.hpp>
#include <modmetrics/gpu.hpp>
#include <modmetrics/gpu_facts.hpp>

namespace {

using namespace modmetrics;

constexpr int kExitOk = 0, kExitParse = 2, kExitValidation = 3, kExitIo = 4, kExitUsage = 64;

// MMGPU_CLI_TIMING=1: phase times on stderr (wall clock, host side)
struct Phase {
    const char* name;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    explicit Phase(const char* n) : name(n) {}
    ~Phase() {
        static const bool on = std::getenv("MMGPU_CLI_TIMING") != nullptr;
        if (on)
            std::fprintf(stderr, "timing %-14s %9.3f ms\n", name,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    }
};

struct Usage : std::runtime_error {
    using std::runtime_error::runtime_error;
};

unsigned default_workers() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : hw;
}

struct RunConfig {
    std::string facts_path, out_path;
    std::string engine = "gpu";
    unsigned workers = default_workers();
    std::string format = "json";
    std::vector<std::string> criteria;
    std::string combine = "union";
    std::optional<double> thr_similarity, thr_lcom, thr_cbo;
    bool all_candidates = false;
    int device = 0;
};

// modmetrics.cpp:61-75
void write_output(const std::string& out_path, const std::string& bytes) {
    if (out_path.empty()) {
        if (std::fwrite(bytes.data(), 1, bytes.size(), stdout) != bytes.size()) throw IoError("write error on stdout");
        std::fflush(stdout);
        return;
    }
    std::ofstream out(out_path, std::ios::binary | std::ios::trunc);
    if (!out) throw IoError("cannot open " + out_path + " for writing");
    out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
    out.flush();
    if (!out) throw IoError("write error on " + out_path);
}

void print_warnings(const std::vector<std::string>& warnings) {
    for (const std::string& w : warnings) std::cerr << "warning: " << w << "\n";
}

std::vector<Criterion> parse_criteria(const std::vector<std::string>& names) {  // modmetrics.cpp:97-107
    if (names.empty()) return {Criterion::Similarity, Criterion::Cohesion, Criterion::Coupling};
    std::vector<Criterion> out;
    for (const std::string& n : names) {
        if (n == "similarity") out.push_back(Criterion::Similarity);
        else if (n == "cohesion") out.push_back(Criterion::Cohesion);
        else if (n == "coupling") out.push_back(Criterion::Coupling);
    }
    return out;
}

// The loaded system and its report from the selected engine.
struct Analysis {
    LoadResult loaded;
    MetricsReport report;
    std::optional<gpu::Engine> engine;  // kept resident for the sweep
};

Analysis analyze_facts(const RunConfig& cfg) {
    Analysis a;
    if (cfg.engine == "gpu") {
        // CUDA context creation (≈ 1-2 s on a fresh process) overlaps the
        // facts load; a facts error still wins, as in the reference's order
        std::exception_ptr ctx_err;
        std::thread init([&] {
            try {
                Phase p("ctx_create");
                a.engine.emplace(cfg.device);
            } catch (...) {
                ctx_err = std::current_exception();
            }
        });
        std::optional<gpu::Facts> facts;
        try {
            Phase p("load_facts");
            facts.emplace(gpu::Facts::load(cfg.facts_path));
        } catch (...) {
            init.join();
            throw;
        }
        {
            Phase p("ctx_wait");
            init.join();
        }
        if (ctx_err) std::rethrow_exception(ctx_err);
        { Phase p("upload"); a.engine->upload(facts->system()); }  // CSR straight from the parse
        { Phase p("load_result"); a.loaded = facts->to_load_result(); }  // names and records for the renderers
        print_warnings(a.loaded.warnings);
        { Phase p("full_report"); a.report = a.engine->full_report(); }
        return a;
    }
    a.loaded = load_facts(cfg.facts_path);
    print_warnings(a.loaded.warnings);
    a.report = cfg.engine == "parallel" ? parallel_full_report(a.loaded.model, a.loaded.deps, cfg.workers)
                                        : full_report(a.loaded.model, a.loaded.deps);
    return a;
}

int cmd_analyze(const RunConfig& cfg) {  // modmetrics.cpp:88-95
    const Analysis a = analyze_facts(cfg);
    Phase p("render+write");
    write_output(cfg.out_path, cfg.format == "text" ? render_report_text(a.loaded.model, a.report)
                                                    : render_report_json(a.loaded.model, a.report));
    return kExitOk;
}

int cmd_suggest(const RunConfig& cfg) {  // modmetrics.cpp:109-131
    Analysis a = analyze_facts(cfg);
    ThresholdOverrides overrides;
    overrides.similarity = cfg.thr_similarity;
    overrides.lcom = cfg.thr_lcom;
    overrides.cbo = cfg.thr_cbo;
    const Thresholds thresholds = compute_thresholds(a.report, overrides);
    const Combine combine = cfg.combine == "intersection" ? Combine::Intersection : Combine::Union;
    SuggestOptions opts;
    opts.all_candidates = cfg.all_candidates;
    const std::vector<Criterion> criteria = parse_criteria(cfg.criteria);
    std::vector<MoveSuggestion> suggestions;
    {
        Phase p("suggest_all");
        suggestions = a.engine ? a.engine->suggest_all(a.report, thresholds, criteria, combine, opts)
                               : suggest_all(a.loaded.model, a.loaded.deps, a.report, thresholds, criteria, combine, opts);
    }
    Phase p("render+write");
    write_output(cfg.out_path, cfg.format == "text" ? render_suggestions_text(a.loaded.model, suggestions, thresholds)
                                                    : render_suggestions_json(a.loaded.model, suggestions, thresholds));
    return kExitOk;
}

int cmd_validate(const std::string& facts_path) {  // modmetrics.cpp:133-141
    const gpu::Facts facts = gpu::Facts::load(facts_path);  // throws on any violation
    print_warnings(facts.warnings());
    const mm_system& s = facts.system();
    write_output("", "ok: " + std::to_string(s.n_classes) + " classes, " + std::to_string(s.n_methods) +
                         " methods, " + std::to_string(s.n_attributes) + " attributes\n");
    return kExitOk;
}

// ---- option parsing (the reference uses CLI11; same names and checks) ----
struct Args {
    std::vector<std::string> v;
    size_t i = 0;
    bool more() const { return i < v.size(); }
    std::string value(const std::string& opt) {
        if (i >= v.size()) throw Usage(opt + ": 1 required argument missing");
        return v[i++];
    }
};

double number(const std::string& opt, const std::string& s, bool non_negative) {
    char* end = nullptr;
    const double d = std::strtod(s.c_str(), &end);
    if (s.empty() || *end) throw Usage(opt + ": value " + s + " is not a number");
    if (non_negative && d < 0) throw Usage(opt + ": value " + s + " not in range [0 - inf]");
    return d;
}

unsigned long long integer(const std::string& opt, const std::string& s, bool positive) {
    char* end = nullptr;
    const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
    if (s.empty() || *end || s[0] == '-') throw Usage(opt + ": value " + s + " is not a non-negative integer");
    if (positive && v == 0) throw Usage(opt + ": value " + s + " not in range [1 - inf]");
    return v;
}

void member(const std::string& opt, const std::string& v, std::initializer_list<const char*> allowed) {
    for (const char* a : allowed)
        if (v == a) return;
    throw Usage(opt + ": " + v + " not in the allowed set");
}

int run(int argc, char** argv) {
    if (argc < 2) throw Usage("A subcommand is required (analyze, suggest, generate, validate)");
    const std::string cmd = argv[1];
    Args a;
    for (int k = 2; k < argc; ++k) a.v.emplace_back(argv[k]);

    if (cmd == "analyze" || cmd == "suggest") {
        RunConfig cfg;
        const bool sug = cmd == "suggest";
        while (a.more()) {
            const std::string o = a.v[a.i++];
            if (o == "--facts") cfg.facts_path = a.value(o);
            else if (o == "--out") cfg.out_path = a.value(o);
            else if (o == "--engine") { cfg.engine = a.value(o); member(o, cfg.engine, {"gpu", "sequential", "parallel"}); }
            else if (o == "--device") cfg.device = int(integer(o, a.value(o), false));
            else if (o == "--workers") cfg.workers = unsigned(integer(o, a.value(o), true));
            else if (o == "--format") { cfg.format = a.value(o); member(o, cfg.format, {"json", "text"}); }
            else if (sug && o == "--criteria") {
                std::string list = a.value(o);
                size_t b = 0;
                for (;;) {
                    const size_t e = list.find(',', b);
                    const std::string item = list.substr(b, e == std::string::npos ? std::string::npos : e - b);
                    member(o, item, {"similarity", "cohesion", "coupling"});
                    cfg.criteria.push_back(item);
                    if (e == std::string::npos) break;
                    b = e + 1;
                }
            } else if (sug && o == "--combine") { cfg.combine = a.value(o); member(o, cfg.combine, {"union", "intersection"}); }
            else if (sug && o == "--threshold-similarity") cfg.thr_similarity = number(o, a.value(o), true);
            else if (sug && o == "--threshold-lcom") cfg.thr_lcom = number(o, a.value(o), true);
            else if (sug && o == "--threshold-cbo") cfg.thr_cbo = number(o, a.value(o), true);
            else if (sug && o == "--all-candidates") cfg.all_candidates = true;
            else throw Usage("The following argument was not expected: " + o);
        }
        if (cfg.facts_path.empty()) throw Usage("--facts is required");
        return sug ? cmd_suggest(cfg) : cmd_analyze(cfg);
    }
    if (cmd == "validate") {
        std::string path;
        while (a.more()) {
            const std::string o = a.v[a.i++];
            if (o == "--facts") path = a.value(o);
            else throw Usage("The following argument was not expected: " + o);
        }
        if (path.empty()) throw Usage("--facts is required");
        return cmd_validate(path);
    }
    if (cmd == "generate") {  // modmetrics.cpp:143-147, defaults :263-265
        GeneratorConfig gen;
        gen.k_max_calls = 4;
        gen.k_max_accesses = 4;
        std::string out;
        bool have_c = false, have_m = false;
        while (a.more()) {
            const std::string o = a.v[a.i++];
            if (o == "--classes") { gen.n_classes = uint32_t(integer(o, a.value(o), true)); have_c = true; }
            else if (o == "--methods") { gen.n_methods = uint32_t(integer(o, a.value(o), false)); have_m = true; }
            else if (o == "--attributes") gen.n_attributes = uint32_t(integer(o, a.value(o), false));
            else if (o == "--kmax-calls") gen.k_max_calls = uint32_t(integer(o, a.value(o), false));
            else if (o == "--kmax-accesses") gen.k_max_accesses = uint32_t(integer(o, a.value(o), false));
            else if (o == "--intra-bias") {
                gen.intra_class_bias = number(o, a.value(o), true);
                if (gen.intra_class_bias > 1.0) throw Usage(o + ": value not in range [0 - 1]");
            } else if (o == "--seed") gen.seed = integer(o, a.value(o), false);
            else if (o == "--out") out = a.value(o);
            else throw Usage("The following argument was not expected: " + o);
        }
        if (!have_c || !have_m || out.empty()) throw Usage("--classes, --methods and --out are required");
        const GeneratedSystem g = generate(gen);
        write_output(out, facts_to_json(g.model, g.deps));
        return kExitOk;
    }
    throw Usage("The following argument was not expected: " + cmd);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        return run(argc, argv);
    } catch (const Usage& e) {
        std::cerr << e.what() << "\nRun with a subcommand: analyze | suggest | generate | validate\n";
        return kExitUsage;
    } catch (const ParseError& e) {  // modmetrics.cpp:331-345
        std::cerr << "error: " << e.what() << "\n";
        return kExitParse;
    } catch (const ValidationError& e) {
        std::cerr << "error: " << e.what() << "\n";
        for (const Violation& v : e.violations()) std::cerr << "  - " << v.message << "\n";
        return kExitValidation;
    } catch (const IoError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitIo;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
