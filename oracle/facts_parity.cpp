// facts_parity.cpp — facts ingest: the reference's parse_facts against the
// engine's streaming CSR reader (include/modmetrics/gpu_facts.hpp, mmfacts.h).
//
// TEST INFRASTRUCTURE. Built by oracle/Makefile from the UNMODIFIED reference
// headers (facts.hpp needs nlohmann/json.hpp, found in the venv) and linked
// against libmmgpu.so; host-only (no device needed). Run by
// tests/test_facts.py. For every document both sides must agree on the
// outcome: on success LoadResult field for field (model ==, deps ==,
// warnings ==) and facts_to_json bytes; on failure the exception TYPE, what()
// verbatim and, for ValidationError, the violations list (kind + message).
//
// Cases: the reference's own test_facts.cpp documents (restated), generated
// systems through the canonical writer, key-shuffled / re-spaced / escaped
// variants, and a seeded mutation fuzz (byte deletes, inserts, replaces,
// truncations) over small documents, which exercises the JSON-error
// line/column path. `--bench` times both parsers on a C4-sized document.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <modmetrics/facts.hpp>
#include <modmetrics/generate.hpp>
#include <modmetrics/gpu_facts.hpp>

using namespace modmetrics;

static int g_fail = 0, g_checks = 0;

struct Outcome {
    std::string type = "none";
    std::string what;
    std::vector<Violation> violations;
    LoadResult r;
};

template <class F>
static Outcome run(F f) {
    Outcome o;
    try {
        o.r = f();
    } catch (const ValidationError& e) {
        o.type = "ValidationError"; o.what = e.what(); o.violations = e.violations();
    } catch (const ParseError& e) {
        o.type = "ParseError"; o.what = e.what();
    } catch (const IoError& e) {
        o.type = "IoError"; o.what = e.what();
    } catch (const nlohmann::json::out_of_range& e) {
        o.type = "json::out_of_range"; o.what = e.what();
    } catch (const std::bad_alloc&) {
        o.type = "bad_alloc";
    } catch (const std::length_error&) {
        o.type = "bad_alloc";  // vector::resize past max_size on absurd ids
    } catch (const std::exception& e) {
        o.type = "other"; o.what = e.what();
    }
    return o;
}

static bool same(const Outcome& a, const Outcome& b, std::string& why) {
    if (a.type != b.type) { why = "type " + a.type + " vs " + b.type + " (" + a.what + " | " + b.what + ")"; return false; }
    if (a.what != b.what) { why = "what '" + a.what + "' vs '" + b.what + "'"; return false; }
    if (!(a.violations == b.violations)) { why = "violations differ"; return false; }
    if (a.type != "none") return true;
    if (!(a.r.model == b.r.model)) { why = "model differs"; return false; }
    if (!(a.r.deps == b.r.deps)) { why = "deps differ"; return false; }
    if (a.r.warnings != b.r.warnings) { why = "warnings differ"; return false; }
    return true;
}

static void check_doc(const std::string& doc, const std::string& label, bool verbose_fail = true) {
    ++g_checks;
    if (std::getenv("FP_TRACE")) std::fprintf(stderr, "%s\n", label.c_str());
    const Outcome ref = run([&] { return parse_facts(doc); });
    const Outcome gpu = run([&] { return gpu::parse_facts(doc); });
    std::string why;
    bool ok = same(ref, gpu, why);
    if (ok && ref.type == "none") {
        // canonical writer bytes
        const std::string want = facts_to_json(ref.r.model, ref.r.deps);
        const std::string got = gpu::Facts::parse(doc).to_json();
        if (want != got) { ok = false; why = "facts_to_json bytes differ"; }
    }
    if (!ok) {
        ++g_fail;
        if (verbose_fail && g_fail <= 25) {
            std::string shown = doc.size() > 300 ? doc.substr(0, 300) + "..." : doc;
            std::printf("FAIL %s: %s\n  doc: %s\n", label.c_str(), why.c_str(), shown.c_str());
        }
    }
}

static const char* kMinimal = R"({
  "schema_version": "1",
  "classes": [
    {"id": 0, "name": "A",
     "attributes": [{"id": 0, "name": "x"}],
     "methods": [{"id": 0, "name": "f", "calls": [1], "accesses": [0]},
                 {"id": 1, "name": "g", "calls": [], "accesses": []}]}
  ]
})";

static std::vector<std::string> handwritten() {
    return {
        kMinimal,
        "{\n  \"schema_version\": \"1\",\n  !\n}",
        "[1,2]",
        R"({"classes": []})",
        R"({"schema_version": "1", "classes": 3})",
        R"({"schema_version": "1", "classes": [{"id": -1, "name": "A", "attributes": [], "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [],
             "methods": [{"id": 0, "name": "f", "calls": [0.5], "accesses": []}]}]})",
        R"({"schema_version": "2", "classes": []})",
        R"({"schema_version": 2, "classes": []})",
        R"({"schema_version": null, "classes": []})",
        R"({"schema_version": "1", "classes": [
            {"id": 0, "name": "A", "attributes": [], "methods": [{"id": 3, "name": "f", "calls": [], "accesses": []}]},
            {"id": 1, "name": "B", "attributes": [], "methods": [{"id": 3, "name": "g", "calls": [], "accesses": []}]}]})",
        R"({"schema_version": "1", "classes": [
            {"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f", "calls": [12], "accesses": []}]}]})",
        R"({"schema_version": "1", "classes": [
            {"id": 0, "name": "A", "attributes": [], "methods": [{"id": 1, "name": "f", "calls": [], "accesses": []}]}]})",
        R"({"schema_version": "1", "classes": [
            {"id": 0, "name": "A", "attributes": [],
             "methods": [{"id": 0, "name": "f", "calls": [0, 1, 0], "accesses": []},
                         {"id": 1, "name": "g", "calls": [], "accesses": []}]}]})",
        R"({"schema_version": "1", "classes": [
            {"id": 0, "name": "A", "attributes": [{"id": 0, "name": "x"}],
             "methods": [{"id": 0, "name": "f", "calls": [1, 1, 1], "accesses": [0, 0]},
                         {"id": 1, "name": "g", "calls": [], "accesses": []}]}]})",
        // shuffled keys (test_facts.cpp:158-179)
        R"({"classes": [{"methods": [{"name": "g", "accesses": [], "id": 1, "calls": []},
                                     {"calls": [1], "accesses": [0], "id": 0, "name": "f"}],
                         "name": "A", "id": 0, "attributes": [{"name": "x", "id": 0}]}],
            "schema_version": "1"})",
        // duplicate keys: last wins
        R"({"schema_version": "2", "schema_version": "1", "classes": [], "classes": [
            {"id": 5, "id": 0, "name": 1, "name": "A", "attributes": 3, "attributes": [],
             "methods": [{"id": 0, "name": "f", "calls": [7], "calls": [], "accesses": []}]}]})",
        // unknown keys, nested junk, escapes and unicode in names
        R"({"x": {"y": [1, 2.5e3, true, false, null, {"z": "w"}]}, "schema_version": "1", "classes": [
            {"id": 0, "name": "A\u00e9\ud83d\ude00\n\"q\"\t\\", "doc": [[], {}], "attributes": [{"id": 0, "name": "\u0001x/\/"}],
             "methods": [{"id": 0, "name": "ü€", "calls": [], "accesses": [0], "extra": -1}]}]})",
        // shape errors at every level
        R"({"schema_version": "1", "classes": [1]})",
        R"({"schema_version": "1", "classes": [{"name": "A", "attributes": [], "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "attributes": [], "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": 3, "attributes": [], "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": {}, "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [7], "methods": 1}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [{"name": "x"}], "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [{"id": 4294967296, "name": "x"}], "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [{"id": 0}], "methods": []}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f"}]}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f", "calls": []}]}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f", "calls": {}, "accesses": []}]}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f", "calls": [], "accesses": ["a"]}]}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f", "calls": [-0], "accesses": []}]}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f", "calls": [18446744073709551616], "accesses": []}]}]})",
        R"({"schema_version": "1", "classes": [{"id": 0, "name": "A", "attributes": [], "methods": [{"id": 0, "name": "f", "calls": [1e0], "accesses": []}]}]})",
        // violations of every kind at once, order matters
        R"({"schema_version": "3", "classes": [
            {"id": 1, "name": "A", "attributes": [{"id": 2, "name": "x"}, {"id": 2, "name": "y"}],
             "methods": [{"id": 0, "name": "f", "calls": [9, 0, 4], "accesses": [7, 2]},
                         {"id": 0, "name": "g", "calls": [99], "accesses": []},
                         {"id": 4, "name": "h", "calls": [], "accesses": [5]}]}]})",
        // a duplicate method's bad calls are never looked at (not pending)
        R"({"schema_version": "1", "classes": [
            {"id": 0, "name": "A", "attributes": [],
             "methods": [{"id": 0, "name": "f", "calls": [], "accesses": []},
                         {"id": 0, "name": "g", "calls": "bad", "accesses": []}]}]})",
        // JSON syntax errors
        "", " ", "{", "{\"a\"", "{\"a\":", "{\"a\":1,}", "[1,]", "{\"a\" 1}", "{1:2}", "tru", "nul", "{\"a\":tx}",
        "{\"a\":01}", "{\"a\":-}", "{\"a\":1.}", "{\"a\":1e}", "{\"a\":1e+}", "{\"a\":\"\\x\"}", "{\"a\":\"\\u12G4\"}",
        "{\"a\":\"\\ud800\"}", "{\"a\":\"\\ud800\\u0041\"}", "{\"a\":\"\\udc00\"}", "{\"a\":\"x\ny\"}",
        "{\"a\":\"\xff\"}", "{\"a\":\"\xe0\x80\x80\"}", "{\"a\":\"\xed\xa0\x80\"}", "{\"a\":\"\xf4\x90\x80\x80\"}",
        "{\"a\":\"\xc3\"}", "{} {}", "{}\n\n  x", "\xef\xbb\xbf{\"schema_version\":\"1\",\"classes\":[]}", "\xef\xbb{}",
        "\xef{}", "{\"schema_version\":\"1\",\"classes\":[]}\n", "{\"a\":[1 2]}", "{\"a\":{\"b\" }}", "{\"a\":}",
        "{\n\"schema_version\": \"1\",\n\"classes\": [\n{\"id\": 0,\n\"name\": \"A\",\n\"attributes\": [],\n\"methods\": [\n{\"id\": 0, \"name\": \"f\", \"calls\": [1,, 2]}]}]}",
        "{\"a\":\"\\",
        "{\"a\":\"\\u00",
        "{\"a\":1e400}", "{\"a\":-1e400, \"b\": !}", "{\"a\":-01}", "{\"a\":--1}", "{\"a\":+1}", "{\"a\":.5}", "{\"a\":1.5e-3}", "{\"a\":[[[[[]]]]]}", "{\"a\":\"\t\"}",
    };
}

static GeneratedSystem gen(uint64_t seed, uint32_t c, uint32_t m, uint32_t a, uint32_t kc, uint32_t ka, double bias) {
    GeneratorConfig cfg;
    cfg.seed = seed; cfg.n_classes = c; cfg.n_methods = m; cfg.n_attributes = a;
    cfg.k_max_calls = kc; cfg.k_max_accesses = ka; cfg.intra_class_bias = bias;
    return generate(cfg);
}

struct Rng {
    uint64_t s;
    uint64_t next() { uint64_t z = (s += 0x9e3779b97f4a7c15ULL); z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL; z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL; return z ^ (z >> 31); }
    size_t below(size_t n) { return n ? next() % n : 0; }
};

static std::string mutate(const std::string& doc, Rng& r) {
    static const char kAlphabet[] = "{}[]:,\"\\ 0123456789-+.eEtrufalsn\nxu\x01\xc3\xa9\xff";
    std::string d = doc;
    const int edits = 1 + int(r.below(3));
    for (int k = 0; k < edits && !d.empty(); ++k) {
        const size_t i = r.below(d.size());
        switch (r.below(5)) {
            case 0: d.erase(i, 1); break;
            case 1: d.insert(d.begin() + i, kAlphabet[r.below(sizeof kAlphabet - 1)]); break;
            case 2: d[i] = kAlphabet[r.below(sizeof kAlphabet - 1)]; break;
            case 3: d.resize(i); break;
            default: {  // swap two digits / ids
                const size_t j = r.below(d.size());
                std::swap(d[i], d[j]);
            }
        }
    }
    return d;
}

static int bench() {
    const GeneratedSystem g = gen(1, 100000, 1000000, 2000000, 4, 4, 0.5);
    const std::string doc = facts_to_json(g.model, g.deps);
    auto t0 = std::chrono::steady_clock::now();
    const LoadResult ref = parse_facts(doc);
    auto t1 = std::chrono::steady_clock::now();
    gpu::Facts f = gpu::Facts::parse(doc);
    auto t2 = std::chrono::steady_clock::now();
    const LoadResult mine = f.to_load_result();
    auto t3 = std::chrono::steady_clock::now();
    const bool eq = ref.model == mine.model && ref.deps == mine.deps;
    const double mb = doc.size() / 1e6;
    const double s_ref = std::chrono::duration<double>(t1 - t0).count();
    const double s_csr = std::chrono::duration<double>(t2 - t1).count();
    const double s_lr = std::chrono::duration<double>(t3 - t2).count();
    std::printf("{\"doc_mb\": %.1f, \"reference_parse_facts_s\": %.3f, \"csr_parse_s\": %.3f, \"csr_to_load_result_s\": %.3f, "
                "\"reference_mb_per_s\": %.1f, \"csr_mb_per_s\": %.1f, \"speedup\": %.1f, \"equal\": %s}\n",
                mb, s_ref, s_csr, s_lr, mb / s_ref, mb / s_csr, s_ref / s_csr, eq ? "true" : "false");
    return eq ? 0 : 1;
}

int main(int argc, char** argv) {
    std::setvbuf(stdout, nullptr, _IONBF, 0);
    if (argc > 1 && std::strcmp(argv[1], "--bench") == 0) return bench();
    if (argc > 2 && std::strcmp(argv[1], "--golden") == 0) {
        // reference outcomes of the handwritten documents, for tests/golden
        // (all strings hex-encoded: several documents are not valid UTF-8)
        auto hex = [](const std::string& x) {
            static const char* d = "0123456789abcdef";
            std::string o;
            for (unsigned char c : x) { o += d[c >> 4]; o += d[c & 15]; }
            return "\"" + o + "\"";
        };
        std::string out = "[\n";
        const std::vector<std::string> docs = handwritten();
        for (size_t i = 0; i < docs.size(); ++i) {
            const Outcome o = run([&] { return parse_facts(docs[i]); });
            out += "{\"doc\":" + hex(docs[i]) + ",\"type\":\"" + o.type + "\",\"what\":" + hex(o.what) + ",\"violations\":[";
            for (size_t k = 0; k < o.violations.size(); ++k)
                out += (k ? "," : "") + std::string("[") + std::to_string(int(o.violations[k].kind)) + "," + hex(o.violations[k].message) + "]";
            out += "],\"warnings\":[";
            for (size_t k = 0; k < o.r.warnings.size(); ++k) out += (k ? "," : "") + hex(o.r.warnings[k]);
            out += "],\"canonical\":" + hex(o.type == "none" ? facts_to_json(o.r.model, o.r.deps) : std::string()) + "}";
            out += i + 1 < docs.size() ? ",\n" : "\n";
        }
        out += "]\n";
        FILE* fp = std::fopen(argv[2], "wb");
        if (!fp) return 2;
        std::fwrite(out.data(), 1, out.size(), fp);
        std::fclose(fp);
        return 0;
    }
    if (argc > 2 && std::strcmp(argv[1], "--write-c4") == 0) {  // C4 document for ingest benchmarks
        const GeneratedSystem g = gen(1, 100000, 1000000, 2000000, 4, 4, 0.5);
        save_facts(g.model, g.deps, argv[2]);
        return 0;
    }
    const int kFuzz = argc > 1 ? std::atoi(argv[1]) : 30000;

    const std::vector<std::string> docs = handwritten();
    for (size_t i = 0; i < docs.size(); ++i) check_doc(docs[i], "handwritten[" + std::to_string(i) + "]");

    // generated systems through the canonical writer, plus a re-spaced variant
    for (uint64_t seed = 0; seed < 40; ++seed) {
        Rng r{seed * 7 + 1};
        const uint32_t c = 1 + uint32_t(r.below(12)), m = uint32_t(r.below(60)), a = uint32_t(r.below(40));
        const GeneratedSystem g = gen(seed, c, m, a, uint32_t(r.below(6)), uint32_t(r.below(6)), double(r.below(11)) / 10);
        const std::string doc = facts_to_json(g.model, g.deps);
        check_doc(doc, "generated seed " + std::to_string(seed));
        std::string spaced;
        for (char ch : doc) {
            spaced += ch;
            if (ch == ',' || ch == ':' || ch == '[' || ch == '{') spaced += r.below(2) ? "\n  " : " \t";
        }
        check_doc(spaced, "generated spaced seed " + std::to_string(seed));
    }
    {
        const GeneratedSystem g = gen(42, 5, 30, 12, 3, 3, 0.6);  // samples/generated.json
        check_doc(facts_to_json(g.model, g.deps), "samples/generated.json system");
        const GeneratedSystem big = gen(1, 1000, 10000, 20000, 4, 4, 0.5);  // C2
        check_doc(facts_to_json(big.model, big.deps), "C2");
    }

    // mutation fuzz
    std::vector<std::string> seeds = docs;
    for (uint64_t seed = 0; seed < 6; ++seed) {
        const GeneratedSystem g = gen(seed + 100, 3, 8, 5, 3, 3, 0.5);
        seeds.push_back(facts_to_json(g.model, g.deps));
    }
    Rng r{12345};

    int fuzz_fail_before = g_fail;
    for (int k = 0; k < kFuzz; ++k) {
        const std::string& base = seeds[r.below(seeds.size())];
        check_doc(mutate(base, r), "fuzz " + std::to_string(k));
    }
    const int fuzz_fail = g_fail - fuzz_fail_before;

    // load_facts: missing file -> IoError with the same message
    {
        ++g_checks;
        const Outcome a = run([] { return load_facts("/nonexistent/facts.json"); });
        const Outcome b = run([] { return gpu::load_facts("/nonexistent/facts.json"); });
        std::string why;
        if (!same(a, b, why)) { ++g_fail; std::printf("FAIL load_facts missing file: %s\n", why.c_str()); }
    }

    std::printf("%d checks, %d failures (%d in the %d-document fuzz)\n", g_checks, g_fail, fuzz_fail, kFuzz);
    std::printf(g_fail ? "FAIL\n" : "PASS\n");
    return g_fail ? 1 : 0;
}
