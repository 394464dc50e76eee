// Facts ingest straight into the engine's CSR.
//
// The reference parses a facts document into an nlohmann DOM, walks it into
// `SystemModel` + `DependencyTable` (vector-of-vectors), then the GPU path
// flattens that again into CSR (parse_facts, /root/reference/proj/include/
// modmetrics/facts.hpp:91-256). Here one streaming pass over the bytes
// captures the schema's fields into flat arrays (no DOM, no per-method heap
// vectors), then a semantic pass replays the reference's checks in the
// reference's order over those arrays and emits mm_system CSR directly.
//
// Behaviour parity with parse_facts:
//  * JSON syntax errors -> MM_E_PARSE "facts: JSON parse error at line L, column C",
//    L/C computed as facts.hpp:51-58 does from the byte count nlohmann's lexer
//    reports (the 1-based position of the last character it consumed);
//  * shape errors (facts.hpp:60-82) in the reference's check order — top level,
//    then class by class: id, name, attributes (each: object, id, name),
//    methods (each: object, id, name); then the second pass (calls, accesses)
//    over the non-duplicate methods — with the same messages;
//  * duplicate object keys: the last one wins (nlohmann's DOM behaviour);
//  * violations (facts.hpp:134-241) with the same kinds, messages and order,
//    and "facts validation failed with N violation(s): <first>" as the error;
//  * warnings for dropped self-calls (facts.hpp:209-212), one per occurrence;
//  * calls/accesses per method sorted unique (facts.hpp:235-240).
// The validate() call at facts.hpp:243-247 cannot add anything once the
// passes above found no violation (every invariant it checks was already
// enforced), so it is not repeated.

#include <algorithm>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <chrono>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/mmgpu.h"
#include "../../include/mmfacts.h"

namespace {

constexpr uint32_t kNone = 0xffffffffu;

// Kind of a captured scalar field.
enum FieldKind : uint8_t { F_MISSING = 0, F_UNSIGNED, F_STRING, F_OTHER, F_ARRAY, F_OBJECT };

struct Span { uint64_t off = 0; uint32_t len = 0; };

struct IdField {
    uint8_t kind = F_MISSING;  // F_UNSIGNED: value fits u64 unsigned
    uint64_t value = 0;
};

struct NameField {
    uint8_t kind = F_MISSING;
    Span s;
};

struct RawAttr {
    uint8_t is_object = 0;
    IdField id;
    NameField name;
};

// per dependency list: first element that is not a valid id
struct DepList {
    uint8_t kind = F_MISSING;  // F_ARRAY or F_OTHER or F_MISSING
    uint64_t begin = 0, end = 0;  // into raw_deps
    int64_t first_bad = -1;
};

struct RawMethod {
    uint8_t is_object = 0;
    IdField id;
    NameField name;
    DepList calls, accesses;
};

struct RawClass {
    uint8_t is_object = 0;
    IdField id;
    NameField name;
    uint8_t attrs_kind = F_MISSING, methods_kind = F_MISSING;
    uint64_t attr_begin = 0, attr_end = 0;
    uint64_t meth_begin = 0, meth_end = 0;
};

struct ParseFail {
    size_t byte;  // nlohmann's chars_read_total at the error
};

struct NumberOverflow {
    std::string token;
};

}  // namespace

struct mm_facts {
    mm_status status = MM_OK;
    std::string error;
    std::vector<std::pair<int, std::string>> violations;
    std::vector<std::string> warnings;

    uint32_t C = 0, M = 0, A = 0;
    std::vector<uint32_t> method_owner, attribute_owner;
    std::vector<uint32_t> cmoff, cmeth, caoff, cattr;
    std::vector<uint32_t> call_off, call_tgt, acc_off, acc_tgt;
    std::vector<uint32_t> class_ids;  // ClassRecord::id (== index once valid)

    std::string blob;  // decoded names
    std::vector<Span> class_name, method_name, attribute_name;
};

namespace {

// ---------------------------------------------------------------------------
// Phase 1: one pass over the text. A strict RFC 8259 reader with nlohmann's
// tokenisation (maximal tokens, error at the last character consumed) that
// records only the facts schema's fields.
// ---------------------------------------------------------------------------
class Reader {
public:
    Reader(const char* t, size_t n, std::string& blob) : s_(reinterpret_cast<const unsigned char*>(t)), n_(n), blob_(blob) {}

    // top level
    uint8_t top_kind = F_MISSING;
    uint8_t version_kind = F_MISSING;
    std::string version_str;   // decoded, when a string
    std::string version_dump;  // nlohmann-style dump of the value
    uint8_t classes_kind = F_MISSING;
    uint64_t cls_begin = 0, cls_end = 0;

    std::vector<RawClass> classes;
    std::vector<RawAttr> attrs;
    std::vector<RawMethod> methods;
    std::vector<uint64_t> deps;  // raw dependency ids (valid ones), kNone64 for invalid

    void run() {
        // Capacity from the smallest JSON each entity can take (a method is at
        // least {"accesses":[],"calls":[],"id":0,"name":""}): virtual space
        // only — untouched pages cost nothing — and no regrowth copies.
        classes.reserve(n_ / 48 + 1);
        methods.reserve(n_ / 44 + 1);
        attrs.reserve(n_ / 20 + 1);
        deps.reserve(n_ / 2 + 1);
        blob_.reserve(n_);
        if (n_ >= 1 && s_[0] == 0xEF) {  // UTF-8 BOM (nlohmann skips it; a partial one is an error)
            if (n_ < 2 || s_[1] != 0xBB) fail_at(2);
            if (n_ < 3 || s_[2] != 0xBF) fail_at(3);
            p_ = 3;
        }
        ws();
        if (peek() == '{') top_object();
        else { top_kind = F_OTHER; skip_value(); }
        ws();
        if (p_ < n_) fail_token();
    }

private:
    const unsigned char* s_;
    size_t n_;
    size_t p_ = 0;
    std::string& blob_;
    std::string key_;

    [[noreturn]] void fail_at(size_t byte) { throw ParseFail{byte}; }
    // error at character index i (0-based) => nlohmann byte i + 1
    [[noreturn]] void fail_idx(size_t i) { fail_at(i + 1); }
    [[noreturn]] void fail_eof() { fail_at(n_ + 1); }

    int peek() const { return p_ < n_ ? s_[p_] : -1; }
    void ws() {
        while (p_ < n_) {
            const unsigned char c = s_[p_];
            if (c == ' ' || c == '\t' || c == '\n' || c == '\r') ++p_;
            else break;
        }
    }

    // Consume the token at p_ (whatever it is) and fail at its last character:
    // nlohmann's "unexpected <token>" errors.
    [[noreturn]] void fail_token() {
        if (p_ >= n_) fail_eof();
        const unsigned char c = s_[p_];
        if (c == '"') { std::string tmp; string_into(tmp); fail_idx(p_ - 1); }
        if (c == '-' || (c >= '0' && c <= '9')) { IdField f; number(f, false); fail_idx(p_ - 1); }
        if (c == 't' || c == 'f' || c == 'n') { literal(); fail_idx(p_ - 1); }
        fail_idx(p_);  // structural char or an invalid one
    }

    void expect(char c) {
        ws();
        if (p_ < n_ && s_[p_] == c) { ++p_; return; }
        fail_token();
    }

    void literal() {
        const char* word = s_[p_] == 't' ? "true" : s_[p_] == 'f' ? "false" : "null";
        for (size_t k = 0; word[k]; ++k) {
            if (p_ >= n_) fail_eof();
            if (s_[p_] != static_cast<unsigned char>(word[k])) fail_idx(p_);
            ++p_;
        }
    }

    // Number token (nlohmann's scan_number). Sets f to F_UNSIGNED (non-negative
    // integer that fits u64) or F_OTHER.
    void number(IdField& f, bool as_value = true) {
        const size_t b = p_;
        bool neg = false, is_int = true;
        if (s_[p_] == '-') { neg = true; ++p_; }
        if (p_ >= n_) fail_eof();
        if (s_[p_] == '0') ++p_;
        else if (s_[p_] >= '1' && s_[p_] <= '9') { while (p_ < n_ && s_[p_] >= '0' && s_[p_] <= '9') ++p_; }
        else fail_idx(p_);
        if (p_ < n_ && s_[p_] == '.') {
            is_int = false; ++p_;
            if (p_ >= n_) fail_eof();
            if (!(s_[p_] >= '0' && s_[p_] <= '9')) fail_idx(p_);
            while (p_ < n_ && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
        }
        if (p_ < n_ && (s_[p_] == 'e' || s_[p_] == 'E')) {
            is_int = false; ++p_;
            if (p_ >= n_) fail_eof();
            if (s_[p_] == '+' || s_[p_] == '-') { ++p_; if (p_ >= n_) fail_eof(); }
            if (!(s_[p_] >= '0' && s_[p_] <= '9')) fail_idx(p_);
            while (p_ < n_ && s_[p_] >= '0' && s_[p_] <= '9') ++p_;
        }
        f.kind = F_OTHER;
        if (!neg && is_int) {
            // strtoull semantics: overflow -> nlohmann falls back to a float
            uint64_t v = 0; bool over = false;
            if (p_ - b <= 19) {  // cannot overflow u64
                for (size_t i = b; i < p_; ++i) v = v * 10 + (s_[i] - '0');
            } else {
                for (size_t i = b; i < p_; ++i) {
                    const uint64_t d = s_[i] - '0';
                    if (v > (UINT64_MAX - d) / 10) { over = true; break; }
                    v = v * 10 + d;
                }
            }
            if (!over) { f.kind = F_UNSIGNED; f.value = v; return; }
        }
        if (neg && is_int) {  // strtoll range: an int64 -> no float conversion
            uint64_t v = 0; bool over = false;
            for (size_t i = b + 1; i < p_; ++i) {
                const uint64_t d = s_[i] - '0';
                if (v > (uint64_t(INT64_MAX) + 1 - d) / 10) { over = true; break; }
                v = v * 10 + d;
            }
            if (!over) return;
        }
        // nlohmann converts every float token it accepts as a value with
        // strtod and rejects overflow with out_of_range.406 (json.hpp parser,
        // value_float case); an unexpected token is a parse error first
        const std::string tok(reinterpret_cast<const char*>(s_ + b), p_ - b);
        if (as_value && !std::isfinite(std::strtod(tok.c_str(), nullptr))) throw NumberOverflow{tok};
    }

    static int hexval(unsigned char c) {
        if (c >= '0' && c <= '9') return c - '0';
        if (c >= 'a' && c <= 'f') return c - 'a' + 10;
        if (c >= 'A' && c <= 'F') return c - 'A' + 10;
        return -1;
    }
    unsigned get4hex() {
        unsigned v = 0;
        for (int k = 0; k < 4; ++k) {
            if (p_ >= n_) fail_eof();
            const int h = hexval(s_[p_]);
            if (h < 0) fail_idx(p_);
            v = v * 16 + h; ++p_;
        }
        return v;
    }
    static void put_utf8(std::string& out, unsigned cp) {
        if (cp < 0x80) out += char(cp);
        else if (cp < 0x800) { out += char(0xC0 | (cp >> 6)); out += char(0x80 | (cp & 0x3F)); }
        else if (cp < 0x10000) { out += char(0xE0 | (cp >> 12)); out += char(0x80 | ((cp >> 6) & 0x3F)); out += char(0x80 | (cp & 0x3F)); }
        else { out += char(0xF0 | (cp >> 18)); out += char(0x80 | ((cp >> 12) & 0x3F)); out += char(0x80 | ((cp >> 6) & 0x3F)); out += char(0x80 | (cp & 0x3F)); }
    }

    // String token at p_ ('"'), decoded and appended to out. UTF-8 checked as
    // nlohmann does (Unicode Table 3-7 ranges).
    void string_into(std::string& out) {
        ++p_;
        for (;;) {
            // fast run of plain ASCII
            size_t q = p_;
            while (q < n_) {
                const unsigned char c = s_[q];
                if (c == '"' || c == '\\' || c < 0x20 || c >= 0x80) break;
                ++q;
            }
            out.append(reinterpret_cast<const char*>(s_ + p_), q - p_);
            p_ = q;
            if (p_ >= n_) fail_eof();
            const unsigned char c = s_[p_];
            if (c == '"') { ++p_; return; }
            if (c < 0x20) fail_idx(p_);
            if (c == '\\') {
                ++p_;
                if (p_ >= n_) fail_eof();
                const unsigned char e = s_[p_++];
                switch (e) {
                    case '"': out += '"'; break;
                    case '\\': out += '\\'; break;
                    case '/': out += '/'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'n': out += '\n'; break;
                    case 'r': out += '\r'; break;
                    case 't': out += '\t'; break;
                    case 'u': {
                        unsigned cp = get4hex();
                        if (cp >= 0xD800 && cp <= 0xDBFF) {
                            if (p_ >= n_) fail_eof();
                            if (s_[p_] != '\\') fail_idx(p_);
                            ++p_;
                            if (p_ >= n_) fail_eof();
                            if (s_[p_] != 'u') fail_idx(p_);
                            ++p_;
                            const unsigned lo = get4hex();
                            if (!(lo >= 0xDC00 && lo <= 0xDFFF)) fail_idx(p_ - 1);
                            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                        } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                            fail_idx(p_ - 1);
                        }
                        put_utf8(out, cp);
                        break;
                    }
                    default: fail_idx(p_ - 1);
                }
                continue;
            }
            // multi-byte UTF-8
            int need; unsigned char lo = 0x80, hi = 0xBF;
            if (c >= 0xC2 && c <= 0xDF) need = 1;
            else if (c == 0xE0) { need = 2; lo = 0xA0; }
            else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) need = 2;
            else if (c == 0xED) { need = 2; hi = 0x9F; }
            else if (c == 0xF0) { need = 3; lo = 0x90; }
            else if (c >= 0xF1 && c <= 0xF3) need = 3;
            else if (c == 0xF4) { need = 3; hi = 0x8F; }
            else fail_idx(p_);
            const size_t b = p_++;
            for (int k = 0; k < need; ++k) {
                if (p_ >= n_) fail_eof();
                const unsigned char d = s_[p_];
                const unsigned char l = k == 0 ? lo : 0x80, h = k == 0 ? hi : 0xBF;
                if (d < l || d > h) fail_idx(p_);
                ++p_;
            }
            out.append(reinterpret_cast<const char*>(s_ + b), p_ - b);
        }
    }

    void name_value(NameField& f) {
        ws();
        if (peek() == '"') {
            const uint64_t off = blob_.size();
            string_into(blob_);
            f.kind = F_STRING; f.s.off = off; f.s.len = uint32_t(blob_.size() - off);
        } else { skip_value(); f.kind = F_OTHER; }
    }

    void id_value(IdField& f) {
        ws();
        const int c = peek();
        if (c == '-' || (c >= '0' && c <= '9')) { number(f); return; }
        skip_value();
        f.kind = F_OTHER; f.value = 0;
    }

    // Generic value (syntax-checked, discarded). Iterative on the container
    // stack so deep nesting cannot overflow the C stack.
    void skip_value() {
        std::vector<char> stack;
        for (;;) {
            ws();
            if (p_ >= n_) fail_eof();
            const unsigned char c = s_[p_];
            bool closed_scalar = true;
            if (c == '{') {
                ++p_; ws();
                if (peek() == '}') { ++p_; }
                else { stack.push_back('{'); skip_key_colon(); closed_scalar = false; }
            } else if (c == '[') {
                ++p_; ws();
                if (peek() == ']') { ++p_; }
                else { stack.push_back('['); closed_scalar = false; }
            } else if (c == '"') { std::string tmp; string_into(tmp); }
            else if (c == '-' || (c >= '0' && c <= '9')) { IdField f; number(f); }
            else if (c == 't' || c == 'f' || c == 'n') literal();
            else fail_idx(p_);
            if (!closed_scalar) continue;
            // after a value: close containers / separators
            for (;;) {
                if (stack.empty()) return;
                ws();
                if (p_ >= n_) fail_eof();
                const unsigned char d = s_[p_];
                if (d == ',') {
                    ++p_;
                    if (stack.back() == '{') skip_key_colon();
                    break;
                }
                if ((d == '}' && stack.back() == '{') || (d == ']' && stack.back() == '[')) {
                    ++p_; stack.pop_back(); continue;
                }
                fail_token();
            }
        }
    }

    enum Key { K_OTHER, K_ID, K_NAME, K_ATTRIBUTES, K_METHODS, K_CALLS, K_ACCESSES, K_SCHEMA, K_CLASSES };
    static int classify(const char* k, size_t n) {
        switch (n) {
            case 2: return std::memcmp(k, "id", 2) == 0 ? K_ID : K_OTHER;
            case 4: return std::memcmp(k, "name", 4) == 0 ? K_NAME : K_OTHER;
            case 5: return std::memcmp(k, "calls", 5) == 0 ? K_CALLS : K_OTHER;
            case 7: return std::memcmp(k, "methods", 7) == 0 ? K_METHODS : std::memcmp(k, "classes", 7) == 0 ? K_CLASSES : K_OTHER;
            case 8: return std::memcmp(k, "accesses", 8) == 0 ? K_ACCESSES : K_OTHER;
            case 10: return std::memcmp(k, "attributes", 10) == 0 ? K_ATTRIBUTES : K_OTHER;
            case 14: return std::memcmp(k, "schema_version", 14) == 0 ? K_SCHEMA : K_OTHER;
            default: return K_OTHER;
        }
    }
    // Object key at p_ ('"'): plain-ASCII keys are matched in place, others
    // (escapes, UTF-8) decoded first so "\u0069d" is "id" as in nlohmann.
    int read_key() {
        size_t q = p_ + 1;
        while (q < n_) {
            const unsigned char c = s_[q];
            if (c == '"' || c == '\\' || c < 0x20 || c >= 0x80) break;
            ++q;
        }
        if (q < n_ && s_[q] == '"') {
            const int k = classify(reinterpret_cast<const char*>(s_ + p_ + 1), q - p_ - 1);
            p_ = q + 1;
            return k;
        }
        key_.clear();
        string_into(key_);
        return classify(key_.data(), key_.size());
    }

    void skip_key_colon() {
        ws();
        if (peek() != '"') fail_token();
        key_.clear();
        string_into(key_);
        expect(':');
    }

    // Iterate an object's members: fn(key) must consume the value.
    template <class Fn>
    void object(Fn&& fn) {
        ++p_;  // '{'
        ws();
        if (peek() == '}') { ++p_; return; }
        for (;;) {
            ws();
            if (peek() != '"') fail_token();
            const int k = read_key();
            expect(':');
            fn(k);
            ws();
            if (p_ >= n_) fail_eof();
            if (s_[p_] == ',') { ++p_; continue; }
            if (s_[p_] == '}') { ++p_; return; }
            fail_token();
        }
    }
    template <class Fn>
    void array(Fn&& fn) {
        ++p_;  // '['
        ws();
        if (peek() == ']') { ++p_; return; }
        for (size_t i = 0;; ++i) {
            fn(i);
            ws();
            if (p_ >= n_) fail_eof();
            if (s_[p_] == ',') { ++p_; continue; }
            if (s_[p_] == ']') { ++p_; return; }
            fail_token();
        }
    }

    void top_object() {
        top_kind = F_OBJECT;
        object([&](int k) {
            if (k == K_SCHEMA) version_value();
            else if (k == K_CLASSES) classes_value();
            else skip_value();
        });
    }

    void version_value() {
        ws();
        const size_t b = p_;
        if (peek() == '"') {
            version_str.clear();
            string_into(version_str);
            version_kind = F_STRING;
            version_dump = dump_string(version_str);
        } else {
            skip_value();
            version_kind = F_OTHER;
            // compact raw text (exact for integers, literals and containers of them)
            version_dump.clear();
            bool in_str = false;
            for (size_t i = b; i < p_; ++i) {
                const char ch = char(s_[i]);
                if (in_str) { version_dump += ch; if (ch == '\\') { version_dump += char(s_[++i]); } else if (ch == '"') in_str = false; continue; }
                if (ch == '"') in_str = true;
                if (ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r') continue;
                version_dump += ch;
            }
        }
    }

    static std::string dump_string(const std::string& s) {
        // nlohmann's dump (ensure_ascii = false)
        std::string o = "\"";
        for (unsigned char ch : s) {
            switch (ch) {
                case '"': o += "\\\""; break;
                case '\\': o += "\\\\"; break;
                case '\b': o += "\\b"; break;
                case '\f': o += "\\f"; break;
                case '\n': o += "\\n"; break;
                case '\r': o += "\\r"; break;
                case '\t': o += "\\t"; break;
                default:
                    if (ch < 0x20 || ch == 0x7F) { char buf[8]; std::snprintf(buf, sizeof buf, "\\u%04x", ch); o += buf; }
                    else o += char(ch);
            }
        }
        return o + "\"";
    }

    void classes_value() {
        ws();
        if (peek() != '[') { skip_value(); classes_kind = F_OTHER; return; }
        classes_kind = F_ARRAY;
        cls_begin = classes.size();
        ++p_;
        ws();
        if (peek() == ']') { ++p_; cls_end = classes.size(); return; }
        for (;;) {
            ws();
            if (splice_ && p_ == splice_->first_start()) {
                const size_t q = splice_->apply(*this);
                if (q == p_) class_element();  // nothing verified: parse it here
                else p_ = q;
            } else class_element();
            ws();
            if (p_ >= n_) fail_eof();
            if (s_[p_] == ',') { ++p_; continue; }
            if (s_[p_] == ']') { ++p_; break; }
            fail_token();
        }
        cls_end = classes.size();
    }

    void class_element() {
        RawClass rc;
        if (peek() != '{') { skip_value(); classes.push_back(rc); return; }
        rc.is_object = 1;
        object([&](int k) {
            if (k == K_ID) id_value(rc.id);
            else if (k == K_NAME) name_value(rc.name);
            else if (k == K_ATTRIBUTES) {
                ws();
                if (peek() != '[') { skip_value(); rc.attrs_kind = F_OTHER; return; }
                rc.attrs_kind = F_ARRAY;
                rc.attr_begin = attrs.size();
                array([&](size_t) { attr_value(); });
                rc.attr_end = attrs.size();
            } else if (k == K_METHODS) {
                ws();
                if (peek() != '[') { skip_value(); rc.methods_kind = F_OTHER; return; }
                rc.methods_kind = F_ARRAY;
                rc.meth_begin = methods.size();
                array([&](size_t) { method_value(); });
                rc.meth_end = methods.size();
            } else skip_value();
        });
        classes.push_back(rc);
    }

public:
    // Speculative chunk of the classes array (parallel ingest): starting at a
    // guessed element start, parse class elements until the next element
    // start at or past `limit`, or the closing ']'. Any failure just means the
    // main reader parses this stretch itself.
    struct Chunk {
        size_t start = 0, next = 0, end_pos = 0;  // next: first element start >= limit; end_pos: after the last element
        bool ok = false, closed = false;          // closed: stopped at the array's ']'
    };
    void run_chunk(Chunk& c, size_t limit) {
        try {
            const size_t span = limit > c.start ? limit - c.start : 0;
            classes.reserve(span / 48 + 16); methods.reserve(span / 44 + 16);
            attrs.reserve(span / 20 + 16); deps.reserve(span / 2 + 16); blob_.reserve(span + 16);
            p_ = c.start;
            for (;;) {
                class_element();
                c.end_pos = p_;
                ws();
                if (p_ >= n_) return;
                if (s_[p_] == ']') { c.closed = true; c.ok = true; return; }
                if (s_[p_] != ',') return;
                ++p_;
                ws();
                if (p_ >= limit) { c.next = p_; c.ok = true; return; }
            }
        } catch (...) {
            c.ok = false;
        }
    }

    // Verified chain of chunks the main reader splices in when it reaches the
    // first chunk's start exactly (which proves that start is a real element
    // start; each verified chunk then proves the next one's).
    struct Splice {
        std::vector<Chunk>* chunks;
        std::vector<Reader*>* readers;
        std::vector<std::thread>* threads;
        size_t first_start() const { return (*chunks)[0].start; }
        size_t apply(Reader& main) {
            for (std::thread& t : *threads) if (t.joinable()) t.join();
            size_t pos = main.p_;
            for (size_t k = 0; k < chunks->size(); ++k) {
                const Chunk& c = (*chunks)[k];
                if (!c.ok || c.start != pos) break;
                main.absorb(*(*readers)[k]);
                pos = c.end_pos;
                if (c.closed || k + 1 == chunks->size() || c.next != (*chunks)[k + 1].start) break;
                pos = c.next;
                // the main loop consumes the ',' between chunks: hand back the
                // end of this chunk unless the next one is verified too
                if (!(*chunks)[k + 1].ok) { pos = c.end_pos; break; }
            }
            main.splice_ = nullptr;
            if (std::getenv("MMGPU_FACTS_DEBUG")) {
                size_t okc = 0;
                for (const Chunk& c : *chunks) okc += c.ok;
                std::fprintf(stderr, "facts splice: %zu chunks, %zu ok, resume at %zu\n", chunks->size(), okc, pos);
            }
            return pos;
        }
    };
    Splice* splice_ = nullptr;

    void absorb(const Reader& w) {
        const uint64_t ab = attrs.size(), mb = methods.size(), db = deps.size(), bb = blob_.size();
        for (RawClass rc : w.classes) {
            rc.attr_begin += ab; rc.attr_end += ab; rc.meth_begin += mb; rc.meth_end += mb; rc.name.s.off += bb;
            classes.push_back(rc);
        }
        for (RawAttr ra : w.attrs) { ra.name.s.off += bb; attrs.push_back(ra); }
        for (RawMethod rm : w.methods) {
            rm.name.s.off += bb;
            rm.calls.begin += db; rm.calls.end += db; rm.accesses.begin += db; rm.accesses.end += db;
            methods.push_back(rm);
        }
        deps.insert(deps.end(), w.deps.begin(), w.deps.end());
        blob_.append(w.blob_);
    }

private:
    void attr_value() {
        ws();
        RawAttr ra;
        if (peek() == '{') {
            ra.is_object = 1;
            object([&](int k) {
                if (k == K_ID) id_value(ra.id);
                else if (k == K_NAME) name_value(ra.name);
                else skip_value();
            });
        } else skip_value();
        attrs.push_back(ra);
    }

    void dep_list(DepList& d) {
        ws();
        if (peek() != '[') { skip_value(); d.kind = F_OTHER; return; }
        d.kind = F_ARRAY;
        d.begin = deps.size();
        d.first_bad = -1;
        array([&](size_t i) {
            IdField f;
            id_value(f);
            const bool ok = f.kind == F_UNSIGNED && f.value <= 0xffffffffULL;
            if (!ok && d.first_bad < 0) d.first_bad = int64_t(i);
            deps.push_back(ok ? f.value : ~uint64_t(0));
        });
        d.end = deps.size();
    }

    void method_value() {
        ws();
        RawMethod rm;
        if (peek() == '{') {
            rm.is_object = 1;
            object([&](int k) {
                if (k == K_ID) id_value(rm.id);
                else if (k == K_NAME) name_value(rm.name);
                else if (k == K_CALLS) dep_list(rm.calls);
                else if (k == K_ACCESSES) dep_list(rm.accesses);
                else skip_value();
            });
        } else skip_value();
        methods.push_back(rm);
    }
};

struct FactsError {
    mm_status status;
    std::string msg;
};

[[noreturn]] void parse_error(const std::string& m) { throw FactsError{MM_E_PARSE, "facts: " + m}; }

bool valid_id(const IdField& f) { return f.kind == F_UNSIGNED && f.value <= 0xffffffffULL; }

uint32_t id_of(const IdField& f, const std::string& where, const std::string& field_where) {
    if (f.kind == F_MISSING) parse_error(where + ": missing \"id\"");
    if (!valid_id(f)) parse_error(field_where + ": expected a non-negative id");
    return uint32_t(f.value);
}

void name_check(const NameField& f, const std::string& where, const std::string& field_where) {
    if (f.kind == F_MISSING) parse_error(where + ": missing \"name\"");
    if (f.kind != F_STRING) parse_error(field_where + ": expected a string name");
}

size_t env_size(const char* name, size_t dflt) {
    const char* v = std::getenv(name);
    return v && *v ? size_t(std::strtoull(v, nullptr, 10)) : dflt;
}

void dbg_mark(const char* what) {
    static const bool on = std::getenv("MMGPU_FACTS_DEBUG") != nullptr;
    if (!on) return;
    static std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  build mark %-12s +%.1f ms\n", what, std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}

// Phase 2: the reference's semantic walk (facts.hpp:100-254) over the arrays.
void build(Reader& r, mm_facts& f, bool parallel_ok) {
    if (r.top_kind != F_OBJECT) parse_error("top level must be an object");
    auto& V = f.violations;
    enum { NonDenseClassIds = MM_VK_NON_DENSE_CLASS_IDS, DupMethod = MM_VK_DUPLICATE_METHOD_MEMBERSHIP,
           DupAttr = MM_VK_DUPLICATE_ATTRIBUTE_MEMBERSHIP, UnownedMethod = MM_VK_UNOWNED_METHOD,
           UnownedAttr = MM_VK_UNOWNED_ATTRIBUTE, DanglingCall = MM_VK_DANGLING_CALL_TARGET,
           DanglingAccess = MM_VK_DANGLING_ACCESS_TARGET, Schema = MM_VK_UNSUPPORTED_SCHEMA_VERSION };

    if (r.version_kind == F_MISSING) parse_error("top level: missing \"schema_version\"");
    if (!(r.version_kind == F_STRING && r.version_str == "1"))
        V.push_back({Schema, "schema_version must be \"1\", got " + r.version_dump});
    if (r.classes_kind == F_MISSING) parse_error("top level: missing \"classes\"");
    if (r.classes_kind != F_ARRAY) parse_error("classes: expected an array");

    const uint64_t nc = r.cls_end - r.cls_begin;
    if (nc > 0xffffffffULL) parse_error("classes: too many classes");
    f.C = uint32_t(nc);
    // Id spaces grow to max id + 1 (facts.hpp:146-149). Guard against a
    // pathological sparse id forcing a multi-GB table.
    const uint64_t id_cap = std::max<uint64_t>(16 * (uint64_t(r.methods.size()) + r.attrs.size()) + (1u << 20), 1u << 25);

    std::vector<uint32_t>& mown = f.method_owner;
    std::vector<uint32_t>& aown = f.attribute_owner;
    f.class_ids.resize(nc);
    f.class_name.resize(nc);
    f.cmoff.assign(nc + 1, 0);
    f.caoff.assign(nc + 1, 0);
    f.cmeth.clear(); f.cattr.clear();
    f.cmeth.reserve(r.methods.size()); f.cattr.reserve(r.attrs.size());
    struct Pending { uint32_t id; uint64_t raw; uint32_t ci, mi; };
    std::vector<Pending> pending;
    pending.reserve(r.methods.size());

    dbg_mark("start");
    bool presized = false;
    {   // size the id spaces once: max valid id + 1 over the declarations the
        // walk below will visit (it grows them the same way, facts.hpp:146-149)
        // per class range: (max attr id + 1, max method id + 1, stopped at a non-object class?)
        auto scan = [&](uint64_t c0, uint64_t c1, uint64_t& ma, uint64_t& mm) {
            for (uint64_t ci = c0; ci < c1; ++ci) {
                const RawClass& rc = r.classes[r.cls_begin + ci];
                if (!rc.is_object) return true;
                if (rc.attrs_kind == F_ARRAY)
                    for (uint64_t i = rc.attr_begin; i < rc.attr_end; ++i)
                        if (valid_id(r.attrs[i].id)) ma = std::max(ma, r.attrs[i].id.value + 1);
                if (rc.methods_kind == F_ARRAY)
                    for (uint64_t i = rc.meth_begin; i < rc.meth_end; ++i)
                        if (valid_id(r.methods[i].id)) mm = std::max(mm, r.methods[i].id.value + 1);
            }
            return false;
        };
        const size_t TS = parallel_ok && nc >= 2 ? size_t(16) : size_t(1);
        std::vector<uint64_t> pa(TS, 0), pm(TS, 0);
        std::vector<char> stop(TS, 0);
        {
            std::vector<std::thread> th;
            for (size_t k = 1; k < TS; ++k)
                th.emplace_back([&, k] { stop[k] = scan(nc * k / TS, nc * (k + 1) / TS, pa[k], pm[k]); });
            stop[0] = scan(0, nc / TS, pa[0], pm[0]);
            for (std::thread& t : th) t.join();
        }
        uint64_t ma = 0, mm = 0;
        bool any_stop = false;
        for (size_t k = 0; k < TS; ++k) {  // ranges in order, up to the first non-object class
            ma = std::max(ma, pa[k]);
            mm = std::max(mm, pm[k]);
            if (stop[k]) { any_stop = true; break; }
        }
        // a non-object class element ends the reference's walk there (a
        // ParseError): the tables are sized only up to it, so the optimistic
        // parallel walk — which visits every range — must not run
        if (any_stop) parallel_ok = false;
        if (ma < id_cap && mm < id_cap) {
            // the final sizes are exactly these (max visited id + 1), so
            // growing to them up front is the same as growing id by id
            aown.assign(ma, kNone); f.attribute_name.resize(ma);
            mown.assign(mm, kNone); f.method_name.resize(mm);
            presized = true;
        }
    }
    // Optimistic parallel walk for the common case — every field well-formed,
    // class ids dense, no id declared twice — over class ranges (ownership
    // claimed with compare-and-swap). Its result is then exactly the
    // sequential walk's. Any deviation anywhere: undo and walk sequentially,
    // which produces the reference's errors in the reference's order.
    dbg_mark("presize");
    bool walked = false;
    const size_t TW = parallel_ok && presized && nc >= 2
        ? std::min<size_t>(env_size("MMGPU_FACTS_THREADS", std::min<size_t>(16, std::max(1u, std::thread::hardware_concurrency()))), 16)
        : 1;
    if (TW > 1) {
        std::vector<uint32_t> apre(nc + 1, 0), mpre(nc + 1, 0);
        for (uint64_t ci = 0; ci < nc; ++ci) {
            const RawClass& rc = r.classes[r.cls_begin + ci];
            apre[ci + 1] = apre[ci] + uint32_t(rc.attrs_kind == F_ARRAY ? rc.attr_end - rc.attr_begin : 0);
            mpre[ci + 1] = mpre[ci] + uint32_t(rc.methods_kind == F_ARRAY ? rc.meth_end - rc.meth_begin : 0);
        }
        f.cattr.assign(apre[nc], 0);
        f.cmeth.assign(mpre[nc], 0);
        pending.assign(mpre[nc], Pending{});
        int bad = 0;
        auto claim = [](uint32_t* slot, uint32_t v) {
            uint32_t want = kNone;
            return __atomic_compare_exchange_n(slot, &want, v, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED);
        };
        auto walk = [&](uint64_t c0, uint64_t c1) {
            for (uint64_t ci = c0; ci < c1; ++ci) {
                if (__atomic_load_n(&bad, __ATOMIC_RELAXED)) return;
                const RawClass& rc = r.classes[r.cls_begin + ci];
                if (!rc.is_object || !valid_id(rc.id) || rc.id.value != ci || rc.name.kind != F_STRING ||
                    rc.attrs_kind != F_ARRAY || rc.methods_kind != F_ARRAY) { __atomic_store_n(&bad, 1, __ATOMIC_RELAXED); return; }
                f.class_ids[ci] = uint32_t(ci);
                f.class_name[ci] = rc.name.s;
                uint32_t* ca = f.cattr.data() + apre[ci];
                for (uint64_t ai = 0; ai < rc.attr_end - rc.attr_begin; ++ai) {
                    const RawAttr& ra = r.attrs[rc.attr_begin + ai];
                    if (!ra.is_object || !valid_id(ra.id) || ra.name.kind != F_STRING || ra.id.value >= aown.size() ||
                        !claim(&aown[ra.id.value], uint32_t(ci))) { __atomic_store_n(&bad, 1, __ATOMIC_RELAXED); return; }
                    f.attribute_name[ra.id.value] = ra.name.s;
                    ca[ai] = uint32_t(ra.id.value);
                }
                if (!std::is_sorted(ca, f.cattr.data() + apre[ci + 1])) std::sort(ca, f.cattr.data() + apre[ci + 1]);
                uint32_t* cm = f.cmeth.data() + mpre[ci];
                for (uint64_t mi = 0; mi < rc.meth_end - rc.meth_begin; ++mi) {
                    const RawMethod& rm = r.methods[rc.meth_begin + mi];
                    if (!rm.is_object || !valid_id(rm.id) || rm.name.kind != F_STRING || rm.id.value >= mown.size() ||
                        !claim(&mown[rm.id.value], uint32_t(ci))) { __atomic_store_n(&bad, 1, __ATOMIC_RELAXED); return; }
                    f.method_name[rm.id.value] = rm.name.s;
                    cm[mi] = uint32_t(rm.id.value);
                    pending[mpre[ci] + mi] = Pending{uint32_t(rm.id.value), rc.meth_begin + mi, uint32_t(ci), uint32_t(mi)};
                }
                if (!std::is_sorted(cm, f.cmeth.data() + mpre[ci + 1])) std::sort(cm, f.cmeth.data() + mpre[ci + 1]);
            }
        };
        {
            std::vector<std::thread> th;
            for (size_t k = 0; k < TW; ++k) th.emplace_back([&, k] { walk(nc * k / TW, nc * (k + 1) / TW); });
            for (std::thread& t : th) t.join();
        }
        dbg_mark(bad ? "pwalk_bad" : "pwalk_ok");
        if (!bad) {
            f.caoff.swap(apre);
            f.cmoff.swap(mpre);
            walked = true;
        } else {  // undo: the sequential walk starts from the presized, unowned tables
            std::fill(aown.begin(), aown.end(), kNone);
            std::fill(mown.begin(), mown.end(), kNone);
            f.cattr.clear();
            f.cmeth.clear();
            pending.clear();
        }
    }
    for (uint64_t ci = 0; ci < nc && !walked; ++ci) {
        const RawClass& rc = r.classes[r.cls_begin + ci];
        const std::string cw = "classes[" + std::to_string(ci) + "]";
        if (!rc.is_object) parse_error(cw + ": expected an object");
        const uint32_t cid = id_of(rc.id, cw, cw + ".id");
        name_check(rc.name, cw, cw + ".name");
        f.class_ids[ci] = cid;
        f.class_name[ci] = rc.name.s;
        if (cid != ci)
            V.push_back({NonDenseClassIds, cw + " has id " + std::to_string(cid) + ", expected " + std::to_string(ci)});

        if (rc.attrs_kind == F_MISSING) parse_error(cw + ": missing \"attributes\"");
        if (rc.attrs_kind != F_ARRAY) parse_error(cw + ".attributes: expected an array");
        const size_t abeg = f.cattr.size();
        for (uint64_t ai = 0; ai < rc.attr_end - rc.attr_begin; ++ai) {
            const RawAttr& ra = r.attrs[rc.attr_begin + ai];
            if (!ra.is_object || ra.id.kind == F_MISSING || !valid_id(ra.id) || ra.name.kind != F_STRING) {
                const std::string aw = cw + ".attributes[" + std::to_string(ai) + "]";
                if (!ra.is_object) parse_error(aw + ": expected an object");
                id_of(ra.id, aw, aw + ".id");
                name_check(ra.name, aw, aw + ".name");
            }
            const uint32_t id = uint32_t(ra.id.value);
            if (id >= aown.size()) {
                if (id >= id_cap) throw FactsError{MM_E_OOM, "facts: attribute id " + std::to_string(id) + " exceeds the id-space guard"};
                aown.resize(uint64_t(id) + 1, kNone);
                f.attribute_name.resize(uint64_t(id) + 1);
            }
            if (aown[id] != kNone) {
                V.push_back({DupAttr, "attribute " + std::to_string(id) + " declared more than once"});
            } else {
                aown[id] = uint32_t(ci);
                f.attribute_name[id] = ra.name.s;
                f.cattr.push_back(id);
            }
        }
        if (!std::is_sorted(f.cattr.begin() + abeg, f.cattr.end())) std::sort(f.cattr.begin() + abeg, f.cattr.end());
        f.caoff[ci + 1] = uint32_t(f.cattr.size());

        if (rc.methods_kind == F_MISSING) parse_error(cw + ": missing \"methods\"");
        if (rc.methods_kind != F_ARRAY) parse_error(cw + ".methods: expected an array");
        const size_t mbeg = f.cmeth.size();
        for (uint64_t mi = 0; mi < rc.meth_end - rc.meth_begin; ++mi) {
            const RawMethod& rm = r.methods[rc.meth_begin + mi];
            if (!rm.is_object || rm.id.kind == F_MISSING || !valid_id(rm.id) || rm.name.kind != F_STRING) {
                const std::string mw = cw + ".methods[" + std::to_string(mi) + "]";
                if (!rm.is_object) parse_error(mw + ": expected an object");
                id_of(rm.id, mw, mw + ".id");
                name_check(rm.name, mw, mw + ".name");
            }
            const uint32_t id = uint32_t(rm.id.value);
            if (id >= mown.size()) {
                if (id >= id_cap) throw FactsError{MM_E_OOM, "facts: method id " + std::to_string(id) + " exceeds the id-space guard"};
                mown.resize(uint64_t(id) + 1, kNone);
                f.method_name.resize(uint64_t(id) + 1);
            }
            if (mown[id] != kNone) {
                V.push_back({DupMethod, "method " + std::to_string(id) + " declared more than once"});
            } else {
                mown[id] = uint32_t(ci);
                f.method_name[id] = rm.name.s;
                f.cmeth.push_back(id);
                pending.push_back({id, rc.meth_begin + mi, uint32_t(ci), uint32_t(mi)});
            }
        }
        if (!std::is_sorted(f.cmeth.begin() + mbeg, f.cmeth.end())) std::sort(f.cmeth.begin() + mbeg, f.cmeth.end());
        f.cmoff[ci + 1] = uint32_t(f.cmeth.size());
    }

    dbg_mark("class_walk");
    for (uint64_t p = 0; p < mown.size(); ++p)
        if (mown[p] == kNone) {
            V.push_back({UnownedMethod, "method id " + std::to_string(p) + " is never declared"});
            mown[p] = 0;
        }
    for (uint64_t a = 0; a < aown.size(); ++a)
        if (aown[a] == kNone) {
            V.push_back({UnownedAttr, "attribute id " + std::to_string(a) + " is never declared"});
            aown[a] = 0;
        }
    f.M = uint32_t(mown.size());
    f.A = uint32_t(aown.size());
    const uint64_t M = f.M, A = f.A;

    dbg_mark("unowned");
    // Second pass (facts.hpp:200-241): shape checks, self-call repair,
    // dangling targets; rows gathered into CSR by method id.
    std::vector<uint32_t> ccount(M + 1, 0), acount(M + 1, 0);
    bool counted = false;
    if (parallel_ok && pending.size() >= 2) {
        // optimistic: no shape error, self-call or dangling target anywhere
        // (each pending method owns its counters); otherwise recount below
        int bad = 0;
        const size_t TP = 16, n = pending.size();
        std::vector<std::thread> th;
        for (size_t k = 0; k < TP; ++k)
            th.emplace_back([&, k] {
                for (size_t j = n * k / TP; j < n * (k + 1) / TP; ++j) {
                    const Pending& pm = pending[j];
                    const RawMethod& rm = r.methods[pm.raw];
                    if (rm.calls.kind != F_ARRAY || rm.accesses.kind != F_ARRAY) { __atomic_store_n(&bad, 1, __ATOMIC_RELAXED); return; }
                    for (uint64_t i = rm.calls.begin; i < rm.calls.end; ++i) {
                        const uint64_t t = r.deps[i];
                        if (t >= M || t == pm.id) { __atomic_store_n(&bad, 1, __ATOMIC_RELAXED); return; }
                    }
                    for (uint64_t i = rm.accesses.begin; i < rm.accesses.end; ++i)
                        if (r.deps[i] >= A) { __atomic_store_n(&bad, 1, __ATOMIC_RELAXED); return; }
                    ccount[pm.id] = uint32_t(rm.calls.end - rm.calls.begin);
                    acount[pm.id] = uint32_t(rm.accesses.end - rm.accesses.begin);
                }
            });
        for (std::thread& t : th) t.join();
        if (!bad) counted = true;
        else {
            std::fill(ccount.begin(), ccount.end(), 0u);
            std::fill(acount.begin(), acount.end(), 0u);
        }
    }
    for (const Pending& pm : pending) {
        if (counted) break;
        const RawMethod& rm = r.methods[pm.raw];
        auto where = [&] { return "classes[" + std::to_string(pm.ci) + "].methods[" + std::to_string(pm.mi) + "]"; };
        auto shape = [&](const DepList& d, const char* nm) {
            if (d.kind == F_MISSING) parse_error(where() + ": missing \"" + nm + "\"");
            if (d.kind != F_ARRAY) parse_error(where() + "." + nm + ": expected an array");
        };
        shape(rm.calls, "calls");
        for (uint64_t i = rm.calls.begin; i < rm.calls.end; ++i) {
            const uint64_t t = r.deps[i];
            if (t == ~uint64_t(0))
                parse_error(where() + ".calls[" + std::to_string(i - rm.calls.begin) + "]: expected a non-negative id");
            if (t == pm.id) {
                f.warnings.push_back("method " + std::to_string(pm.id) + " calls itself; self-call dropped");
            } else if (t >= M) {
                V.push_back({DanglingCall, "method " + std::to_string(pm.id) + " calls unknown method " + std::to_string(t)});
            } else ++ccount[pm.id];
        }
        shape(rm.accesses, "accesses");
        for (uint64_t i = rm.accesses.begin; i < rm.accesses.end; ++i) {
            const uint64_t t = r.deps[i];
            if (t == ~uint64_t(0))
                parse_error(where() + ".accesses[" + std::to_string(i - rm.accesses.begin) + "]: expected a non-negative id");
            if (t >= A) {
                V.push_back({DanglingAccess, "method " + std::to_string(pm.id) + " accesses unknown attribute " + std::to_string(t)});
            } else ++acount[pm.id];
        }
    }

    dbg_mark("pass2_loop");
    if (!V.empty()) {
        throw FactsError{MM_E_VALIDATION, "facts validation failed with " + std::to_string(V.size()) +
                                              " violation(s): " + V.front().second};
    }

    // CSR rows: scatter, then sort-unique each row in place and compact.
    // Rows land where their method id says; each pending method owns its
    // row, so threads over ranges of `pending` never touch the same words.
    const size_t T = parallel_ok ? std::max<size_t>(1, std::min<size_t>(
        env_size("MMGPU_FACTS_THREADS", std::min<size_t>(16, std::max(1u, std::thread::hardware_concurrency()))), 16)) : 1;
    auto parallel_pending = [&](auto&& body) {
        const size_t n = pending.size();
        if (T <= 1 || n < 2 * T) { body(size_t(0), n); return; }
        std::vector<std::thread> th;
        for (size_t k = 0; k < T; ++k) th.emplace_back([&, k] { body(n * k / T, n * (k + 1) / T); });
        for (std::thread& t : th) t.join();
    };
    auto scatter = [&](std::vector<uint32_t>& cnt, std::vector<uint32_t>& off, std::vector<uint32_t>& tgt, bool calls) {
        off.assign(M + 1, 0);
        for (uint64_t p = 0; p < M; ++p) off[p + 1] = off[p] + cnt[p];
        tgt.resize(off[M]);
        // fill each row, sort-unique it in place, keep its final length
        std::vector<uint32_t> len(M, 0);
        parallel_pending([&](size_t b, size_t e) {
            for (size_t k = b; k < e; ++k) {
                const Pending& pm = pending[k];
                const RawMethod& rm = r.methods[pm.raw];
                const DepList& d = calls ? rm.calls : rm.accesses;
                uint32_t* row = tgt.data() + off[pm.id];
                uint32_t* w = row;
                for (uint64_t i = d.begin; i < d.end; ++i) {
                    const uint64_t t = r.deps[i];
                    if (calls && t == pm.id) continue;
                    *w++ = uint32_t(t);
                }
                bool sorted = true;
                for (uint32_t* q = row + 1; q < w; ++q) if (q[-1] >= q[0]) { sorted = false; break; }
                if (!sorted) { std::sort(row, w); w = std::unique(row, w); }
                len[pm.id] = uint32_t(w - row);
            }
        });
        std::vector<uint32_t> noff(M + 1, 0);
        for (uint64_t p = 0; p < M; ++p) noff[p + 1] = noff[p] + len[p];
        if (noff[M] != off[M]) {  // duplicates collapsed: compact into a fresh array
            std::vector<uint32_t> packed(noff[M]);
            parallel_pending([&](size_t b, size_t e) {
                for (size_t k = b; k < e; ++k) {
                    const uint32_t p = pending[k].id;
                    std::copy(tgt.begin() + off[p], tgt.begin() + off[p] + len[p], packed.begin() + noff[p]);
                }
            });
            tgt.swap(packed);
        }
        off.swap(noff);
    };
    dbg_mark("pass2");
    scatter(ccount, f.call_off, f.call_tgt, true);
    scatter(acount, f.acc_off, f.acc_tgt, false);
    dbg_mark("scatter_acc");
}

// ---------------------------------------------------------------------------
// Parallel ingest: the classes array is cut into chunks parsed speculatively
// on worker threads while the main reader parses the head. Chunk starts are
// guessed from a parallel bracket-depth scan (the first '{' at depth 2 after
// each split point); the main reader only splices a chunk in when it reaches
// that chunk's start exactly at an element boundary, and each spliced chunk
// must end exactly where the next one starts. Anything else — a wrong guess,
// an error inside a chunk — is simply parsed by the main reader, so results
// and errors are the sequential reader's by construction.
// ---------------------------------------------------------------------------
struct Parallel {
    std::vector<Reader::Chunk> chunks;
    std::vector<std::string> blobs;
    std::vector<std::unique_ptr<Reader>> owned;
    std::vector<Reader*> readers;
    std::vector<std::thread> threads;
    Reader::Splice splice{};
    ~Parallel() {
        for (std::thread& t : threads) if (t.joinable()) t.join();
    }
};


// depth change over [b, e), assuming the segment starts outside a string
int64_t depth_delta(const unsigned char* s, size_t b, size_t e) {
    int64_t d = 0;
    bool in_str = false;
    for (size_t i = b; i < e; ++i) {
        const unsigned char c = s[i];
        if (in_str) {
            if (c == '\\') ++i;
            else if (c == '"') in_str = false;
        } else if (c == '"') in_str = true;
        else if (c == '{' || c == '[') ++d;
        else if (c == '}' || c == ']') --d;
    }
    return d;
}

// first '{' opened at depth 2 at or after b (a class element of the top-level classes array)
size_t element_start(const unsigned char* s, size_t n, size_t b, int64_t depth) {
    bool in_str = false;
    for (size_t i = b; i < n; ++i) {
        const unsigned char c = s[i];
        if (in_str) {
            if (c == '\\') ++i;
            else if (c == '"') in_str = false;
        } else if (c == '"') in_str = true;
        else if (c == '{') { if (depth == 2) return i; ++depth; }
        else if (c == '[') ++depth;
        else if (c == '}' || c == ']') --depth;
    }
    return n;
}

// next "}" ws "," ws "{" at or after b: the '{' (a likely object-element
// start, outside any string in any sane document)
size_t resync(const unsigned char* s, size_t n, size_t b) {
    auto ws = [](unsigned char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; };
    for (size_t i = b; i < n; ++i) {
        if (s[i] != '}') continue;
        size_t j = i + 1;
        while (j < n && ws(s[j])) ++j;
        if (j >= n || s[j] != ',') continue;
        ++j;
        while (j < n && ws(s[j])) ++j;
        if (j < n && s[j] == '{') return j;
    }
    return n;
}

void plan_parallel(Parallel& P, Reader& main, const char* text, size_t len) {
    const size_t min_len = env_size("MMGPU_FACTS_PAR_MIN", size_t(8) << 20);
    size_t T = env_size("MMGPU_FACTS_THREADS", std::min<size_t>(16, std::max(1u, std::thread::hardware_concurrency())));
    if (len < min_len || T < 2) return;
    T = std::min<size_t>(T, std::max<size_t>(2, len / std::max<size_t>(min_len / 8, 1)));
    const unsigned char* s = reinterpret_cast<const unsigned char*>(text);
    // segment boundaries at likely element starts (outside strings), so each
    // segment's depth change can be counted independently
    std::vector<size_t> bound{0};
    for (size_t k = 1; k < T; ++k) {
        const size_t b = resync(s, len, std::max(len * k / T, bound.back() + 1));
        if (b >= len) break;
        bound.push_back(b);
    }
    bound.push_back(len);
    const size_t S = bound.size() - 1;
    std::vector<int64_t> delta(S, 0);
    {
        std::vector<std::thread> th;
        for (size_t k = 0; k < S; ++k) th.emplace_back([&, k] { delta[k] = depth_delta(s, bound[k], bound[k + 1]); });
        for (std::thread& t : th) t.join();
    }
    int64_t depth = 0;
    std::vector<size_t> starts;
    for (size_t k = 1; k < S; ++k) {
        depth += delta[k - 1];
        const size_t st = element_start(s, len, bound[k], depth);
        if (st < len && (starts.empty() || st > starts.back())) starts.push_back(st);
    }
    if (starts.empty()) return;
    const size_t C = starts.size();
    P.chunks.resize(C);
    P.blobs.resize(C);
    for (size_t k = 0; k < C; ++k) {
        P.chunks[k].start = starts[k];
        P.owned.emplace_back(new Reader(text, len, P.blobs[k]));
        P.readers.push_back(P.owned.back().get());
    }
    for (size_t k = 0; k < C; ++k) {
        const size_t limit = k + 1 < C ? starts[k + 1] : len;
        P.threads.emplace_back([&P, k, limit] { P.readers[k]->run_chunk(P.chunks[k], limit); });
    }
    P.splice = Reader::Splice{&P.chunks, &P.readers, &P.threads};
    main.splice_ = &P.splice;
}

mm_status finish(mm_facts* f, const char* text, size_t len) {
    try {
        Reader rd(text, len, f->blob);
        Parallel par;
        try {
            try {
                plan_parallel(par, rd, text, len);
            } catch (...) {  // no threads: the sequential reader alone
                rd.splice_ = nullptr;
            }
            const auto t0 = std::chrono::steady_clock::now();
            rd.run();
            if (std::getenv("MMGPU_FACTS_DEBUG"))
                std::fprintf(stderr, "facts read %.1f ms\n",
                             std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        } catch (const ParseFail& pf) {
            // facts.hpp:51-58 applied to nlohmann's byte count
            size_t line = 1, col = 1;
            for (size_t i = 0; i + 1 < pf.byte && i < len; ++i) {
                if (text[i] == '\n') { ++line; col = 1; } else ++col;
            }
            throw FactsError{MM_E_PARSE, "facts: JSON parse error at line " + std::to_string(line) +
                                             ", column " + std::to_string(col)};
        } catch (const NumberOverflow& no) {
            // json::out_of_range 406, escapes parse_facts unwrapped
            throw FactsError{MM_E_RANGE, "number overflow parsing '" + no.token + "'"};
        }
        const auto t1 = std::chrono::steady_clock::now();
        build(rd, *f, len >= env_size("MMGPU_FACTS_PAR_MIN", size_t(8) << 20));
        if (std::getenv("MMGPU_FACTS_DEBUG"))
            std::fprintf(stderr, "facts build %.1f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count());
        f->status = MM_OK;
    } catch (const FactsError& e) {
        f->status = e.status;
        f->error = e.msg;
        if (e.status != MM_E_VALIDATION) f->violations.clear();
        f->warnings.clear();
    } catch (const std::bad_alloc&) {
        f->status = MM_E_OOM;
        f->error = "facts: out of host memory";
    }
    return f->status;
}

const char* name_ptr(const mm_facts* f, const Span& s, size_t* len) {
    if (len) *len = s.len;
    return f->blob.data() + s.off;
}

// canonical writer pieces (json_writer.hpp:23-76)
void quote(std::string& o, const char* s, size_t n) {
    o += '"';
    for (size_t i = 0; i < n; ++i) {
        const char ch = s[i];
        switch (ch) {
            case '"': o += "\\\""; break;
            case '\\': o += "\\\\"; break;
            case '\n': o += "\\n"; break;
            case '\r': o += "\\r"; break;
            case '\t': o += "\\t"; break;
            default:
                if (static_cast<unsigned char>(ch) < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", ch);
                    o += buf;
                } else o += ch;
        }
    }
    o += '"';
}
void put_u(std::string& o, uint64_t v) {
    char buf[24];
    char* e = buf + sizeof buf;
    char* q = e;
    do { *--q = char('0' + v % 10); v /= 10; } while (v);
    o.append(q, e - q);
}

}  // namespace

extern "C" {

mm_status mm_facts_parse(const char* text, size_t len, mm_facts** out) {
    if (!out || (!text && len)) return MM_E_ARG;
    mm_facts* f = new (std::nothrow) mm_facts();
    if (!f) return MM_E_OOM;
    *out = f;
    return finish(f, text ? text : "", len);
}

mm_status mm_facts_load(const char* path, mm_facts** out) {
    if (!out || !path) return MM_E_ARG;
    mm_facts* f = new (std::nothrow) mm_facts();
    if (!f) return MM_E_OOM;
    *out = f;
    // facts.hpp:258-265. A regular file is mapped, not copied: the reader
    // threads fault its pages in in parallel. Other files are read to EOF.
    const int fd = ::open(path, O_RDONLY);
    if (fd < 0) { f->status = MM_E_IO; f->error = std::string("cannot open ") + path; return f->status; }
    struct stat st;
    if (::fstat(fd, &st) == 0 && S_ISDIR(st.st_mode)) {
        // std::ifstream opens a directory and then reads nothing (no badbit):
        // the reference parses "" -> JSON parse error at line 1, column 1
        ::close(fd);
        return finish(f, "", 0);
    }
    if (S_ISREG(st.st_mode) && st.st_size > 0) {
        const size_t n = size_t(st.st_size);
        void* m = ::mmap(nullptr, n, PROT_READ, MAP_PRIVATE, fd, 0);
        if (m != MAP_FAILED) {
            ::close(fd);
            ::madvise(m, n, MADV_SEQUENTIAL);
            const mm_status r = finish(f, static_cast<const char*>(m), n);
            ::munmap(m, n);
            return r;
        }
    }
    std::string text;
    char buf[1 << 16];
    for (;;) {
        const ssize_t got = ::read(fd, buf, sizeof buf);
        if (got > 0) { text.append(buf, size_t(got)); continue; }
        if (got == 0) break;
        if (errno == EINTR) continue;
        ::close(fd);
        f->status = MM_E_IO;
        f->error = std::string("read error on ") + path;
        return f->status;
    }
    ::close(fd);
    return finish(f, text.data(), text.size());
}

void mm_facts_free(mm_facts* f) { delete f; }

mm_status mm_facts_status(const mm_facts* f) { return f ? f->status : MM_E_ARG; }

const char* mm_facts_error(const mm_facts* f) { return f ? f->error.c_str() : "null facts"; }

mm_status mm_facts_system(const mm_facts* f, mm_system* sys) {
    if (!f || !sys) return MM_E_ARG;
    if (f->status != MM_OK) return MM_E_STATE;
    sys->n_classes = f->C;
    sys->n_methods = f->M;
    sys->n_attributes = f->A;
    sys->reserved = 0;
    sys->method_owner = f->method_owner.data();
    sys->attribute_owner = f->attribute_owner.data();
    sys->class_method_off = f->cmoff.data();
    sys->class_methods = f->cmeth.data();
    sys->class_attr_off = f->caoff.data();
    sys->class_attrs = f->cattr.data();
    sys->call_off = f->call_off.data();
    sys->call_tgt = f->call_tgt.data();
    sys->acc_off = f->acc_off.data();
    sys->acc_tgt = f->acc_tgt.data();
    return MM_OK;
}

uint32_t mm_facts_violation_count(const mm_facts* f) { return f ? uint32_t(f->violations.size()) : 0; }

mm_status mm_facts_violation(const mm_facts* f, uint32_t i, int* kind, const char** message) {
    if (!f || i >= f->violations.size()) return MM_E_RANGE;
    if (kind) *kind = f->violations[i].first;
    if (message) *message = f->violations[i].second.c_str();
    return MM_OK;
}

uint32_t mm_facts_warning_count(const mm_facts* f) { return f ? uint32_t(f->warnings.size()) : 0; }

const char* mm_facts_warning(const mm_facts* f, uint32_t i) {
    return (f && i < f->warnings.size()) ? f->warnings[i].c_str() : nullptr;
}

const char* mm_facts_class_name(const mm_facts* f, uint32_t c, size_t* len) {
    if (!f || f->status != MM_OK || c >= f->C) return nullptr;
    return name_ptr(f, f->class_name[c], len);
}
const char* mm_facts_method_name(const mm_facts* f, uint32_t p, size_t* len) {
    if (!f || f->status != MM_OK || p >= f->M) return nullptr;
    return name_ptr(f, f->method_name[p], len);
}
const char* mm_facts_attribute_name(const mm_facts* f, uint32_t a, size_t* len) {
    if (!f || f->status != MM_OK || a >= f->A) return nullptr;
    return name_ptr(f, f->attribute_name[a], len);
}

// facts_to_json (facts.hpp:270-320): canonical, keys sorted, trailing newline.
mm_status mm_facts_to_json(const mm_facts* f, char* out, size_t cap, size_t* n_out) {
    if (!f || !n_out) return MM_E_ARG;
    if (f->status != MM_OK) return MM_E_STATE;
    std::string o;
    o.reserve(size_t(f->M) * 48 + size_t(f->A) * 24 + f->blob.size() + 64);
    o += "{\"classes\":[";
    for (uint32_t c = 0; c < f->C; ++c) {
        if (c) o += ',';
        o += "{\"attributes\":[";
        for (uint32_t i = f->caoff[c]; i < f->caoff[c + 1]; ++i) {
            const uint32_t a = f->cattr[i];
            if (i != f->caoff[c]) o += ',';
            o += "{\"id\":"; put_u(o, a);
            o += ",\"name\":"; quote(o, f->blob.data() + f->attribute_name[a].off, f->attribute_name[a].len);
            o += '}';
        }
        o += "],\"id\":"; put_u(o, f->class_ids[c]);
        o += ",\"methods\":[";
        for (uint32_t i = f->cmoff[c]; i < f->cmoff[c + 1]; ++i) {
            const uint32_t p = f->cmeth[i];
            if (i != f->cmoff[c]) o += ',';
            o += "{\"accesses\":[";
            for (uint32_t k = f->acc_off[p]; k < f->acc_off[p + 1]; ++k) { if (k != f->acc_off[p]) o += ','; put_u(o, f->acc_tgt[k]); }
            o += "],\"calls\":[";
            for (uint32_t k = f->call_off[p]; k < f->call_off[p + 1]; ++k) { if (k != f->call_off[p]) o += ','; put_u(o, f->call_tgt[k]); }
            o += "],\"id\":"; put_u(o, p);
            o += ",\"name\":"; quote(o, f->blob.data() + f->method_name[p].off, f->method_name[p].len);
            o += '}';
        }
        o += "],\"name\":"; quote(o, f->blob.data() + f->class_name[c].off, f->class_name[c].len);
        o += '}';
    }
    o += "],\"schema_version\":\"1\"}\n";
    *n_out = o.size();
    if (!out || cap < o.size()) return MM_E_CAPACITY;
    std::memcpy(out, o.data(), o.size());
    return MM_OK;
}

}  // extern "C"
