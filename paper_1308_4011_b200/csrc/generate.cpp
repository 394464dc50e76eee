// Host-side synthetic system generators (input synthesis, not the hot path).
//
// mm_generate with zipf_s == 0 reproduces the reference generator
// generate() (/root/reference/proj/include/modmetrics/generate.hpp:94-164)
// draw for draw: the same SplitMix64 stream (generate.hpp:17-37), round-robin
// ownership (:109-122), per-method call/access counts uniform in [0, k]
// (:131, :141), intra-class bias coin (:133, :143), pick rules
// pick_excluding / pick_foreign (:57-84), skipped draws and sort+unique
// (:155-160). tests/test_abi_cpu.py:50-71 pins it against the reference
// compiled in oracle/_ref and against committed golden hashes.
//
// zipf_s > 0 is the skewed variant used for config C3: class
// sizes ∝ 1/rank^s (min 1), ids shuffled across classes, dependencies drawn
// with the same rules as above. It is new (the reference has no Zipf
// generator); its output passes the reference validate().

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <new>
#include <vector>

#include "../../include/mmgpu.h"

namespace {

struct Rng {  // SplitMix64 (generate.hpp:17-37)
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        s += 0x9e3779b97f4a7c15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    uint64_t below(uint64_t n) { return next() % n; }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

}  // namespace

struct mm_host_system {
    std::vector<uint32_t> method_owner, attribute_owner;
    std::vector<uint32_t> class_method_off, class_methods, class_attr_off, class_attrs;
    std::vector<uint32_t> call_off, call_tgt, acc_off, acc_tgt;
    mm_system view{};
    void refresh() {
        view.n_classes = static_cast<uint32_t>(class_method_off.size() - 1);
        view.n_methods = static_cast<uint32_t>(method_owner.size());
        view.n_attributes = static_cast<uint32_t>(attribute_owner.size());
        view.method_owner = method_owner.data();
        view.attribute_owner = attribute_owner.data();
        view.class_method_off = class_method_off.data();
        view.class_methods = class_methods.data();
        view.class_attr_off = class_attr_off.data();
        view.class_attrs = class_attrs.data();
        view.call_off = call_off.data();
        view.call_tgt = call_tgt.data();
        view.acc_off = acc_off.data();
        view.acc_tgt = acc_tgt.data();
    }
};

namespace {

// Class-local pools: members of each class, sorted ascending (CSR).
struct Pools {
    std::vector<uint32_t> off, ids;
    const uint32_t* begin(uint32_t c) const { return ids.data() + off[c]; }
    uint32_t size(uint32_t c) const { return off[c + 1] - off[c]; }
};

Pools pools_from_owner(const std::vector<uint32_t>& owner, uint32_t n_classes) {
    Pools p;
    p.off.assign(n_classes + 1, 0);
    for (uint32_t o : owner) ++p.off[o + 1];
    for (uint32_t c = 0; c < n_classes; ++c) p.off[c + 1] += p.off[c];
    p.ids.resize(owner.size());
    std::vector<uint32_t> cur(p.off.begin(), p.off.end() - 1);
    for (uint32_t id = 0; id < owner.size(); ++id) p.ids[cur[owner[id]]++] = id;  // ascending
    return p;
}

// A member of `pool` other than `self` (generate.hpp:57-68 semantics: the
// index is drawn over the pool minus self, then shifted past self).
bool pick_other(Rng& rng, const uint32_t* pool, uint32_t n, uint32_t self, uint32_t& out) {
    const uint32_t* it = std::lower_bound(pool, pool + n, self);
    const bool has_self = it != pool + n && *it == self;
    const uint64_t avail = n - (has_self ? 1 : 0);
    if (avail == 0) return false;
    uint64_t k = rng.below(avail);
    if (has_self && k >= static_cast<uint64_t>(it - pool)) ++k;
    out = pool[k];
    return true;
}

// Rejection sampling for an entity owned elsewhere, 64 tries (generate.hpp:73-84).
bool pick_elsewhere(Rng& rng, const std::vector<uint32_t>& owner, uint32_t home, uint32_t& out) {
    if (owner.empty()) return false;
    for (int t = 0; t < 64; ++t) {
        const uint32_t cand = static_cast<uint32_t>(rng.below(owner.size()));
        if (owner[cand] != home) {
            out = cand;
            return true;
        }
    }
    return false;
}

void sort_unique(std::vector<uint32_t>& v) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
}

// Class sizes ∝ 1/(rank+1)^s summing to n, at least one per class when n >= c.
std::vector<uint32_t> zipf_sizes(uint32_t n, uint32_t c, double s) {
    std::vector<double> w(c);
    double W = 0.0;
    for (uint32_t r = 0; r < c; ++r) W += (w[r] = 1.0 / std::pow(double(r) + 1.0, s));
    std::vector<uint32_t> sz(c);
    uint64_t total = 0;
    const uint32_t floor_sz = n >= c ? 1u : 0u;
    for (uint32_t r = 0; r < c; ++r) {
        sz[r] = std::max<uint32_t>(floor_sz, static_cast<uint32_t>(std::floor(double(n) * w[r] / W)));
        total += sz[r];
    }
    for (uint32_t r = 0; total > n; r = (r + 1) % c)  // shave the biggest first
        if (sz[r] > floor_sz) { --sz[r]; --total; }
    for (uint32_t r = 0; total < n; r = (r + 1) % c) { ++sz[r]; ++total; }
    return sz;
}

std::vector<uint32_t> zipf_owner(uint32_t n, uint32_t c, double s, Rng& shuffle) {
    std::vector<uint32_t> perm(n);
    for (uint32_t i = 0; i < n; ++i) perm[i] = i;
    for (uint32_t i = n; i > 1; --i) std::swap(perm[i - 1], perm[shuffle.below(i)]);
    const std::vector<uint32_t> sz = zipf_sizes(n, c, s);
    std::vector<uint32_t> owner(n);
    uint32_t at = 0;
    for (uint32_t r = 0; r < c; ++r)
        for (uint32_t k = 0; k < sz[r]; ++k) owner[perm[at++]] = r;
    return owner;
}

}  // namespace

extern "C" mm_status mm_generate(const mm_gen_config* cfg, mm_host_system** out) {
    if (!cfg || !out) return MM_E_ARG;
    *out = nullptr;
    if (cfg->n_classes == 0) return MM_E_ARG;                                   // generate.hpp:96
    if (!(cfg->intra_class_bias >= 0.0 && cfg->intra_class_bias <= 1.0)) return MM_E_ARG;  // :98
    if (cfg->zipf_s < 0.0) return MM_E_ARG;
    mm_host_system* h = new (std::nothrow) mm_host_system();
    if (!h) return MM_E_OOM;
    try {
        const uint32_t C = cfg->n_classes, M = cfg->n_methods, A = cfg->n_attributes;
        if (cfg->zipf_s > 0.0) {
            Rng shuffle(cfg->seed ^ 0x5a17f00dd15ea5e5ULL);
            h->method_owner = zipf_owner(M, C, cfg->zipf_s, shuffle);
            h->attribute_owner = zipf_owner(A, C, cfg->zipf_s, shuffle);
        } else {
            h->method_owner.resize(M);
            h->attribute_owner.resize(A);
            for (uint32_t p = 0; p < M; ++p) h->method_owner[p] = p % C;   // round-robin
            for (uint32_t a = 0; a < A; ++a) h->attribute_owner[a] = a % C;
        }
        const Pools mp = pools_from_owner(h->method_owner, C);
        const Pools ap = pools_from_owner(h->attribute_owner, C);
        h->class_method_off = mp.off;
        h->class_methods = mp.ids;
        h->class_attr_off = ap.off;
        h->class_attrs = ap.ids;

        Rng rng(cfg->seed);
        h->call_off.assign(M + 1, 0);
        h->acc_off.assign(M + 1, 0);
        std::vector<uint32_t> calls, accs;
        for (uint32_t p = 0; p < M; ++p) {
            const uint32_t home = h->method_owner[p];
            calls.clear();
            accs.clear();
            const uint64_t nc = cfg->k_max_calls ? rng.below(uint64_t(cfg->k_max_calls) + 1) : 0;
            for (uint64_t i = 0; i < nc; ++i) {
                const bool stay = rng.unit() < cfg->intra_class_bias;
                uint32_t t;
                const bool ok = stay ? pick_other(rng, mp.begin(home), mp.size(home), p, t)
                                     : pick_elsewhere(rng, h->method_owner, home, t);
                if (ok) calls.push_back(t);
            }
            const uint64_t na = cfg->k_max_accesses ? rng.below(uint64_t(cfg->k_max_accesses) + 1) : 0;
            for (uint64_t i = 0; i < na; ++i) {
                const bool stay = rng.unit() < cfg->intra_class_bias;
                uint32_t t;
                if (stay) {
                    const uint32_t n = ap.size(home);
                    if (n == 0) continue;
                    t = ap.begin(home)[rng.below(n)];
                } else if (!pick_elsewhere(rng, h->attribute_owner, home, t)) {
                    continue;
                }
                accs.push_back(t);
            }
            sort_unique(calls);
            sort_unique(accs);
            h->call_tgt.insert(h->call_tgt.end(), calls.begin(), calls.end());
            h->acc_tgt.insert(h->acc_tgt.end(), accs.begin(), accs.end());
            h->call_off[p + 1] = static_cast<uint32_t>(h->call_tgt.size());
            h->acc_off[p + 1] = static_cast<uint32_t>(h->acc_tgt.size());
        }
        h->refresh();
    } catch (const std::bad_alloc&) {
        delete h;
        return MM_E_OOM;
    }
    *out = h;
    return MM_OK;
}

extern "C" const mm_system* mm_host_system_view(const mm_host_system* h) { return h ? &h->view : nullptr; }

extern "C" void mm_host_system_free(mm_host_system* h) { delete h; }
