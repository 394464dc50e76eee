// k_sweep.cu — the move-method candidate sweep and the single what-if.
//
// Replaces suggest_by_cohesion (suggest.hpp:239-259), suggest_by_coupling
// (:266-294), their merge in suggest_all (:303-350) and what_if_move
// (:87-122). Instead of re-running four LCOM and four CBO passes per
// candidate (the reference's what_if_move), every (u, d) pair is scored in
// O(|used(u)|·log|U[d]|) from the class tables of the metric pass
// (SURVEY.md Appendix A):
//   lcom_origin_after = lcom(A_o, M_o − 1, H_o − h_u(o))
//   lcom_dest_after   = lcom(A_d, M_d + 1, H_d + h_u(d))
//   cbo_origin_after  = cbo_o − #{X ∈ used(u)\{o} : U[o][X] == 1}
//   cbo_dest_after    = cbo_d + #{X ∈ used(u)\{d} : X ∉ U[d]}
// Ownership stays frozen as in the reference. Gates, predicates, keys and
// the (key, d) argmin with lowest-d tie-break follow suggest.hpp:165-196 and
// :285-290 bit for bit.
//
// One thread per method, methods in class-segment order (origin ascending,
// method id ascending within a class — the order suggest_all sorts into), so
// the emitted records come out already in (origin, method, destination)
// order. Output offsets come from a single-pass decoupled look-back scan over
// 256-method tiles: no atomics on the data, deterministic placement.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "mm_device.cuh"
#include "mm_kernels.h"

#ifndef MMGPU_SCORE_MINB
#define MMGPU_SCORE_MINB 4
#endif
#ifndef MMGPU_FAST_MINB
#define MMGPU_FAST_MINB 6
#endif
namespace mmg {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// Per-thread used list staged in shared memory (column-major over the tile
// so thread t's k-th entry sits at [k * kSweepTile + t]: conflict-free).
// Dynamic loops keep the kernel small and its register count low.
template <int S>
struct SmemEnumT {  // a method's used list in shared memory, stride S (the block size)
    static constexpr int kStride = S;
    uint32_t* X;
    uint32_t* H;
    int n;
    template <class F>
    __device__ __forceinline__ void each(F f) const {
#pragma unroll 1
        for (int k = 0; k < n; ++k) f(k, X[k * S], H[k * S]);
    }
    __device__ __forceinline__ uint32_t hits(uint32_t v) const {
        for (int k = 0; k < n; ++k)
            if (X[k * S] == v) return H[k * S];
        return 0;
    }
    // returns false when a new class would exceed `cap` distinct entries
    __device__ __forceinline__ bool insert(uint32_t v, uint32_t acc, int cap) {
        int k = 0;
        while (k < n && X[k * S] < v) ++k;
        if (k < n && X[k * S] == v) {
            H[k * S] += acc;
            return true;
        }
        if (n >= cap) return false;
        for (int j = n; j > k; --j) {
            X[j * S] = X[(j - 1) * S];
            H[j * S] = H[(j - 1) * S];
        }
        X[k * S] = v;
        H[k * S] = acc;
        ++n;
        return true;
    }
    // distinct used classes of p from the CSR (any degree); false if more than cap
    __device__ __forceinline__ bool build(const DevModel& s, uint32_t p, int cap) {
        n = 0;
        const uint32_t cb = __ldg(s.call_off + p), ce = __ldg(s.call_off + p + 1);
        for (uint32_t e = cb; e < ce; ++e)
            if (!insert(__ldg(s.method_owner + __ldg(s.call_tgt + e)), 0, cap)) return false;
        const uint32_t ab = __ldg(s.acc_off + p), ae = __ldg(s.acc_off + p + 1);
        for (uint32_t e = ab; e < ae; ++e)
            if (!insert(__ldg(s.attribute_owner + __ldg(s.acc_tgt + e)), 1, cap)) return false;
        return true;
    }
};
using SmemEnum = SmemEnumT<kSweepTile>;

struct StreamEnum {
    StreamUsed S;
    template <class F>
    __device__ __forceinline__ void each(F f) const {
        uint32_t prev = kNone, h = 0;
        for (int k = 0;; ++k) {
            const uint32_t x = S.next(prev, h);
            if (x == kNone) break;
            f(k, x, h);
            prev = x;
        }
    }
    __device__ __forceinline__ uint32_t hits(uint32_t v) const { return S.hits(v); }
};

struct Origin {
    ClassRec ro;
    double lo_b, lo_a;   // exact doubles (always filled; cheap: once per method)
    uint32_t co_b, co_a;
    bool odeg;
    bool coh_ok;         // lcom_origin_after < lcom_origin_before
};

struct Dest {
    double ld_b, ld_a;
    uint32_t cd_b, cd_a;
    bool ddeg;
};

constexpr uint64_t kExact53 = 1ull << 53;

// lcom(A, M−1, H−ho) < lcom(A, M, H) as the reference compares the doubles
// (suggest.hpp:189-192). Exact-rational pre-test: the rounded map q -> lcom is
// monotone, so q_after ≤ q_before already decides "false" without division.
__device__ __forceinline__ Origin make_origin(const ClassRec& ro, uint32_t ho, uint32_t removed) {
    Origin g;
    g.ro = ro;
    g.lo_b = lcom_of(ro.A, ro.M, ro.H);
    g.lo_a = lcom_of(ro.A, (uint64_t)ro.M - 1, (uint64_t)ro.H - ho);
    g.coh_ok = g.lo_a < g.lo_b;
    g.co_b = ro.cbo;
    g.co_a = ro.cbo - removed;
    g.odeg = ro.M <= 1 || ro.A == 0;  // origin_after.empty() || attrs empty (suggest.hpp:118-120)
    return g;
}

// The origin for scoring only (best / top-k / all-passing decisions): the
// exact-rational pre-test decides "lcom(origin) cannot drop" without a
// division (A == 0, or M ≥ 2 with exact denominators and H ≤ h·M); otherwise
// lo_a by the reference's formula and lo_b = lcom[o] from the metric pass
// (the same double). Emission uses make_origin (every field exact).
__device__ __forceinline__ Origin make_origin_score(const ClassRec& ro, uint32_t ho, uint32_t removed,
                                                   const double* __restrict__ dlcom, uint32_t o) {
    Origin g;
    g.ro = ro;
    g.lo_b = 0.0;
    g.lo_a = 0.0;
    g.coh_ok = false;
    bool maybe = ro.A != 0 && ro.M != 0;
    if (maybe && ro.M >= 2 && (uint64_t)ro.A * ro.M < kExact53) maybe = (uint64_t)ho * ro.M < ro.H;
    if (maybe) {
        g.lo_a = lcom_of(ro.A, (uint64_t)ro.M - 1, (uint64_t)ro.H - ho);
        g.lo_b = __ldg(dlcom + o);
        g.coh_ok = g.lo_a < g.lo_b;
    }
    g.co_b = ro.cbo;
    g.co_a = ro.cbo - removed;
    g.odeg = ro.M <= 1 || ro.A == 0;
    return g;
}

// lcom(A_d, M_d+1, H_d+h) < lcom(A_d, M_d, H_d): integer pre-test h·M > H
// (q_after > q_before), doubles only when it holds.
__device__ __forceinline__ bool coh_dest(const ClassRec& rd, uint32_t h, double& ld_a,
                                         const double* __restrict__ dlcom = nullptr, uint32_t d = 0) {
    if (rd.A == 0 || rd.M == 0) return false;  // before is 0.0 (degenerate): nothing is < 0
    const bool exact_denoms = (uint64_t)rd.A * ((uint64_t)rd.M + 1) < kExact53;
    if (exact_denoms && !((uint64_t)h * rd.M > rd.H)) return false;
    ld_a = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + h);
    // lcom_dest_before: the metric pass's lcom[d] (the same double) when given
    return ld_a < (dlcom ? __ldg(dlcom + d) : lcom_of(rd.A, rd.M, rd.H));
}

// X ∈ U[d]? Exact bitmap for dense rows; else the Bloom signature (a clear
// bit proves absence), then the row.
__device__ __forceinline__ bool in_urow(const ClassRec* __restrict__ rec, uint32_t d, const ClassRec& rd,
                                        const uint32_t* __restrict__ ux, const uint32_t* __restrict__ dense,
                                        uint32_t X) {
    if (rd.dense != kNone) return (__ldg(dense + rd.dense + (X >> 5)) >> (X & 31)) & 1u;
    if (!sig_maybe(rec, d, X)) return false;
    return urow_find(ux, rd.ubase, rd.cbo, X) >= 0;
}

// coupling predicate for destination d given co_a < co_b: cd_after <= cd_before
// ⟺ every X ∈ used(u) \ {d} is already in U[d] (miss == 0).
template <class E>
__device__ __forceinline__ bool coup_dest(const ClassRec* __restrict__ rec, const ClassRec& rd,
                                          const uint32_t* __restrict__ ux, const uint32_t* __restrict__ dense,
                                          const E& en, uint32_t d) {
    bool ok = true;
    en.each([&](int, uint32_t X, uint32_t) {
        if (ok && X != d && !in_urow(rec, d, rd, ux, dense, X)) ok = false;
    });
    return ok;
}

template <class E>
__device__ __forceinline__ Dest eval_dest(const ClassRec* __restrict__ rec, const uint32_t* __restrict__ ux,
                                          const uint32_t* __restrict__ dense, const E& en, uint32_t d, uint32_t hd) {
    const ClassRec rd = load_rec(rec, d);
    Dest r;
    r.ld_b = lcom_of(rd.A, rd.M, rd.H);
    r.ld_a = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + hd);
    uint32_t miss = 0;
    en.each([&](int, uint32_t X, uint32_t) {
        if (X != d && !in_urow(rec, d, rd, ux, dense, X)) ++miss;
    });
    r.cd_b = rd.cbo;
    r.cd_a = rd.cbo + miss;
    r.ddeg = rd.A == 0;
    return r;
}

// #{X ∈ used(u) \ {o} : U[o][X] == 1} from the rows (methods whose record
// could not carry it); a dense origin row answers from its singleton bitmap
template <class E>
__device__ __forceinline__ uint32_t removed_count(const ClassRec& ro, const uint32_t* __restrict__ ux,
                                                  const uint32_t* __restrict__ un,
                                                  const uint32_t* __restrict__ dense, uint32_t C, const E& en,
                                                  uint32_t o) {
    uint32_t removed = 0;
    if (ro.dense != kNone) {
        const uint32_t* single = dense + ro.dense + (C + 31) / 32;
        en.each([&](int, uint32_t X, uint32_t) {
            if (X != o) removed += (__ldg(single + (X >> 5)) >> (X & 31)) & 1u;
        });
        return removed;
    }
    en.each([&](int, uint32_t X, uint32_t) {
        if (X != o) {
            const int pos = urow_find(ux, ro.ubase, ro.cbo, X);
            if (pos >= 0 && __ldg(un + ro.ubase + pos) == 1u) ++removed;
        }
    });
    return removed;
}

// #{X ∈ list \ {o} : U[o][X] == 1} for a packed used list (records whose
// removed count the class pass did not fill in)
__device__ __forceinline__ uint32_t removed_from_list(const ClassRec& ro, const uint32_t* __restrict__ ux,
                                                      const uint32_t* __restrict__ un,
                                                      const uint32_t* __restrict__ dense, uint32_t C,
                                                      const uint32_t* ent, uint32_t n, uint32_t o) {
    uint32_t removed = 0;
    for (uint32_t k = 0; k < n; ++k) {
        const uint32_t X = ent[k] >> 8;
        if (X == o) continue;
        if (ro.dense != kNone) {
            removed += (__ldg(dense + ro.dense + (C + 31) / 32 + (X >> 5)) >> (X & 31)) & 1u;
        } else {
            const int p = urow_find(ux, ro.ubase, ro.cbo, X);
            if (p >= 0 && __ldg(un + ro.ubase + p) == 1u) ++removed;
        }
    }
    return removed;
}

// Both predicates and keys of one candidate (the shared core of the modes).
template <class E>
__device__ __forceinline__ void score(const SweepArgs& a, const E& en, const Origin& org, uint32_t d, uint32_t hd,
                                      bool& pcoh, double& kcoh, bool& pcoup, uint32_t& kcoup) {
    pcoh = pcoup = false;
    if (!org.coh_ok && org.co_a >= org.co_b) return;  // neither criterion can pass
    const ClassRec rd = load_rec(a.rec, d);
    double ld_a;
    if (org.coh_ok && coh_dest(rd, hd, ld_a, a.dlcom, d)) {
        pcoh = true;
        kcoh = __dadd_rn(org.lo_a, ld_a);  // lcom_key, suggest.hpp:194-196
    }
    if (org.co_a < org.co_b && coup_dest(a.rec, rd, a.ux, a.dense, en, d)) {
        pcoup = true;
        kcoup = rd.cbo;  // cbo_dest_after == cbo_dest_before when it passes
    }
}

// the next passing (key, index) strictly above (pk, pi) in lexicographic
// order for one criterion (top-k extension; k ≤ 8 rounds)
template <class E>
__device__ __forceinline__ int select_next(const SweepArgs& a, const E& en, uint32_t o, const Origin& org,
                                           bool coh, bool have_prev, double pk, int pi, double& out_key) {
    int best = -1;
    double bk = 0.0;
    en.each([&](int k, uint32_t d, uint32_t hd) {
        if (d == o) return;
        bool pc, pp;
        double kc = 0.0;
        uint32_t kp = 0;
        score(a, en, org, d, hd, pc, kc, pp, kp);
        const bool pass = coh ? pc : pp;
        const double key = coh ? kc : (double)kp;
        if (!pass) return;
        if (have_prev && !(key > pk || (key == pk && k > pi))) return;
        if (best < 0 || key < bk) { best = k; bk = key; }
    });
    out_key = bk;
    return best;
}

// Top-k / all-candidates modes keep the passing destinations as bit masks over
// the method's used-list index (bits 0..30). A method whose list has 32 or
// more entries ("wide", e.g. a hub calling into 100+ classes) instead keeps
// three counts — destinations passing only cohesion, only coupling, both —
// in a side table; k_offsets turns them into its record count under the
// class gates and k_write re-scores its candidates to emit them. No cap on
// the number of classes a method uses.
constexpr uint32_t kMaskBits = 31;
constexpr uint32_t kWideMark = 0x80000000u;  // res.x marker of a wide method (never a mask bit)
constexpr int kTopMax = 8;
// res.w of a best-only result whose method record is complete (entries,
// own-access and removed counts): k_offsets writes its records itself;
// 0 = k_write re-derives them from the CSR
constexpr uint32_t kResFull = 1u << 31;
constexpr uint32_t kEmitFast = 1u << 31;  // emitter list: written by k_write_best (positions < 2^31)

// records of a top-k / all-candidates method from its pass counts under the
// class gates: union = every gated pass, intersection = passes of both
__device__ __forceinline__ uint32_t wide_count(uint32_t n_co, uint32_t n_cp, uint32_t n_both, bool gcoh, bool gcoup,
                                               bool inter) {
    if (inter) return (gcoh && gcoup) ? n_both : 0u;
    return (gcoh ? n_co + n_both : 0u) + (gcoup ? n_cp + n_both : 0u) - ((gcoh && gcoup) ? n_both : 0u);
}

struct MethodResult {
    uint32_t count;
    uint32_t cands;
    uint32_t gated;
    uint32_t bd_coh, bd_coup;             // best-only mode
    unsigned long long m_coh, m_coup;     // top-k / all mode (bits over list index, narrow lists)
    uint32_t n_co, n_cp, n_both;          // top-k / all mode: passing only cohesion / only coupling / both
    uint32_t n_list;                      // used-list length (own class included)
};

// the k best passing list indices of one criterion, ascending by (key, index)
// (top-k extension; k ≤ kTopMax rounds of select_next)
template <class E>
__device__ __forceinline__ int select_topk(const SweepArgs& a, const E& en, uint32_t o, const Origin& org, bool coh,
                                           int* sel) {
    double pk = 0.0;
    int pi = -1, n = 0;
    for (uint32_t t = 0; t < a.topk && t < (uint32_t)kTopMax; ++t) {
        double key;
        const int k = select_next(a, en, o, org, coh, pi >= 0, pk, pi, key);
        if (k < 0) break;
        sel[n++] = k;
        pk = key;
        pi = k;
    }
    return n;
}

__device__ __forceinline__ bool in_sel(const int* sel, int n, int k) {
    bool f = false;
    for (int i = 0; i < n; ++i) f |= sel[i] == k;
    return f;
}

template <class E>
__device__ __forceinline__ MethodResult evaluate(const SweepArgs& a, const E& en, uint32_t o,
                                                 const Origin& org, bool gcoh, bool gcoup) {
    MethodResult r;
    r.bd_coh = r.bd_coup = kNone;
    r.m_coh = r.m_coup = 0;
    r.n_co = r.n_cp = r.n_both = 0;
    uint32_t cands = 0, n_list = 0;
    double best_coh = 0.0;
    uint32_t best_coup = 0;
    // every candidate is scored for both criteria (ungated); the class gates
    // only decide what is emitted
    en.each([&](int k, uint32_t d, uint32_t hd) {
        n_list = (uint32_t)k + 1;
        if (d == o) return;
        ++cands;
        bool pcoh, pcoup;
        double kc = 0.0;
        uint32_t kp = 0;
        score(a, en, org, d, hd, pcoh, kc, pcoup, kp);
        // argmin over (key, d), d ascending, strict < : lowest d wins ties (suggest.hpp:180-184)
        if (pcoh && (r.bd_coh == kNone || kc < best_coh)) { r.bd_coh = d; best_coh = kc; }
        if (pcoup && (r.bd_coup == kNone || kp < best_coup)) { r.bd_coup = d; best_coup = kp; }
        if (a.mode == 2) {
            if (k < (int)kMaskBits) {
                if (pcoh) r.m_coh |= 1ull << k;
                if (pcoup) r.m_coup |= 1ull << k;
            }
            r.n_both += pcoh && pcoup;
            r.n_co += pcoh && !pcoup;
            r.n_cp += pcoup && !pcoh;
        }
    });
    r.n_list = n_list;
    if (a.mode == 1) {
        int sc[kTopMax], sp[kTopMax];
        const int nc = gcoh ? select_topk(a, en, o, org, true, sc) : 0;
        const int np = gcoup ? select_topk(a, en, o, org, false, sp) : 0;
        for (int i = 0; i < nc; ++i)
            if (sc[i] < (int)kMaskBits) r.m_coh |= 1ull << sc[i];
        for (int i = 0; i < np; ++i)
            if (sp[i] < (int)kMaskBits) r.m_coup |= 1ull << sp[i];
        uint32_t both = 0;
        for (int i = 0; i < nc; ++i) both += in_sel(sp, np, sc[i]);
        r.n_both = both;
        r.n_co = (uint32_t)nc - both;
        r.n_cp = (uint32_t)np - both;
    }
    if (!gcoh) { r.bd_coh = kNone; r.m_coh = 0; }
    if (!gcoup) { r.bd_coup = kNone; r.m_coup = 0; }
    r.cands = cands;
    r.gated = cands * ((gcoh ? 1u : 0u) + (gcoup ? 1u : 0u));
    const bool both = (a.crit & MM_CRIT_COHESION) && (a.crit & MM_CRIT_COUPLING);
    const bool inter = a.combine == MM_COMBINE_INTERSECTION && both;
    uint32_t count;
    if (a.mode == 0) {
        const bool same = r.bd_coh != kNone && r.bd_coh == r.bd_coup;
        count = inter ? (same ? 1u : 0u)
                      : (uint32_t)(r.bd_coh != kNone) + (uint32_t)(r.bd_coup != kNone) - (same ? 1u : 0u);
    } else {
        count = wide_count(r.n_co, r.n_cp, r.n_both, gcoh, gcoup, inter);
    }
    r.count = count;
    return r;
}

__device__ __forceinline__ void store_record(mm_suggestion* dst, const mm_suggestion& s) {
    const uint4* src = reinterpret_cast<const uint4*>(&s);
    uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) d[i] = src[i];
}

// wide == true (top-k / all modes, lists of ≥ 32 entries): the passing
// destinations are re-derived here; r.m_coh / r.m_coup then hold the class
// gates (bit 0) instead of masks
template <class E>
__device__ __forceinline__ void emit(const SweepArgs& a, const E& en, uint32_t p, uint32_t o,
                                     const Origin& org, const MethodResult& r, uint64_t at, bool wide = false) {
    const bool both = (a.crit & MM_CRIT_COHESION) && (a.crit & MM_CRIT_COUPLING);
    const bool inter = a.combine == MM_COMBINE_INTERSECTION && both;
    int sc[kTopMax], sp[kTopMax], nc = 0, np = 0;
    if (wide && a.mode == 1) {
        if (r.m_coh) nc = select_topk(a, en, o, org, true, sc);
        if (r.m_coup) np = select_topk(a, en, o, org, false, sp);
    }
    en.each([&](int k, uint32_t d, uint32_t hd) {
        if (d == o) return;
        bool tcoh, tcoup;
        if (a.mode == 0) {
            tcoh = d == r.bd_coh;
            tcoup = d == r.bd_coup;
        } else if (!wide) {
            tcoh = k < (int)kMaskBits && ((r.m_coh >> k) & 1ull);
            tcoup = k < (int)kMaskBits && ((r.m_coup >> k) & 1ull);
        } else if (a.mode == 1) {
            tcoh = in_sel(sc, nc, k);
            tcoup = in_sel(sp, np, k);
        } else {
            bool pcoh, pcoup;
            double kc;
            uint32_t kp;
            score(a, en, org, d, hd, pcoh, kc, pcoup, kp);
            tcoh = pcoh && r.m_coh;
            tcoup = pcoup && r.m_coup;
        }
        if (inter ? !(tcoh && tcoup) : !(tcoh || tcoup)) return;
        const Dest dv = eval_dest(a.rec, a.ux, a.dense, en, d, hd);
        mm_suggestion s;
        s.lcom_origin_before = org.lo_b;
        s.lcom_origin_after = org.lo_a;
        s.lcom_dest_before = dv.ld_b;
        s.lcom_dest_after = dv.ld_a;
        s.method = p;
        s.origin = o;
        s.destination = d;
        s.cbo_origin_before = org.co_b;
        s.cbo_origin_after = org.co_a;
        s.cbo_dest_before = dv.cd_b;
        s.cbo_dest_after = dv.cd_a;
        s.criteria = (uint8_t)((tcoh ? MM_CRIT_COHESION : 0u) | (tcoup ? MM_CRIT_COUPLING : 0u));
        s.origin_degenerate_after = org.odeg;
        s.dest_degenerate_after = dv.ddeg;
        s.pad = 0;
        store_record(a.out + at, s);
        ++at;
    });
}

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += y;
    }
    return v;
}

// Fills `ren` (shared-memory list) or `sen` (streaming) with method p's used
// list and returns the origin-side values. Record path when the method pass
// could pack the list; CSR otherwise.
template <int K, bool SCORE = false, class REN>
__device__ __forceinline__ bool load_method(const SweepArgs& a, uint32_t pos, uint32_t p, uint32_t o,
                                            REN& ren, StreamEnum& sen, Origin& org) {
    const uint4* rp = reinterpret_cast<const uint4*>(a.recs + pos);
    const uint4 r0 = rp[0], r1 = rp[1];
    const uint32_t hdr = rec_hdrs(a.recs, a.s.M)[pos];
    const ClassRec ro = load_rec(a.rec, o);
    if (!(hdr & kRecOverflow)) {
        const uint32_t ent[kRecMaxEnt] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        const uint32_t n = rec_n(hdr);
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k)
            if (k < (int)n) { ren.X[k * REN::kStride] = ent[k] >> 8; ren.H[k * REN::kStride] = ent[k] & 0xffu; }
        ren.n = (int)n;
        const uint32_t removed = (hdr & kRecRemovedValid) ? rec_removed(hdr)
                                                           : removed_count(ro, a.ux, a.un, a.dense, a.s.C, ren, o);
        org = SCORE ? make_origin_score(ro, rec_hown(hdr), removed, a.dlcom, o) : make_origin(ro, rec_hown(hdr), removed);
        return true;
    }
    if (ren.build(a.s, p, K)) {  // ≤ K distinct classes (any degree): shared-memory list
        org = make_origin(ro, ren.hits(o), removed_count(ro, a.ux, a.un, a.dense, a.s.C, ren, o));
        return true;
    }
    sen.S.init(a.s, p);
    org = make_origin(ro, sen.hits(o), removed_count(ro, a.ux, a.un, a.dense, a.s.C, sen, o));
    return false;
}

// Pass 1: score every candidate of every method (ungated, both criteria) and
// keep the per-method best / top-k / all-passing destinations. Independent
// of the thresholds, so it overlaps the threshold kernel on another stream.
// One method per thread, its used list in shared memory: small per-thread
// state and high occupancy measured faster on C4 than a warp-flattened
// variant (one candidate per lane), the round-1 profiles show why — every
// kernel here is latency-bound, so resident warps matter most. Blocks of
// kScoreTile threads: per-method work is uneven (C5: up to 16 used classes,
// each destination checked against the others), and a block keeps its shared
// memory and registers until its slowest warp ends, so small blocks keep more
// warps resident (C5 at 256 threads: 14.8 of 32 possible warps per SM).
#ifndef MMGPU_SCORE_TILE
#define MMGPU_SCORE_TILE 64
#endif
constexpr int kScoreTile = MMGPU_SCORE_TILE;
static_assert(kSweepTile % kScoreTile == 0, "score tile divides the sweep tile");
template <int K, bool LIST = false>
__global__ void __launch_bounds__(kScoreTile, MMGPU_SCORE_MINB * (kSweepTile / kScoreTile)) k_score_thread(SweepArgs a) {
    __shared__ uint32_t s_X[K * kScoreTile], s_H[K * kScoreTile];
    uint64_t pos;
    bool live;
    if (LIST) {  // the methods k_score_fast handed over (record overflow)
        const uint32_t i = blockIdx.x * kScoreTile + threadIdx.x;
        live = i < *a.n_fallback;
        pos = live ? a.fallback[i] : 0;
    } else {
        pos = (uint64_t)a.pos_begin + (uint64_t)blockIdx.x * kScoreTile + threadIdx.x;
        live = pos < a.pos_end;
    }
    uint32_t cands = 0;
    if (live) {
        const uint32_t p = __ldg(a.s.cls_methods + pos);
        const uint32_t o = __ldg(a.pos_owner + pos);
        SmemEnumT<kScoreTile> ren{s_X + threadIdx.x, s_H + threadIdx.x, 0};
        StreamEnum sen;
        Origin org;
        MethodResult r;
        uint32_t fw = 0;
        const uint32_t hdr = rec_hdrs(a.recs, a.s.M)[pos];
        if (load_method<K, true>(a, (uint32_t)pos, p, o, ren, sen, org)) r = evaluate(a, ren, o, org, true, true);
        else r = evaluate(a, sen, o, org, true, true);
        // the record writer can work from the method's record alone
        if (!(hdr & kRecOverflow) && (hdr & kRecRemovedValid)) fw = kResFull;
        cands = r.cands;
        uint4 out;
        if (a.mode == 0) {
            out = make_uint4(r.bd_coh, r.bd_coup, r.cands, fw);
        } else if (r.n_list > kMaskBits) {  // wide: counts in the side table
            const uint32_t slot = atomicAdd(a.n_wide, 1u);
            a.wide_cnt[slot] = make_uint4(r.n_co, r.n_cp, r.n_both, (uint32_t)pos);
            out = make_uint4(kWideMark | slot, 0u, r.cands, 0);
        } else {
            out = make_uint4((uint32_t)r.m_coh, (uint32_t)r.m_coup, r.cands, 0);
        }
        a.res[pos] = out;
    }
    const uint32_t wc = __reduce_add_sync(0xffffffffu, cands);
    if ((threadIdx.x & 31) == 0 && wc) atomicAdd(a.stats + 0, (unsigned long long)wc);
}

// Pass 1, best-only mode (the reference's default and the bench step), for
// every method whose record the metric pass completed (≤ 8 used classes,
// own-access and removed counts valid — every method of the generator's
// k ≤ 4 + 4 configurations): one method per thread, everything in registers.
// The packed used list (class order: one coalesced 32-byte record), the
// origin's counts (neighbouring threads share them: L1), the exact-rational
// origin pre-test h·M < H before the one lcom_origin_after division, then per
// destination d (ascending): d's counts, the cohesion pre-test h_u(d)·M_d > H_d
// before the lcom_dest_after division, and — when the method can lower its
// origin's cbo (removed > 0) — every other used class checked against U[d]
// (exact bitmap of a dense row, else the Bloom signature, the row only on a
// positive). Argmin over (key, d) with strict < in ascending d
// (suggest.hpp:180-184). Incomplete records go to k_score_thread's list.
#ifndef MMGPU_FAST_TILE
#define MMGPU_FAST_TILE 64
#endif
constexpr int kFastTile = MMGPU_FAST_TILE;  // block size of k_score_fast (64: C4 scoring 62.5 -> 60 us against 256, uneven per-method work)
static_assert(kSweepTile % kFastTile == 0, "fast-score tile divides the sweep tile");
__global__ void __launch_bounds__(kFastTile, MMGPU_FAST_MINB * (kSweepTile / kFastTile)) k_score_fast(SweepArgs a) {
    // the used list column-major in shared memory (thread t's k-th entry at
    // [k][t]: conflict-free), so the candidate and membership loops stay
    // rolled: small code, lanes of a warp in step
    __shared__ uint32_t s_ent[kRecMaxEnt][kFastTile];
    const uint32_t pos = a.pos_begin + blockIdx.x * kFastTile + threadIdx.x;
    const bool live = pos < a.pos_end;
    const int lane = threadIdx.x & 31;
    uint32_t hdr = kRecOverflow;
    if (live) hdr = rec_hdrs(a.recs, a.s.M)[pos];
    const bool fb = live && ((hdr & kRecOverflow) || !(hdr & kRecRemovedValid));
    const uint32_t fbm = __ballot_sync(0xffffffffu, fb);
    if (fbm) {  // the general per-thread kernel takes these (CSR path)
        uint32_t base = 0;
        if (lane == __ffs(fbm) - 1) base = atomicAdd(a.n_fallback, (uint32_t)__popc(fbm));
        base = __shfl_sync(0xffffffffu, base, __ffs(fbm) - 1);
        if (fb) a.fallback[base + __popc(fbm & ((1u << lane) - 1u))] = pos;
    }
    uint32_t cands = 0;
    if (live && !fb) {
        const uint4* rp = reinterpret_cast<const uint4*>(a.recs + pos);
        const uint4 r0 = rp[0], r1 = rp[1];
        const uint32_t o = __ldg(a.pos_owner + pos);
        const uint4 ro = __ldg(reinterpret_cast<const uint4*>(a.rec + o));  // A, M, H, cbo
        const uint32_t n = rec_n(hdr), hown = rec_hown(hdr);
        uint32_t* E = &s_ent[0][threadIdx.x];
        E[0 * kFastTile] = r0.x; E[1 * kFastTile] = r0.y; E[2 * kFastTile] = r0.z; E[3 * kFastTile] = r0.w;
        E[4 * kFastTile] = r1.x; E[5 * kFastTile] = r1.y; E[6 * kFastTile] = r1.z; E[7 * kFastTile] = r1.w;
        // origin side (make_origin_score)
        bool coh_ok = false;
        double lo_a = 0.0;
        if (ro.x != 0 && ro.y != 0) {
            bool maybe = true;
            if (ro.y >= 2 && (uint64_t)ro.x * ro.y < kExact53) maybe = (uint64_t)hown * ro.y < ro.z;
            if (maybe) {
                lo_a = lcom_of(ro.x, (uint64_t)ro.y - 1, (uint64_t)ro.z - hown);
                coh_ok = lo_a < __ldg(a.dlcom + o);
            }
        }
        const bool can_coup = rec_removed(hdr) > 0;
        uint32_t bd_coh = kNone, bd_coup = kNone, bkp = 0;
        double bkc = 0.0;
#pragma unroll 1
        for (uint32_t k = 0; k < n; ++k) {
            const uint32_t d = E[k * kFastTile] >> 8;
            if (d == o) continue;
            ++cands;
            if (!coh_ok && !can_coup) continue;
            const uint32_t h = E[k * kFastTile] & 0xffu;
            // the first other used class's two signature words requested with d's
            // record (their addresses need only d and X): the common coupling
            // rejection then costs one memory round trip, not two
            uint32_t X0 = kNone, sw1 = 0, sw2 = 0, sb1 = 0, sb2 = 0;
            if (can_coup) {
                X0 = E[0] >> 8;
                if (X0 == d) X0 = n > 1 ? E[kFastTile] >> 8 : kNone;
                if (X0 != kNone) {
                    sb1 = bloom_h1(X0);
                    sb2 = bloom_h2(X0);
                    sw1 = __ldg(a.rec[d].sig + (sb1 >> 5));
                    sw2 = __ldg(a.rec[d].sig + (sb2 >> 5));
                }
            }
            const ClassRec rd = load_rec(a.rec, d);
            if (coh_ok && rd.A != 0 && rd.M != 0) {  // coh_dest
                const bool exact = (uint64_t)rd.A * ((uint64_t)rd.M + 1) < kExact53;
                if (!exact || (uint64_t)h * rd.M > rd.H) {
                    const double ld_a = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + h);
                    if (ld_a < __ldg(a.dlcom + d)) {
                        const double kc = __dadd_rn(lo_a, ld_a);  // lcom_key
                        if (bd_coh == kNone || kc < bkc) { bd_coh = d; bkc = kc; }
                    }
                }
            }
            if (can_coup && (bd_coup == kNone || rd.cbo < bkp)) {  // cbo_dest_after == cbo_d when it passes
                // a clear prefetched Bloom bit proves X0 ∉ U[d] (Bloom rows only)
                bool okc = X0 == kNone || rd.dense != kNone || (((sw1 >> (sb1 & 31)) & (sw2 >> (sb2 & 31)) & 1u) != 0);
#pragma unroll 1
                for (uint32_t j = 0; j < n && okc; ++j) {
                    const uint32_t X = E[j * kFastTile] >> 8;
                    if (X != d) okc = in_urow(a.rec, d, rd, a.ux, a.dense, X);
                }
                if (okc) { bd_coup = d; bkp = rd.cbo; }
            }
        }
        a.res[pos] = make_uint4(bd_coh, bd_coup, cands, kResFull);
    }
    const uint32_t wc = __reduce_add_sync(0xffffffffu, cands);
    if (lane == 0 && wc) atomicAdd(a.stats + 0, (unsigned long long)wc);
}

// Pass 2: apply the class gates (suggest.hpp:246, :273) and the criteria
// merge (union / intersection, :315-341) to each method's pass-1 result,
// then a tile scan + decoupled look-back gives every EMITTING method a slot in
// a compact emitter list — (position, gated selection, offset of its first
// record) — both counts travel packed in one 64-bit look-back word. 1024
// methods per tile (4 per thread) keep the look-back chain short; res is only
// read.
// Best-only records of one method straight from its pass-1 result (kResFull):
// the method's packed used list, the origin's and destinations' class
// records, the two lcom divisions, and cbo_dest_after = cbo_d + #{X ∈
// used(u) \ {d} : X ∉ U[d]} (0 for a coupling pass; exact bitmap, or Bloom
// then the row). Records in ascending destination order (suggest.hpp:343-349).
__device__ __forceinline__ void write_best(const SweepArgs& a, uint32_t pos, uint32_t dc, uint32_t dp, uint64_t at) {
    // every load that depends only on the emitter first (one memory round trip)
    const uint32_t o = __ldg(a.pos_owner + pos), p = __ldg(a.s.cls_methods + pos);
    const uint32_t hdr = rec_hdrs(a.recs, a.s.M)[pos];
    const uint4* rp = reinterpret_cast<const uint4*>(a.recs + pos);
    const uint4 r0 = rp[0], r1 = rp[1];
    const uint32_t d1 = dc != kNone ? dc : dp;                       // first destination in the record order
    const uint32_t d2 = (dc != kNone && dp != kNone && dc != dp) ? dp : kNone;
    const uint32_t da = (d2 != kNone && d2 < d1) ? d2 : d1, db = (d2 != kNone && d2 < d1) ? d1 : d2;
    const ClassRec ra = load_rec(a.rec, da);
    ClassRec rb = ra;
    double lb_b = 0.0;
    if (db != kNone) { rb = load_rec(a.rec, db); lb_b = __ldg(a.dlcom + db); }
    const double la_b = __ldg(a.dlcom + da);
    const uint4 ro = __ldg(reinterpret_cast<const uint4*>(a.rec + o));
    const double lo_b = __ldg(a.dlcom + o);
    const uint32_t ent[kRecMaxEnt] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    const uint32_t n = rec_n(hdr);
    mm_suggestion s;
    s.lcom_origin_before = lo_b;
    s.lcom_origin_after = lcom_of(ro.x, (uint64_t)ro.y - 1, (uint64_t)ro.z - rec_hown(hdr));
    s.method = p;
    s.origin = o;
    s.cbo_origin_before = ro.w;
    s.cbo_origin_after = ro.w - rec_removed(hdr);
    s.origin_degenerate_after = ro.y <= 1 || ro.x == 0;
    s.pad = 0;
    auto one = [&](uint32_t d, const ClassRec& rd, double ld_b) {
        const bool coh = d == dc, coup = d == dp;
        uint32_t h = 0, miss = 0;
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k) {
            if ((uint32_t)k >= n) break;
            const uint32_t X = ent[k] >> 8;
            if (X == d) { h = ent[k] & 0xffu; continue; }
            if (!coup && !in_urow(a.rec, d, rd, a.ux, a.dense, X)) ++miss;  // a coupling pass has none
        }
        s.lcom_dest_before = ld_b;
        s.lcom_dest_after = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + h);
        s.destination = d;
        s.cbo_dest_before = rd.cbo;
        s.cbo_dest_after = rd.cbo + miss;
        s.criteria = (uint8_t)((coh ? MM_CRIT_COHESION : 0u) | (coup ? MM_CRIT_COUPLING : 0u));
        s.dest_degenerate_after = rd.A == 0;
        store_record(a.out + at, s);
        ++at;
    };
    // records in ascending destination order (suggest.hpp:343-349); the count
    // k_offsets made excludes the intersection case where dc != dp
    one(da, ra, la_b);
    if (db != kNone) one(db, rb, lb_b);
}

#ifndef MMGPU_OFF_ITEMS
#define MMGPU_OFF_ITEMS 8
#endif
constexpr int kOffItems = MMGPU_OFF_ITEMS;  // 8: 2048-position tiles (489 for 1M methods; 16 measured 1.7 µs slower on C4, 5 µs on C5: fewer resident warps)
constexpr uint32_t kOffTile = kSweepTile * kOffItems;

// one method's pass-1 result under the class gates and the criteria merge:
// the emitter's selection words and the record count
__device__ __forceinline__ uint4 gate_result(const SweepArgs& a, uint4 v, bool gcoh, bool gcoup, bool inter,
                                             uint32_t& count) {
    if (a.mode == 0) {
        const uint32_t bc = gcoh ? v.x : kNone, bp = gcoup ? v.y : kNone;
        const bool same = bc != kNone && bc == bp;
        count = inter ? (same ? 1u : 0u) : (uint32_t)(bc != kNone) + (uint32_t)(bp != kNone) - (same ? 1u : 0u);
        v.x = bc;
        v.y = bp;
    } else if (v.x & kWideMark) {
        const uint4 wc = a.wide_cnt[v.x & ~kWideMark];
        count = wide_count(wc.x, wc.y, wc.z, gcoh, gcoup, inter);
        v.x = kWideMark | (gcoh ? 1u : 0u);  // k_write re-derives the destinations under these gates
        v.y = gcoup ? 1u : 0u;
    } else {
        v.x = gcoh ? v.x : 0u;
        v.y = gcoup ? v.y : 0u;
        count = __popc(inter ? (v.x & v.y) : (v.x | v.y));
    }
    return v;
}

__global__ void __launch_bounds__(kSweepTile) k_offsets(SweepArgs a) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_warp[kSweepTile / 32];
    __shared__ unsigned long long s_excl;
    __shared__ unsigned long long s_red[2][kSweepTile / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t pos0 = (uint64_t)a.pos_begin + (uint64_t)tile * kOffTile + (uint64_t)threadIdx.x * kOffItems;

    double thr_l = a.thr_lcom, thr_c = a.thr_cbo;
    if (a.thr_device) { thr_l = a.dthr->lcom; thr_c = a.dthr->cbo; }
    const bool both = (a.crit & MM_CRIT_COHESION) && (a.crit & MM_CRIT_COUPLING);
    const bool inter = a.combine == MM_COMBINE_INTERSECTION && both;

    // pass A: counts (the gated results are recomputed in pass C from the
    // same reads — cache hits — instead of holding 16 of them in registers)
    uint32_t cnt[kOffItems];
    uint32_t gates = 0;  // bit 2·it: cohesion gate, bit 2·it + 1: coupling gate
    unsigned long long mine = 0, gated = 0, nvalid = 0;  // packed (emitters << 32) | records
#pragma unroll
    for (int it = 0; it < kOffItems; ++it) {
        const uint64_t pos = pos0 + it;
        cnt[it] = 0;
        if (pos >= a.pos_end) continue;
        ++nvalid;
        const uint4 v = a.res[pos];
        const uint32_t o = __ldg(a.pos_owner + pos);
        const bool gcoh = (a.crit & MM_CRIT_COHESION) && __ldg(a.lcom + o) > thr_l;
        const bool gcoup = (a.crit & MM_CRIT_COUPLING) && (double)__ldg(a.cbo + o) > thr_c;
        gates |= ((gcoh ? 1u : 0u) | (gcoup ? 2u : 0u)) << (2 * it);
        gated += v.z * ((gcoh ? 1u : 0u) + (gcoup ? 1u : 0u));
        uint32_t count;
        gate_result(a, v, gcoh, gcoup, inter, count);
        cnt[it] = count;
        mine += count + (count ? (1ull << 32) : 0ull);
    }
    // pass B: block scan of the packed pair, decoupled look-back
    unsigned long long inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    {
        unsigned long long g0 = gated, g1 = nvalid;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            g0 += __shfl_down_sync(0xffffffffu, g0, d);
            g1 += __shfl_down_sync(0xffffffffu, g1, d);
        }
        if (lane == 0) { s_red[0][warp] = g0; s_red[1][warp] = g1; }
    }
    __syncthreads();
    unsigned long long before = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kSweepTile / 32; ++w) {
        if (w < warp) before += s_warp[w];
        agg += s_warp[w];
    }
    const unsigned long long texcl = before + inc - mine;
    // warp 0 inspects 32 predecessor tiles per step (relaxed gpu-scope loads;
    // flag and value share one 64-bit word)
    if (warp == 0) {
        unsigned long long excl = 0;
        if (tile == 0) {
            if (lane == 0) st_relaxed_u64(a.tile_state, kFlagPrefix | agg);
        } else {
            if (lane == 0) st_relaxed_u64(a.tile_state + tile, kFlagAgg | agg);
            int base = (int)tile - 1;
            while (true) {
                const int j = base - lane;
                const unsigned long long v = j >= 0 ? ld_relaxed_u64(a.tile_state + j) : kFlagPrefix;
                const unsigned long long f = v & ~kValMask;
                const uint32_t bP = __ballot_sync(0xffffffffu, f == kFlagPrefix);
                const uint32_t bZ = __ballot_sync(0xffffffffu, f == 0);
                const int lim = bP ? __ffs(bP) - 1 : 31;
                const uint32_t need = lim == 31 ? 0xffffffffu : ((2u << lim) - 1);
                if (bZ & need) continue;
                unsigned long long part = lane <= lim ? (v & kValMask) : 0ull;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) part += __shfl_down_sync(0xffffffffu, part, d);
                excl += __shfl_sync(0xffffffffu, part, 0);
                if (bP) break;
                base -= 32;
            }
            if (lane == 0) st_relaxed_u64(a.tile_state + tile, kFlagPrefix | (excl + agg));
        }
        if (lane == 0) {
            s_excl = excl;
            unsigned long long t0 = 0, t1 = 0;
            for (int w = 0; w < kSweepTile / 32; ++w) { t0 += s_red[0][w]; t1 += s_red[1][w]; }
            atomicAdd(a.stats + 1, t0);
            atomicAdd(a.stats + 2, agg & 0xffffffffull);
            atomicAdd(a.stats + 3, t1);
            atomicAdd(a.n_emit, (uint32_t)(agg >> 32));
        }
    }
    __syncthreads();
    // pass C: the emitters' compact records
    unsigned long long at = s_excl + texcl;
#pragma unroll
    for (int it = 0; it < kOffItems; ++it) {
        const uint64_t pos = pos0 + it;
        if (pos >= a.pos_end) continue;
        if (cnt[it]) {  // (position | fast flag, gated selection, first record)
            uint32_t count;
            const uint4 v = gate_result(a, a.res[pos], (gates >> (2 * it)) & 1u, (gates >> (2 * it + 1)) & 1u, inter,
                                        count);
            // best-only results whose method record is complete: k_write_best
            const uint32_t fast = (a.mode == 0 && (v.w & kResFull)) ? kEmitFast : 0u;
            a.emitters[at >> 32] = make_uint4((uint32_t)pos | fast, v.x, v.y, (uint32_t)(at & 0xffffffffull));
        }
        at += cnt[it] + (cnt[it] ? (1ull << 32) : 0ull);
    }
}

// Pass 3: the emitting methods (compact list from pass 2) write their
// records — exact what-if values — at their offsets. One thread per emitter.
template <int K>
__global__ void __launch_bounds__(kSweepTile) k_write(SweepArgs a) {
    __shared__ uint32_t s_X[K * kSweepTile], s_H[K * kSweepTile];
    const uint32_t n = *a.n_emit;
    for (uint32_t i = blockIdx.x * kSweepTile + threadIdx.x; i < n; i += gridDim.x * kSweepTile) {
        const uint4 em = a.emitters[i];
        if (em.x & kEmitFast) continue;  // k_write_best
        const uint32_t pos = em.x;
        const uint4 r = make_uint4(em.y, em.z, 0u, em.w);
        const uint32_t o = __ldg(a.pos_owner + pos);
        const uint32_t p = __ldg(a.s.cls_methods + pos);
        MethodResult res{};
        const bool wide = a.mode != 0 && (r.x & kWideMark);
        if (a.mode == 0) { res.bd_coh = r.x; res.bd_coup = r.y; }
        else if (wide) { res.m_coh = r.x & 1u; res.m_coup = r.y & 1u; }
        else { res.m_coh = r.x; res.m_coup = r.y; }
        SmemEnum ren{s_X + threadIdx.x, s_H + threadIdx.x, 0};
        StreamEnum sen;
        Origin org;
        if (load_method<K>(a, pos, p, o, ren, sen, org)) emit(a, ren, p, o, org, res, r.w, wide);
        else emit(a, sen, p, o, org, res, r.w, wide);
    }
}

// Pass 3, best-only records of complete-record methods (kEmitFast): one
// thread per emitter, register-light (write_best).
__global__ void __launch_bounds__(kSweepTile) k_write_best(SweepArgs a) {
    const uint32_t n = *a.n_emit;
    for (uint32_t i = blockIdx.x * kSweepTile + threadIdx.x; i < n; i += gridDim.x * kSweepTile) {
        const uint4 em = a.emitters[i];
        if (!(em.x & kEmitFast)) continue;
        write_best(a, em.x & ~kEmitFast, em.y, em.z, em.w);
    }
}

__global__ void k_what_if(DevModel s, const ClassRec* __restrict__ rec, const uint32_t* __restrict__ ux,
                          const uint32_t* __restrict__ un, const uint32_t* __restrict__ dense, uint32_t u,
                          uint32_t o, uint32_t d, mm_whatif* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (s.method_owner[u] != o) {  // not a member of the origin: invalid_argument (suggest.hpp:93-96)
        mm_whatif w{};
        w.pad[0] = 1;
        *out = w;
        return;
    }
    StreamEnum en;
    en.S.init(s, u);
    const ClassRec ro = load_rec(rec, o);
    const Origin org = make_origin(ro, en.hits(o), removed_count(ro, ux, un, dense, s.C, en, o));
    const Dest dv = eval_dest(rec, ux, dense, en, d, en.hits(d));
    mm_whatif w;
    w.lcom_origin_before = org.lo_b;
    w.lcom_origin_after = org.lo_a;
    w.lcom_dest_before = dv.ld_b;
    w.lcom_dest_after = dv.ld_a;
    w.cbo_origin_before = org.co_b;
    w.cbo_origin_after = org.co_a;
    w.cbo_dest_before = dv.cd_b;
    w.cbo_dest_after = dv.cd_a;
    w.origin_degenerate_after = org.odeg;
    w.dest_degenerate_after = dv.ddeg;
    for (int i = 0; i < 6; ++i) w.pad[i] = 0;
    *out = w;
}

// ---- the similarity criterion (suggest_by_similarity, suggest.hpp:200-232) ----
// A stored pair above the threshold whose methods live in different classes
// makes both methods candidates; each candidate's destinations are the other
// method's class plus the owners of what it calls, and a move passes when it
// strictly lowers both lcoms (lcom_improves, key lcom_key — the cohesion
// test). lcom_dest_after < lcom_dest_before needs h_u(d)·M_d > H_d, so only
// destinations that own an attribute u accesses can pass: the candidates are
// the used-list entries with h > 0 that are a partner's class or a callee's.

// partners: per method, the classes of its above-threshold partners
__global__ void k_sim_partner_count(const mm_similarity* __restrict__ tab, uint64_t n, double thr,
                                    const uint32_t* __restrict__ owner, uint32_t* __restrict__ cnt) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const mm_similarity e = tab[k];
        if (!(e.value > thr) || owner[e.first] == owner[e.second]) continue;  // suggest.hpp:217-218
        atomicAdd(cnt + e.first, 1u);
        atomicAdd(cnt + e.second, 1u);
    }
}

__global__ void k_sim_partner_fill(const mm_similarity* __restrict__ tab, uint64_t n, double thr,
                                   const uint32_t* __restrict__ owner, uint32_t* __restrict__ cur,
                                   uint32_t* __restrict__ part) {
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const mm_similarity e = tab[k];
        const uint32_t of = owner[e.first], os = owner[e.second];
        if (!(e.value > thr) || of == os) continue;
        part[atomicAdd(cur + e.first, 1u)] = os;
        part[atomicAdd(cur + e.second, 1u)] = of;
    }
}

struct SimCrit {
    const uint32_t* part_off;  // by method id
    const uint32_t* part;
    uint32_t* rec_cnt;         // pass 0: records per method id
    const uint32_t* rec_off;   // pass 1: first record of each method id
    uint32_t all_candidates;
};

// pass 0 counts each candidate method's records, pass 1 writes them (the
// reference's order: methods ascending, destinations ascending)
template <int K, int PASS>
__global__ void __launch_bounds__(kSweepTile) k_sim_emit(SweepArgs a, SimCrit sc) {
    __shared__ uint32_t s_X[K * kSweepTile], s_H[K * kSweepTile];
    const uint64_t pos = (uint64_t)a.pos_begin + (uint64_t)blockIdx.x * kSweepTile + threadIdx.x;
    if (pos >= a.pos_end) return;
    const uint32_t p = __ldg(a.s.cls_methods + pos);
    const uint32_t pb = sc.part_off[p], pe = sc.part_off[p + 1];
    if (pb == pe) return;  // no partner above the threshold
    const uint32_t o = __ldg(a.pos_owner + pos);
    SmemEnum ren{s_X + threadIdx.x, s_H + threadIdx.x, 0};
    StreamEnum sen;
    Origin org;
    const bool smem = load_method<K>(a, (uint32_t)pos, p, o, ren, sen, org);
    const uint32_t cb = __ldg(a.s.call_off + p), ce = __ldg(a.s.call_off + p + 1);
    auto run = [&](const auto& en) {
        uint32_t n = 0, best = kNone, best_h = 0;
        double best_key = 0.0;
        uint64_t at = PASS ? sc.rec_off[p] : 0;
        auto emit_one = [&](uint32_t d, uint32_t hd) {
            const Dest dv = eval_dest(a.rec, a.ux, a.dense, en, d, hd);
            mm_suggestion r;
            r.lcom_origin_before = org.lo_b;
            r.lcom_origin_after = org.lo_a;
            r.lcom_dest_before = dv.ld_b;
            r.lcom_dest_after = dv.ld_a;
            r.method = p;
            r.origin = o;
            r.destination = d;
            r.cbo_origin_before = org.co_b;
            r.cbo_origin_after = org.co_a;
            r.cbo_dest_before = dv.cd_b;
            r.cbo_dest_after = dv.cd_a;
            r.criteria = (uint8_t)MM_CRIT_SIMILARITY;
            r.origin_degenerate_after = org.odeg;
            r.dest_degenerate_after = dv.ddeg;
            r.pad = 0;
            store_record(a.out + at, r);
            ++at;
        };
        if (org.coh_ok)
            en.each([&](int, uint32_t d, uint32_t hd) {
                if (d == o || hd == 0) return;
                bool cand = false;
                for (uint32_t k = pb; k < pe && !cand; ++k) cand = __ldg(sc.part + k) == d;
                for (uint32_t e = cb; e < ce && !cand; ++e) cand = __ldg(a.s.method_owner + __ldg(a.s.call_tgt + e)) == d;
                if (!cand) return;
                const ClassRec rd = load_rec(a.rec, d);
                double ld_a;
                if (!coh_dest(rd, hd, ld_a)) return;  // lcom_improves (suggest.hpp:189-192)
                if (sc.all_candidates) {
                    ++n;
                    if (PASS) emit_one(d, hd);
                    return;
                }
                const double key = __dadd_rn(org.lo_a, ld_a);  // lcom_key; d ascending, strict <
                if (best == kNone || key < best_key) { best = d; best_h = hd; best_key = key; }
            });
        if (!sc.all_candidates && best != kNone) {
            n = 1;
            if (PASS) emit_one(best, best_h);
        }
        if (!PASS) sc.rec_cnt[p] = n;
    };
    if (smem) run(ren);
    else run(sen);
}

}  // namespace

void launch_score(const SweepArgs& a, uint32_t n_tiles, cudaStream_t st) {
    if (!n_tiles) return;
    const uint32_t blocks = n_tiles * (kSweepTile / kScoreTile);
    if (a.maxdeg_fast <= 8) k_score_thread<8><<<blocks, kScoreTile, 0, st>>>(a);
    else k_score_thread<16><<<blocks, kScoreTile, 0, st>>>(a);
}

uint32_t offsets_tiles(uint64_t npos) { return (uint32_t)((npos + kOffTile - 1) / kOffTile); }

void launch_score_fast(const SweepArgs& a, uint32_t n_tiles, uint32_t fallback_tiles, cudaStream_t st) {
    if (n_tiles) k_score_fast<<<n_tiles * (kSweepTile / kFastTile), kFastTile, 0, st>>>(a);
    if (!fallback_tiles) return;  // incomplete records (their list is built above)
    const uint32_t blocks = fallback_tiles * (kSweepTile / kScoreTile);
    if (a.maxdeg_fast <= 8) k_score_thread<8, true><<<blocks, kScoreTile, 0, st>>>(a);
    else k_score_thread<16, true><<<blocks, kScoreTile, 0, st>>>(a);
}

void launch_offsets(const SweepArgs& a, uint32_t n_tiles, cudaStream_t st) {
    if (!n_tiles) return;
    k_offsets<<<n_tiles, kSweepTile, 0, st>>>(a);
}

void launch_write(const SweepArgs& a, uint32_t n_tiles, bool fast_list, cudaStream_t st) {
    if (!n_tiles) return;
    const uint32_t grid = std::min<uint32_t>(n_tiles, 148 * 8);  // grid-stride over the emitter list
    if (a.mode == 0 && fast_list) k_write_best<<<grid, kSweepTile, 0, st>>>(a);
    if (a.maxdeg_fast <= 8) k_write<8><<<grid, kSweepTile, 0, st>>>(a);
    else k_write<16><<<grid, kSweepTile, 0, st>>>(a);
}

void launch_sim_partners(const mm_similarity* tab, uint64_t n, double thr, const uint32_t* owner, uint32_t M,
                         uint32_t* cnt, uint32_t* off, uint32_t* cur, uint32_t* part, uint32_t* totals, uint32_t* grand,
                         cudaStream_t st) {
    cudaMemsetAsync(cnt, 0, 4ull * (M + 1), st);
    const uint32_t grid = 148 * 8;
    if (n) k_sim_partner_count<<<grid, 256, 0, st>>>(tab, n, thr, owner, cnt);
    launch_scan(cnt, off, M + 1, totals, grand, st);
    cudaMemcpyAsync(cur, off, 4ull * (M + 1), cudaMemcpyDeviceToDevice, st);
    if (n) k_sim_partner_fill<<<grid, 256, 0, st>>>(tab, n, thr, owner, cur, part);
}

void launch_sim_emit(const SweepArgs& a, int pass, const uint32_t* part_off, const uint32_t* part, uint32_t* rec_cnt,
                     const uint32_t* rec_off, uint32_t all_candidates, cudaStream_t st) {
    const uint64_t npos = a.pos_end - a.pos_begin;
    if (!npos) return;
    const uint32_t n_tiles = (uint32_t)((npos + kSweepTile - 1) / kSweepTile);
    const SimCrit sc{part_off, part, rec_cnt, rec_off, all_candidates};
    if (a.maxdeg_fast <= 8) {
        if (pass == 0) k_sim_emit<8, 0><<<n_tiles, kSweepTile, 0, st>>>(a, sc);
        else k_sim_emit<8, 1><<<n_tiles, kSweepTile, 0, st>>>(a, sc);
    } else {
        if (pass == 0) k_sim_emit<16, 0><<<n_tiles, kSweepTile, 0, st>>>(a, sc);
        else k_sim_emit<16, 1><<<n_tiles, kSweepTile, 0, st>>>(a, sc);
    }
}

void launch_what_if(const DevModel& s, const ClassRec* rec, const uint32_t* ux, const uint32_t* un,
                    const uint32_t* dense, uint32_t u, uint32_t o, uint32_t d, mm_whatif* out, cudaStream_t st) {
    k_what_if<<<1, 32, 0, st>>>(s, rec, ux, un, dense, u, o, d, out);
}

}  // namespace mmg
