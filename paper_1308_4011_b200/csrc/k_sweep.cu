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
#define MMGPU_SCORE_MINB 6
#endif
#ifndef MMGPU_FAST_MINB
#define MMGPU_FAST_MINB 8
#endif
namespace mmg {

namespace {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPrefix = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

// Per-thread used list staged in shared memory (column-major over the tile
// so thread t's k-th entry sits at [k * kSweepTile + t]: conflict-free).
// Dynamic loops keep the kernel small and its register count low.
struct SmemEnum {
    uint32_t* X;
    uint32_t* H;
    int n;
    template <class F>
    __device__ __forceinline__ void each(F f) const {
#pragma unroll 1
        for (int k = 0; k < n; ++k) f(k, X[k * kSweepTile], H[k * kSweepTile]);
    }
    __device__ __forceinline__ uint32_t hits(uint32_t v) const {
        for (int k = 0; k < n; ++k)
            if (X[k * kSweepTile] == v) return H[k * kSweepTile];
        return 0;
    }
    // returns false when a new class would exceed `cap` distinct entries
    __device__ __forceinline__ bool insert(uint32_t v, uint32_t acc, int cap) {
        int k = 0;
        while (k < n && X[k * kSweepTile] < v) ++k;
        if (k < n && X[k * kSweepTile] == v) {
            H[k * kSweepTile] += acc;
            return true;
        }
        if (n >= cap) return false;
        for (int j = n; j > k; --j) {
            X[j * kSweepTile] = X[(j - 1) * kSweepTile];
            H[j * kSweepTile] = H[(j - 1) * kSweepTile];
        }
        X[k * kSweepTile] = v;
        H[k * kSweepTile] = acc;
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
template <int K, bool SCORE = false>
__device__ __forceinline__ bool load_method(const SweepArgs& a, uint32_t pos, uint32_t p, uint32_t o,
                                            SmemEnum& ren, StreamEnum& sen, Origin& org) {
    const uint4* rp = reinterpret_cast<const uint4*>(a.recs + pos);
    const uint4 r0 = rp[0], r1 = rp[1];
    const uint32_t hdr = rec_hdrs(a.recs, a.s.M)[pos];
    const ClassRec ro = load_rec(a.rec, o);
    if (!(hdr & kRecOverflow)) {
        const uint32_t ent[kRecMaxEnt] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
        const uint32_t n = rec_n(hdr);
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k)
            if (k < (int)n) { ren.X[k * kSweepTile] = ent[k] >> 8; ren.H[k * kSweepTile] = ent[k] & 0xffu; }
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
// kernel here is latency-bound, so resident warps matter most.
template <int K, bool LIST = false>
__global__ void __launch_bounds__(kSweepTile, MMGPU_SCORE_MINB) k_score_thread(SweepArgs a) {
    __shared__ uint32_t s_X[K * kSweepTile], s_H[K * kSweepTile];
    uint64_t pos;
    bool live;
    if (LIST) {  // the methods k_score_fast / k_screen handed over (record overflow)
        const uint32_t i = blockIdx.x * kSweepTile + threadIdx.x;
        live = i < *a.n_fallback;
        pos = live ? a.fallback[i] : 0;
    } else {
        pos = (uint64_t)a.pos_begin + (uint64_t)blockIdx.x * kSweepTile + threadIdx.x;
        live = pos < a.pos_end;
    }
    uint32_t cands = 0;
    if (live) {
        const uint32_t p = __ldg(a.s.cls_methods + pos);
        const uint32_t o = __ldg(a.pos_owner + pos);
        SmemEnum ren{s_X + threadIdx.x, s_H + threadIdx.x, 0};
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
__global__ void __launch_bounds__(kSweepTile, MMGPU_FAST_MINB) k_score_fast(SweepArgs a) {
    // the used list column-major in shared memory (thread t's k-th entry at
    // [k][t]: conflict-free), so the candidate and membership loops stay
    // rolled: small code, lanes of a warp in step
    __shared__ uint32_t s_ent[kRecMaxEnt][kSweepTile];
    const uint32_t pos = a.pos_begin + blockIdx.x * kSweepTile + threadIdx.x;
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
        E[0 * kSweepTile] = r0.x; E[1 * kSweepTile] = r0.y; E[2 * kSweepTile] = r0.z; E[3 * kSweepTile] = r0.w;
        E[4 * kSweepTile] = r1.x; E[5 * kSweepTile] = r1.y; E[6 * kSweepTile] = r1.z; E[7 * kSweepTile] = r1.w;
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
            const uint32_t d = E[k * kSweepTile] >> 8;
            if (d == o) continue;
            ++cands;
            if (!coh_ok && !can_coup) continue;
            const uint32_t h = E[k * kSweepTile] & 0xffu;
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
                bool okc = true;
#pragma unroll 1
                for (uint32_t j = 0; j < n && okc; ++j) {
                    const uint32_t X = E[j * kSweepTile] >> 8;
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

// Pass 1, best-only mode (the reference's default and the bench step): a
// flattened candidate screen. Each warp takes 32 consecutive class-order
// positions (one method per lane) and then spreads the warp's candidates
// (u, d) over its lanes, one candidate per lane and iteration, so lanes never
// idle on a neighbour's longer list. Per method (its own lane): the packed
// used list from the method pass's record, the origin's counts, and — only
// when the exact-rational pre-test h·M < H allows lcom(origin) to drop — the
// two origin doubles. Per candidate lane: d's counts and lcom, the integer
// pre-test h_u(d)·M_d > H_d (then the one fp64 division of lcom_dest_after),
// and, if the method can lower the origin's cbo, the membership of every
// other used class in U[d] (exact bitmap, or Bloom then the row). Per-method
// argmin over (key, d) in ascending-d order with strict < (lowest d wins
// ties, suggest.hpp:180-184) reads the candidates' results back from shared
// memory. Methods whose used list did not fit their record are evaluated
// afterwards by the whole warp, one at a time (screen_coop).
constexpr int kScreenWarps = kSweepTile / 32;
constexpr int kScreenSlots = 32 * kRecMaxEnt;  // candidates of one warp: ≤ 8 per method

struct ScreenSmem {
    uint32_t ent[kScreenWarps][32][kRecMaxEnt];   // the methods' used lists (X << 8 | h), own class included
    uint8_t cm[kScreenWarps][kScreenSlots];       // candidate slot -> method lane
    uint8_t ck[kScreenWarps][kScreenSlots];       // candidate slot -> list index
    double kc[kScreenWarps][kScreenSlots];        // cohesion key (passing) or -1
    uint32_t kp[kScreenWarps][kScreenSlots];      // coupling key cbo_d (passing) or kNone
};

// ascending bitonic sort of buf[0, N) (N a power of two), one warp
__device__ __forceinline__ void warp_sort_u32(uint32_t* buf, uint32_t N, int lane) {
    for (uint32_t k = 2; k <= N; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < N; i += 32) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t x = buf[i], y = buf[ixj];
                    if ((x > y) == ((i & k) == 0)) { buf[i] = y; buf[ixj] = x; }
                }
            }
            __syncwarp();
        }
}

constexpr uint32_t kCoopMaxDeg = 128;  // methods with more edges (hubs) take one lane's streaming path

// Best-only evaluation of ONE method whose used list did not fit its record,
// by the whole warp (all lanes call it with the same pos): the used list from
// the CSR (lane per edge, warp sort, run-length -> classes and own-access
// counts), the origin's removed count over lanes, then one destination per
// lane and a warp argmin over (key, list index). `scr` holds ≥ 3·kCoopMaxDeg
// words of this warp's shared memory.
__device__ __noinline__ void screen_coop(const SweepArgs& a, uint32_t pos, uint32_t* scr, int lane, uint4& out) {
    const uint32_t p = __ldg(a.s.cls_methods + pos), o = __ldg(a.pos_owner + pos);
    const uint32_t cb = __ldg(a.s.call_off + p), nc = __ldg(a.s.call_off + p + 1) - cb;
    const uint32_t ab = __ldg(a.s.acc_off + p), na = __ldg(a.s.acc_off + p + 1) - ab;
    const uint32_t deg = nc + na;
    uint32_t* key = scr;                      // owner << 1 | is_access, sorted
    uint32_t* LX = scr + kCoopMaxDeg;         // distinct used classes, ascending
    uint32_t* LH = scr + 2 * kCoopMaxDeg;     // accesses of the method owned by each
    uint32_t N = 32;
    while (N < deg) N <<= 1;
    for (uint32_t k = lane; k < N; k += 32) {
        uint32_t v = kNone;
        if (k < nc) v = __ldg(a.s.method_owner + __ldg(a.s.call_tgt + cb + k)) << 1;
        else if (k < deg) v = (__ldg(a.s.attr_info + __ldg(a.s.acc_tgt + ab + (k - nc))).x << 1) | 1u;
        key[k] = v;
    }
    __syncwarp();
    warp_sort_u32(key, N, lane);
    uint32_t n = 0;
    for (uint32_t k0 = 0; k0 < deg; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool head = k < deg && (k == 0 || (key[k] >> 1) != (key[k - 1] >> 1));
        const uint32_t hb = __ballot_sync(0xffffffffu, head);
        if (head) {
            const uint32_t X = key[k] >> 1;
            uint32_t h = 0, e = k;
            while (e < deg && (key[e] >> 1) == X) h += key[e++] & 1u;
            const uint32_t idx = n + __popc(hb & ((1u << lane) - 1));
            LX[idx] = X;
            LH[idx] = h;
        }
        n += __popc(hb);
    }
    __syncwarp();
    // origin: own-access count, removed count (U[o][X] == 1) over lanes
    const ClassRec ro = load_rec(a.rec, o);
    uint32_t hown = 0, removed = 0, own_used = 0;
    for (uint32_t k = lane; k < n; k += 32) {
        const uint32_t X = LX[k];
        if (X == o) { hown = LH[k]; own_used = 1; continue; }
        if (ro.dense != kNone) {
            removed += (__ldg(a.dense + ro.dense + (a.s.C + 31) / 32 + (X >> 5)) >> (X & 31)) & 1u;
        } else {
            const int q = urow_find(a.ux, ro.ubase, ro.cbo, X);
            if (q >= 0 && __ldg(a.un + ro.ubase + q) == 1u) ++removed;
        }
    }
    hown = __reduce_max_sync(0xffffffffu, hown);
    removed = __reduce_add_sync(0xffffffffu, removed);
    own_used = __reduce_or_sync(0xffffffffu, own_used);
    const Origin org = make_origin(ro, hown, removed);
    const bool can_coup = org.co_a < org.co_b;
    // destinations: one per lane
    double bk = 0.0;
    uint32_t bki = kNone, bp = 0, bpi = kNone;
    if (org.coh_ok || can_coup)
        for (uint32_t k = lane; k < n; k += 32) {
            const uint32_t d = LX[k];
            if (d == o) continue;
            const ClassRec rd = load_rec(a.rec, d);
            double ld_a;
            if (org.coh_ok && coh_dest(rd, LH[k], ld_a)) {
                const double kc = __dadd_rn(org.lo_a, ld_a);
                if (bki == kNone || kc < bk) { bk = kc; bki = k; }
            }
            if (can_coup) {
                bool ok = true;
                for (uint32_t j = 0; j < n && ok; ++j) {
                    const uint32_t X = LX[j];
                    if (X != d && !in_urow(a.rec, d, rd, a.ux, a.dense, X)) ok = false;
                }
                if (ok && (bpi == kNone || rd.cbo < bp)) { bp = rd.cbo; bpi = k; }
            }
        }
    // warp argmin over (key, list index): lowest d wins ties (suggest.hpp:180-184)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ok_ = __shfl_xor_sync(0xffffffffu, bk, off);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bki, off);
        if (oi != kNone && (bki == kNone || ok_ < bk || (ok_ == bk && oi < bki))) { bk = ok_; bki = oi; }
        const uint32_t op = __shfl_xor_sync(0xffffffffu, bp, off);
        const uint32_t opi = __shfl_xor_sync(0xffffffffu, bpi, off);
        if (opi != kNone && (bpi == kNone || op < bp || (op == bp && opi < bpi))) { bp = op; bpi = opi; }
    }
    out = make_uint4(bki == kNone ? kNone : LX[bki], bpi == kNone ? kNone : LX[bpi], n - own_used, 0);
    __syncwarp();
}

// one hub method (more than kCoopMaxDeg edges) on one lane, streaming used list
__device__ __noinline__ uint4 screen_stream_one(const SweepArgs& a, uint32_t ps, uint32_t pm) {
    const uint32_t o = __ldg(a.pos_owner + ps);
    StreamEnum sen;
    sen.S.init(a.s, pm);
    const ClassRec ro = load_rec(a.rec, o);
    const Origin org = make_origin(ro, sen.hits(o), removed_count(ro, a.ux, a.un, a.dense, a.s.C, sen, o));
    const MethodResult r = evaluate(a, sen, o, org, true, true);
    return make_uint4(r.bd_coh, r.bd_coup, r.cands, 0);
}

// the warp's methods whose used list did not fit their record (ovf lanes):
// one at a time by the whole warp; hubs beyond kCoopMaxDeg edges by their own
// lane on the streaming used list. Returns this lane's (bd_coh, bd_coup,
// candidates) when it is an ovf lane.
__device__ __forceinline__ uint4 screen_overflow(const SweepArgs& a, bool ovf, uint64_t pos, uint32_t* scr,
                                                 int lane) {
    uint4 mine = make_uint4(kNone, kNone, 0, 0);
    uint32_t ob = __ballot_sync(0xffffffffu, ovf);
    while (ob) {
        const int src = __ffs(ob) - 1;
        ob &= ob - 1;
        const uint32_t ps = __shfl_sync(0xffffffffu, (uint32_t)pos, src);
        const uint32_t pm = __ldg(a.s.cls_methods + ps);
        const uint32_t deg = (__ldg(a.s.call_off + pm + 1) - __ldg(a.s.call_off + pm)) +
                             (__ldg(a.s.acc_off + pm + 1) - __ldg(a.s.acc_off + pm));
        if (deg <= kCoopMaxDeg) {
            uint4 r;
            screen_coop(a, ps, scr, lane, r);
            if (lane == src) mine = r;
        } else if (lane == src) {
            mine = screen_stream_one(a, ps, pm);
        }
        __syncwarp();
    }
    return mine;
}

__global__ void __launch_bounds__(kSweepTile, 4) k_screen(SweepArgs a) {
    __shared__ ScreenSmem sm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t pos = (uint64_t)a.pos_begin + (uint64_t)blockIdx.x * kSweepTile + threadIdx.x;
    const bool live = pos < a.pos_end;
    uint32_t (*ent)[kRecMaxEnt] = sm.ent[warp];
    uint8_t* cm = sm.cm[warp];
    uint8_t* ck = sm.ck[warp];
    double* kc = sm.kc[warp];
    uint32_t* kp = sm.kp[warp];

    // ---- per method (this lane)
    uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);
    uint32_t o = 0, hdr = 0;
    if (live) {
        const uint4* rp = reinterpret_cast<const uint4*>(a.recs + pos);
        r0 = rp[0];
        r1 = rp[1];
        hdr = rec_hdrs(a.recs, a.s.M)[pos];
        o = __ldg(a.pos_owner + pos);
    }
    const bool ovf = live && (hdr & kRecOverflow);
    const uint32_t n = (live && !ovf) ? rec_n(hdr) : 0u;
    {
        const uint32_t e7[kRecMaxEnt] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k) ent[lane][k] = e7[k];
    }
    uint32_t nc = 0;  // candidates: list entries other than the own class
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k) nc += (k < (int)n && (ent[lane][k] >> 8) != o);
    // origin
    bool coh_ok = false, can_coup = false;
    double lo_a = 0.0;
    if (n) {
        const ClassRec ro = load_rec(a.rec, o);
        const uint32_t h = rec_hown(hdr);
        const uint32_t removed = (hdr & kRecRemovedValid) ? rec_removed(hdr)
                                                            : removed_from_list(ro, a.ux, a.un, a.dense, a.s.C,
                                                                                ent[lane], n, o);
        can_coup = removed > 0;  // cbo_origin_after < cbo_origin_before
        // lcom(A, M-1, H-h) < lcom(A, M, H): impossible when A == 0 (both 0.0)
        // or, with exact denominators and M ≥ 2, when (H-h)·M ≤ H·(M-1)
        bool maybe = ro.A != 0 && ro.M != 0;
        if (maybe && ro.M >= 2 && (uint64_t)ro.A * ro.M < kExact53) maybe = (uint64_t)h * ro.M < ro.H;
        if (maybe) {
            lo_a = lcom_of(ro.A, (uint64_t)ro.M - 1, (uint64_t)ro.H - h);
            coh_ok = lo_a < __ldg(a.dlcom + o);
        }
    }
    // candidate slots: this method's at [excl, excl + nc), list order (d ascending)
    uint32_t incl = nc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    const uint32_t excl = incl - nc;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    {
        uint32_t w = excl;
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k)
            if (k < (int)n && (ent[lane][k] >> 8) != o) {
                cm[w] = (uint8_t)lane;
                ck[w] = (uint8_t)k;
                ++w;
            }
    }
    const uint32_t flags = (coh_ok ? 1u : 0u) | (can_coup ? 2u : 0u);
    __syncwarp();

    // ---- per candidate (one per lane and round)
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
        const uint32_t c = c0 + lane;
        const bool act = c < total;
        const uint32_t m = act ? cm[c] : 0u;
        const uint32_t mflags = __shfl_sync(0xffffffffu, flags, m);
        const double m_lo_a = __shfl_sync(0xffffffffu, lo_a, m);
        const uint32_t m_n = __shfl_sync(0xffffffffu, n, m);
        if (!act) continue;
        const uint32_t e = ent[m][ck[c]];
        const uint32_t d = e >> 8, hd = e & 0xffu;
        double key = -1.0;
        uint32_t kpv = kNone;
        if (mflags) {
            const ClassRec rd = load_rec(a.rec, d);
            if ((mflags & 1u) && rd.A != 0 && rd.M != 0) {
                const bool exact = (uint64_t)rd.A * ((uint64_t)rd.M + 1) < kExact53;
                if (!exact || (uint64_t)hd * rd.M > rd.H) {
                    const double ld_a = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + hd);
                    if (ld_a < __ldg(a.dlcom + d)) key = __dadd_rn(m_lo_a, ld_a);  // lcom_key, suggest.hpp:194-196
                }
            }
            if (mflags & 2u) {
                bool ok = true;
                for (uint32_t j = 0; j < m_n && ok; ++j) {
                    const uint32_t X = ent[m][j] >> 8;
                    if (X != d && !in_urow(a.rec, d, rd, a.ux, a.dense, X)) ok = false;
                }
                if (ok) kpv = rd.cbo;  // cbo_dest_after == cbo_dest_before when it passes
            }
        }
        kc[c] = key;
        kp[c] = kpv;
    }
    __syncwarp();

    // ---- per method: argmin over its slots (d ascending, strict <)
    uint32_t bd_coh = kNone, bd_coup = kNone;
    double bk = 0.0;
    uint32_t bp = 0;
    for (uint32_t j = 0; j < nc; ++j) {
        const uint32_t slot = excl + j;
        const double kcv = kc[slot];
        const uint32_t kpv = kp[slot];
        if (kcv >= 0.0 || kpv != kNone) {
            const uint32_t d = ent[lane][ck[slot]] >> 8;
            if (kcv >= 0.0 && (bd_coh == kNone || kcv < bk)) { bd_coh = d; bk = kcv; }
            if (kpv != kNone && (bd_coup == kNone || kpv < bp)) { bd_coup = d; bp = kpv; }
        }
    }
    if (live && !ovf) a.res[pos] = make_uint4(bd_coh, bd_coup, nc, 0);
    const uint32_t wc = __reduce_add_sync(0xffffffffu, nc);
    if (lane == 0 && wc) atomicAdd(a.stats + 0, (unsigned long long)wc);
    __syncwarp();
    const uint4 ov = screen_overflow(a, ovf, pos, reinterpret_cast<uint32_t*>(kc), lane);  // kc: free now
    if (ovf) {
        a.res[pos] = ov;
        if (ov.z) atomicAdd(a.stats + 0, (unsigned long long)ov.z);
    }
}

// Variant 2 of the screen (MMGPU_SCREEN=2): the same decisions with the
// memory round trips overlapped — the origin's record is requested before the
// candidate slots are built, the first round's destination records before the
// origin's doubles are computed, and the Bloom words of every other used class
// are requested together (predicated, no early exit), the U rows only probed
// for Bloom positives.
#ifndef MMGPU_SCREEN_MINB
#define MMGPU_SCREEN_MINB 4
#endif
__device__ __forceinline__ bool bloom_word_test(const ClassRec* __restrict__ rec, uint32_t d, uint32_t X) {
    const uint32_t b1 = bloom_h1(X), b2 = bloom_h2(X);
    const uint32_t w1 = __ldg(rec[d].sig + (b1 >> 5)), w2 = __ldg(rec[d].sig + (b2 >> 5));
    return ((w1 >> (b1 & 31)) & (w2 >> (b2 & 31)) & 1u) != 0;
}

__global__ void __launch_bounds__(kSweepTile, MMGPU_SCREEN_MINB) k_screen2(SweepArgs a) {
    __shared__ ScreenSmem sm;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t pos = (uint64_t)a.pos_begin + (uint64_t)blockIdx.x * kSweepTile + threadIdx.x;
    const bool live = pos < a.pos_end;
    uint32_t (*ent)[kRecMaxEnt] = sm.ent[warp];
    uint8_t* cm = sm.cm[warp];
    uint8_t* ck = sm.ck[warp];
    double* kc = sm.kc[warp];
    uint32_t* kp = sm.kp[warp];

    uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);
    uint32_t o = 0, hdr = 0;
    if (live) {
        const uint4* rp = reinterpret_cast<const uint4*>(a.recs + pos);
        r0 = rp[0];
        r1 = rp[1];
        hdr = rec_hdrs(a.recs, a.s.M)[pos];
        o = __ldg(a.pos_owner + pos);
    }
    const bool ovf = live && (hdr & kRecOverflow);
    const uint32_t n = (live && !ovf) ? rec_n(hdr) : 0u;
    // the origin's record and lcom: in flight while the slots are built
    ClassRec ro{};
    double dlo = 0.0;
    if (n) {
        ro = load_rec(a.rec, o);
        dlo = __ldg(a.dlcom + o);
    }
    {
        const uint32_t e7[kRecMaxEnt] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k) ent[lane][k] = e7[k];
    }
    uint32_t nc = 0;
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k) nc += (k < (int)n && (ent[lane][k] >> 8) != o);
    uint32_t incl = nc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    const uint32_t excl = incl - nc;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    {
        uint32_t w = excl;
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k)
            if (k < (int)n && (ent[lane][k] >> 8) != o) {
                cm[w] = (uint8_t)lane;
                ck[w] = (uint8_t)k;
                ++w;
            }
    }
    __syncwarp();
    // the first round's destination: record and lcom requested before the origin math
    uint32_t c = lane, m = 0, d = 0, hd = 0;
    ClassRec rd{};
    double dld = 0.0;
    auto fetch = [&]() {
        if (c < total) {
            m = cm[c];
            const uint32_t e = ent[m][ck[c]];
            d = e >> 8;
            hd = e & 0xffu;
            rd = load_rec(a.rec, d);
            dld = __ldg(a.dlcom + d);
        }
    };
    fetch();
    // origin (this lane's method)
    bool coh_ok = false, can_coup = false;
    double lo_a = 0.0;
    if (n) {
        const uint32_t h = rec_hown(hdr);
        const uint32_t removed = (hdr & kRecRemovedValid) ? rec_removed(hdr)
                                                            : removed_from_list(ro, a.ux, a.un, a.dense, a.s.C,
                                                                                ent[lane], n, o);
        can_coup = removed > 0;
        bool maybe = ro.A != 0 && ro.M != 0;
        if (maybe && ro.M >= 2 && (uint64_t)ro.A * ro.M < kExact53) maybe = (uint64_t)h * ro.M < ro.H;
        if (maybe) {
            lo_a = lcom_of(ro.A, (uint64_t)ro.M - 1, (uint64_t)ro.H - h);
            coh_ok = lo_a < dlo;
        }
    }
    const uint32_t flags = (coh_ok ? 1u : 0u) | (can_coup ? 2u : 0u);
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
        const bool act = c < total;
        const uint32_t mflags = __shfl_sync(0xffffffffu, flags, act ? m : 0);
        const double m_lo_a = __shfl_sync(0xffffffffu, lo_a, act ? m : 0);
        const uint32_t m_n = __shfl_sync(0xffffffffu, n, act ? m : 0);
        if (act) {
            double key = -1.0;
            uint32_t kpv = kNone;
            if ((mflags & 1u) && rd.A != 0 && rd.M != 0) {
                const bool exact = (uint64_t)rd.A * ((uint64_t)rd.M + 1) < kExact53;
                if (!exact || (uint64_t)hd * rd.M > rd.H) {
                    const double ld_a = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + hd);
                    if (ld_a < dld) key = __dadd_rn(m_lo_a, ld_a);  // lcom_key, suggest.hpp:194-196
                }
            }
            if (mflags & 2u) {
                // every other used class must be in U[d]: all Bloom words at once
                bool ok = true;
                uint32_t probe = 0;
                if (rd.dense != kNone) {
#pragma unroll
                    for (int j = 0; j < kRecMaxEnt; ++j)
                        if (j < (int)m_n) {
                            const uint32_t X = ent[m][j] >> 8;
                            if (X != d) ok &= ((__ldg(a.dense + rd.dense + (X >> 5)) >> (X & 31)) & 1u) != 0;
                        }
                } else {
#pragma unroll
                    for (int j = 0; j < kRecMaxEnt; ++j)
                        if (j < (int)m_n) {
                            const uint32_t X = ent[m][j] >> 8;
                            if (X != d) {
                                if (bloom_word_test(a.rec, d, X)) probe |= 1u << j;
                                else ok = false;
                            }
                        }
                    for (int j = 0; ok && probe; ++j, probe >>= 1)
                        if (probe & 1u) ok = urow_find(a.ux, rd.ubase, rd.cbo, ent[m][j] >> 8) >= 0;
                }
                if (ok) kpv = rd.cbo;
            }
            kc[c] = key;
            kp[c] = kpv;
        }
        c += 32;
        fetch();
    }
    __syncwarp();
    uint32_t bd_coh = kNone, bd_coup = kNone;
    double bk = 0.0;
    uint32_t bp = 0;
    for (uint32_t j = 0; j < nc; ++j) {
        const uint32_t slot = excl + j;
        const double kcv = kc[slot];
        const uint32_t kpv = kp[slot];
        if (kcv >= 0.0 || kpv != kNone) {
            const uint32_t dd = ent[lane][ck[slot]] >> 8;
            if (kcv >= 0.0 && (bd_coh == kNone || kcv < bk)) { bd_coh = dd; bk = kcv; }
            if (kpv != kNone && (bd_coup == kNone || kpv < bp)) { bd_coup = dd; bp = kpv; }
        }
    }
    if (live && !ovf) a.res[pos] = make_uint4(bd_coh, bd_coup, nc, 0);
    const uint32_t wc = __reduce_add_sync(0xffffffffu, nc);
    if (lane == 0 && wc) atomicAdd(a.stats + 0, (unsigned long long)wc);
    __syncwarp();
    const uint4 ov = screen_overflow(a, ovf, pos, reinterpret_cast<uint32_t*>(kc), lane);  // kc: free now
    if (ovf) {
        a.res[pos] = ov;
        if (ov.z) atomicAdd(a.stats + 0, (unsigned long long)ov.z);
    }
}

// ---- best-only mode, fused: screen + gates + offsets + records in one pass
//
// The class gates need the threshold means, which the metric pass now
// computes before the sweep, so the whole best-only sweep runs as one kernel:
// each CTA takes the next 256 class-order positions (dynamic tile id), screens
// them exactly as k_screen, applies the gates (suggest.hpp:246, :273) and the
// criteria merge (:315-341) per method, scans the record counts over the CTA
// and a decoupled look-back over the preceding tiles (relaxed gpu-scope
// 64-bit words: flag | emitters << 32 | records), publishes its inclusive
// prefix, and only then writes its records (what-if values recomputed from the
// class tables, suggest.hpp:87-122): emission never delays a successor's
// look-back. No per-method result array, no emitter list, no extra launch.

// decoupled look-back by warp 0 of the CTA: returns (lane 0) the exclusive
// prefix of this tile and publishes tile_state[tile] = prefix | (excl + agg)
__device__ __forceinline__ unsigned long long tile_lookback(const SweepArgs& a, uint32_t tile, unsigned long long agg,
                                                            int lane) {
    unsigned long long excl = 0;
    if (tile == 0) {
        if (lane == 0) st_relaxed_u64(a.tile_state, kFlagPrefix | agg);
        return 0;
    }
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
    return excl;
}

// one method's records (best-only; destinations bdc / bdp gated already) from
// its packed used list; destinations ascending, suggest_all's tags
__device__ __noinline__ void emit_best(const SweepArgs& a, uint32_t pos, uint32_t o, uint32_t hdr, const uint32_t* ent,
                                       uint32_t n, uint32_t bdc, uint32_t bdp, bool inter, uint64_t at) {
    const uint32_t p = __ldg(a.s.cls_methods + pos);
    const ClassRec ro = load_rec(a.rec, o);
    const uint32_t removed = (hdr & kRecRemovedValid) ? rec_removed(hdr)
                                                       : removed_from_list(ro, a.ux, a.un, a.dense, a.s.C, ent, n, o);
    const Origin org = make_origin(ro, rec_hown(hdr), removed);
    uint32_t ds[2];
    int nd = 0;
    if (inter) {
        ds[nd++] = bdc;  // bdc == bdp here
    } else {
        const uint32_t x = bdc < bdp ? bdc : bdp, y = bdc < bdp ? bdp : bdc;  // kNone sorts last
        if (x != kNone) ds[nd++] = x;
        if (y != kNone && y != x) ds[nd++] = y;
    }
    for (int i = 0; i < nd; ++i) {
        const uint32_t d = ds[i];
        uint32_t hd = 0;
        for (uint32_t k = 0; k < n; ++k)
            if ((ent[k] >> 8) == d) hd = ent[k] & 0xffu;
        const ClassRec rd = load_rec(a.rec, d);
        uint32_t miss = 0;
        for (uint32_t k = 0; k < n; ++k) {
            const uint32_t X = ent[k] >> 8;
            if (X != d && !in_urow(a.rec, d, rd, a.ux, a.dense, X)) ++miss;
        }
        mm_suggestion r;
        r.lcom_origin_before = org.lo_b;
        r.lcom_origin_after = org.lo_a;
        r.lcom_dest_before = lcom_of(rd.A, rd.M, rd.H);
        r.lcom_dest_after = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + hd);
        r.method = p;
        r.origin = o;
        r.destination = d;
        r.cbo_origin_before = org.co_b;
        r.cbo_origin_after = org.co_a;
        r.cbo_dest_before = rd.cbo;
        r.cbo_dest_after = rd.cbo + miss;
        r.criteria = (uint8_t)((d == bdc ? MM_CRIT_COHESION : 0u) | (d == bdp ? MM_CRIT_COUPLING : 0u));
        r.origin_degenerate_after = org.odeg;
        r.dest_degenerate_after = rd.A == 0;
        r.pad = 0;
        store_record(a.out + at + i, r);
    }
}

// the same for a method whose used list overflowed its record (streaming list)
__device__ __noinline__ void emit_best_stream(const SweepArgs& a, uint32_t pos, uint32_t o, uint32_t bdc,
                                              uint32_t bdp, uint64_t at) {
    const uint32_t p = __ldg(a.s.cls_methods + pos);
    StreamEnum sen;
    sen.S.init(a.s, p);
    const ClassRec ro = load_rec(a.rec, o);
    const Origin org = make_origin(ro, sen.hits(o), removed_count(ro, a.ux, a.un, a.dense, a.s.C, sen, o));
    MethodResult res{};
    res.bd_coh = bdc;
    res.bd_coup = bdp;
    emit(a, sen, p, o, org, res, at);
}

__global__ void __launch_bounds__(kSweepTile, 4) k_sweep_best(SweepArgs a) {
    __shared__ ScreenSmem sm;
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_warp[kScreenWarps], s_red[2][kScreenWarps];
    __shared__ unsigned long long s_excl;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t pos = (uint64_t)a.pos_begin + (uint64_t)tile * kSweepTile + threadIdx.x;
    const bool live = pos < a.pos_end;
    uint32_t (*ent)[kRecMaxEnt] = sm.ent[warp];
    uint8_t* cm = sm.cm[warp];
    uint8_t* ck = sm.ck[warp];
    double* kc = sm.kc[warp];
    uint32_t* kp = sm.kp[warp];

    // ---- screen (as k_screen)
    uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);
    uint32_t o = 0, hdr = 0;
    if (live) {
        const uint4* rp = reinterpret_cast<const uint4*>(a.recs + pos);
        r0 = rp[0];
        r1 = rp[1];
        hdr = rec_hdrs(a.recs, a.s.M)[pos];
        o = __ldg(a.pos_owner + pos);
    }
    const bool ovf = live && (hdr & kRecOverflow);
    const uint32_t n = (live && !ovf) ? rec_n(hdr) : 0u;
    {
        const uint32_t e8[kRecMaxEnt] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k) ent[lane][k] = e8[k];
    }
    uint32_t nc = 0;
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k) nc += (k < (int)n && (ent[lane][k] >> 8) != o);
    bool coh_ok = false, can_coup = false;
    double lo_a = 0.0;
    if (n) {
        const ClassRec ro = load_rec(a.rec, o);
        const uint32_t h = rec_hown(hdr);
        const uint32_t removed = (hdr & kRecRemovedValid) ? rec_removed(hdr)
                                                           : removed_from_list(ro, a.ux, a.un, a.dense, a.s.C,
                                                                               ent[lane], n, o);
        can_coup = removed > 0;
        bool maybe = ro.A != 0 && ro.M != 0;
        if (maybe && ro.M >= 2 && (uint64_t)ro.A * ro.M < kExact53) maybe = (uint64_t)h * ro.M < ro.H;
        if (maybe) {
            lo_a = lcom_of(ro.A, (uint64_t)ro.M - 1, (uint64_t)ro.H - h);
            coh_ok = lo_a < __ldg(a.dlcom + o);
        }
    }
    uint32_t incl = nc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
    }
    const uint32_t excl_c = incl - nc;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    {
        uint32_t w = excl_c;
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k)
            if (k < (int)n && (ent[lane][k] >> 8) != o) {
                cm[w] = (uint8_t)lane;
                ck[w] = (uint8_t)k;
                ++w;
            }
    }
    const uint32_t flags = (coh_ok ? 1u : 0u) | (can_coup ? 2u : 0u);
    __syncwarp();
    for (uint32_t c0 = 0; c0 < total; c0 += 32) {
        const uint32_t c = c0 + lane;
        const bool act = c < total;
        const uint32_t m = act ? cm[c] : 0u;
        const uint32_t mflags = __shfl_sync(0xffffffffu, flags, m);
        const double m_lo_a = __shfl_sync(0xffffffffu, lo_a, m);
        const uint32_t m_n = __shfl_sync(0xffffffffu, n, m);
        if (!act) continue;
        const uint32_t e = ent[m][ck[c]];
        const uint32_t d = e >> 8, hd = e & 0xffu;
        double key = -1.0;
        uint32_t kpv = kNone;
        if (mflags) {
            const ClassRec rd = load_rec(a.rec, d);
            if ((mflags & 1u) && rd.A != 0 && rd.M != 0) {
                const bool exact = (uint64_t)rd.A * ((uint64_t)rd.M + 1) < kExact53;
                if (!exact || (uint64_t)hd * rd.M > rd.H) {
                    const double ld_a = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + hd);
                    if (ld_a < __ldg(a.dlcom + d)) key = __dadd_rn(m_lo_a, ld_a);
                }
            }
            if (mflags & 2u) {
                bool ok = true;
                for (uint32_t j = 0; j < m_n && ok; ++j) {
                    const uint32_t X = ent[m][j] >> 8;
                    if (X != d && !in_urow(a.rec, d, rd, a.ux, a.dense, X)) ok = false;
                }
                if (ok) kpv = rd.cbo;
            }
        }
        kc[c] = key;
        kp[c] = kpv;
    }
    __syncwarp();
    uint32_t bdc = kNone, bdp = kNone;
    {
        double bk = 0.0;
        uint32_t bp = 0;
        for (uint32_t j = 0; j < nc; ++j) {
            const uint32_t slot = excl_c + j;
            const double kcv = kc[slot];
            const uint32_t kpv = kp[slot];
            if (kcv >= 0.0 || kpv != kNone) {
                const uint32_t dd = ent[lane][ck[slot]] >> 8;
                if (kcv >= 0.0 && (bdc == kNone || kcv < bk)) { bdc = dd; bk = kcv; }
                if (kpv != kNone && (bdp == kNone || kpv < bp)) { bdp = dd; bp = kpv; }
            }
        }
    }
    __syncwarp();
    uint32_t cands = nc;
    {
        const uint4 ov = screen_overflow(a, ovf, pos, reinterpret_cast<uint32_t*>(kc), lane);
        if (ovf) { bdc = ov.x; bdp = ov.y; cands = ov.z; }
    }
    // ---- gates and the criteria merge
    double thr_l = a.thr_lcom, thr_c = a.thr_cbo;
    if (a.thr_device) { thr_l = a.dthr->lcom; thr_c = a.dthr->cbo; }
    const bool both = (a.crit & MM_CRIT_COHESION) && (a.crit & MM_CRIT_COUPLING);
    const bool inter = a.combine == MM_COMBINE_INTERSECTION && both;
    uint32_t count = 0;
    unsigned long long gated = 0;
    if (live) {
        const bool gcoh = (a.crit & MM_CRIT_COHESION) && __ldg(a.lcom + o) > thr_l;
        const bool gcoup = (a.crit & MM_CRIT_COUPLING) && (double)__ldg(a.cbo + o) > thr_c;
        gated = (unsigned long long)cands * ((gcoh ? 1u : 0u) + (gcoup ? 1u : 0u));
        if (!gcoh) bdc = kNone;
        if (!gcoup) bdp = kNone;
        const bool same = bdc != kNone && bdc == bdp;
        count = inter ? (same ? 1u : 0u) : (uint32_t)(bdc != kNone) + (uint32_t)(bdp != kNone) - (same ? 1u : 0u);
    }
    // ---- CTA scan of (emitters << 32 | records), look-back, publish
    const unsigned long long mine = count + (count ? (1ull << 32) : 0ull);
    unsigned long long inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) s_warp[warp] = inc;
    {
        unsigned long long g0 = gated, g1 = cands;
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
    for (int w = 0; w < kScreenWarps; ++w) {
        if (w < warp) before += s_warp[w];
        agg += s_warp[w];
    }
    if (warp == 0) {
        const unsigned long long ex = tile_lookback(a, tile, agg, lane);
        if (lane == 0) {
            s_excl = ex;
            unsigned long long t0 = 0, t1 = 0;
            for (int w = 0; w < kScreenWarps; ++w) { t0 += s_red[0][w]; t1 += s_red[1][w]; }
            if (t1) atomicAdd(a.stats + 0, t1);
            if (t0) atomicAdd(a.stats + 1, t0);
            if (agg & 0xffffffffull) atomicAdd(a.stats + 2, agg & 0xffffffffull);
            const uint64_t t0pos = (uint64_t)a.pos_begin + (uint64_t)tile * kSweepTile;
            const uint64_t rest = a.pos_end > t0pos ? a.pos_end - t0pos : 0;
            const uint64_t nvalid = rest < kSweepTile ? rest : (uint64_t)kSweepTile;
            atomicAdd(a.stats + 3, (unsigned long long)nvalid);
            atomicAdd(a.n_emit, (uint32_t)(agg >> 32));
        }
    }
    __syncthreads();
    // ---- records (the tile's prefix is already published)
    if (count) {
        const uint64_t at = (s_excl + before + inc - mine) & 0xffffffffull;
        if (!ovf) emit_best(a, (uint32_t)pos, o, hdr, ent[lane], n, bdc, bdp, inter, at);
        else emit_best_stream(a, (uint32_t)pos, o, bdc, bdp, at);
    }
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

constexpr int kOffItems = 16;  // 4096-position tiles: ≤ 245 tiles for 1M methods, one resident wave
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

void launch_sweep_best(const SweepArgs& a, uint32_t n_tiles, cudaStream_t st) {
    if (!n_tiles) return;
    k_sweep_best<<<n_tiles, kSweepTile, 0, st>>>(a);
}

void launch_score(const SweepArgs& a, uint32_t n_tiles, uint32_t fallback_tiles, cudaStream_t st) {
    if (!n_tiles) return;
    if (a.mode == 0 && !a.no_screen) {
        if (a.screen_variant == 1) k_screen<<<n_tiles, kSweepTile, 0, st>>>(a);
        else k_screen2<<<n_tiles, kSweepTile, 0, st>>>(a);
        (void)fallback_tiles;  // record-overflow methods are handled inside the screen (warp-cooperative)
        return;
    }
    if (a.maxdeg_fast <= 8) k_score_thread<8><<<n_tiles, kSweepTile, 0, st>>>(a);
    else k_score_thread<16><<<n_tiles, kSweepTile, 0, st>>>(a);
}

uint32_t offsets_tiles(uint64_t npos) { return (uint32_t)((npos + kOffTile - 1) / kOffTile); }

void launch_score_fast(const SweepArgs& a, uint32_t n_tiles, uint32_t fallback_tiles, cudaStream_t st) {
    if (n_tiles) k_score_fast<<<n_tiles, kSweepTile, 0, st>>>(a);
    if (!fallback_tiles) return;  // incomplete records (their list is built above)
    if (a.maxdeg_fast <= 8) k_score_thread<8, true><<<fallback_tiles, kSweepTile, 0, st>>>(a);
    else k_score_thread<16, true><<<fallback_tiles, kSweepTile, 0, st>>>(a);
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
