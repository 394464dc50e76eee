// mm_device.cuh — device-side data layout and shared device functions.
//
// HBM layout (one copy per context, all u32 unless noted):
//   model (uploaded verbatim from mm_system):
//     method_owner[m], attribute_owner[a], cls_moff[c+1], cls_methods[m],
//     cls_aoff[c+1], cls_attrs[a], call_off[m+1], call_tgt[E_c],
//     acc_off[m+1], acc_tgt[E_a]
//   derived by the metric pass:
//     attr_local[a]      index of attribute a inside its class's sorted list
//     rec[c]             ClassRec, 32 B: the per-class table the sweep gathers
//     lcom[c] (f64), lcom_ck[c] (u64), cbo[c]   dense outputs (D2H, thresholds)
//     ux[], un[]         U rows: for class c, ux[rec.ubase .. +rec.cbo) is the
//                        sorted set {X != c : some member of c uses X} and
//                        un[] the member counts U[c][X]
#pragma once
#include <cstdint>

#include "../../include/mmgpu.h"

namespace mmg {

constexpr uint32_t kNone = 0xffffffffu;
constexpr int kSmallMaxMembers = 32;  // warp path: one lane per member
constexpr int kSmallMaxAttrs = 64;    // own-attribute set fits a u64 mask
constexpr int kSmallMaxDeg = 16;      // per-member used list fits registers
constexpr uint32_t kSmallRowCap = kSmallMaxDeg;  // U-row slots reserved per member of a small class
// class kinds (upload plan): warp path with ≤ 32 U-row keys, CTA path, warp
// path with more keys (shared-memory sort)
constexpr uint32_t kKindLean = 0, kKindCta = 1, kKindWarpBig = 2;

struct DevModel {
    uint32_t C, M, A;
    const uint32_t* __restrict__ method_owner;
    const uint32_t* __restrict__ attribute_owner;
    const uint32_t* __restrict__ cls_moff;
    const uint32_t* __restrict__ cls_methods;
    const uint32_t* __restrict__ cls_aoff;
    const uint32_t* __restrict__ cls_attrs;
    const uint32_t* __restrict__ call_off;
    const uint32_t* __restrict__ call_tgt;
    const uint32_t* __restrict__ acc_off;
    const uint32_t* __restrict__ acc_tgt;
    const uint2* __restrict__ attr_info;  // derived at upload: (owner, position in the owner's attribute list)
    // the dependency rows again, in class order (row k = the method at
    // class-order position k), laid out at upload so the method pass streams
    // them coalesced: offsets [M+1], targets [E]
    const uint32_t* __restrict__ pc_off;
    const uint32_t* __restrict__ pc_tgt;
    const uint32_t* __restrict__ pa_off;
    const uint32_t* __restrict__ pa_tgt;
};

constexpr int kSigWords = 10;               // 320-bit Bloom signature
constexpr uint32_t kSigBits = 32 * kSigWords;

// Per-class table, one 64-byte half line: the counts the sweep needs and a
// 320-bit two-hash Bloom signature of the U row (a clear bit proves X ∉ U[c];
// false-positive rate ≈ 1.4% at the C4 row length of 20).
struct __align__(64) ClassRec {
    uint32_t A;      // |attrs(c)|
    uint32_t M;      // |methods(c)|
    uint32_t H;      // Σ_{p∈c} |acc(p) ∩ attrs(c)|
    uint32_t cbo;    // |U row|
    uint32_t ubase;  // U row start in ux/un
    uint32_t dense;  // word offset of an exact class bitmap of the U row (dense rows), or kNone
    uint32_t sig[kSigWords];
};
constexpr uint32_t kDenseRowMin = 64;  // rows longer than this get an exact bitmap (CTA path)

__device__ __forceinline__ uint32_t bloom_h1(uint32_t x) {
    return (uint32_t)(((uint64_t)(x * 0x9E3779B1u) * kSigBits) >> 32);
}
__device__ __forceinline__ uint32_t bloom_h2(uint32_t x) {
    return (uint32_t)(((uint64_t)((x ^ 0x5bd1e995u) * 0x85EBCA6Bu) * kSigBits) >> 32);
}

// Compact per-method record, stored at the method's class-order position by
// the method pass (one 32-byte sector): the sorted used list (owner classes
// of calls ∪ accesses, own class included) packed as X << 8 | h, with h the
// number of accesses owned by X — up to 8 classes, so a method with ≤ 8
// edges (every method of the k ≤ 4 + 4 generator configs) always fits. The
// record's 32-bit header lives in a separate array right after the records
// (rec_hdrs): readers load it coalesced beside the entries.
constexpr int kRecMaxEnt = 8;
struct __align__(32) MethRec {
    uint32_t ent[kRecMaxEnt];
};
__host__ __device__ __forceinline__ uint32_t* rec_hdrs(MethRec* recs, uint32_t M) {
    return reinterpret_cast<uint32_t*>(recs + M);
}
__host__ __device__ __forceinline__ const uint32_t* rec_hdrs(const MethRec* recs, uint32_t M) {
    return reinterpret_cast<const uint32_t*>(recs + M);
}
constexpr uint32_t kRecN = 0xfu;            // bits 0-3   number of entries (≤ 8)
constexpr int kRecHownShift = 8;            // bits 8-15  |acc(p) ∩ attrs(own)|
constexpr int kRecRemovedShift = 16;        // bits 16-23 #{X ≠ own : U[own][X] == 1} (class pass)
constexpr uint32_t kRecOverflow = 1u << 24; // list not representable: consumers use the CSR
constexpr uint32_t kRecRemovedValid = 1u << 25;

__device__ __forceinline__ uint32_t rec_n(uint32_t hdr) { return hdr & kRecN; }
__device__ __forceinline__ uint32_t rec_hown(uint32_t hdr) { return (hdr >> kRecHownShift) & 0xffu; }
__device__ __forceinline__ uint32_t rec_removed(uint32_t hdr) { return (hdr >> kRecRemovedShift) & 0xffu; }
static_assert(sizeof(ClassRec) == 64, "ClassRec must be 64 bytes");

struct DevThresholds {
    double lcom;   // mean of lcom (sequential-sum semantics)
    double cbo;    // mean of cbo
    uint32_t fast_path_ok;  // 1 if the parallel exact summation verified
    uint32_t pad;
};

// lcom_normalized_over's arithmetic (metrics.hpp:114-126) on counts:
// 0.0 if A == 0 or M == 0, else 1.0 - (double)H / ((double)A * (double)M).
// Explicit _rn intrinsics: no contraction, IEEE round-to-nearest like x86-64 SSE2.
__device__ __forceinline__ double lcom_of(uint64_t A, uint64_t M, uint64_t H) {
    if (A == 0 || M == 0) return 0.0;
    const double denom = __dmul_rn(static_cast<double>(A), static_cast<double>(M));
    return __dsub_rn(1.0, __ddiv_rn(static_cast<double>(H), denom));
}

// Sorted unique list of the classes a method uses (owners of calls ∪
// accesses, own class included) with h[k] = number of accesses owned by X[k]
// — used_classes (suggest.hpp:152-159) plus the per-class hit counts of
// intersection_count (metrics.hpp:121-123), in registers.
template <int K>
struct UsedList {
    uint32_t X[K];
    uint32_t h[K];
    int n;

    __device__ __forceinline__ void clear() {
#pragma unroll
        for (int k = 0; k < K; ++k) { X[k] = kNone; h[k] = 0; }
        n = 0;
    }
    // Insert owner v; acc = 1 for an access edge. Fully unrolled, register-only.
    __device__ __forceinline__ void insert(uint32_t v, uint32_t acc) {
        bool found = false;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (X[k] == v) { h[k] += acc; found = true; }
        if (!found) {
            uint32_t cv = v, ch = acc;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                if (cv < X[k]) {
                    const uint32_t tx = X[k], th = h[k];
                    X[k] = cv; h[k] = ch;
                    cv = tx; ch = th;
                }
            }
            ++n;
        }
    }
    __device__ __forceinline__ uint32_t hits(uint32_t v) const {
        uint32_t r = 0;
#pragma unroll
        for (int k = 0; k < K; ++k)
            if (X[k] == v) r = h[k];
        return r;
    }
    __device__ __forceinline__ bool has(uint32_t v) const {
        bool r = false;
#pragma unroll
        for (int k = 0; k < K; ++k) r |= (X[k] == v);
        return r;
    }
};

// Streaming used list for methods whose degree exceeds the register list:
// distinct owners are enumerated in ascending order by repeated min-scans of
// the method's edges. O(deg) per step; correct for any degree.
struct StreamUsed {
    const DevModel* s;
    uint32_t cb, ce, ab, ae;
    __device__ __forceinline__ void init(const DevModel& m, uint32_t p) {
        s = &m;
        cb = __ldg(m.call_off + p); ce = __ldg(m.call_off + p + 1);
        ab = __ldg(m.acc_off + p);  ae = __ldg(m.acc_off + p + 1);
    }
    // smallest owner > prev (prev = kNone means "from the start"); kNone if none
    __device__ __forceinline__ uint32_t next(uint32_t prev, uint32_t& h) const {
        uint32_t best = kNone;
        h = 0;
        for (uint32_t e = cb; e < ce; ++e) {
            const uint32_t o = __ldg(s->method_owner + __ldg(s->call_tgt + e));
            if ((prev == kNone || o > prev) && o < best) best = o;
        }
        for (uint32_t e = ab; e < ae; ++e) {
            const uint32_t o = __ldg(s->attribute_owner + __ldg(s->acc_tgt + e));
            if ((prev == kNone || o > prev) && o < best) best = o;
        }
        if (best != kNone)
            for (uint32_t e = ab; e < ae; ++e)
                h += (__ldg(s->attribute_owner + __ldg(s->acc_tgt + e)) == best);
        return best;
    }
    __device__ __forceinline__ uint32_t hits(uint32_t v) const {
        uint32_t r = 0;
        for (uint32_t e = ab; e < ae; ++e) r += (__ldg(s->attribute_owner + __ldg(s->acc_tgt + e)) == v);
        return r;
    }
    __device__ __forceinline__ bool has(uint32_t v) const {
        for (uint32_t e = cb; e < ce; ++e)
            if (__ldg(s->method_owner + __ldg(s->call_tgt + e)) == v) return true;
        for (uint32_t e = ab; e < ae; ++e)
            if (__ldg(s->attribute_owner + __ldg(s->acc_tgt + e)) == v) return true;
        return false;
    }
};

// Position of X in U row [base, base+len), or -1. Short rows (any order: the
// warp path leaves rows of ≤ 32 entries unsorted) are scanned with independent
// loads, one memory round trip per 8 entries instead of one per binary-search
// probe; long rows (always sorted) are binary searched.
__device__ __forceinline__ int urow_find(const uint32_t* __restrict__ ux, uint32_t base, uint32_t len,
                                         uint32_t X) {
    if (len <= 48) {
        for (uint32_t k0 = 0; k0 < len; k0 += 8) {
            uint32_t v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = (k0 + j < len) ? __ldg(ux + base + k0 + j) : kNone;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (v[j] == X) return (int)(k0 + j);
        }
        return -1;
    }
    uint32_t lo = 0, hi = len;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        const uint32_t v = __ldg(ux + base + mid);
        if (v < X) lo = mid + 1;
        else hi = mid;
    }
    return (lo < len && __ldg(ux + base + lo) == X) ? static_cast<int>(lo) : -1;
}

__device__ __forceinline__ ClassRec load_rec(const ClassRec* __restrict__ rec, uint32_t c) {
    const uint4* p = reinterpret_cast<const uint4*>(rec + c);
    const uint4 a = __ldg(p), b = __ldg(p + 1);
    ClassRec r;
    r.A = a.x; r.M = a.y; r.H = a.z; r.cbo = a.w;
    r.ubase = b.x; r.dense = b.y;  // sig words stay in memory: read on demand (same cache line)
    return r;
}

// Bloom test against class c's U-row signature (L1 hits once c's record line is loaded)
__device__ __forceinline__ bool sig_maybe(const ClassRec* __restrict__ rec, uint32_t c, uint32_t x) {
    const uint32_t b1 = bloom_h1(x), b2 = bloom_h2(x);
    const uint32_t w1 = __ldg(rec[c].sig + (b1 >> 5)), w2 = __ldg(rec[c].sig + (b2 >> 5));
    return ((w1 >> (b1 & 31)) & (w2 >> (b2 & 31)) & 1u) != 0;
}

}  // namespace mmg
