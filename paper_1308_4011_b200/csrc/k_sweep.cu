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

#include <cstdint>

#include "mm_device.cuh"
#include "mm_kernels.h"

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
    __device__ __forceinline__ void insert(uint32_t v, uint32_t acc) {
        int k = 0;
        while (k < n && X[k * kSweepTile] < v) ++k;
        if (k < n && X[k * kSweepTile] == v) {
            H[k * kSweepTile] += acc;
            return;
        }
        for (int j = n; j > k; --j) {
            X[j * kSweepTile] = X[(j - 1) * kSweepTile];
            H[j * kSweepTile] = H[(j - 1) * kSweepTile];
        }
        X[k * kSweepTile] = v;
        H[k * kSweepTile] = acc;
        ++n;
    }
    __device__ __forceinline__ void build(const DevModel& s, uint32_t p) {
        n = 0;
        const uint32_t cb = __ldg(s.call_off + p), ce = __ldg(s.call_off + p + 1);
        for (uint32_t e = cb; e < ce; ++e) insert(__ldg(s.method_owner + __ldg(s.call_tgt + e)), 0);
        const uint32_t ab = __ldg(s.acc_off + p), ae = __ldg(s.acc_off + p + 1);
        for (uint32_t e = ab; e < ae; ++e) insert(__ldg(s.attribute_owner + __ldg(s.acc_tgt + e)), 1);
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
    double lo_b, lo_a;
    uint32_t co_b, co_a;
    bool odeg;
};

struct Dest {
    double ld_b, ld_a;
    uint32_t cd_b, cd_a;
    bool ddeg;
};

template <class E>
__device__ __forceinline__ Origin eval_origin(const ClassRec& ro, const uint32_t* __restrict__ ux,
                                              const uint32_t* __restrict__ un, const E& en, uint32_t o) {
    Origin r;
    const uint32_t ho = en.hits(o);
    r.lo_b = ro.lcom;
    r.lo_a = lcom_of(ro.A, (uint64_t)ro.M - 1, (uint64_t)ro.H - ho);
    uint32_t removed = 0;
    en.each([&](int, uint32_t X, uint32_t) {
        if (X != o) {
            const int pos = urow_find(ux, ro.ubase, ro.cbo, X);
            if (pos >= 0 && __ldg(un + ro.ubase + pos) == 1u) ++removed;
        }
    });
    r.co_b = ro.cbo;
    r.co_a = ro.cbo - removed;
    r.odeg = ro.M <= 1 || ro.A == 0;  // origin_after.empty() || attrs empty (suggest.hpp:118-120)
    return r;
}

template <class E>
__device__ __forceinline__ Dest eval_dest(const ClassRec* __restrict__ rec, const uint32_t* __restrict__ ux,
                                          const E& en, uint32_t d, uint32_t hd) {
    const ClassRec rd = load_rec(rec, d);
    Dest r;
    r.ld_b = rd.lcom;
    r.ld_a = lcom_of(rd.A, (uint64_t)rd.M + 1, (uint64_t)rd.H + hd);
    uint32_t miss = 0;
    en.each([&](int, uint32_t X, uint32_t) {
        if (X != d && urow_find(ux, rd.ubase, rd.cbo, X) < 0) ++miss;
    });
    r.cd_b = rd.cbo;
    r.cd_a = rd.cbo + miss;
    r.ddeg = rd.A == 0;
    return r;
}

struct MethodResult {
    uint32_t count;
    uint32_t cands;
    uint32_t gated;
    uint32_t bd_coh, bd_coup;             // best-only mode
    unsigned long long m_coh, m_coup;     // top-k / all mode (bits over list index)
};

// k-th smallest passing (key, index) for one criterion, found by selection:
// the next (key, idx) strictly above (pk, pi) in lexicographic order. Used by
// the top-k extension only; keys are recomputed (k ≤ 8 rounds).
template <class E>
__device__ __forceinline__ int select_next(const SweepArgs& a, const E& en, uint32_t o, const Origin& org,
                                           bool coh, bool have_prev, double pk, int pi, double& out_key) {
    int best = -1;
    double bk = 0.0;
    en.each([&](int k, uint32_t d, uint32_t hd) {
        if (d == o) return;
        const Dest dv = eval_dest(a.rec, a.ux, en, d, hd);
        bool pass;
        double key;
        if (coh) {
            pass = org.lo_a < org.lo_b && dv.ld_a < dv.ld_b;
            key = __dadd_rn(org.lo_a, dv.ld_a);
        } else {
            pass = org.co_a < org.co_b && dv.cd_a <= dv.cd_b;
            key = (double)dv.cd_a;
        }
        if (!pass) return;
        if (have_prev && !(key > pk || (key == pk && k > pi))) return;
        if (best < 0 || key < bk) { best = k; bk = key; }
    });
    out_key = bk;
    return best;
}

template <class E>
__device__ __forceinline__ MethodResult evaluate(const SweepArgs& a, const E& en, uint32_t o,
                                                 const Origin& org, bool gcoh, bool gcoup) {
    MethodResult r;
    r.bd_coh = r.bd_coup = kNone;
    r.m_coh = r.m_coup = 0;
    uint32_t cands = 0;
    double best_coh = 0.0;
    uint32_t best_coup = 0;
    // every candidate is scored for both criteria (ungated); the class gates
    // only decide what is emitted
    en.each([&](int k, uint32_t d, uint32_t hd) {
        if (d == o) return;
        ++cands;
        const Dest dv = eval_dest(a.rec, a.ux, en, d, hd);
        const bool pcoh = org.lo_a < org.lo_b && dv.ld_a < dv.ld_b;    // suggest.hpp:189-192
        const bool pcoup = org.co_a < org.co_b && dv.cd_a <= dv.cd_b;  // :285-287
        const double kc = __dadd_rn(org.lo_a, dv.ld_a);                // :194-196
        // argmin over (key, d), d ascending, strict < : lowest d wins ties (:180-184)
        if (pcoh && (r.bd_coh == kNone || kc < best_coh)) { r.bd_coh = d; best_coh = kc; }
        if (pcoup && (r.bd_coup == kNone || dv.cd_a < best_coup)) { r.bd_coup = d; best_coup = dv.cd_a; }
        if (a.mode == 2 && k < 64) {
            if (pcoh) r.m_coh |= 1ull << k;
            if (pcoup) r.m_coup |= 1ull << k;
        } else if (a.mode == 2 && (pcoh || pcoup)) {
            atomicOr(a.err, 2u);
        }
    });
    if (a.mode == 1) {
        for (int c = 0; c < 2; ++c) {
            const bool coh = c == 0;
            if (coh ? !gcoh : !gcoup) continue;
            double pk = 0.0;
            int pi = -1;
            unsigned long long m = 0;
            for (uint32_t t = 0; t < a.topk; ++t) {
                double key;
                const int k = select_next(a, en, o, org, coh, pi >= 0, pk, pi, key);
                if (k < 0) break;
                if (k >= 64) { atomicOr(a.err, 2u); break; }
                m |= 1ull << k;
                pk = key;
                pi = k;
            }
            (coh ? r.m_coh : r.m_coup) = m;
        }
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
        count = __popcll(inter ? (r.m_coh & r.m_coup) : (r.m_coh | r.m_coup));
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

template <class E>
__device__ __forceinline__ void emit(const SweepArgs& a, const E& en, uint32_t p, uint32_t o,
                                     const Origin& org, const MethodResult& r, uint64_t at) {
    const bool both = (a.crit & MM_CRIT_COHESION) && (a.crit & MM_CRIT_COUPLING);
    const bool inter = a.combine == MM_COMBINE_INTERSECTION && both;
    en.each([&](int k, uint32_t d, uint32_t hd) {
        if (d == o) return;
        bool tcoh, tcoup;
        if (a.mode == 0) {
            tcoh = d == r.bd_coh;
            tcoup = d == r.bd_coup;
        } else {
            tcoh = k < 64 && ((r.m_coh >> k) & 1ull);
            tcoup = k < 64 && ((r.m_coup >> k) & 1ull);
        }
        if (inter ? !(tcoh && tcoup) : !(tcoh || tcoup)) return;
        const Dest dv = eval_dest(a.rec, a.ux, en, d, hd);
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

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += y;
    }
    return v;
}

template <int K>
__global__ void __launch_bounds__(kSweepTile) k_sweep(SweepArgs a) {
    __shared__ uint32_t s_X[K * kSweepTile], s_H[K * kSweepTile];
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_warp[kSweepTile / 32];
    __shared__ unsigned long long s_excl;
    __shared__ unsigned long long s_red[3][kSweepTile / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(a.tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = s_tile;
    const uint64_t pos = (uint64_t)a.pos_begin + (uint64_t)tile * kSweepTile + threadIdx.x;
    const bool valid = pos < a.pos_end;

    double thr_l = a.thr_lcom, thr_c = a.thr_cbo;
    if (a.thr_device) { thr_l = a.dthr->lcom; thr_c = a.dthr->cbo; }

    uint32_t p = 0, o = 0;
    bool fast = true;
    SmemEnum ren;
    ren.X = s_X + threadIdx.x;
    ren.H = s_H + threadIdx.x;
    ren.n = 0;
    StreamEnum sen;
    Origin org{};
    MethodResult res{};
    if (valid) {
        p = __ldg(a.s.cls_methods + pos);
        o = __ldg(a.s.method_owner + p);
        const uint32_t deg = (__ldg(a.s.call_off + p + 1) - __ldg(a.s.call_off + p)) +
                             (__ldg(a.s.acc_off + p + 1) - __ldg(a.s.acc_off + p));
        fast = deg <= (uint32_t)K;
        const ClassRec ro = load_rec(a.rec, o);
        // gates: lcom[c] > thr.lcom (suggest.hpp:246), (double)cbo[c] > thr.cbo (:273)
        const bool gcoh = (a.crit & MM_CRIT_COHESION) && ro.lcom > thr_l;
        const bool gcoup = (a.crit & MM_CRIT_COUPLING) && (double)ro.cbo > thr_c;
        if (fast) {
            ren.build(a.s, p);
            org = eval_origin(ro, a.ux, a.un, ren, o);
            res = evaluate(a, ren, o, org, gcoh, gcoup);
        } else {
            sen.S.init(a.s, p);
            org = eval_origin(ro, a.ux, a.un, sen, o);
            res = evaluate(a, sen, o, org, gcoh, gcoup);
        }
    }

    // tile-wide exclusive scan of record counts
    const uint32_t inc = warp_incl_scan(res.count, lane);
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    uint32_t before = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kSweepTile / 32; ++w) {
        if (w < warp) before += s_warp[w];
        agg += s_warp[w];
    }
    const uint32_t texcl = before + inc - res.count;

    // decoupled look-back for the tile's global offset
    if (threadIdx.x == 0) {
        unsigned long long excl = 0;
        if (tile == 0) {
            __threadfence();
            atomicExch(a.tile_state, kFlagPrefix | agg);
        } else {
            __threadfence();
            atomicExch(a.tile_state + tile, kFlagAgg | agg);
            int j = (int)tile - 1;
            while (true) {
                const unsigned long long v = *reinterpret_cast<volatile unsigned long long*>(a.tile_state + j);
                const unsigned long long f = v & ~kValMask;
                if (f == 0) continue;
                excl += v & kValMask;
                if (f == kFlagPrefix) break;
                --j;
            }
            __threadfence();
            atomicExch(a.tile_state + tile, kFlagPrefix | (excl + agg));
        }
        s_excl = excl;
    }
    // stats (one atomic per tile per counter)
    {
        unsigned long long c0 = res.cands, c1 = res.gated, c2 = valid ? 1ull : 0ull;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            c0 += __shfl_down_sync(0xffffffffu, c0, d);
            c1 += __shfl_down_sync(0xffffffffu, c1, d);
            c2 += __shfl_down_sync(0xffffffffu, c2, d);
        }
        if (lane == 0) { s_red[0][warp] = c0; s_red[1][warp] = c1; s_red[2][warp] = c2; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t0 = 0, t1 = 0, t2 = 0;
        for (int w = 0; w < kSweepTile / 32; ++w) { t0 += s_red[0][w]; t1 += s_red[1][w]; t2 += s_red[2][w]; }
        atomicAdd(a.stats + 0, t0);
        atomicAdd(a.stats + 1, t1);
        atomicAdd(a.stats + 2, (unsigned long long)agg);
        atomicAdd(a.stats + 3, t2);
    }
    if (valid && res.count) {
        const uint64_t at = s_excl + texcl;
        if (fast) emit(a, ren, p, o, org, res, at);
        else emit(a, sen, p, o, org, res, at);
    }
}

__global__ void k_what_if(DevModel s, const ClassRec* __restrict__ rec, const uint32_t* __restrict__ ux,
                          const uint32_t* __restrict__ un, uint32_t u, uint32_t o, uint32_t d,
                          mm_whatif* __restrict__ out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    StreamEnum en;
    en.S.init(s, u);
    const ClassRec ro = load_rec(rec, o);
    const Origin org = eval_origin(ro, ux, un, en, o);
    const Dest dv = eval_dest(rec, ux, en, d, en.hits(d));
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

}  // namespace

void launch_sweep(const SweepArgs& a, uint32_t n_tiles, cudaStream_t st) {
    if (!n_tiles) return;
    if (a.maxdeg_fast <= 8) k_sweep<8><<<n_tiles, kSweepTile, 0, st>>>(a);
    else k_sweep<16><<<n_tiles, kSweepTile, 0, st>>>(a);
}

void launch_what_if(const DevModel& s, const ClassRec* rec, const uint32_t* ux, const uint32_t* un, uint32_t u,
                    uint32_t o, uint32_t d, mm_whatif* out, cudaStream_t st) {
    k_what_if<<<1, 32, 0, st>>>(s, rec, ux, un, u, o, d, out);
}

}  // namespace mmg
