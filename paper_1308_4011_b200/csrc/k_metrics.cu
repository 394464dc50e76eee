// k_metrics.cu — the class metric pass (LCOM normalized, LCOM-CK, CBO + the
// class×class use-count rows U) and the threshold means.
//
// Replaces the per-class loop of full_report (metrics.hpp:253-261) and
// parallel_class_metrics / parallel_lcom_ck (parallel.hpp:149-174). Results
// are bit-identical to the reference:
//   lcom    : H = Σ_p |acc(p) ∩ attrs(c)| counted as accesses whose owner is c
//             (same integer as intersection_count, metrics.hpp:121-123 for a
//             validated model), then the reference's single-division formula.
//   lcom_ck : Q = #pairs (i<j) whose own-attribute sets intersect; with
//             P = C(M,2) - Q the reference returns P > Q ? P - Q : 0
//             (metrics.hpp:147-156).
//   cbo     : |{owner(t) : t ∈ calls ∪ accesses of members} \ {c}|
//             (metrics.hpp:167-185), built as the sorted U row with counts.
#include <cuda_runtime.h>

#include <atomic>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "mm_device.cuh"
#include "mm_kernels.h"

namespace mmg {

// ---------------------------------------------------------------------------
// upload-time: range validation and class planning
// ---------------------------------------------------------------------------

__global__ void k_validate_ids(const uint32_t* __restrict__ v, uint64_t n, uint32_t bound,
                               uint32_t* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (v[i] >= bound) atomicOr(bad, 1u);
}

// offsets must be non-decreasing, start at 0 and end at `total`
__global__ void k_validate_offsets(const uint32_t* __restrict__ off, uint64_t n_plus_1, uint32_t total,
                                   uint32_t* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_plus_1;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (i == 0 && off[0] != 0) atomicOr(bad, 2u);
        if (i + 1 == n_plus_1 && off[i] != total) atomicOr(bad, 2u);
        if (i + 1 < n_plus_1 && off[i] > off[i + 1]) atomicOr(bad, 2u);
    }
}

// fan_out[p] = |calls(p)| (metrics.hpp:87-93); fan_in[t] += 1 per call-list
// occurrence of t (metrics.hpp:79-85) — integer atomics, so the counts are
// exact and order-free. Thread per method: its own row, then its targets.
// Also the largest call and access sets (estimate_workload's k_m / k_a,
// metrics.hpp:228-233): a warp max, then one atomic per warp.
__global__ void k_fan(DevModel s, uint32_t* __restrict__ fan_in, uint32_t* __restrict__ fan_out,
                      uint32_t* __restrict__ kmax) {
    const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t nc = 0, na = 0;
    if (p < s.M) {
        const uint32_t cb = s.call_off[p], ce = s.call_off[p + 1];
        nc = ce - cb;
        na = s.acc_off[p + 1] - s.acc_off[p];
        if (fan_out) fan_out[p] = nc;
        if (fan_in)
            for (uint32_t e = cb; e < ce; ++e) atomicAdd(fan_in + __ldg(s.call_tgt + e), 1u);
    }
    nc = __reduce_max_sync(0xffffffffu, nc);
    na = __reduce_max_sync(0xffffffffu, na);
    if ((threadIdx.x & 31) == 0 && kmax) {
        atomicMax(kmax, nc);
        atomicMax(kmax + 1, na);
    }
}

// Upload-time expansion of the membership lists, one thread per list
// position (method positions, then attribute positions), its class found by a
// binary search of the class offsets (warps hold consecutive positions, so
// they walk the same search path; a warp per class serialised Zipf giants):
//   pos_owner[k]  = class of method position k (the class-order owner table
//                   every pass reads instead of gathering method_owner)
//   attr_info[t]  = (owner(t), position of t in its owner's attribute list):
//                   one 8-byte gather gives the method pass the owner and the
//                   LCOM-CK mask bit
//   method_owner / attribute_owner, when the caller omitted them
// Every index is clamped or bounds-checked: this runs before validation's
// verdict is known.
__device__ __forceinline__ uint32_t class_of(const uint32_t* __restrict__ off, uint32_t C, uint32_t k) {
    uint32_t lo = 0, hi = C - 1;  // the largest c with off[c] <= k
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (__ldg(off + mid) <= k) lo = mid; else hi = mid - 1;
    }
    return lo;
}
__global__ void k_expand(DevModel s, uint32_t* __restrict__ mo_out, uint32_t* __restrict__ ao_out,
                         uint32_t* __restrict__ pos_owner, uint2* __restrict__ info) {
    const uint64_t n = (uint64_t)s.M + s.A;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (i < s.M) {
            const uint32_t k = (uint32_t)i;
            const uint32_t c = class_of(s.cls_moff, s.C, k);
            pos_owner[k] = c;
            if (mo_out) {
                const uint32_t p = s.cls_methods[k];
                if (p < s.M) mo_out[p] = c;
            }
        } else {
            const uint32_t k = (uint32_t)(i - s.M);
            const uint32_t c = class_of(s.cls_aoff, s.C, k);
            const uint32_t t = s.cls_attrs[k];
            if (t >= s.A) continue;
            if (ao_out) ao_out[t] = c;
            info[t] = make_uint2(ao_out ? c : s.attribute_owner[t], k - min(__ldg(s.cls_aoff + c), k));
        }
    }
}

// Upload-time layout: the call / access rows in class order, in three
// kernels over 256-position tiles: per-tile degree sums, one block scanning
// the tile sums, then the row pass below (its block scan + the tile base give
// the class-order offsets, written beside the rows). Indices are
// bounds-checked (this runs before the validation verdict is known).
constexpr uint32_t kPosTile = 256;

struct PosRow {
    uint32_t p, cb, ce, ab, ae;
};
__device__ __forceinline__ PosRow pos_row(const DevModel& s, uint32_t k, uint32_t Ec, uint32_t Ea) {
    PosRow r{s.M, 0, 0, 0, 0};
    if (k >= s.M) return r;
    r.p = s.cls_methods[k];
    if (r.p >= s.M) return r;
    r.cb = min(s.call_off[r.p], Ec); r.ce = min(max(s.call_off[r.p + 1], r.cb), Ec);
    r.ab = min(s.acc_off[r.p], Ea); r.ae = min(max(s.acc_off[r.p + 1], r.ab), Ea);
    return r;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= (uint32_t)d) v += u;
    }
    return v;
}

__global__ void __launch_bounds__(kPosTile) k_pos_tile_sums(DevModel s, uint32_t* __restrict__ tsum) {
    __shared__ uint32_t ws[2][kPosTile / 32];
    const uint32_t Ec = s.call_off[s.M], Ea = s.acc_off[s.M];
    const PosRow r = pos_row(s, blockIdx.x * kPosTile + threadIdx.x, Ec, Ea);
    const uint32_t sc = __reduce_add_sync(0xffffffffu, r.ce - r.cb), sa = __reduce_add_sync(0xffffffffu, r.ae - r.ab);
    if ((threadIdx.x & 31) == 0) { ws[0][threadIdx.x >> 5] = sc; ws[1][threadIdx.x >> 5] = sa; }
    __syncthreads();
    if (threadIdx.x < 2) {
        uint32_t v = 0;
        for (int w = 0; w < (int)(kPosTile / 32); ++w) v += ws[threadIdx.x][w];
        tsum[threadIdx.x * gridDim.x + blockIdx.x] = v;
    }
}

// one block: exclusive scans of both tile-sum arrays in place (4 consecutive
// tiles per thread, both arrays in the same pass), and the totals into
// pc_off[M] / pa_off[M]
__global__ void __launch_bounds__(1024) k_pos_tile_scan(uint32_t* __restrict__ tsum, uint32_t ntiles,
                                                        uint32_t* __restrict__ pc_off, uint32_t* __restrict__ pa_off,
                                                        uint32_t M) {
    __shared__ uint32_t ws[2][32];
    const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t carry[2] = {0u, 0u};
    for (uint32_t base = 0; base < ntiles; base += 4096) {
        const uint32_t i0 = base + 4 * threadIdx.x;
        uint32_t v[2][4], s[2] = {0u, 0u};
#pragma unroll
        for (int arr = 0; arr < 2; ++arr)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[arr][j] = i0 + j < ntiles ? tsum[arr * ntiles + i0 + j] : 0u;
                s[arr] += v[arr][j];
            }
        uint32_t incl[2];
#pragma unroll
        for (int arr = 0; arr < 2; ++arr) {
            incl[arr] = warp_incl_scan(s[arr], lane);
            if (lane == 31) ws[arr][w] = incl[arr];
        }
        __syncthreads();
        if (w < 2) ws[w][lane] = warp_incl_scan(ws[w][lane], lane);
        __syncthreads();
#pragma unroll
        for (int arr = 0; arr < 2; ++arr) {
            uint32_t x = carry[arr] + (w ? ws[arr][w - 1] : 0u) + incl[arr] - s[arr];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (i0 + j < ntiles) tsum[arr * ntiles + i0 + j] = x;
                x += v[arr][j];
            }
            carry[arr] += ws[arr][31];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        pc_off[M] = carry[0];
        pa_off[M] = carry[1];
    }
}

// The row pass: one warp per 32 consecutive class-order positions, whose rows
// are flattened (warp scan of the degrees) and copied one element per lane
// (two per iteration, loads issued before use), so the class-order writes are
// fully coalesced and short rows do not idle lanes. Beside each target: the
// member index of its position within the class (255 past that), which the
// lean class kernel reads instead of searching the members' row starts. The
// same pass folds the class plan's per-member inputs (formerly a separate
// per-method pass): the foreign-edge count and the largest degree per class,
// and the number of methods whose used list can outgrow a method record.
__device__ __forceinline__ uint32_t flat_pos(uint32_t excl, uint32_t i) {
    uint32_t j = 0;  // the position holding element i: the largest j with excl_j <= i
#pragma unroll
    for (int step = 16; step; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, excl, j + step);
        if (v <= i) j += step;
    }
    return j;
}
__device__ __forceinline__ void flat_rows(uint32_t lane, uint32_t b, uint32_t excl, uint32_t total, uint32_t dst0,
                                          uint32_t limit, const uint32_t* __restrict__ src,
                                          const uint32_t* __restrict__ owner, uint32_t bound, uint32_t c,
                                          uint32_t mi, uint32_t* __restrict__ tgt, uint8_t* __restrict__ mem,
                                          uint32_t* __restrict__ fr) {
    for (uint32_t base = 0; base < total; base += 64) {
        const uint32_t i0 = base + lane, i1 = i0 + 32;
        const uint32_t j0 = flat_pos(excl, i0), j1 = flat_pos(excl, i1);
        const uint32_t e0 = __shfl_sync(0xffffffffu, excl, j0), e1 = __shfl_sync(0xffffffffu, excl, j1);
        const uint32_t b0 = __shfl_sync(0xffffffffu, b, j0), b1 = __shfl_sync(0xffffffffu, b, j1);
        const uint32_t c0 = __shfl_sync(0xffffffffu, c, j0), c1 = __shfl_sync(0xffffffffu, c, j1);
        const uint32_t m0 = __shfl_sync(0xffffffffu, mi, j0), m1 = __shfl_sync(0xffffffffu, mi, j1);
        const uint32_t o0 = dst0 + i0, o1 = dst0 + i1;
        const bool v0 = i0 < total && o0 < limit, v1 = i1 < total && o1 < limit;
        const uint32_t x0 = v0 ? __ldg(src + b0 + (i0 - e0)) : 0u;
        const uint32_t x1 = v1 ? __ldg(src + b1 + (i1 - e1)) : 0u;
        const uint32_t w0 = v0 && x0 < bound ? __ldg(owner + x0) : kNone;
        const uint32_t w1 = v1 && x1 < bound ? __ldg(owner + x1) : kNone;
        if (v0) {
            tgt[o0] = x0;
            mem[o0] = (uint8_t)m0;
            if (w0 != c0) atomicAdd_block(fr + j0, 1u);
        }
        if (v1) {
            tgt[o1] = x1;
            mem[o1] = (uint8_t)m1;
            if (w1 != c1) atomicAdd_block(fr + j1, 1u);
        }
    }
}

__global__ void __launch_bounds__(kPosTile) k_pos_rows(DevModel s, const uint32_t* __restrict__ pos_owner,
                                                       const uint32_t* __restrict__ tsum, uint32_t* __restrict__ pc_off,
                                                       uint32_t* __restrict__ pa_off, uint32_t* __restrict__ pc_tgt,
                                                       uint32_t* __restrict__ pa_tgt, uint8_t* __restrict__ pc_mem,
                                                       uint8_t* __restrict__ pa_mem, uint32_t* __restrict__ foreign,
                                                       uint32_t* __restrict__ cmaxdeg, uint32_t* __restrict__ n_hideg) {
    __shared__ uint32_t fr_s[kPosTile / 32][32];
    __shared__ uint32_t ws[2][kPosTile / 32];
    const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const uint32_t k = blockIdx.x * kPosTile + threadIdx.x;
    uint32_t* fr = fr_s[wib];
    fr[lane] = 0;
    const uint32_t Ec = s.call_off[s.M], Ea = s.acc_off[s.M];
    const PosRow r = pos_row(s, k, Ec, Ea);
    uint32_t c = kNone, mi = 255u;
    if (k < s.M) {
        c = pos_owner[k];
        mi = c < s.C ? min(k - min(s.cls_moff[c], k), 255u) : 255u;
    }
    const uint32_t nc = r.ce - r.cb, na = r.ae - r.ab;
    const uint32_t ic = warp_incl_scan(nc, lane), ia = warp_incl_scan(na, lane);
    if (lane == 31) { ws[0][wib] = ic; ws[1][wib] = ia; }
    __syncthreads();
    uint32_t wc = tsum[blockIdx.x], wa = tsum[gridDim.x + blockIdx.x];
    for (uint32_t w = 0; w < wib; ++w) { wc += ws[0][w]; wa += ws[1][w]; }
    if (k < s.M) { pc_off[k] = wc + ic - nc; pa_off[k] = wa + ia - na; }
    const uint32_t tc = __shfl_sync(0xffffffffu, ic, 31), ta = __shfl_sync(0xffffffffu, ia, 31);
    flat_rows(lane, r.cb, ic - nc, tc, wc, Ec, s.call_tgt, s.method_owner, s.M, c, mi, pc_tgt, pc_mem, fr);
    flat_rows(lane, r.ab, ia - na, ta, wa, Ea, s.acc_tgt, s.attribute_owner, s.A, c, mi, pa_tgt, pa_mem, fr);
    __syncwarp();
    // plan inputs, one atomic per class present in the warp
    const bool member = k < s.M && r.p < s.M && c < s.C;
    const uint32_t deg = nc + na;
    const uint32_t hi = __ballot_sync(0xffffffffu, member && deg > (uint32_t)kRecMaxEnt);
    if (hi && lane == 0) atomicAdd(n_hideg, __popc(hi));
    const uint32_t grp = __match_any_sync(0xffffffffu, member ? c : kNone);
    const uint32_t fsum = __reduce_add_sync(grp, member ? fr[lane] : 0u);
    const uint32_t dmax = __reduce_max_sync(grp, member ? deg : 0u);
    if (member && lane == (uint32_t)(__ffs(grp) - 1)) {
        if (fsum) atomicAdd(foreign + c, fsum);
        atomicMax(cmaxdeg + c, dmax);
    }
}

// classify into the warp path (small) or the CTA path (large)
__global__ void k_plan_classes(DevModel s, const uint32_t* __restrict__ cmaxdeg, const uint32_t* __restrict__ foreign,
                               uint4* __restrict__ cplan, uint4* __restrict__ cedge, uint32_t* __restrict__ large_list,
                               uint32_t* __restrict__ n_large, uint32_t* __restrict__ big_list,
                               uint32_t* __restrict__ n_big, uint32_t* __restrict__ max_deg) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= s.C) return;
    const uint32_t mb = min(s.cls_moff[c], s.M), me = min(max(s.cls_moff[c + 1], mb), s.M);
    const uint32_t A = s.cls_aoff[c + 1] - s.cls_aoff[c];
    const uint32_t mdeg = cmaxdeg[c];
    const bool small = (me - mb) <= kSmallMaxMembers && A <= kSmallMaxAttrs && mdeg <= kSmallMaxDeg &&
                       s.C < (1u << 27);  // warp path packs X << 5 | member into 32 bits
    // warp path: ≤ 32 foreign edges (so ≤ 32 U-row keys) take the lean
    // register-sort variant, the rest the shared-memory one (listed)
    const uint32_t kind = !small ? kKindCta : (foreign[c] <= 32 ? kKindLean : kKindWarpBig);
    cplan[c] = make_uint4(mb, me - mb, A, kind);
    // the class's edge ranges in the class-order rows
    cedge[c] = make_uint4(s.pc_off[mb], s.pc_off[me], s.pa_off[mb], s.pa_off[me]);
    if (kind == kKindCta) large_list[atomicAdd(n_large, 1u)] = c;
    if (kind == kKindWarpBig) big_list[atomicAdd(n_big, 1u)] = c;
    atomicMax(max_deg, mdeg);
}

// Method pass in class order: thread i handles the method at class-order
// position i. CSR rows are gathered (sector-sized random reads); every write
// — the 32-byte MethRec, the own-attribute mask, the owner — is coalesced
// (random partial-sector writes would cost a DRAM read-modify-write each).
// Each method's sorted used list with per-class access counts is packed into
// its MethRec; the own-attribute mask has bit k for the k-th attribute of the
// own class (classes with ≤ 64 attributes).
constexpr int kChunkBuckets = 8;  // k_method regrouping: 0..6 chunks, 7 = more or past the end

#ifndef MMGPU_METHOD_MINB
#define MMGPU_METHOD_MINB 4
#endif
template <int K, bool REGROUP>
__global__ void __launch_bounds__(256, MMGPU_METHOD_MINB)
k_method(DevModel s, MethRec* __restrict__ recs, uint64_t* __restrict__ own_mask,
         const uint32_t* __restrict__ pos_owner, const uint32_t* __restrict__ plist, uint32_t n_pos) {
    // Blocks holding methods of more than one chunk (dense shapes like C5)
    // first regroup their positions by chunk count (a counting sort in shared
    // memory), so a warp's threads loop the same number of chunks instead of
    // all waiting for the warp's longest row. Writes stay inside the block's
    // own position range (whole 32-byte records; L2 merges the masks).
    __shared__ uint32_t s_cnt[kChunkBuckets], s_perm[256];
    uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
    if (plist) pos = pos < n_pos ? __ldg(plist + pos) : kNone;  // only the listed positions (non-lean classes)
    if (REGROUP) {
        const bool live = pos < s.M;
        uint32_t nch = 0;
        if (live) {
            const uint32_t d = (__ldg(s.pc_off + pos + 1) - __ldg(s.pc_off + pos)) +
                               (__ldg(s.pa_off + pos + 1) - __ldg(s.pa_off + pos));
            nch = (d + K - 1) / K;
        }
        if (threadIdx.x < kChunkBuckets) s_cnt[threadIdx.x] = 0;
        if (__syncthreads_or(nch > 1)) {
            const uint32_t b = live ? min(nch, (uint32_t)kChunkBuckets - 1) : kChunkBuckets - 1;
            const int lane = threadIdx.x & 31;
            const uint32_t grp = __match_any_sync(0xffffffffu, b);
            const int lead = __ffs(grp) - 1;
            uint32_t base = 0;
            if (lane == lead) base = atomicAdd(&s_cnt[b], __popc(grp));
            base = __shfl_sync(0xffffffffu, base, lead) + __popc(grp & ((1u << lane) - 1));
            __syncthreads();
            if (threadIdx.x == 0) {  // bucket starts (exclusive prefix)
                uint32_t acc = 0;
                for (int k = 0; k < kChunkBuckets; ++k) {
                    const uint32_t c = s_cnt[k];
                    s_cnt[k] = acc;
                    acc += c;
                }
            }
            __syncthreads();
            s_perm[s_cnt[b] + base] = live ? pos : kNone;
            __syncthreads();
            pos = s_perm[threadIdx.x];
        }
    }
    if (pos >= s.M) return;
    const uint32_t own = __ldg(pos_owner + pos);
    // this position's rows, laid out in class order at upload: coalesced
    const uint32_t cb = __ldg(s.pc_off + pos), ce = __ldg(s.pc_off + pos + 1);
    const uint32_t ab = __ldg(s.pa_off + pos), ae = __ldg(s.pa_off + pos + 1);
    const uint32_t oab = __ldg(s.cls_aoff + own), oae = __ldg(s.cls_aoff + own + 1);
    uint32_t hdr = kRecOverflow;
    uint32_t ent[kRecMaxEnt];
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k) ent[k] = 0;
    uint64_t mask = 0;
    const uint32_t nc = ce - cb, na = ae - ab, deg = nc + na;
    // edges in chunks of K: all targets of a chunk, then all their owner
    // gathers — two memory round trips per chunk instead of two per edge.
    // The list keeps kRecMaxEnt + 1 slots: a 9th distinct class means the
    // record cannot hold the list (consumers then read the CSR).
    UsedList<kRecMaxEnt + 1> L;
    L.clear();
    uint32_t hown = 0;
    bool own_used = false;
    // masks feed LCOM-CK of every class with ≤ 64 attributes (both class paths)
    const bool small_attrs = oae - oab <= 64;
    auto chunk = [&](uint32_t e0) {
        uint32_t tg[K], ow[K], rk[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t e = e0 + k;
            const bool isc = e < nc, isa = !isc && e < deg;
            tg[k] = isc ? __ldg(s.pc_tgt + cb + e) : (isa ? __ldg(s.pa_tgt + ab + (e - nc)) : 0u);
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t e = e0 + k;
            const bool isc = e < nc, isa = !isc && e < deg;
            if (isc) {
                ow[k] = __ldg(s.method_owner + tg[k]);
            } else if (isa) {
                const uint2 ai = __ldg(s.attr_info + tg[k]);
                ow[k] = ai.x;
                rk[k] = ai.y;
            } else {
                ow[k] = kNone;
            }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const uint32_t e = e0 + k;
            const bool isa = e >= nc && e < deg;
            if (e >= deg) continue;
            if (ow[k] == own) {  // own class: counted here, inserted once below (cheap for intra-class edges)
                own_used = true;
                if (isa) {
                    if (small_attrs) mask |= 1ull << rk[k];
                    ++hown;
                }
            } else {
                L.insert(ow[k], isa ? 1u : 0u);
            }
        }
    };
    if (deg <= (uint32_t)K) chunk(0);  // the common case: one straight-line chunk
    else
        for (uint32_t e0 = 0; e0 < deg; e0 += K) chunk(e0);
    if (own_used) L.insert(own, hown);
    bool fits = L.n <= kRecMaxEnt && hown < 256;
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k)
        if (k < L.n) {
            fits = fits && L.X[k] < (1u << 24) && L.h[k] < 256;
            ent[k] = (L.X[k] << 8) | L.h[k];
        }
    if (fits) hdr = (uint32_t)L.n | (hown << kRecHownShift);
    uint4* dst = reinterpret_cast<uint4*>(recs + pos);
    dst[0] = make_uint4(ent[0], ent[1], ent[2], ent[3]);
    dst[1] = make_uint4(ent[4], ent[5], ent[6], ent[7]);
    rec_hdrs(recs, s.M)[pos] = hdr;
    own_mask[pos] = mask;
}

// ---------------------------------------------------------------------------
// warp path: one warp per class, one lane per member (M ≤ 32, A ≤ 64, deg ≤ 16)
// ---------------------------------------------------------------------------

constexpr int kWarpsPerBlock = 8;
constexpr int kSmallEntries = kSmallMaxMembers * kSmallMaxDeg;  // 512

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) { return __reduce_add_sync(0xffffffffu, v); }

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, int lane) {
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    return x - v;
}

// ascending bitonic sort of buf[0, N) (N a power of two ≥ 2), one warp
__device__ __forceinline__ void warp_bitonic_u32(uint32_t* buf, int N, int lane) {
    for (int k = 2; k <= N; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < N; i += 32) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t a = buf[i], b = buf[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { buf[i] = b; buf[ixj] = a; }
                }
            }
            __syncwarp();
        }
}

// One warp per class, one lane per member. Members' used lists come from the
// method pass records (coalesced: a class's members are contiguous in class
// order); a member whose list overflowed its record is rebuilt from the CSR.
template <bool BIG>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, BIG ? 1 : 6)
k_class_small(DevModel s, const uint4* __restrict__ cplan, const uint32_t* __restrict__ list, uint32_t n_list,
              MethRec* __restrict__ recs, const uint64_t* __restrict__ own_mask, ClassRec* __restrict__ rec,
              double* __restrict__ lcom_out, uint64_t* __restrict__ ck_out, uint32_t* __restrict__ cbo_out,
              uint32_t* __restrict__ ux, uint32_t* __restrict__ un) {
    constexpr int kBuf = BIG ? kSmallEntries : 32;
    __shared__ uint32_t sbuf[kWarpsPerBlock][kBuf];
    __shared__ uint32_t scnt[kWarpsPerBlock][BIG ? kSmallEntries : 1];
    __shared__ uint32_t srem[kWarpsPerBlock][32];
    __shared__ uint32_t ssig[kWarpsPerBlock][kSigWords];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t wid = blockIdx.x * kWarpsPerBlock + warp;
    uint32_t c;
    if (BIG) {
        if (wid >= n_list) return;
        c = list[wid];
    } else {
        c = wid;
        if (c >= s.C) return;
    }
    const uint4 cp = cplan[c];  // (first member position, M, A, kind): one load
    if (!BIG && cp.w != kKindLean) return;  // warp-uniform exit
    const uint32_t mb = cp.x, M = cp.y, A = cp.z;
    const bool active = lane < (int)M;
    const uint32_t pos = mb + lane;

    UsedList<kSmallMaxDeg> L;  // only for overflowed records
    L.clear();
    uint4 r0 = make_uint4(0, 0, 0, 0), r1 = make_uint4(0, 0, 0, 0);
    uint32_t hdr = kRecOverflow;
    uint64_t mask = 0;
    uint32_t hown = 0;
    uint32_t* hdrs = rec_hdrs(recs, s.M);
    if (active) {
        const uint4* src = reinterpret_cast<const uint4*>(recs + pos);
        r0 = src[0];
        r1 = src[1];
        hdr = hdrs[pos];
        mask = own_mask[pos];
    }
    const bool ovf = active && (hdr & kRecOverflow);
    const uint32_t ent[kRecMaxEnt] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    uint32_t nent = active && !ovf ? rec_n(hdr) : 0;
    if (active && !ovf) hown = rec_hown(hdr);
    if (ovf) {
        const uint32_t p = s.cls_methods[pos];
        const uint32_t cb = __ldg(s.call_off + p), ce = __ldg(s.call_off + p + 1);
        for (uint32_t e = cb; e < ce; ++e) L.insert(__ldg(s.method_owner + __ldg(s.call_tgt + e)), 0);
        const uint32_t ab = __ldg(s.acc_off + p), ae = __ldg(s.acc_off + p + 1);
        mask = 0;
        for (uint32_t e = ab; e < ae; ++e) {
            const uint2 ai = __ldg(s.attr_info + __ldg(s.acc_tgt + e));
            L.insert(ai.x, 1);
            if (ai.x == c) {
                mask |= 1ull << ai.y;
                ++hown;
            }
        }
    }
    const uint32_t H = warp_sum(hown);

    // LCOM-CK: Q = #pairs (i<j) with intersecting own sets
    uint32_t q = 0;
    for (uint32_t k = 0; k < M; ++k) {
        const uint64_t mk = __shfl_sync(0xffffffffu, mask, k);
        if ((uint32_t)lane < k && (mask & mk)) ++q;
    }
    const uint32_t Q = warp_sum(q);

    // U row: multiset union of the members' used classes other than c, as
    // keys X << 5 | member so that a run of length 1 names the one member that
    // alone uses X (that member's cbo_origin_after drops by one, App. A)
    uint32_t cnt = 0;
    if (ovf) cnt = (uint32_t)L.n - (L.has(c) ? 1u : 0u);
    else
#pragma unroll
        for (int k = 0; k < kRecMaxEnt; ++k) cnt += (k < (int)nent && (ent[k] >> 8) != c);
    const uint32_t off = warp_excl_scan(cnt, lane);
    const uint32_t T = __shfl_sync(0xffffffffu, off + cnt, 31);
    uint32_t* buf = sbuf[warp];
    uint32_t* rcnt = scnt[warp];
    const uint32_t ubase = kSmallRowCap * mb;
    {
        uint32_t w = off;
        if (ovf) {
#pragma unroll
            for (int k = 0; k < kSmallMaxDeg; ++k)
                if (k < L.n && L.X[k] != c) buf[w++] = (L.X[k] << 5) | lane;
        } else {
#pragma unroll
            for (int k = 0; k < kRecMaxEnt; ++k)
                if (k < (int)nent && (ent[k] >> 8) != c) buf[w++] = ((ent[k] >> 8) << 5) | lane;
        }
    }
    uint32_t* rem = srem[warp];  // per-member removed counters (smem path)
    uint32_t* sig = ssig[warp];   // Bloom signature of the U row
    if (lane < kSigWords) sig[lane] = 0;
    rem[lane] = 0;
    __syncwarp();
    uint32_t cbo = 0;
    uint32_t removed_me = 0;
    if (T <= 32) {
        // one key per lane; lanes holding the same class X form a match group:
        // its size is U[c][X], a group of one names the member that alone uses
        // X. Rows this short are scanned linearly by every consumer, so they
        // stay in lane order — no sort.
        const uint32_t v = lane < (int)T ? buf[lane] : kNone;
        const uint32_t X = v >> 5;  // X < 2^27 - 1 < kNone >> 5: padding lanes never join a real group
        const uint32_t grp = __match_any_sync(0xffffffffu, X);
        const bool head = lane < (int)T && (uint32_t)(__ffs(grp) - 1) == (uint32_t)lane;
        const uint32_t hb = __ballot_sync(0xffffffffu, head);
        cbo = __popc(hb);
        if (head) {
            const uint32_t n = __popc(grp);
            if (n == 1) atomicAdd(rem + (v & 31u), 1u);  // the member named by the key loses X
            const uint32_t idx = __popc(hb & ((1u << lane) - 1));
            ux[ubase + idx] = X;
            un[ubase + idx] = n;
            const uint32_t b1 = bloom_h1(X), b2 = bloom_h2(X);
            atomicOr(sig + (b1 >> 5), 1u << (b1 & 31));
            atomicOr(sig + (b2 >> 5), 1u << (b2 & 31));
        }
    } else if (BIG) {
        int N = 64;
        while (N < (int)T) N <<= 1;
        for (int i = (int)T + lane; i < N; i += 32) buf[i] = kNone;
        __syncwarp();
        warp_bitonic_u32(buf, N, lane);
        uint32_t nh = 0;
        for (uint32_t base = 0; base < T; base += 32) {  // heads compacted into rcnt (positions)
            const uint32_t i = base + lane;
            const bool head = i < T && (i == 0 || (buf[i] >> 5) != (buf[i - 1] >> 5));
            const uint32_t b = __ballot_sync(0xffffffffu, head);
            if (head) {
                rcnt[nh + __popc(b & ((1u << lane) - 1))] = i;
                const uint32_t b1 = bloom_h1(buf[i] >> 5), b2 = bloom_h2(buf[i] >> 5);
                atomicOr(sig + (b1 >> 5), 1u << (b1 & 31));
                atomicOr(sig + (b2 >> 5), 1u << (b2 & 31));
            }
            nh += __popc(b);
        }
        __syncwarp();
        cbo = nh;
        // (X, count) into buf/rcnt in place: head k sits at position ≥ k
        for (uint32_t k0 = 0; k0 < cbo; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t x = 0, cn = 0, key = 0;
            if (k < cbo) {
                const uint32_t h0 = rcnt[k];
                const uint32_t h1 = k + 1 < cbo ? rcnt[k + 1] : T;
                key = buf[h0];
                x = key >> 5;
                cn = h1 - h0;
            }
            __syncwarp();
            if (k < cbo) {
                buf[k] = x;
                rcnt[k] = cn;
                if (cn == 1) atomicAdd(rem + (key & 31u), 1u);
            }
            __syncwarp();
        }
        // static row slot: a small class has at most kSmallRowCap foreign classes
        // per member, so rows placed at kSmallRowCap · (first member position)
        // never overlap — no contended global atomic per class
        for (uint32_t k = lane; k < cbo; k += 32) {
            ux[ubase + k] = buf[k];
            un[ubase + k] = rcnt[k];
        }
    }
    __syncwarp();
    removed_me = rem[lane];
    // per member: #{X ≠ c : U[c][X] == 1} — the sweep's cbo_origin_after
    if (active && !ovf) hdrs[pos] = hdr | (removed_me << kRecRemovedShift) | kRecRemovedValid;
    if (lane == 0) {
        const double l = lcom_of(A, M, H);
        const uint64_t pairs = (uint64_t)M * (M - 1) / 2;
        const uint64_t P = pairs - Q;
        ClassRec r;
        r.A = A; r.M = M; r.H = H; r.cbo = cbo; r.ubase = ubase; r.dense = kNone;
        for (int w = 0; w < kSigWords; ++w) r.sig[w] = sig[w];
        rec[c] = r;
        lcom_out[c] = l;
        ck_out[c] = P > Q ? P - Q : 0;
        cbo_out[c] = cbo;
    }
}

// ---------------------------------------------------------------------------
// CTA path: one CTA per large class (any M, A, degree)
// ---------------------------------------------------------------------------

constexpr int kLargeThreads = 256;     // default CTA size; the largest classes launch with 1024
constexpr int kMaxWarps = 32;

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v, uint64_t* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    uint64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) t += red[w];
    __syncthreads();
    return t;
}

// exclusive block scan of one u32 per thread; returns total in *total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* red, uint32_t* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t inc = warp_excl_scan(v, lane) + v;
    __syncthreads();
    if (lane == 31) red[warp] = inc;
    __syncthreads();
    uint32_t before = 0, all = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
        if (w < warp) before += red[w];
        all += red[w];
    }
    __syncthreads();
    *total = all;
    return before + inc - v;
}

__device__ void block_bitonic_u32(uint32_t* buf, uint32_t N) {
    for (uint32_t k = 2; k <= N; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t a = buf[i], b = buf[ixj];
                    const bool up = (i & k) == 0;
                    if ((a > b) == up) { buf[i] = b; buf[ixj] = a; }
                }
            }
            __syncthreads();
        }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Member i's distinct used classes, ascending (record entries, or a streaming
// enumeration of the CSR row when the record overflowed); f(X, h).
template <class F>
__device__ __forceinline__ void member_used(const DevModel& s, const MethRec* recs, uint32_t pos, uint32_t p, F f) {
    const uint32_t hdr = rec_hdrs(recs, s.M)[pos];
    if (!(hdr & kRecOverflow)) {
        for (uint32_t k = 0; k < rec_n(hdr); ++k) {
            const uint32_t e = recs[pos].ent[k];
            f(e >> 8, e & 0xffu);
        }
        return;
    }
    StreamUsed S;
    S.init(s, p);
    uint32_t prev = kNone, h = 0;
    for (;;) {
        const uint32_t x = S.next(prev, h);
        if (x == kNone) break;
        f(x, h);
        prev = x;
    }
}

// Phase 1 of a giant CTA-path class (≥ kGiantMembers members, histogram U
// row, attribute bitmaps in global scratch) spread over many CTAs, one
// member per thread: foreign used classes counted into the giant's global
// histogram, own accesses into H and the attribute bitmaps. k_class_large
// then starts from the histogram instead of walking 10k members itself.
__global__ void __launch_bounds__(kGiantChunk)
k_giant_p1(DevModel s, const uint32_t* __restrict__ large_list, const LargePlan* __restrict__ plan,
           const uint2* __restrict__ items, const MethRec* __restrict__ recs, uint32_t* __restrict__ gcnt,
           unsigned long long* __restrict__ gH, uint32_t* __restrict__ grows) {
    __shared__ uint64_t red64[kGiantChunk / 32];
    const uint2 it = items[blockIdx.x];  // (index into the large list, first member)
    const uint32_t c = large_list[it.x];
    const LargePlan pl = plan[it.x];
    const uint32_t mb = s.cls_moff[c];
    const uint32_t M = s.cls_moff[c + 1] - mb;
    const uint32_t W = (M + 31) / 32;
    uint32_t* hist = gcnt + (uint64_t)pl.pre_slot * s.C;
    uint32_t* rows = grows + pl.rows_off;
    const uint32_t i = it.y + threadIdx.x;
    uint64_t hown = 0;
    if (i < M) {
        const uint32_t pos = mb + i;
        const uint32_t p = s.cls_methods[pos];
        member_used(s, recs, pos, p, [&](uint32_t X, uint32_t) {
            if (X != c) atomicAdd(hist + X, 1u);
        });
        const uint32_t ab = __ldg(s.acc_off + p), ae = __ldg(s.acc_off + p + 1);
        for (uint32_t e = ab; e < ae; ++e) {
            const uint2 ai = __ldg(s.attr_info + __ldg(s.acc_tgt + e));
            if (ai.x != c) continue;
            ++hown;
            atomicOr(rows + (uint64_t)ai.y * W + (i >> 5), 1u << (i & 31));
        }
    }
    const uint64_t h = block_sum_u64(hown, red64);
    if (threadIdx.x == 0 && h) atomicAdd(gH + pl.pre_slot, (unsigned long long)h);
}

// One CTA per class outside the warp path (Zipf giants, C5's 500-method
// classes). Dynamic shared memory holds, when they fit (host plan): a
// histogram over all C classes (cnt[X] = U[c][X]) or the foreign-class keys
// (one per member and used class — members' lists are already distinct, so a
// run length IS the member count U[c][X]), and the LCOM-CK structure
// (own-attribute positions come from attr_info, no searches): per-member own-attribute masks (A ≤ 256: pairs tested by
// word ANDs) or per-attribute member bitmaps (sparse giants).
__global__ void __launch_bounds__(1024)
k_class_large(DevModel s, const uint32_t* __restrict__ large_list, const LargePlan* __restrict__ plan,
              MethRec* __restrict__ recs, const uint64_t* __restrict__ own_mask, ClassRec* __restrict__ rec,
              double* __restrict__ lcom_out, uint64_t* __restrict__ ck_out, uint32_t* __restrict__ cbo_out,
              uint32_t* __restrict__ ux, uint32_t* __restrict__ un, uint32_t* __restrict__ ucursor,
              uint32_t* __restrict__ gkeys, uint32_t* __restrict__ grows, uint32_t* __restrict__ dense,
              uint32_t dense_cap, uint32_t* __restrict__ dense_cursor, const uint32_t* __restrict__ gcnt,
              const unsigned long long* __restrict__ gH) {
    extern __shared__ __align__(16) unsigned char dsm[];
    __shared__ uint64_t red64[kMaxWarps];
    __shared__ uint32_t red32[kMaxWarps];
    __shared__ uint32_t s_nk, s_ubase, s_dense;
    __shared__ uint32_t s_sig[kSigWords];
    const uint32_t c = large_list[blockIdx.x];
    const LargePlan pl = plan[blockIdx.x];
    const uint32_t mb = s.cls_moff[c];
    const uint32_t M = s.cls_moff[c + 1] - mb;
    const uint32_t ab0 = s.cls_aoff[c];
    const uint32_t A = s.cls_aoff[c + 1] - ab0;
    const uint32_t W = (M + 31) / 32;        // rows mode: words per attribute bitmap
    const uint32_t WA = (A + 63) / 64;       // masks mode: u64 words per member
    unsigned char* cur = dsm;
    // foreign classes: a per-class histogram cnt[X] = U[c][X] over all C
    // classes when it fits (few classes, many keys: no sort, no searches),
    // else the keys sorted in place
    uint32_t* cnt = pl.hist ? reinterpret_cast<uint32_t*>(cur) : nullptr;
    if (pl.hist) cur += (4ull * s.C + 15) & ~15ull;
    uint32_t* keys = pl.keys_in_smem ? reinterpret_cast<uint32_t*>(cur) : gkeys + pl.keys_off;
    if (pl.keys_in_smem) cur += (4ull * pl.keys_cap + 15) & ~15ull;  // keep the u64 masks aligned
    uint64_t* masks = reinterpret_cast<uint64_t*>(cur);  // masks mode (always in smem)
    uint32_t* rows = pl.ck_masks ? nullptr : (pl.rows_in_smem ? reinterpret_cast<uint32_t*>(cur) : grows + pl.rows_off);
    const uint64_t ck_words = pl.ck_masks ? (uint64_t)M * WA * 2 : (uint64_t)A * W;
    uint32_t* ckz = pl.ck_masks ? reinterpret_cast<uint32_t*>(masks) : rows;
    if (threadIdx.x == 0) s_nk = 0;
    if (threadIdx.x < kSigWords) s_sig[threadIdx.x] = 0;
    // (global-scratch bitmaps are cleared by one cudaMemsetAsync before the launch)
    if (pl.ck_masks || pl.rows_in_smem)
        for (uint64_t i = threadIdx.x; i < ck_words; i += blockDim.x) ckz[i] = 0;
    if (pl.hist && pl.pre_slot == kNone)
        for (uint32_t i = threadIdx.x; i < s.C; i += blockDim.x) cnt[i] = 0;
    __syncthreads();

    // phase 1: members' foreign used classes -> keys; H; own-attribute sets.
    // Giants had it done by k_giant_p1 over many CTAs: load their histogram.
    const bool pre = pl.pre_slot != kNone;
    if (pre)
        for (uint32_t k = threadIdx.x; k < s.C; k += blockDim.x) cnt[k] = gcnt[(uint64_t)pl.pre_slot * s.C + k];
    uint64_t hown = 0;
    for (uint32_t i = pre ? M : threadIdx.x; i < M; i += blockDim.x) {
        const uint32_t pos = mb + i;
        const uint32_t p = s.cls_methods[pos];
        if (pl.hist)
            member_used(s, recs, pos, p, [&](uint32_t X, uint32_t) {
                if (X != c) atomicAdd(cnt + X, 1u);
            });
        else
            member_used(s, recs, pos, p, [&](uint32_t X, uint32_t) {
                if (X != c) keys[atomicAdd(&s_nk, 1u)] = X;
            });
        const uint32_t mh = rec_hdrs(recs, s.M)[pos];
        if (A <= 64 && pl.ck_masks && !(mh & kRecOverflow)) {
            // the method pass already built this member's mask and own-hit count
            masks[i] = own_mask[pos];
            hown += rec_hown(mh);
            continue;
        }
        const uint32_t ab = __ldg(s.acc_off + p), ae = __ldg(s.acc_off + p + 1);
        for (uint32_t e = ab; e < ae; ++e) {
            const uint2 ai = __ldg(s.attr_info + __ldg(s.acc_tgt + e));
            if (ai.x != c) continue;
            ++hown;
            const uint32_t a = ai.y;
            if (pl.ck_masks) masks[(uint64_t)i * WA + (a >> 6)] |= 1ull << (a & 63);  // member i: this thread only
            else atomicOr(rows + (uint64_t)a * W + (i >> 5), 1u << (i & 31));
        }
    }
    const uint64_t H = pre ? gH[pl.pre_slot] : block_sum_u64(hown, red64);  // (includes a __syncthreads)
    if (pre) __syncthreads();
    const uint32_t dwords = (s.C + 31) / 32;
    uint32_t nx = 0, ubase = 0, nk = 0;
    if (pl.hist) {
        // phase 2 (histogram): the nonzero counts, in class order, are the U
        // row. Each warp owns a contiguous range of whole 32-class words:
        // it counts its nonzeros (ballots), one barrier publishes the warp
        // counts (their prefix = the warp's offset in the row), and the warp
        // writes its entries in order — two barriers per class, not two per
        // blockDim classes (C5: 5000 classes scanned by 256 threads had 40)
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
        const uint32_t seg = (s.C + 32u * nwarps - 1) / (32u * nwarps) * 32u;
        const uint32_t k0 = min(s.C, (uint32_t)warp * seg), k1 = min(s.C, k0 + seg);
        uint32_t wcnt = 0;
        for (uint32_t b = k0; b < k1; b += 32) {
            const uint32_t k = b + lane;
            wcnt += __popc(__ballot_sync(0xffffffffu, k < k1 && cnt[k] != 0u));
        }
        if (lane == 0) red32[warp] = wcnt;
        __syncthreads();
        uint32_t woff = 0;
        for (int w2 = 0; w2 < nwarps; ++w2) {
            const uint32_t c2 = red32[w2];
            woff += w2 < warp ? c2 : 0u;
            nx += c2;
        }
        if (threadIdx.x == 0) {
            s_ubase = kSmallRowCap * s.M + (nx ? atomicAdd(ucursor, nx) : 0u);
            s_dense = kNone;
            if (nx > kDenseRowMin && dense) {
                const uint32_t off = atomicAdd(dense_cursor, 2 * dwords);
                if ((uint64_t)off + 2 * dwords <= dense_cap) s_dense = off;
            }
        }
        __syncthreads();
        ubase = s_ubase;
        const uint32_t dn = s_dense;
        uint32_t run = woff;
        for (uint32_t b = k0; b < k1; b += 32) {
            const uint32_t k = b + lane;
            const uint32_t v = k < k1 ? cnt[k] : 0u;
            const uint32_t m = __ballot_sync(0xffffffffu, v != 0u);
            if (v) {
                const uint32_t at = ubase + run + __popc(m & ((1u << lane) - 1u));
                ux[at] = k;
                un[at] = v;
                const uint32_t b1 = bloom_h1(k), b2 = bloom_h2(k);
                atomicOr(s_sig + (b1 >> 5), 1u << (b1 & 31));
                atomicOr(s_sig + (b2 >> 5), 1u << (b2 & 31));
            }
            if (dn != kNone) {  // whole 32-class words: membership, singletons
                const uint32_t one = __ballot_sync(0xffffffffu, v == 1u);
                if (lane == 0) {
                    dense[dn + (b >> 5)] = m;
                    dense[dn + dwords + (b >> 5)] = one;
                }
            }
            run += __popc(m);
        }
    } else {
        nk = s_nk;
        uint32_t N = 1;
        while (N < nk) N <<= 1;
        for (uint32_t i = nk + threadIdx.x; i < N; i += blockDim.x) keys[i] = kNone;
        __syncthreads();
        if (N > 1) block_bitonic_u32(keys, N);

        // phase 2: runs of equal X = one U row entry with count = run length
        for (uint32_t b = 0; b < nk; b += blockDim.x) {
            const uint32_t k = b + threadIdx.x;
            const bool xh = k < nk && (k == 0 || keys[k] != keys[k - 1]);
            uint32_t tot;
            block_excl_scan(xh ? 1u : 0u, red32, &tot);
            nx += tot;
        }
        // large classes reserve their rows past the small-class region (few, so the
        // atomic is uncontended): the paper's atomicAdd slot reservation
        if (threadIdx.x == 0) s_ubase = kSmallRowCap * s.M + (nx ? atomicAdd(ucursor, nx) : 0u);
        __syncthreads();
        ubase = s_ubase;
        uint32_t xcarry = 0;
        for (uint32_t b = 0; b < nk; b += blockDim.x) {
            const uint32_t k = b + threadIdx.x;
            const bool xh = k < nk && (k == 0 || keys[k] != keys[k - 1]);
            uint32_t tot;
            const uint32_t ex = block_excl_scan(xh ? 1u : 0u, red32, &tot);
            if (xh) {
                const uint32_t X = keys[k];
                ux[ubase + xcarry + ex] = X;
                un[ubase + xcarry + ex] = lower_bound_u32(keys, nk, X + 1) - k;  // run length
                const uint32_t b1 = bloom_h1(X), b2 = bloom_h2(X);
                atomicOr(s_sig + (b1 >> 5), 1u << (b1 & 31));
                atomicOr(s_sig + (b2 >> 5), 1u << (b2 & 31));
            }
            xcarry += tot;
        }

        // dense rows also get exact bitmaps over all classes: membership (O(1)
        // in the sweep where a Bloom signature of a long row says "maybe" to all)
        // then the U[c][X] == 1 singletons (the origin's removed count)
        if (threadIdx.x == 0) {
            s_dense = kNone;
            if (nx > kDenseRowMin && dense) {
                const uint32_t off = atomicAdd(dense_cursor, 2 * dwords);
                if ((uint64_t)off + 2 * dwords <= dense_cap) s_dense = off;
            }
        }
        __syncthreads();
        if (s_dense != kNone) {
            for (uint32_t w = threadIdx.x; w < 2 * dwords; w += blockDim.x) dense[s_dense + w] = 0;
            __syncthreads();
            for (uint32_t k = threadIdx.x; k < nx; k += blockDim.x) {
                const uint32_t X = ux[ubase + k];
                atomicOr(dense + s_dense + (X >> 5), 1u << (X & 31));
                if (un[ubase + k] == 1u) atomicOr(dense + s_dense + dwords + (X >> 5), 1u << (X & 31));
            }
        }
    }

    // phase 3: per member, #{X ≠ c : U[c][X] == 1} into its method record
    for (uint32_t i = threadIdx.x; i < M; i += blockDim.x) {
        MethRec* r = recs + mb + i;
        uint32_t* rh = rec_hdrs(recs, s.M) + mb + i;
        const uint32_t hdr = *rh;
        if (hdr & kRecOverflow) continue;
        uint32_t removed = 0;
        for (uint32_t k = 0; k < rec_n(hdr); ++k) {
            const uint32_t X = r->ent[k] >> 8;
            if (X == c) continue;
            if (pl.hist) {
                removed += cnt[X] == 1u;
            } else {
                const uint32_t lo = lower_bound_u32(keys, nk, X);
                removed += (lower_bound_u32(keys, nk, X + 1) - lo) == 1u;
            }
        }
        *rh = hdr | (removed << kRecRemovedShift) | kRecRemovedValid;
    }

    // phase 4: LCOM-CK, Q = #pairs (i<j) sharing an own attribute. Classes
    // whose attribute bitmaps live in global scratch (Zipf giants) are split
    // over many CTAs by k_ck_rows instead (ck_out[c] accumulates Q there).
    const bool split = !pl.ck_masks && !pl.rows_in_smem;
    uint64_t q = 0;
    if (split || pl.ck_mma) {  // another kernel owns this class's LCOM-CK
    } else if (pl.ck_masks) {
        // warp per row i, lanes over j > i: conflict-free consecutive mask
        // loads, no per-thread trip-count imbalance
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
        if (WA == 1) {
            for (uint32_t i = warp; i < M; i += nw) {
                const uint64_t mi = masks[i];
                if (!mi) continue;  // no own attribute: shares with nobody
                for (uint32_t j = i + 1 + lane; j < M; j += 32) q += (mi & masks[j]) != 0;
            }
        } else {
            for (uint32_t i = warp; i < M; i += nw)
                for (uint32_t j = i + 1 + lane; j < M; j += 32) {
                    uint64_t any = 0;
                    for (uint32_t w = 0; w < WA; ++w) any |= masks[(uint64_t)i * WA + w] & masks[(uint64_t)j * WA + w];
                    q += any != 0;
                }
        }
    } else {
        // rows[a] = members using a; member i's sharers = OR of its rows, above i
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
        for (uint32_t i = warp; i < M; i += blockDim.x / 32) {
            const uint32_t p = s.cls_methods[mb + i];
            const uint32_t ab = __ldg(s.acc_off + p), ae = __ldg(s.acc_off + p + 1);
            for (uint32_t wb = 0; wb < W; wb += 32) {
                const uint32_t w = wb + lane;
                uint32_t acc = 0;
                if (w < W && w >= (i >> 5)) {
                    for (uint32_t e = ab; e < ae; ++e) {
                        const uint2 ai = __ldg(s.attr_info + __ldg(s.acc_tgt + e));
                        if (ai.x == c) acc |= rows[(uint64_t)ai.y * W + w];
                    }
                    if (w == (i >> 5)) acc &= ((i & 31) == 31) ? 0u : (~0u << ((i & 31) + 1));
                }
                q += __popc(acc);
            }
        }
    }
    const uint64_t Q = block_sum_u64(q, red64);
    if (threadIdx.x == 0) {
        const double l = lcom_of(A, M, H);
        const uint64_t pairs = (uint64_t)M * (M - 1) / 2;
        const uint64_t P = pairs - Q;
        ClassRec r;
        r.A = A; r.M = M; r.H = (uint32_t)H; r.cbo = nx; r.ubase = ubase; r.dense = s_dense;
        for (int w = 0; w < kSigWords; ++w) r.sig[w] = s_sig[w];
        rec[c] = r;
        lcom_out[c] = l;
        if (!pl.ck_mma) ck_out[c] = split ? 0ull : (P > Q ? P - Q : 0);
        cbo_out[c] = nx;
    }
}

// LCOM-CK of a split class, one CTA per (class, kCkChunk-member chunk): member i's
// sharers above it = OR of the bitmaps rows[a] of its own attributes a.
__global__ void __launch_bounds__(kLargeThreads)
k_ck_rows(DevModel s, const uint32_t* __restrict__ large_list, const LargePlan* __restrict__ plan,
          const uint2* __restrict__ items, const uint32_t* __restrict__ grows, uint64_t* __restrict__ ck_out) {
    __shared__ uint64_t red64[kLargeThreads / 32];
    const uint2 it = items[blockIdx.x];  // (index into the large list, first member)
    const uint32_t c = large_list[it.x];
    const LargePlan pl = plan[it.x];
    const uint32_t mb = s.cls_moff[c];
    const uint32_t M = s.cls_moff[c + 1] - mb;
    const uint32_t ab0 = s.cls_aoff[c];
    const uint32_t A = s.cls_aoff[c + 1] - ab0;
    const uint32_t W = (M + 31) / 32;
    const uint32_t* rows = grows + pl.rows_off;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t iend = min(M, it.y + kCkChunk);
    uint64_t q = 0;
    for (uint32_t i = it.y + warp; i < iend; i += kLargeThreads / 32) {
        const uint32_t p = s.cls_methods[mb + i];
        const uint32_t ab = __ldg(s.acc_off + p), ae = __ldg(s.acc_off + p + 1);
        // the member's own-attribute positions, gathered once (lane-parallel)
        uint32_t mypos = kNone;
        uint32_t nown = 0;
        __shared__ uint32_t spos[kLargeThreads / 32][64];
        for (uint32_t e0 = ab; e0 < ae; e0 += 32) {
            const uint32_t e = e0 + lane;
            bool own = false;
            if (e < ae) {
                const uint2 ai = __ldg(s.attr_info + __ldg(s.acc_tgt + e));
                own = ai.x == c;
                if (own) mypos = ai.y;
            }
            const uint32_t b = __ballot_sync(0xffffffffu, own);
            if (own) {
                const uint32_t at = nown + __popc(b & ((1u << lane) - 1));
                if (at < 64) spos[warp][at] = mypos;
            }
            nown += __popc(b);
        }
        __syncwarp();
        const uint32_t nk = min(nown, 64u);
        for (uint32_t wb = (i >> 5) & ~31u; wb < W; wb += 32) {
            const uint32_t w = wb + lane;
            uint32_t acc = 0;
            if (w < W && w >= (i >> 5)) {
                for (uint32_t k = 0; k < nk; ++k) acc |= __ldg(rows + (uint64_t)spos[warp][k] * W + w);
                if (nown > 64) {  // rare: more own attributes than the staging list
                    for (uint32_t e = ab; e < ae; ++e) {
                        const uint2 ai = __ldg(s.attr_info + __ldg(s.acc_tgt + e));
                        if (ai.x == c) acc |= __ldg(rows + (uint64_t)ai.y * W + w);
                    }
                }
                if (w == (i >> 5)) acc &= ((i & 31) == 31) ? 0u : (~0u << ((i & 31) + 1));
            }
            q += __popc(acc);
        }
        __syncwarp();
    }
    const uint64_t Q = block_sum_u64(q, red64);
    if (threadIdx.x == 0 && Q) atomicAdd(reinterpret_cast<unsigned long long*>(ck_out + c), (unsigned long long)Q);
}

// P = C(M,2) - Q; lcom_ck = P > Q ? P - Q : 0 (metrics.hpp:147-156) for the split classes
__global__ void k_ck_finalize(DevModel s, const uint32_t* __restrict__ split_list, uint32_t n,
                              uint64_t* __restrict__ ck_out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const uint32_t c = split_list[k];
    const uint64_t M = s.cls_moff[c + 1] - s.cls_moff[c];
    const uint64_t Q = ck_out[c];
    const uint64_t P = M * (M - 1) / 2 - Q;
    ck_out[c] = P > Q ? P - Q : 0;
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------

void launch_validate_ids(const uint32_t* v, uint64_t n, uint32_t bound, uint32_t* bad, cudaStream_t st) {
    if (!n) return;
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
    k_validate_ids<<<blocks, 256, 0, st>>>(v, n, bound, bad);
}
void launch_expand(const DevModel& s, uint32_t* mo_out, uint32_t* ao_out, uint32_t* pos_owner, uint2* info,
                   cudaStream_t st) {
    if (!s.C) return;
    if (mo_out && s.M) cudaMemsetAsync(mo_out, 0xff, 4ull * s.M, st);  // unowned ids fail validation
    if (ao_out && s.A) cudaMemsetAsync(ao_out, 0xff, 4ull * s.A, st);
    const uint64_t n = (uint64_t)s.M + s.A;
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
    if (n) k_expand<<<blocks, 256, 0, st>>>(s, mo_out, ao_out, pos_owner, info);
}
void launch_fan(const DevModel& s, uint32_t* fan_in, uint32_t* fan_out, uint32_t* kmax, cudaStream_t st) {
    if (kmax) cudaMemsetAsync(kmax, 0, 8, st);
    if (!s.M) return;
    if (fan_in) cudaMemsetAsync(fan_in, 0, 4ull * s.M, st);
    k_fan<<<(s.M + 255) / 256, 256, 0, st>>>(s, fan_in, fan_out, kmax);
}
void launch_validate_offsets(const uint32_t* off, uint64_t n1, uint32_t total, uint32_t* bad, cudaStream_t st) {
    const uint32_t blocks = (uint32_t)std::min<uint64_t>((n1 + 255) / 256, 148 * 16);
    k_validate_offsets<<<blocks, 256, 0, st>>>(off, n1, total, bad);
}
void launch_plan_classes(const DevModel& s, uint4* cplan, uint4* cedge, uint32_t* large_list,
                         uint32_t* n_large, uint32_t* big_list, uint32_t* n_big, uint32_t* max_deg,
                         const uint32_t* foreign, const uint32_t* cmaxdeg, cudaStream_t st) {
    if (!s.C) return;
    k_plan_classes<<<(s.C + 127) / 128, 128, 0, st>>>(s, cmaxdeg, foreign, cplan, cedge, large_list, n_large, big_list,
                                                       n_big, max_deg);
}
void launch_pos_rows(const DevModel& s, const uint32_t* pos_owner, uint32_t* pc_off, uint32_t* pc_tgt,
                     uint32_t* pa_off, uint32_t* pa_tgt, uint8_t* pc_mem, uint8_t* pa_mem, uint32_t* totals,
                     uint32_t* foreign, uint32_t* cmaxdeg, uint32_t* n_hideg, cudaStream_t st) {
    if (s.C) {
        cudaMemsetAsync(foreign, 0, 4ull * s.C, st);
        cudaMemsetAsync(cmaxdeg, 0, 4ull * s.C, st);
    }
    const uint32_t ntiles = (s.M + kPosTile - 1) / kPosTile;
    if (!ntiles) {  // no positions: empty rows
        cudaMemsetAsync(pc_off, 0, 4, st);
        cudaMemsetAsync(pa_off, 0, 4, st);
        return;
    }
    k_pos_tile_sums<<<ntiles, kPosTile, 0, st>>>(s, totals);
    k_pos_tile_scan<<<1, 1024, 0, st>>>(totals, ntiles, pc_off, pa_off, s.M);
    k_pos_rows<<<ntiles, kPosTile, 0, st>>>(s, pos_owner, totals, pc_off, pa_off, pc_tgt, pa_tgt, pc_mem, pa_mem,
                                            foreign, cmaxdeg, n_hideg);
}

void launch_method(const DevModel& s, MethRec* recs, uint64_t* own_mask, const uint32_t* pos_owner,
                   uint32_t max_deg, const uint32_t* plist, uint32_t n_pos, cudaStream_t st) {
    const uint32_t n = plist ? n_pos : s.M;
    if (!n) return;
    const uint32_t blocks = (n + 255) / 256;
    if (max_deg > 8)  // some method needs several chunks: regroup by chunk count
        k_method<8, true><<<blocks, 256, 0, st>>>(s, recs, own_mask, pos_owner, plist, n_pos);
    else
        k_method<8, false><<<blocks, 256, 0, st>>>(s, recs, own_mask, pos_owner, plist, n_pos);
}
void launch_class_small(const DevModel& s, const uint4* cplan, const uint32_t* big_list, uint32_t n_big,
                        MethRec* recs, const uint64_t* own_mask, ClassRec* rec, double* lcom, uint64_t* ck,
                        uint32_t* cbo, uint32_t* ux, uint32_t* un, bool lean, cudaStream_t st, cudaStream_t st_big) {
    if (!s.C) return;
    if (lean)
        k_class_small<false><<<(s.C + kWarpsPerBlock - 1) / kWarpsPerBlock, kWarpsPerBlock * 32, 0, st>>>(
        s, cplan, nullptr, 0, recs, own_mask, rec, lcom, ck, cbo, ux, un);
    if (n_big)
        k_class_small<true><<<(n_big + kWarpsPerBlock - 1) / kWarpsPerBlock, kWarpsPerBlock * 32, 0, st_big>>>(
            s, cplan, big_list, n_big, recs, own_mask, rec, lcom, ck, cbo, ux, un);
}
void launch_class_large(const DevModel& s, uint32_t n_large, const uint32_t* large_list, const LargePlan* plan,
                        uint32_t smem_bytes, MethRec* recs, const uint64_t* own_mask, ClassRec* rec, double* lcom,
                        uint64_t* ck, uint32_t* cbo, uint32_t* ux, uint32_t* un, uint32_t* ucursor,
                        uint32_t* gkeys, uint32_t* grows, uint32_t* dense, uint32_t dense_cap,
                        uint32_t* dense_cursor, const uint32_t* gcnt, const unsigned long long* gH,
                        uint32_t threads, cudaStream_t st) {
    if (!n_large) return;
    k_class_large<<<n_large, threads, smem_bytes, st>>>(s, large_list, plan, recs, own_mask, rec, lcom, ck, cbo, ux,
                                                              un, ucursor, gkeys, grows, dense, dense_cap,
                                                              dense_cursor, gcnt, gH);
}
void launch_ck_rows(const DevModel& s, const uint32_t* large_list, const LargePlan* plan, const uint2* items,
                    uint32_t n_items, const uint32_t* grows, const uint32_t* split_list, uint32_t n_split,
                    uint64_t* ck, cudaStream_t st) {
    if (!n_items) return;
    k_ck_rows<<<n_items, kLargeThreads, 0, st>>>(s, large_list, plan, items, grows, ck);
    k_ck_finalize<<<(n_split + 127) / 128, 128, 0, st>>>(s, split_list, n_split, ck);
}
void launch_giant_p1(const DevModel& s, const uint32_t* large_list, const LargePlan* plan, const uint2* items,
                     uint32_t n_items, const MethRec* recs, uint32_t* gcnt, unsigned long long* gH, uint32_t* grows,
                     cudaStream_t st) {
    if (!n_items) return;
    k_giant_p1<<<n_items, kGiantChunk, 0, st>>>(s, large_list, plan, items, recs, gcnt, gH, grows);
}
// The attribute belongs to the function, process-wide, not to a context: a
// later upload of a smaller system (another engine, another thread) must not
// lower it under a launch planned with more. Raised only, never lowered.
cudaError_t set_class_large_smem(uint32_t bytes) {
    static std::atomic<int> granted{0};
    int cur = granted.load(std::memory_order_relaxed);
    while ((int)bytes > cur) {
        const cudaError_t e = cudaFuncSetAttribute(k_class_large, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return e;
        if (granted.compare_exchange_weak(cur, (int)bytes, std::memory_order_relaxed)) break;
    }
    return cudaSuccess;
}

}  // namespace mmg
