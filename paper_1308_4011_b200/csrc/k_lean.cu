// k_lean.cu — method pass and class pass fused for warp-path ("lean") classes.
//
// Replaces, for every class of kind kKindLean (M ≤ 32 members, A ≤ 64
// attributes, member degree ≤ 16, ≤ 32 foreign edges), the two-kernel chain
// k_method (thread per method, register used lists) → k_class_small (warp per
// class). One warp owns one class and walks the class's dependency edges one
// EDGE per lane: the class's rows are contiguous in the class-order CSR
// (pc_tgt / pa_tgt), so 32 call and 32 access edges load coalesced per step
// beside their member indices (pc_mem / pa_mem, laid out at upload), and each
// lane gathers its targets' owners: three dependent memory round trips per
// class (plan, edges, owners). Everything the two kernels
// computed comes out of one pass:
//   * H, lcom (metrics.hpp:114-126), LCOM-CK from the members' own-attribute
//     masks (metrics.hpp:135-157), cbo = |U row| (metrics.hpp:167-185);
//   * the U row {X ≠ c : some member uses X} with member counts U[c][X] and
//     its Bloom signature, in lane order at the static slot 16·(first member
//     position) (same layout k_class_small wrote);
//   * each member's MethRec — its used classes (own class included) sorted by
//     class id with own-access counts, used_classes + intersection_count
//     (suggest.hpp:152-159, metrics.hpp:121-123) — and its header with the
//     removed count #{X ≠ c : U[c][X] == 1 and the member uses X}, i.e. the
//     sweep's cbo_origin_after.
// Foreign edges (≤ 32) are deduplicated with two __match_any_sync rounds:
// (X, member) pairs, then classes X among the pair heads; a member's list is
// ranked by class id with shuffles over its match group. Records are
// assembled in shared memory and written as whole 32-byte sectors.
#include <cuda_runtime.h>

#include <cstdint>

#include "mm_device.cuh"
#include "mm_kernels.h"

namespace mmg {

namespace {

constexpr int kLeanWarps = 8;
constexpr uint32_t kFull = 0xffffffffu;

struct __align__(16) LeanWarp {
    uint32_t ent[32][kRecMaxEnt];  // member records being assembled (class-order positions mb..mb+M)
    uint32_t hown[32];             // accesses owned by c, per member
    uint32_t mlo[32], mhi[32];     // own-attribute masks (bit k = k-th attribute of c)
    uint32_t used[32];             // member uses its own class
    uint32_t low[32];              // distinct foreign classes below c, per member (own entry's rank)
    uint32_t nfor[32];             // distinct foreign classes, per member
    uint32_t rem[32];              // foreign classes this member alone uses
    uint32_t ovf[32];              // record cannot hold the list
    uint32_t kx[32], km[32];       // compacted foreign edges: class, member | is_access << 5
    uint32_t sig[kSigWords];
};

__global__ void __launch_bounds__(kLeanWarps * 32)
k_class_lean(DevModel s, const uint4* __restrict__ cplan, const uint4* __restrict__ cedge,
             const uint8_t* __restrict__ pc_mem, const uint8_t* __restrict__ pa_mem, MethRec* __restrict__ recs,
             ClassRec* __restrict__ rec, double* __restrict__ lcom_out, uint64_t* __restrict__ ck_out,
             uint32_t* __restrict__ cbo_out, uint32_t* __restrict__ ux, uint32_t* __restrict__ un,
             const uint32_t* __restrict__ list, uint32_t n_list) {
    __shared__ LeanWarp sw[kLeanWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t wi = blockIdx.x * kLeanWarps + warp;
    if (wi >= (list ? n_list : s.C)) return;
    const uint32_t c = list ? __ldg(list + wi) : wi;
    const uint4 cp = cplan[c];  // (first member position, M, A, kind)
    const uint4 ce = cedge[c];  // call edges [x, y), access edges [z, w) in the class-order rows
    if (cp.w != kKindLean) return;  // warp-uniform
    LeanWarp& w = sw[warp];
    const uint32_t mb = cp.x, M = cp.y, A = cp.z;
    const uint32_t lt = (1u << lane) - 1u;

    w.hown[lane] = 0; w.mlo[lane] = 0; w.mhi[lane] = 0; w.used[lane] = 0;
    w.low[lane] = 0; w.nfor[lane] = 0; w.rem[lane] = 0; w.ovf[lane] = 0;
    if (lane < kSigWords) w.sig[lane] = 0;
    uint4* ent4 = reinterpret_cast<uint4*>(&w.ent[0][0]);
    ent4[lane] = make_uint4(0, 0, 0, 0);
    ent4[lane + 32] = make_uint4(0, 0, 0, 0);
    __syncwarp();

    // ---- edges, one call and one access edge per lane and round ----
    uint32_t T = 0;  // foreign edges so far (≤ 32 for a lean class)
    const uint32_t nC = ce.y - ce.x, nA = ce.w - ce.z, nmax = max(nC, nA);
    for (uint32_t b = 0; b < nmax; b += 32) {
        const uint32_t j = b + lane;
        const bool lc = j < nC, la = j < nA;
        uint32_t tc = 0, ta = 0, mc = 0, ma = 0;
        if (lc) { tc = __ldg(s.pc_tgt + ce.x + j); mc = __ldg(pc_mem + ce.x + j); }
        if (la) { ta = __ldg(s.pa_tgt + ce.z + j); ma = __ldg(pa_mem + ce.z + j); }
        const uint32_t Xc = lc ? __ldg(s.method_owner + tc) : c;
        const uint2 ai = la ? __ldg(s.attr_info + ta) : make_uint2(c, 0u);
        mc &= 31u;
        ma &= 31u;
        if (lc && Xc == c) w.used[mc] = 1u;
        if (la && ai.x == c) {
            w.used[ma] = 1u;
            atomicAdd(&w.hown[ma], 1u);
            atomicOr(ai.y < 32 ? &w.mlo[ma] : &w.mhi[ma], 1u << (ai.y & 31u));
        }
        const bool fc = Xc != c, fa = ai.x != c;
        const uint32_t bc = __ballot_sync(kFull, fc), ba = __ballot_sync(kFull, fa);
        if (fc) {
            const uint32_t i = T + __popc(bc & lt);
            if (i < 32) { w.kx[i] = Xc; w.km[i] = mc; }
        }
        T += __popc(bc);
        if (fa) {
            const uint32_t i = T + __popc(ba & lt);
            if (i < 32) { w.kx[i] = ai.x; w.km[i] = ma | 32u; }
        }
        T += __popc(ba);
    }
    __syncwarp();

    // ---- foreign edges, one per lane: U row, removed counts, member lists ----
    const uint32_t ubase = kSmallRowCap * mb;
    const bool fv = (uint32_t)lane < T;
    const uint32_t vmask = __ballot_sync(kFull, fv);
    uint32_t cbo = 0;
    if (fv) {
        const uint32_t X = w.kx[lane], km = w.km[lane];
        const uint32_t mi = km & 31u;
        const uint32_t amask = __ballot_sync(vmask, km >> 5);
        const uint32_t g1 = __match_any_sync(vmask, (X << 5) | mi);  // same (class, member)
        const bool h1 = (uint32_t)(__ffs(g1) - 1) == (uint32_t)lane;
        const uint32_t h1mask = __ballot_sync(vmask, h1);
        cbo = 0;
        if (h1) {
            const uint32_t g2 = __match_any_sync(h1mask, X);  // members using X
            const bool h2 = (uint32_t)(__ffs(g2) - 1) == (uint32_t)lane;
            const uint32_t h2mask = __ballot_sync(h1mask, h2);
            cbo = __popc(h2mask);
            if (h2) {
                const uint32_t n2 = __popc(g2);
                const uint32_t idx = __popc(h2mask & lt);
                ux[ubase + idx] = X;
                un[ubase + idx] = n2;
                if (n2 == 1) atomicAdd(&w.rem[mi], 1u);  // the one member that loses X when it leaves
                const uint32_t b1 = bloom_h1(X), b2 = bloom_h2(X);
                atomicOr(&w.sig[b1 >> 5], 1u << (b1 & 31u));
                atomicOr(&w.sig[b2 >> 5], 1u << (b2 & 31u));
            }
            // the member's distinct foreign classes: rank by class id inside its group
            const uint32_t g3 = __match_any_sync(h1mask, mi);
            uint32_t rest = g3 & ~(1u << lane);
            const uint32_t rounds = __reduce_max_sync(h1mask, (uint32_t)__popc(rest));
            uint32_t r = 0;
            for (uint32_t it = 0; it < rounds; ++it) {
                const int src = rest ? __ffs(rest) - 1 : lane;
                rest &= rest - 1u;
                const uint32_t Xs = __shfl_sync(h1mask, X, src);
                r += (src != lane && Xs < X) ? 1u : 0u;
            }
            if (X < c) atomicAdd(&w.low[mi], 1u);
            if ((uint32_t)(__ffs(g3) - 1) == (uint32_t)lane) w.nfor[mi] = __popc(g3);
            if (X >= (1u << 24)) w.ovf[mi] = 1u;
            const uint32_t at = r + ((w.used[mi] && c < X) ? 1u : 0u);
            if (at < (uint32_t)kRecMaxEnt) w.ent[mi][at] = (X << 8) | __popc(g1 & amask);
        }
    }
    cbo = __reduce_max_sync(kFull, cbo);
    __syncwarp();

    // ---- members: own entry, header, LCOM-CK ----
    const bool act = (uint32_t)lane < M;
    uint32_t hown = 0, hdr = 0, q = 0;
    if (act) {
        hown = w.hown[lane];
        const uint32_t u = w.used[lane];
        const uint32_t n = w.nfor[lane] + u;
        if (u && w.low[lane] < (uint32_t)kRecMaxEnt) w.ent[lane][w.low[lane]] = (c << 8) | hown;
        const bool ovf = n > (uint32_t)kRecMaxEnt || w.ovf[lane] || (u && c >= (1u << 24)) || hown >= 256u;
        hdr = ovf ? kRecOverflow
                  : (n | (hown << kRecHownShift) | (w.rem[lane] << kRecRemovedShift) | kRecRemovedValid);
        const uint64_t mk = ((uint64_t)w.mhi[lane] << 32) | w.mlo[lane];
        for (uint32_t k = 0; k < (uint32_t)lane; ++k) {
            const uint64_t o = ((uint64_t)w.mhi[k] << 32) | w.mlo[k];
            q += (mk & o) ? 1u : 0u;
        }
    }
    const uint32_t H = __reduce_add_sync(kFull, hown);
    const uint32_t Q = __reduce_add_sync(kFull, q);
    __syncwarp();

    // ---- outputs: whole records, headers, the class record ----
    uint4* dst = reinterpret_cast<uint4*>(recs + mb);
    for (uint32_t j = lane; j < 2 * M; j += 32) dst[j] = ent4[j];
    if (act) rec_hdrs(recs, s.M)[mb + lane] = hdr;
    if (lane < 16) {
        uint32_t v;
        switch (lane) {
            case 0: v = A; break;
            case 1: v = M; break;
            case 2: v = H; break;
            case 3: v = cbo; break;
            case 4: v = ubase; break;
            case 5: v = kNone; break;
            default: v = w.sig[lane - 6]; break;
        }
        reinterpret_cast<uint32_t*>(rec + c)[lane] = v;
    }
    if (lane == 0) {
        lcom_out[c] = lcom_of(A, M, H);
        const uint64_t pairs = (uint64_t)M * (M ? M - 1 : 0) / 2;
        const uint64_t P = pairs - Q;
        ck_out[c] = P > Q ? P - Q : 0;
        cbo_out[c] = cbo;
    }
}

// ---------------------------------------------------------------------------
// Groups of whole lean classes per warp (the C4 shape: ~10 members per class).
// A warp-per-class pass leaves two thirds of its lanes idle and pays its fixed
// per-class code once per ~10 methods; here one warp takes a run of
// consecutive lean classes whose members fit the 32 lanes (≤ 32 members, ≤ 64
// foreign edges, member degree ≤ 8; planned at upload), one MEMBER per lane:
//   * its ≤ 8 edges gathered (targets, then owners: two round trips), keys
//     (owner << 1 | is_access) sorted by a 19-comparator network in registers
//     and run-length encoded into the sorted used list with own-access counts
//     (used_classes + intersection_count, suggest.hpp:152-159,
//     metrics.hpp:121-123) — no per-method insertion sorts;
//   * every (class, foreign X, member) key of the group (≤ 64) sorted by one
//     bitonic network over the warp's registers (two keys per lane): runs of
//     (class, X) are the group's U rows in ascending X with U[c][X] = run
//     length (metrics.hpp:167-185), their Bloom signatures, and a run of one
//     names the member that alone uses X (the sweep's cbo_origin_after);
//   * H, LCOM-CK (pairwise own-mask ANDs inside each class's lane segment,
//     metrics.hpp:135-157) and lcom (metrics.hpp:114-126) per class.
// Outputs are the same arrays k_class_lean writes (records, headers, class
// records, lcom / LCOM-CK / cbo, U rows at 16·(first member position)).
#ifndef MMGPU_GROUP_WARPS
#define MMGPU_GROUP_WARPS 4
#endif
constexpr int kGroupWarps = MMGPU_GROUP_WARPS;
constexpr uint32_t kGroupKeys = 64;  // (class, foreign X, member) keys per group (the plan bounds foreign edges)

struct __align__(16) GroupWarp {
    uint32_t ent[32][kRecMaxEnt];      // member records
    uint32_t keys[kGroupKeys];         // (class index << 27) | (X << 5) | member, before the sort
    uint32_t csig[32][kSigWords];      // per class of the group: Bloom signature
    unsigned long long mask[32];       // member own-attribute masks
    uint32_t ccnt[32], cH[32], cQ[32], cmb[32];  // per class: U-row length, H, LCOM-CK pairs, first position
    uint32_t rem[32];                  // per member: classes it alone uses
};

__device__ __forceinline__ void cas_sort(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
}

#ifndef MMGPU_GROUP_MINB
#define MMGPU_GROUP_MINB 12
#endif
__global__ void __launch_bounds__(kGroupWarps * 32, MMGPU_GROUP_MINB)
k_class_group(DevModel s, const uint4* __restrict__ cplan, const uint2* __restrict__ groups, uint32_t n_groups,
              const uint32_t* __restrict__ pos_owner, MethRec* __restrict__ recs, ClassRec* __restrict__ rec,
              double* __restrict__ lcom_out, uint64_t* __restrict__ ck_out, uint32_t* __restrict__ cbo_out,
              uint32_t* __restrict__ ux, uint32_t* __restrict__ un) {
    __shared__ GroupWarp sw[kGroupWarps];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t gi = blockIdx.x * kGroupWarps + warp;
    if (gi >= n_groups) return;
    GroupWarp& w = sw[warp];
    const uint2 g = groups[gi];  // (first class, number of classes)
    const uint32_t c0 = g.x, nc = g.y;
    uint4 cp = make_uint4(0, 0, 0, 0);
    if ((uint32_t)lane < nc) cp = cplan[c0 + lane];
    const uint32_t P0 = __shfl_sync(kFull, cp.x, 0);
    const uint32_t Pend = __shfl_sync(kFull, cp.x + cp.y, nc - 1);
    const uint32_t nm = Pend - P0;  // ≤ 32 by the plan
    const bool act = (uint32_t)lane < nm;
    const uint32_t pos = P0 + lane;
    // member rows (class-order offsets) and class
    uint32_t co = 0, co1 = 0, ao = 0, ao1 = 0, c = 0;
    if (act) {
        co = __ldg(s.pc_off + pos); co1 = __ldg(s.pc_off + pos + 1);
        ao = __ldg(s.pa_off + pos); ao1 = __ldg(s.pa_off + pos + 1);
        c = __ldg(pos_owner + pos);
    }
    // shared state
    w.keys[lane] = kNone;
    w.keys[lane + 32] = kNone;
    w.ccnt[lane] = 0; w.cH[lane] = 0; w.cQ[lane] = 0; w.rem[lane] = 0;
    w.cmb[lane] = cp.x;
    for (uint32_t j = lane; j < nc * kSigWords; j += 32) (&w.csig[0][0])[j] = 0;
    reinterpret_cast<uint4*>(w.ent[lane])[0] = make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(w.ent[lane])[1] = make_uint4(0, 0, 0, 0);
    // ---- edges: all targets, then all owners (branch-free: selected addresses, predicated loads) ----
    const uint32_t ncall = co1 - co, deg = ncall + (ao1 - ao);
    uint32_t key[kRecMaxEnt];
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k) {
        const uint32_t e = (uint32_t)k;
        const uint32_t* src = e < ncall ? s.pc_tgt + co + e : s.pa_tgt + ao + (e - ncall);
        key[k] = 0;
        if (e < deg) key[k] = __ldg(src);
    }
    unsigned long long mask = 0;
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k) {
        const uint32_t e = (uint32_t)k;
        const bool isa = e >= ncall;
        uint2 ai = make_uint2(kNone, 0u);
        if (e < ncall) ai.x = __ldg(s.method_owner + key[k]);
        if (isa && e < deg) ai = __ldg(s.attr_info + key[k]);
        if (isa && ai.x == c) mask |= 1ull << ai.y;  // lean: A ≤ 64
        key[k] = e < deg ? (ai.x << 1) | (isa ? 1u : 0u) : kNone;
    }
    // ---- sort (19-comparator network for 8), run-length encode ----
    cas_sort(key[0], key[2]); cas_sort(key[1], key[3]); cas_sort(key[4], key[6]); cas_sort(key[5], key[7]);
    cas_sort(key[0], key[4]); cas_sort(key[1], key[5]); cas_sort(key[2], key[6]); cas_sort(key[3], key[7]);
    cas_sort(key[0], key[1]); cas_sort(key[2], key[3]); cas_sort(key[4], key[5]); cas_sort(key[6], key[7]);
    cas_sort(key[2], key[4]); cas_sort(key[3], key[5]);
    cas_sort(key[1], key[4]); cas_sort(key[3], key[6]);
    cas_sort(key[1], key[2]); cas_sort(key[3], key[4]); cas_sort(key[5], key[6]);
    __syncwarp();
    const uint32_t ci = c - c0;
    uint32_t n = 0, hown = 0, h = 0, own_seen = 0;
    bool ovf = false;
#pragma unroll
    for (int k = 0; k < kRecMaxEnt; ++k) {
        if (key[k] == kNone) break;
        const uint32_t X = key[k] >> 1;
        h += key[k] & 1u;
        if (k + 1 < kRecMaxEnt && key[k + 1] != kNone && (key[k + 1] >> 1) == X) continue;  // run continues
        w.ent[lane][n++] = (X << 8) | h;
        ovf |= X >= (1u << 24);
        if (X == c) { hown = h; own_seen = 1; }
        h = 0;
    }
    // every (class, foreign X, member) once: compacted into 64 slots
    const uint32_t nf = n - own_seen;
    uint32_t fo = nf;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, fo, d);
        if (lane >= d) fo += y;
    }
    fo -= nf;
#pragma unroll 1
    for (uint32_t k = 0; k < n; ++k) {
        const uint32_t X = w.ent[lane][k] >> 8;
        if (X == c) continue;
        if (fo < kGroupKeys) w.keys[fo] = (ci << 27) | (X << 5) | (uint32_t)lane;
        ++fo;
    }
    if (act) {
        atomicAdd(&w.cH[ci], hown);
        w.mask[lane] = mask;
    }
    __syncwarp();
    // ---- bitonic sort of the 64 keys over the warp (element e = lane + 32 r) ----
    uint32_t v0 = w.keys[lane], v1 = w.keys[lane + 32];
#pragma unroll
    for (uint32_t k = 2; k <= kGroupKeys; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {  // partner in the same lane (only for k == 64: ascending)
                const uint32_t lo = min(v0, v1), hi = max(v0, v1);
                v0 = lo;
                v1 = hi;
            } else {
                const uint32_t p0 = __shfl_xor_sync(kFull, v0, j), p1 = __shfl_xor_sync(kFull, v1, j);
                const bool lower = ((uint32_t)lane & j) == 0;
                const bool up0 = ((uint32_t)lane & k) == 0, up1 = (((uint32_t)lane + 32u) & k) == 0;
                v0 = (lower == up0) ? min(v0, p0) : max(v0, p0);
                v1 = (lower == up1) ? min(v1, p1) : max(v1, p1);
            }
        }
    }
    // ---- runs of (class, X): U rows (ascending X), counts, Bloom, sole users ----
    const uint32_t prev0 = __shfl_up_sync(kFull, v0, 1), last0 = __shfl_sync(kFull, v0, 31);
    const uint32_t prev1 = __shfl_up_sync(kFull, v1, 1);
    const bool val0 = v0 != kNone, val1 = v1 != kNone;
    const bool hd0 = val0 && (lane == 0 || (prev0 >> 5) != (v0 >> 5));
    const bool hd1 = val1 && ((lane == 0 ? last0 : prev1) >> 5) != (v1 >> 5);
    const bool ch0 = val0 && (lane == 0 || (prev0 >> 27) != (v0 >> 27));   // first key of its class
    const bool ch1 = val1 && ((lane == 0 ? last0 : prev1) >> 27) != (v1 >> 27);
    const unsigned long long H = (unsigned long long)__ballot_sync(kFull, hd0) |
                                 ((unsigned long long)__ballot_sync(kFull, hd1) << 32);
    const unsigned long long CH = (unsigned long long)__ballot_sync(kFull, ch0) |
                                  ((unsigned long long)__ballot_sync(kFull, ch1) << 32);
    const uint32_t F = min(__shfl_sync(kFull, fo, 31), kGroupKeys);  // keys in use
#pragma unroll
    for (int r = 0; r < 2; ++r) {
        const bool hd = r ? hd1 : hd0;
        if (!hd) continue;
        const uint32_t v = r ? v1 : v0;
        const uint32_t e = (uint32_t)lane + 32u * r;
        const unsigned long long below = (1ull << e) - 1ull;
        const unsigned long long after = H & ~(below | (1ull << e));
        const uint32_t next = after ? (uint32_t)(__ffsll((long long)after) - 1) : F;
        const uint32_t cnt = next - e;                           // members using X
        const unsigned long long cb = CH & (below | (1ull << e));
        const uint32_t cs = 63u - (uint32_t)__clzll((long long)cb);  // the class's first key
        const uint32_t idx = (uint32_t)__popcll(H & below) - (uint32_t)__popcll(H & ((1ull << cs) - 1ull));
        const uint32_t cj = v >> 27, X = (v >> 5) & ((1u << 22) - 1u);
        const uint32_t ub = kSmallRowCap * w.cmb[cj];
        ux[ub + idx] = X;
        un[ub + idx] = cnt;
        atomicAdd(&w.ccnt[cj], 1u);
        if (cnt == 1) atomicAdd(&w.rem[v & 31u], 1u);
        const uint32_t b1 = bloom_h1(X), b2 = bloom_h2(X);
        atomicOr(&w.csig[cj][b1 >> 5], 1u << (b1 & 31u));
        atomicOr(&w.csig[cj][b2 >> 5], 1u << (b2 & 31u));
    }
    // ---- LCOM-CK: pairs inside each class's lane segment ----
    const uint32_t seg0 = act ? w.cmb[ci] - P0 : (uint32_t)lane;
    const uint32_t span = __reduce_max_sync(kFull, (uint32_t)lane - seg0);
    uint32_t q = 0;
    for (uint32_t d = 1; d <= span; ++d) {
        const uint32_t j = (uint32_t)lane - d;
        if (d <= (uint32_t)lane - seg0 && (mask & w.mask[j])) ++q;
    }
    if (act && q) atomicAdd(&w.cQ[ci], q);
    __syncwarp();
    // ---- outputs: records, headers, class records ----
    if (act) {
        const bool bad = ovf || hown >= 256u;
        const uint32_t hdr = bad ? kRecOverflow
                                 : (n | (hown << kRecHownShift) | (w.rem[lane] << kRecRemovedShift) | kRecRemovedValid);
        rec_hdrs(recs, s.M)[pos] = hdr;
    }
    {
        const uint4* src = reinterpret_cast<const uint4*>(&w.ent[0][0]);
        uint4* dst = reinterpret_cast<uint4*>(recs + P0);
        for (uint32_t j = lane; j < 2 * nm; j += 32) dst[j] = src[j];
    }
    if ((uint32_t)lane < nc) {
        const uint32_t cc = c0 + lane, M = cp.y, A = cp.z, H = w.cH[lane], Q = w.cQ[lane], cbo = w.ccnt[lane];
        uint4* rp = reinterpret_cast<uint4*>(rec + cc);
        const uint32_t* sg = w.csig[lane];
        rp[0] = make_uint4(A, M, H, cbo);
        rp[1] = make_uint4(kSmallRowCap * cp.x, kNone, sg[0], sg[1]);
        rp[2] = make_uint4(sg[2], sg[3], sg[4], sg[5]);
        rp[3] = make_uint4(sg[6], sg[7], sg[8], sg[9]);
        lcom_out[cc] = lcom_of(A, M, H);
        const uint64_t pairs = (uint64_t)M * (M ? M - 1 : 0) / 2;
        const uint64_t P = pairs - Q;
        ck_out[cc] = P > Q ? P - Q : 0;
        cbo_out[cc] = cbo;
    }
}

// Upload plan: runs of consecutive lean classes per warp of k_class_group
// (≤ 32 members, ≤ 64 foreign edges, ≤ 32 classes, member degree ≤ 8, fewer
// than 2^22 classes),
// greedily inside blocks of 16 classes (one thread per block); lean classes
// with a member of degree 9..16 go to k_class_lean's list.
__global__ void k_plan_groups(const uint4* __restrict__ cplan, const uint32_t* __restrict__ foreign,
                              const uint32_t* __restrict__ cmaxdeg, uint32_t C, uint2* __restrict__ groups,
                              uint32_t* __restrict__ n_groups, uint32_t* __restrict__ solo,
                              uint32_t* __restrict__ n_solo) {
    const uint32_t cb = (blockIdx.x * blockDim.x + threadIdx.x) * 16u;
    if (cb >= C) return;
    const uint32_t ce = min(cb + 16u, C);
    uint32_t g0 = 0, gn = 0, gm = 0, gf = 0;
    auto close = [&]() {
        if (gn) groups[atomicAdd(n_groups, 1u)] = make_uint2(g0, gn);
        gn = gm = gf = 0;
    };
    // the block's 16 plans first (independent loads), then the greedy walk on registers
    uint32_t kind[16], mem[16], fr[16], md[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t c = cb + k;
        kind[k] = kNone;
        if (c < ce) {
            const uint4 cp = cplan[c];
            kind[k] = cp.w;
            mem[k] = cp.y;
            fr[k] = foreign[c];
            md[k] = cmaxdeg[c];
        }
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        const uint32_t c = cb + k;
        if (c >= ce) break;
        if (kind[k] != kKindLean) { close(); continue; }
        // (group keys pack the class id in 22 bits)
        if (md[k] > (uint32_t)kRecMaxEnt || C >= (1u << 22)) { close(); solo[atomicAdd(n_solo, 1u)] = c; continue; }
        const uint4 cp = make_uint4(0, mem[k], 0, 0);
        const uint32_t f = fr[k];
        if (gn && (gm + cp.y > 32u || gf + f > 64u || gn == 32u)) close();
        if (!gn) g0 = c;
        ++gn; gm += cp.y; gf += f;
    }
    close();
}

// Upload plan: the class-order positions of every class that is not lean
// (k_method's list when both kinds exist), compacted on the device.
__global__ void k_nl_positions(const uint32_t* __restrict__ pos_owner, const uint4* __restrict__ cplan, uint32_t M,
                               uint32_t* __restrict__ out, uint32_t* __restrict__ n) {
    const uint32_t pos = blockIdx.x * blockDim.x + threadIdx.x;
    const bool keep = pos < M && cplan[pos_owner[pos]].w != kKindLean;
    const uint32_t b = __ballot_sync(kFull, keep);
    if (!b) return;
    const int lane = threadIdx.x & 31, lead = __ffs(b) - 1;
    uint32_t base = 0;
    if (lane == lead) base = atomicAdd(n, (uint32_t)__popc(b));
    base = __shfl_sync(kFull, base, lead);
    if (keep) out[base + __popc(b & ((1u << lane) - 1u))] = pos;
}

}  // namespace

void launch_class_group(const DevModel& s, const uint4* cplan, const uint2* groups, uint32_t n_groups,
                        const uint32_t* pos_owner, MethRec* recs, ClassRec* rec, double* lcom, uint64_t* ck,
                        uint32_t* cbo, uint32_t* ux, uint32_t* un, cudaStream_t st) {
    if (!n_groups) return;
    k_class_group<<<(n_groups + kGroupWarps - 1) / kGroupWarps, kGroupWarps * 32, 0, st>>>(
        s, cplan, groups, n_groups, pos_owner, recs, rec, lcom, ck, cbo, ux, un);
}

void launch_class_lean(const DevModel& s, const uint4* cplan, const uint4* cedge, const uint8_t* pc_mem,
                       const uint8_t* pa_mem, MethRec* recs, ClassRec* rec, double* lcom, uint64_t* ck, uint32_t* cbo,
                       uint32_t* ux, uint32_t* un, const uint32_t* list, uint32_t n_list, cudaStream_t st) {
    const uint32_t n = list ? n_list : s.C;
    if (!n) return;
    k_class_lean<<<(n + kLeanWarps - 1) / kLeanWarps, kLeanWarps * 32, 0, st>>>(s, cplan, cedge, pc_mem, pa_mem,
                                                                                  recs, rec, lcom, ck, cbo, ux, un,
                                                                                  list, n_list);
}

void launch_nl_positions(const uint32_t* pos_owner, const uint4* cplan, uint32_t M, uint32_t* out, uint32_t* n,
                         cudaStream_t st) {
    if (M) k_nl_positions<<<(M + 255) / 256, 256, 0, st>>>(pos_owner, cplan, M, out, n);
}

void launch_plan_groups(const uint4* cplan, const uint32_t* foreign, const uint32_t* cmaxdeg, uint32_t C,
                        uint2* groups, uint32_t* n_groups, uint32_t* solo, uint32_t* n_solo, cudaStream_t st) {
    if (!C) return;
    const uint32_t threads = (C + 15) / 16;
    k_plan_groups<<<(threads + 127) / 128, 128, 0, st>>>(cplan, foreign, cmaxdeg, C, groups, n_groups, solo, n_solo);
}

}  // namespace mmg
