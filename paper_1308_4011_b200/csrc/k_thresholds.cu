// k_thresholds.cu — compute_thresholds' means (suggest.hpp:46-61) with the
// reference's SEQUENTIAL double-sum semantics, computed in parallel.
//
// The reference sums per-class lcom left to right in double precision:
// s_{i+1} = RN(s_i + x_i). Reassociating would change the last bits, so a
// plain tree reduction is not bit-exact. A serial loop on the GPU is exact but
// costs ~3 ms for 100k classes (one dependent fp64 add chain). Instead:
//
// * Every lcom value is k·2^-53 with k ∈ [0, 2^53] (1 − q with q ∈ [0,1]:
//   exact when q ≥ 1/2 by Sterbenz, else rounded in [1/2, 1] whose ulp is
//   2^-53). So the state is an exact integer T = s·2^53 (< 2^85) and one step
//   is T' = RNE53(T + X): round to 53 significant bits, ties to even.
// * While the exact sum stays in one binade (granularity g = 2^e), a step on a
//   state that is a multiple of g is T' = T + g·inc where inc depends on X and
//   only on the PARITY of T/g (ties to even). Each element is therefore a
//   function on one bit of state — {p -> (inc_p, p'_p)} — and those compose
//   associatively: a segmented block scan yields, for every chunk of elements,
//   the composed function since its binade segment began. The first element
//   of each segment (where g doubles) is applied exactly; segments are at
//   most ~34, chained by one thread.
// * That gives every chunk's starting state S_t. Each thread then replays its
//   chunk with exact RNE arithmetic from S_t, and the result is accepted only
//   if every chunk's end state equals the next chunk's S_{t+1} (induction from
//   S_0 = 0): the answer is then provably the sequential sum, bit for bit.
//   Any violated precondition or mismatch falls back to the serial loop in
//   the same kernel.
//
// cbo's mean sums integers: exact in u64, and (double)Σ equals the
// reference's running double sum while Σ < 2^53 (checked; else serial).
#include <cuda_runtime.h>

#include <atomic>

#include <cooperative_groups.h>

#include <cstdint>
#include <cstdlib>

#include "mm_async.cuh"
#include "mm_device.cuh"
#include "mm_kernels.h"

namespace mmg {

namespace {

typedef unsigned __int128 u128;
constexpr int kThrThreads = 1024;
constexpr int kMaxSegs = 64;

__device__ __forceinline__ int bitlen128(u128 v) {
    const uint64_t hi = (uint64_t)(v >> 64), lo = (uint64_t)v;
    return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

__device__ __forceinline__ int gran_exp(u128 v) {  // e with ulp(v·2^-53) = 2^e units
    const int b = bitlen128(v);
    return b > 53 ? b - 53 : 0;
}

__device__ __forceinline__ u128 rne53(u128 v) {
    const int e = gran_exp(v);
    if (e == 0) return v;
    const u128 g = (u128)1 << e, half = g >> 1, r = v & (g - 1);
    u128 q = v >> e;
    if (r > half || (r == half && (q & 1))) q += 1;
    return q << e;
}

// element function on one bit of state: p -> (inc[p], par bit (p' of p) in bits)
struct Fn {
    uint64_t inc0, inc1;
    uint32_t bits;  // bit0: p'(0), bit1: p'(1), bit2: segment-start flag (scan carrier)
};

__device__ __forceinline__ Fn fn_id() { return {0, 0, 0b10u}; }

__device__ __forceinline__ Fn fn_elem(uint64_t X, int e) {
    uint64_t i0, i1;
    if (e == 0) {
        i0 = i1 = X;
    } else {
        const uint64_t q = X >> e, r = X & ((1ull << e) - 1), half = 1ull << (e - 1);
        if (r < half) i0 = i1 = q;
        else if (r > half) i0 = i1 = q + 1;
        else {  // tie: the result multiple must be even
            i0 = (q & 1) ? q + 1 : q;        // p = 0
            i1 = (q & 1) ? q : q + 1;        // p = 1
        }
    }
    return {i0, i1, (uint32_t)((0 + i0) & 1) | ((uint32_t)((1 + i1) & 1) << 1)};
}

__device__ __forceinline__ int fpar(const Fn& f, int p) { return (f.bits >> p) & 1; }
__device__ __forceinline__ uint64_t finc(const Fn& f, int p) { return p ? f.inc1 : f.inc0; }

// a then b (flags: the result carries a's|b's flag; segmented combine handled by caller)
__device__ __forceinline__ Fn compose(const Fn& a, const Fn& b) {
    const int a0 = fpar(a, 0), a1 = fpar(a, 1);
    Fn c;
    c.inc0 = a.inc0 + finc(b, a0);
    c.inc1 = a.inc1 + finc(b, a1);
    c.bits = (uint32_t)fpar(b, a0) | ((uint32_t)fpar(b, a1) << 1);
    return c;
}

// segmented combine of (L, R): flag = L|R; F = R.flag ? R.F : L.F ∘ R.F
__device__ __forceinline__ Fn seg_combine(const Fn& L, const Fn& R) {
    Fn c = (R.bits & 4u) ? R : compose(L, R);
    c.bits = (c.bits & 3u) | ((L.bits | R.bits) & 4u);
    return c;
}

__device__ __forceinline__ Fn shfl_up_fn(const Fn& f, int d) {
    Fn o;
    o.inc0 = __shfl_up_sync(0xffffffffu, f.inc0, d);
    o.inc1 = __shfl_up_sync(0xffffffffu, f.inc1, d);
    o.bits = __shfl_up_sync(0xffffffffu, f.bits, d);
    return o;
}

__device__ __forceinline__ u128 shfl_up_u128(u128 v, int d) {
    const uint64_t lo = __shfl_up_sync(0xffffffffu, (uint64_t)v, d);
    const uint64_t hi = __shfl_up_sync(0xffffffffu, (uint64_t)(v >> 64), d);
    return ((u128)hi << 64) | lo;
}

__device__ __forceinline__ bool lcom_units(double x, uint64_t& X) {
    if (!(x >= 0.0 && x <= 1.0)) return false;
    const double y = x * 0x1p53;  // exact (power-of-two scaling)
    X = (uint64_t)y;
    return (double)X == y;
}

constexpr int kTT = 256;                  // threads per CTA
constexpr int kItems = 8;                 // consecutive elements per thread
constexpr int kTile = kTT * kItems;       // 2048 elements: one tile per CTA
constexpr int kSlot = kMaxSegs + 1;       // piece slots per tile

// A tile's run of one binade: the continuation piece (first = 0: its function
// covers elements from the tile start) or a real segment piece (first = 1:
// X of its first element is applied exactly, the function covers the rest).
struct Piece {
    Fn f;
    uint64_t x_first;
    int e;
    int first;
};

struct Scratch {              // global scratch, sized for the grid
    u128* tile_sum;           // [tiles] exact Σ X
    u128* tile_entry;         // [tiles] chained entry state
    u128* tile_exit;          // [tiles] replayed exit state
    Piece* pieces;            // [tiles * kSlot]
    int* n_pieces;            // [tiles]
    unsigned long long* cbo_sum;
    int* bad;
};

struct TileShared {
    u128 warp_u128[kTT / 32];
    Fn warp_fn[kTT / 32];
    u128 start_state[kTT];
    u128 end_state[kTT];
    uint32_t seg_pos[kMaxSegs];
    int seg_e[kMaxSegs];
    uint64_t seg_x[kMaxSegs];
    Fn seg_total[kMaxSegs + 1];
    u128 seg_first[kMaxSegs];
    u128 seg_end[kMaxSegs + 1];
    u128 entry;
    u128 prefix;
    int n_segs;
};

__device__ __forceinline__ u128 blk_excl_u128(u128 v, TileShared& sh, u128* total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u128 inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u128 y = shfl_up_u128(inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) sh.warp_u128[warp] = inc;
    __syncthreads();
    u128 pre = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kTT / 32; ++w) {
        if (w < warp) pre += sh.warp_u128[w];
        all += sh.warp_u128[w];
    }
    *total = all;
    __syncthreads();
    return pre + inc - v;
}

__device__ __forceinline__ Fn blk_excl_fn(const Fn& agg, TileShared& sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Fn x = agg;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Fn y = shfl_up_fn(x, d);
        if (lane >= d) x = seg_combine(y, x);
    }
    if (lane == 31) sh.warp_fn[warp] = x;
    const Fn xin = shfl_up_fn(x, 1);
    __syncthreads();
    Fn wp = fn_id();
#pragma unroll
    for (int w = 0; w < kTT / 32; ++w)
        if (w < warp) wp = seg_combine(wp, sh.warp_fn[w]);
    __syncthreads();
    return lane == 0 ? wp : seg_combine(wp, xin);
}

// Cooperative kernel: one 2048-element tile per CTA, three grid-wide phases.
__global__ void __launch_bounds__(kTT)
k_thresholds_coop(const double* __restrict__ lcom, const uint32_t* __restrict__ cbo, uint32_t n,
                  Scratch g, DevThresholds* __restrict__ out) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    __shared__ TileShared sh;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t tile = blockIdx.x, n_tiles = gridDim.x;
    const uint32_t base = tile * kTile;
    const uint32_t my = base + (uint32_t)t * kItems;
    const int cnt = my < n ? (int)min((uint32_t)kItems, n - my) : 0;
    const uint32_t tile_end = min(n, base + kTile);

    // ---- phase 1: load, preconditions, exact tile sum, cbo sum
    uint64_t X[kItems];
    int bad = 0;
    uint64_t cs = 0;
    if (cnt == kItems && ((reinterpret_cast<uintptr_t>(lcom + my) & 15) == 0)) {
        const double2* p2 = reinterpret_cast<const double2*>(lcom + my);
#pragma unroll
        for (int j = 0; j < kItems / 2; ++j) {
            const double2 v = p2[j];
            bad |= !lcom_units(v.x, X[2 * j]);
            bad |= !lcom_units(v.y, X[2 * j + 1]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            X[j] = 0;
            if (j < cnt) bad |= !lcom_units(lcom[my + j], X[j]);
        }
    }
    if (cbo) {
#pragma unroll
        for (int j = 0; j < kItems; ++j)
            if (j < cnt) cs += cbo[my + j];
    }
    if (bad) atomicOr(g.bad, 1);
    u128 S = 0;
#pragma unroll
    for (int j = 0; j < kItems; ++j) S += X[j];
    u128 tsum;
    const u128 excl_sum = blk_excl_u128(S, sh, &tsum);
    {
        unsigned long long cw = cs;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) cw += __shfl_down_sync(0xffffffffu, cw, d);
        if (lane == 0 && cw) atomicAdd(g.cbo_sum, cw);
    }
    if (t == 0) g.tile_sum[tile] = tsum;
    grid.sync();

    // ---- phase 2: exact prefix, binade segments, per-thread compositions, tile pieces
    {
        u128 part = 0;
        for (uint32_t j = t; j < tile; j += kTT) part += g.tile_sum[j];
        u128 dummy;
        const u128 ex = blk_excl_u128(part, sh, &dummy);
        (void)ex;
        if (t == 0) { sh.prefix = dummy; sh.n_segs = 0; }
        __syncthreads();
    }
    const u128 P_tile = sh.prefix;
    const u128 P_my = P_tile + excl_sum;
    const int e_cont = base == 0 ? -1 : gran_exp(P_tile);
    int e_el[kItems];
    uint32_t starts = 0;
    Fn agg = fn_id();
    {
        u128 P = P_my;
        int e_prev = my == 0 ? -1 : gran_exp(P_my);
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            e_el[j] = 0;
            if (j < cnt) {
                P += X[j];
                const int e = gran_exp(P);
                e_el[j] = e;
                if (e != e_prev) {
                    starts |= 1u << j;
                    const int k = atomicAdd(&sh.n_segs, 1);
                    if (k < kMaxSegs) { sh.seg_pos[k] = my + j; sh.seg_e[k] = e; sh.seg_x[k] = X[j]; }
                    agg = fn_id();
                    agg.bits |= 4u;
                } else {
                    const uint32_t fl = agg.bits & 4u;
                    agg = compose(agg, fn_elem(X[j], e));
                    agg.bits |= fl;
                }
                e_prev = e;
            }
        }
    }
    const Fn excl = blk_excl_fn(agg, sh);
    if (t == 0) {
        if (sh.n_segs > kMaxSegs) atomicOr(g.bad, 4);
        const int ns = min(sh.n_segs, kMaxSegs);
        for (int a = 1; a < ns; ++a)
            for (int b = a; b > 0 && sh.seg_pos[b - 1] > sh.seg_pos[b]; --b) {
                const uint32_t tp = sh.seg_pos[b]; sh.seg_pos[b] = sh.seg_pos[b - 1]; sh.seg_pos[b - 1] = tp;
                const int te = sh.seg_e[b]; sh.seg_e[b] = sh.seg_e[b - 1]; sh.seg_e[b - 1] = te;
                const uint64_t tx = sh.seg_x[b]; sh.seg_x[b] = sh.seg_x[b - 1]; sh.seg_x[b - 1] = tx;
            }
        sh.seg_total[0] = fn_id();
    }
    __syncthreads();
    const int ns = min(sh.n_segs, kMaxSegs);
    int kb = -1;  // local segment active just before `my` (-1: continuation)
    for (int k = 0; k < ns; ++k)
        if (sh.seg_pos[k] < my) kb = k;
    if (cnt > 0) {
        Fn run = excl;
        int k = kb;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            if (j < cnt) {
                if (starts & (1u << j)) {
                    if (k + 1 <= kMaxSegs) sh.seg_total[k + 1] = run;
                    ++k;
                    run = fn_id();
                } else {
                    run = compose(run, fn_elem(X[j], e_el[j]));
                }
            }
        }
        if (my + cnt == tile_end && k + 1 <= kMaxSegs) sh.seg_total[k + 1] = run;
    }
    __syncthreads();
    const bool has_cont = !(ns > 0 && sh.seg_pos[0] == base);
    if (t == 0) {
        Piece* pc = g.pieces + (size_t)tile * kSlot;
        int np = 0;
        if (has_cont) pc[np++] = Piece{sh.seg_total[0], 0, e_cont, 0};
        for (int k = 0; k < ns; ++k) pc[np++] = Piece{sh.seg_total[k + 1], sh.seg_x[k], sh.seg_e[k], 1};
        g.n_pieces[tile] = np;
    }
    grid.sync();

    // ---- phase 3: chain all earlier pieces -> tile entry state; derive chunk
    // starts; exact replay; verify chunk joins
    if (t == 0) {
        u128 T = 0;
        for (uint32_t b = 0; b < tile; ++b) {
            const Piece* pc = g.pieces + (size_t)b * kSlot;
            const int np = g.n_pieces[b];
            for (int i = 0; i < np; ++i) {
                const Piece q = pc[i];
                if (q.first) T = rne53(T + q.x_first);
                if (q.e >= 0) T += (u128)finc(q.f, (int)((T >> q.e) & 1)) << q.e;
            }
        }
        sh.entry = T;
        g.tile_entry[tile] = T;
        // this tile's segment states
        if (has_cont && e_cont >= 0) T += (u128)finc(sh.seg_total[0], (int)((T >> e_cont) & 1)) << e_cont;
        sh.seg_end[0] = T;
        for (int k = 0; k < ns; ++k) {
            const int e = sh.seg_e[k];
            T = rne53(T + sh.seg_x[k]);
            sh.seg_first[k] = T;
            T += (u128)finc(sh.seg_total[k + 1], (int)((T >> e) & 1)) << e;
            sh.seg_end[k + 1] = T;
        }
    }
    __syncthreads();
    const u128 T_entry = sh.entry;
    u128 S0 = T_entry;
    if (cnt > 0) {
        if (starts & 1u) {
            S0 = sh.seg_end[kb + 1];
        } else if (kb >= 0) {
            const int e = sh.seg_e[kb];
            const u128 F = sh.seg_first[kb];
            S0 = F + ((u128)finc(excl, (int)((F >> e) & 1)) << e);
        } else if (e_cont >= 0) {
            S0 = T_entry + ((u128)finc(excl, (int)((T_entry >> e_cont) & 1)) << e_cont);
        }
    }
    sh.start_state[t] = S0;
    u128 T = S0;
#pragma unroll
    for (int j = 0; j < kItems; ++j)
        if (j < cnt) T = rne53(T + X[j]);
    sh.end_state[t] = T;
    __syncthreads();
    if (cnt > 0) {
        if (my == base && S0 != T_entry) atomicOr(g.bad, 2);
        const bool last = my + cnt == tile_end;
        if (!last && sh.start_state[t + 1] != T) atomicOr(g.bad, 2);
        if (last) g.tile_exit[tile] = T;
    }
    grid.sync();

    // ---- phase 4: tile joins, final mean (or the serial fallback)
    if (tile == 0 && t == 0) {
        int b = *g.bad;
        for (uint32_t j = 1; j < n_tiles; ++j)
            if (g.tile_exit[j - 1] != g.tile_entry[j]) b |= 2;
        double mean_l;
        uint32_t fast = 1;
        if (b || n == 0) {
            fast = 0;
            double s = 0.0;
            for (uint32_t i = 0; i < n; ++i) s = __dadd_rn(s, lcom[i]);
            mean_l = n ? __ddiv_rn(s, (double)n) : 0.0;
        } else {
            const u128 Tn = g.tile_exit[n_tiles - 1];
            const int bl = bitlen128(Tn);
            const int sft = bl > 53 ? bl - 53 : 0;
            mean_l = __ddiv_rn(ldexp((double)(uint64_t)(Tn >> sft), sft - 53), (double)n);
        }
        const unsigned long long csum = *g.cbo_sum;
        double mean_c;
        if (csum < (1ull << 53)) {
            mean_c = n ? __ddiv_rn((double)csum, (double)n) : 0.0;
        } else {
            fast = 0;
            double sc = 0.0;
            for (uint32_t i = 0; i < n; ++i) sc = __dadd_rn(sc, cbo ? (double)cbo[i] : 0.0);
            mean_c = n ? __ddiv_rn(sc, (double)n) : 0.0;
        }
        out->lcom = mean_l;
        out->cbo = mean_c;
        out->fast_path_ok = fast;
    }
}

// ---- one-CTA variant (n ≤ kBlockMax): the same exact emulation without grid
// syncs, so it runs on a single SM next to the candidate scoring instead of
// holding every SM through three grid-wide barriers. 1024 threads, each owning
// a contiguous chunk of ⌈n/1024⌉ values: (1) exact chunk sums (u128 in 2^-53
// units) and a block scan give each chunk's exact prefix; (2) a chunk whose
// prefix stays in one binade (all but ≤ ~34 chunks) composes its elements'
// one-bit-state functions in one straight pass, the few chunks where a binade
// starts walk element by element and record the segment starts; a segmented
// block scan of the functions and one thread chaining the segments give every
// chunk's start state; (3) every chunk is replayed with IEEE double adds from
// its start state and must end exactly on the next chunk's start (induction
// from 0): the result is then the sequential sum. Anything else -> serial.
constexpr int kBT = 1024;
constexpr uint32_t kBlockMax = kBT * 256;

struct BlockShared {
    u128 warp_u128[kBT / 32];
    Fn warp_fn[kBT / 32];
    unsigned long long warp_c[kBT / 32];
    double start[kBT];
    uint32_t seg_pos[kMaxSegs];
    int seg_e[kMaxSegs];
    uint64_t seg_x[kMaxSegs];
    Fn seg_total[kMaxSegs + 1];
    u128 seg_first[kMaxSegs];
    u128 seg_end[kMaxSegs + 1];
    int n_segs;
    int bad;
};

template <class SH>
__device__ __forceinline__ u128 blk1k_excl_u128(u128 v, SH& sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u128 inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u128 y = shfl_up_u128(inc, d);
        if (lane >= d) inc += y;
    }
    if (lane == 31) sh.warp_u128[warp] = inc;
    __syncthreads();
    if (warp == 0) {  // scan of the 32 warp totals
        u128 w = sh.warp_u128[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u128 y = shfl_up_u128(w, d);
            if (lane >= d) w += y;
        }
        sh.warp_u128[lane] = w;
    }
    __syncthreads();
    return (warp ? sh.warp_u128[warp - 1] : (u128)0) + inc - v;
}

template <class SH>
__device__ __forceinline__ Fn blk1k_excl_fn(const Fn& agg, SH& sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Fn x = agg;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Fn y = shfl_up_fn(x, d);
        if (lane >= d) x = seg_combine(y, x);
    }
    if (lane == 31) sh.warp_fn[warp] = x;
    const Fn xin = shfl_up_fn(x, 1);
    __syncthreads();
    if (warp == 0) {
        Fn w = sh.warp_fn[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const Fn y = shfl_up_fn(w, d);
            if (lane >= d) w = seg_combine(y, w);
        }
        sh.warp_fn[lane] = w;
    }
    __syncthreads();
    const Fn wp = warp ? sh.warp_fn[warp - 1] : fn_id();
    return lane == 0 ? wp : seg_combine(wp, xin);
}

__device__ __forceinline__ double u128_to_double(u128 T) {  // T·2^-53, exact for ≤ 53 significant bits
    const int bl = bitlen128(T);
    const int sft = bl > 64 ? bl - 64 : 0;
    return ldexp((double)(uint64_t)(T >> sft), sft - 53);
}

__global__ void __launch_bounds__(kBT, 1)
k_thresholds_block(const double* __restrict__ lcom, const uint32_t* __restrict__ cbo, uint32_t n,
                   DevThresholds* __restrict__ out) {
    __shared__ BlockShared sh;
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const uint32_t E = (n + kBT - 1) / kBT;
    const uint32_t my = (uint32_t)t * E;
    const uint32_t cnt = my < n ? min(E, n - my) : 0u;
    if (t == 0) { sh.n_segs = 0; sh.bad = 0; }
    // (1) preconditions, exact chunk sum, cbo sum
    u128 S = 0;
    unsigned long long cs = 0;
    int bad = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
        uint64_t X;
        bad |= !lcom_units(__ldg(lcom + my + j), X);
        S += X;
        if (cbo) cs += __ldg(cbo + my + j);
    }
    {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) cs += __shfl_down_sync(0xffffffffu, cs, d);
        if (lane == 0) sh.warp_c[warp] = cs;
    }
    if (__syncthreads_or(bad)) {  // outside the fast path's precondition: serial
        if (warp == 0) {
            double sl = 0.0;
            for (uint32_t b = 0; b < n; b += 32) {
                const uint32_t i = b + lane;
                const double v = i < n ? lcom[i] : 0.0;
                const uint32_t m = min(32u, n - b);
                for (uint32_t k = 0; k < m; ++k) sl = __dadd_rn(sl, __shfl_sync(0xffffffffu, v, k));
            }
            if (lane == 0) sh.seg_first[0] = (u128)0, sh.start[0] = sl;
        }
        __syncthreads();
        if (t == 0) {
            unsigned long long csum = 0;
            for (int w = 0; w < kBT / 32; ++w) csum += sh.warp_c[w];
            out->lcom = n ? __ddiv_rn(sh.start[0], (double)n) : 0.0;
            double mc;
            if (csum < (1ull << 53)) {
                mc = n ? __ddiv_rn((double)csum, (double)n) : 0.0;
            } else {
                double sc = 0.0;
                for (uint32_t i = 0; i < n; ++i) sc = __dadd_rn(sc, cbo ? (double)cbo[i] : 0.0);
                mc = n ? __ddiv_rn(sc, (double)n) : 0.0;
            }
            out->cbo = mc;
            out->fast_path_ok = 0;
        }
        return;
    }
    const u128 P_my = blk1k_excl_u128(S, sh);
    // (2) binade segments and per-chunk functions
    const int e_prev = my == 0 ? -1 : gran_exp(P_my);
    const bool has_start = cnt > 0 && gran_exp(P_my + S) != e_prev;
    Fn agg = fn_id();
    if (cnt > 0 && !has_start) {
        for (uint32_t j = 0; j < cnt; ++j) {
            uint64_t X;
            lcom_units(__ldg(lcom + my + j), X);
            agg = compose(agg, fn_elem(X, e_prev));
        }
    } else if (has_start) {
        u128 P = P_my;
        int ep = e_prev;
        for (uint32_t j = 0; j < cnt; ++j) {
            uint64_t X;
            lcom_units(__ldg(lcom + my + j), X);
            P += X;
            const int e = gran_exp(P);
            if (e != ep) {
                const int k = atomicAdd(&sh.n_segs, 1);
                if (k < kMaxSegs) { sh.seg_pos[k] = my + j; sh.seg_e[k] = e; sh.seg_x[k] = X; }
                agg = fn_id();
                agg.bits |= 4u;
            } else {
                const uint32_t fl = agg.bits & 4u;
                agg = compose(agg, fn_elem(X, e));
                agg.bits |= fl;
            }
            ep = e;
        }
    }
    const Fn excl = blk1k_excl_fn(agg, sh);
    if (t == 0) {
        if (sh.n_segs > kMaxSegs) sh.bad = 1;
        const int ns = min(sh.n_segs, kMaxSegs);
        for (int a = 1; a < ns; ++a)
            for (int b = a; b > 0 && sh.seg_pos[b - 1] > sh.seg_pos[b]; --b) {
                const uint32_t tp = sh.seg_pos[b]; sh.seg_pos[b] = sh.seg_pos[b - 1]; sh.seg_pos[b - 1] = tp;
                const int te = sh.seg_e[b]; sh.seg_e[b] = sh.seg_e[b - 1]; sh.seg_e[b - 1] = te;
                const uint64_t tx = sh.seg_x[b]; sh.seg_x[b] = sh.seg_x[b - 1]; sh.seg_x[b - 1] = tx;
            }
    }
    __syncthreads();
    const int ns = min(sh.n_segs, kMaxSegs);
    int kb = -1;  // the segment active just before this chunk
    for (int k = 0; k < ns; ++k)
        if (sh.seg_pos[k] < my) kb = k;
    // segment totals: closed by the chunk holding the next segment's start, or the last chunk
    if (has_start) {
        Fn run = excl;
        int k = kb;
        u128 P = P_my;
        int ep = e_prev;
        for (uint32_t j = 0; j < cnt; ++j) {
            uint64_t X;
            lcom_units(__ldg(lcom + my + j), X);
            P += X;
            const int e = gran_exp(P);
            if (e != ep) {
                if (k + 1 <= kMaxSegs) sh.seg_total[k + 1] = run;
                ++k;
                run = fn_id();
            } else {
                run = compose(run, fn_elem(X, e));
            }
            ep = e;
        }
        if (my + cnt == n && k + 1 <= kMaxSegs) sh.seg_total[k + 1] = run;
    } else if (cnt > 0 && my + cnt == n && kb + 1 <= kMaxSegs) {
        sh.seg_total[kb + 1] = compose(excl, agg);
    }
    __syncthreads();
    if (t == 0) {  // chain the segments from S_0 = 0
        u128 T = 0;
        sh.seg_end[0] = T;
        for (int k = 0; k < ns; ++k) {
            const int e = sh.seg_e[k];
            T = rne53(T + sh.seg_x[k]);
            sh.seg_first[k] = T;
            T += (u128)finc(sh.seg_total[k + 1], (int)((T >> e) & 1)) << e;
            sh.seg_end[k + 1] = T;
        }
    }
    __syncthreads();
    // start state of this chunk
    u128 S0 = 0;
    if (cnt > 0) {
        if (has_start && sh.seg_pos[kb + 1] == my) {
            S0 = sh.seg_end[kb + 1];
        } else if (kb >= 0) {
            const int e = sh.seg_e[kb];
            const u128 F = sh.seg_first[kb];
            S0 = F + ((u128)finc(excl, (int)((F >> e) & 1)) << e);
        }
    }
    const double s0 = u128_to_double(S0);
    sh.start[t] = s0;
    __syncthreads();
    // (3) exact replay in IEEE doubles; every join must hold
    double sv = s0;
    for (uint32_t j = 0; j < cnt; ++j) sv = __dadd_rn(sv, __ldg(lcom + my + j));
    int jb = 0;
    if (cnt > 0 && my + cnt < n && sh.start[t + 1] != sv) jb = 1;
    if (my == 0 && cnt > 0 && s0 != 0.0) jb = 1;
    if (cnt > 0 && my + cnt == n) sh.start[0] = sv;  // the last chunk's end: the sequential sum (t ≥ 1 or n small)
    const int any_bad = __syncthreads_or(jb | sh.bad);
    if (t == 0) {
        unsigned long long csum = 0;
        for (int w = 0; w < kBT / 32; ++w) csum += sh.warp_c[w];
        double ml;
        uint32_t fast = 1;
        if (any_bad) {
            fast = 0;
            double sl = 0.0;
            for (uint32_t i = 0; i < n; ++i) sl = __dadd_rn(sl, lcom[i]);
            ml = n ? __ddiv_rn(sl, (double)n) : 0.0;
        } else {
            ml = n ? __ddiv_rn(sh.start[0], (double)n) : 0.0;
        }
        double mc;
        if (csum < (1ull << 53)) {
            mc = n ? __ddiv_rn((double)csum, (double)n) : 0.0;
        } else {
            fast = 0;
            double sc = 0.0;
            for (uint32_t i = 0; i < n; ++i) sc = __dadd_rn(sc, cbo ? (double)cbo[i] : 0.0);
            mc = n ? __ddiv_rn(sc, (double)n) : 0.0;
        }
        out->lcom = ml;
        out->cbo = mc;
        out->fast_path_ok = fast;
    }
}

// ---- cluster variant (n ≤ kClusterMax): the one-CTA algorithm spread over a
// thread-block cluster of 8 CTAs (8 SMs) whose shared memory holds every value:
// one coalesced load per value into the owning CTA's shared memory, then the
// three phases read shared memory only; the block-level scans are combined
// across the cluster through distributed shared memory, with cluster barriers
// (hardware) between phases. Segment chaining (≤ kMaxSegs starts, in rank
// order) is done by one thread of CTA 0, which publishes the chained states.
constexpr int kCC = 8;                                  // CTAs per cluster (portable)
constexpr int kCPer = 17;                               // values per thread (max): (8 + 4) B each in shared memory
constexpr uint32_t kClusterMax = (uint32_t)kCC * kBT * kCPer;  // 139,264 values

struct ClusterShared {
    u128 warp_u128[kBT / 32];
    Fn warp_fn[kBT / 32];
    unsigned long long warp_c[kBT / 32];
    double start[kBT];
    // this CTA's segment starts (local list), each with the function of the
    // segment it closes (the previous one)
    uint32_t seg_pos[kMaxSegs];
    int seg_e[kMaxSegs];
    uint64_t seg_x[kMaxSegs];
    Fn seg_close[kMaxSegs];
    int n_segs;
    int bad;
    u128 cta_total;
    Fn cta_agg;
    unsigned long long cta_cbo;
    Fn final_total;   // the last segment's function (written by the CTA owning the last value)
    int has_final;
    double final_sum;
    uint64_t bar;     // the bulk copies' mbarrier
    // cluster-wide chained segment table (filled in CTA 0, copied by every CTA)
    int g_n;
    uint32_t g_pos[kMaxSegs];
    int g_e[kMaxSegs];
    u128 g_first[kMaxSegs];
    u128 g_end[kMaxSegs + 1];
    // CTA 0's gather of every CTA's starts (unsorted), then sorted x / closing functions
    uint32_t seg_pos_all[kMaxSegs];
    int seg_e_all[kMaxSegs];
    uint64_t seg_x_all[kMaxSegs];
    Fn seg_close_all[kMaxSegs];
    uint64_t g_x[kMaxSegs];
    Fn g_close[kMaxSegs];
};

__global__ void __cluster_dims__(kCC, 1, 1) __launch_bounds__(kBT, 1)
k_thresholds_cluster(const double* __restrict__ lcom, const uint32_t* __restrict__ cbo, uint32_t n,
                     DevThresholds* __restrict__ out) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ ClusterShared sh;
    extern __shared__ double vals[];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int rank = (int)cluster.block_rank();
    const uint32_t E = (n + kCC * kBT - 1) / (kCC * kBT);
    const uint32_t base = (uint32_t)rank * kBT * E;
    const uint32_t len = base < n ? min((uint32_t)kBT * E, n - base) : 0u;
    const uint32_t lo = (uint32_t)t * E;                  // local chunk start
    const uint32_t cnt = lo < len ? min(E, len - lo) : 0u;
    const uint32_t my = base + lo;                        // global chunk start
    // ---- this CTA's values and cbo counts into shared memory: one bulk (TMA)
    // copy each, completing on an mbarrier; the odd tail by plain loads
    uint32_t* cvals = reinterpret_cast<uint32_t*>(vals + (size_t)kBT * E);
    const uint32_t lb = (len * 8u) & ~15u, cb = cbo ? (len * 4u) & ~15u : 0u;
    if (t == 0) {
        sh.n_segs = 0; sh.bad = 0; sh.has_final = 0;
        mbar_init(&sh.bar, 1);
    }
    __syncthreads();
    if (t == 0) {
        mbar_expect_tx(&sh.bar, lb + cb);
        if (lb) bulk_g2s(vals, lcom + base, lb, &sh.bar);
        if (cb) bulk_g2s(cvals, cbo + base, cb, &sh.bar);
    }
    for (uint32_t i = lb / 8 + t; i < len; i += kBT) vals[i] = __ldg(lcom + base + i);
    if (cbo)
        for (uint32_t i = cb / 4 + t; i < len; i += kBT) cvals[i] = __ldg(cbo + base + i);
    mbar_wait(&sh.bar, 0);
    __syncthreads();
    unsigned long long cs = 0;
    if (cbo)
        for (uint32_t j = 0; j < cnt; ++j) cs += cvals[lo + j];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) cs += __shfl_down_sync(0xffffffffu, cs, d);
    if (lane == 0) sh.warp_c[warp] = cs;
    // ---- (1) preconditions, exact chunk sums, cluster prefix
    u128 S = 0;
    int bad = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
        uint64_t X;
        bad |= !lcom_units(vals[lo + j], X);
        S += X;
    }
    bad = __syncthreads_or(bad);
    const u128 ex_blk = blk1k_excl_u128(S, sh);
    if (t == kBT - 1) sh.cta_total = ex_blk + S;
    if (t == 0) {
        unsigned long long c = 0;
        for (int w = 0; w < kBT / 32; ++w) c += sh.warp_c[w];
        sh.cta_cbo = c;
        sh.bad = bad;
    }
    cluster.sync();
    int any_bad = 0;
    u128 cta_prefix = 0;
    for (int r = 0; r < kCC; ++r) {
        ClusterShared* o = cluster.map_shared_rank(&sh, r);
        any_bad |= o->bad;
        if (r < rank) cta_prefix += o->cta_total;
    }
    if (any_bad) {  // outside the fast path's precondition: CTA 0 sums serially
        if (rank == 0 && warp == 0) {
            double sl = 0.0;
            for (uint32_t b = 0; b < n; b += 32) {
                const uint32_t i = b + lane;
                const double v = i < n ? lcom[i] : 0.0;
                const uint32_t m = min(32u, n - b);
                for (uint32_t k = 0; k < m; ++k) sl = __dadd_rn(sl, __shfl_sync(0xffffffffu, v, k));
            }
            if (lane == 0) {
                unsigned long long csum = 0;
                for (int r = 0; r < kCC; ++r) csum += cluster.map_shared_rank(&sh, r)->cta_cbo;
                out->lcom = n ? __ddiv_rn(sl, (double)n) : 0.0;
                double mc;
                if (csum < (1ull << 53)) {
                    mc = n ? __ddiv_rn((double)csum, (double)n) : 0.0;
                } else {
                    double sc = 0.0;
                    for (uint32_t i = 0; i < n; ++i) sc = __dadd_rn(sc, cbo ? (double)cbo[i] : 0.0);
                    mc = n ? __ddiv_rn(sc, (double)n) : 0.0;
                }
                out->cbo = mc;
                out->fast_path_ok = 0;
            }
        }
        cluster.sync();  // no CTA leaves while its shared memory may still be read
        return;
    }
    const u128 P_my = cta_prefix + ex_blk;
    // ---- (2) binade segments and per-chunk functions
    const int e_prev = my == 0 ? -1 : gran_exp(P_my);
    const bool has_start = cnt > 0 && gran_exp(P_my + S) != e_prev;
    Fn agg = fn_id();
    if (cnt > 0 && !has_start) {
        for (uint32_t j = 0; j < cnt; ++j) {
            uint64_t X;
            lcom_units(vals[lo + j], X);
            agg = compose(agg, fn_elem(X, e_prev));
        }
    } else if (has_start) {
        u128 P = P_my;
        int ep = e_prev;
        for (uint32_t j = 0; j < cnt; ++j) {
            uint64_t X;
            lcom_units(vals[lo + j], X);
            P += X;
            const int e = gran_exp(P);
            if (e != ep) {
                agg = fn_id();
                agg.bits |= 4u;
            } else {
                const uint32_t fl = agg.bits & 4u;
                agg = compose(agg, fn_elem(X, e));
                agg.bits |= fl;
            }
            ep = e;
        }
    }
    const Fn ex_fn = blk1k_excl_fn(agg, sh);
    if (t == kBT - 1) sh.cta_agg = seg_combine(ex_fn, agg);
    cluster.sync();
    Fn cta_in = fn_id();
    for (int r = 0; r < rank; ++r) cta_in = seg_combine(cta_in, cluster.map_shared_rank(&sh, r)->cta_agg);
    // the function since the last segment start before this chunk
    const Fn excl = seg_combine(cta_in, ex_fn);
    if (has_start) {  // record starts with the function of the segment each closes
        Fn run = excl;
        u128 P = P_my;
        int ep = e_prev;
        for (uint32_t j = 0; j < cnt; ++j) {
            uint64_t X;
            lcom_units(vals[lo + j], X);
            P += X;
            const int e = gran_exp(P);
            if (e != ep) {
                const int k = atomicAdd(&sh.n_segs, 1);
                if (k < kMaxSegs) {
                    sh.seg_pos[k] = my + j; sh.seg_e[k] = e; sh.seg_x[k] = X; sh.seg_close[k] = run;
                } else {
                    sh.bad = 1;
                }
                run = fn_id();
            } else {
                run = compose(run, fn_elem(X, e));
            }
            ep = e;
        }
        if (my + cnt == n) { sh.final_total = run; sh.has_final = 1; }
    } else if (cnt > 0 && my + cnt == n) {
        sh.final_total = compose(excl, agg);
        sh.has_final = 1;
    }
    cluster.sync();
    if (rank == 0 && warp == 0) {
        // chain every segment, in position order, from S_0 = 0. The segment
        // lists of the 8 CTAs are gathered over the lanes (independent remote
        // reads instead of one dependent chain of them), ordered by position
        // with a rank count, then chained by lane 0 (local arithmetic only).
        int ns = 0, rbad = 0, rfin = 0;
        if (lane < kCC) {
            ClusterShared* o = cluster.map_shared_rank(&sh, lane);
            ns = o->n_segs;
            rbad = o->bad;
            rfin = o->has_final;
        }
        int bad_seg = __reduce_or_sync(0xffffffffu, rbad | (ns > kMaxSegs ? 1 : 0));
        ns = min(ns, kMaxSegs);
        int incl = ns;
#pragma unroll
        for (int d = 1; d < kCC; d <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, d);
            if (lane >= d) incl += y;
        }
        const int K = __shfl_sync(0xffffffffu, incl, kCC - 1);
        if (K > kMaxSegs) bad_seg = 1;
        const int Kc = min(K, kMaxSegs);
        const int fin_rank = __ffs(__ballot_sync(0xffffffffu, lane < kCC && rfin)) - 1;
        // gathered (unsorted) entries in this CTA's g_* arrays; g_end[k+1] / g_first[k] reused below
        int inc_r[kCC];
#pragma unroll
        for (int q = 0; q < kCC; ++q) inc_r[q] = __shfl_sync(0xffffffffu, incl, q);
        for (int idx = lane; idx < Kc; idx += 32) {
            int r = 0, before = 0;
#pragma unroll
            for (int q = 0; q < kCC - 1; ++q)
                if (idx >= inc_r[q]) { r = q + 1; before = inc_r[q]; }
            ClusterShared* o = cluster.map_shared_rank(&sh, r);
            const int a = idx - before;
            sh.seg_pos_all[idx] = o->seg_pos[a];
            sh.seg_e_all[idx] = o->seg_e[a];
            sh.seg_x_all[idx] = o->seg_x[a];
            sh.seg_close_all[idx] = o->seg_close[a];
        }
        __syncwarp();
        // position order (positions are distinct): rank of each entry
        for (int idx = lane; idx < Kc; idx += 32) {
            const uint32_t p = sh.seg_pos_all[idx];
            int rk = 0;
            for (int j = 0; j < Kc; ++j) rk += sh.seg_pos_all[j] < p;
            sh.g_pos[rk] = p;
            sh.g_e[rk] = sh.seg_e_all[idx];
            sh.g_x[rk] = sh.seg_x_all[idx];
            sh.g_close[rk] = sh.seg_close_all[idx];
        }
        Fn fin = fn_id();
        if (fin_rank >= 0 && lane == 0) fin = cluster.map_shared_rank(&sh, fin_rank)->final_total;
        __syncwarp();
        if (lane == 0) {
            u128 T = 0;
            sh.g_end[0] = T;
            for (int k = 0; k < Kc; ++k) {
                const Fn tot = k + 1 < Kc ? sh.g_close[k + 1] : fin;  // segment k closes at start k+1 (or the end)
                const int e = sh.g_e[k];
                T = rne53(T + sh.g_x[k]);
                sh.g_first[k] = T;
                T += (u128)finc(tot, (int)((T >> e) & 1)) << e;
                sh.g_end[k + 1] = T;
            }
            sh.g_n = Kc;
            sh.bad = bad_seg;
        }
    }
    cluster.sync();
    if (rank != 0) {  // the chained table into this CTA's shared memory (one remote read each)
        ClusterShared* z = cluster.map_shared_rank(&sh, 0);
        const int K0 = z->g_n;
        if (t == 0) sh.g_n = K0;
        for (int k = t; k < K0; k += kBT) {
            sh.g_pos[k] = z->g_pos[k];
            sh.g_e[k] = z->g_e[k];
            sh.g_first[k] = z->g_first[k];
            sh.g_end[k + 1] = z->g_end[k + 1];
        }
        __syncthreads();
    }
    const int K = sh.g_n;
    int kb = -1;
    for (int k = 0; k < K; ++k)
        if (sh.g_pos[k] < my) kb = k;
    u128 S0 = 0;
    if (cnt > 0) {
        if (has_start && kb + 1 < K && sh.g_pos[kb + 1] == my) {
            S0 = sh.g_end[kb + 1];
        } else if (kb >= 0) {
            const int e = sh.g_e[kb];
            const u128 F = sh.g_first[kb];
            S0 = F + ((u128)finc(excl, (int)((F >> e) & 1)) << e);
        }
    }
    const double s0 = u128_to_double(S0);
    sh.start[t] = s0;
    cluster.sync();
    // ---- (3) exact replay in IEEE doubles from shared memory; every join must hold
    double sv = s0;
    for (uint32_t j = 0; j < cnt; ++j) sv = __dadd_rn(sv, vals[lo + j]);
    int jb = 0;
    if (cnt > 0 && my + cnt < n) {
        const double next = t + 1 < kBT ? sh.start[t + 1] : cluster.map_shared_rank(&sh, rank + 1)->start[0];
        if (next != sv) jb = 1;
    }
    if (my == 0 && cnt > 0 && s0 != 0.0) jb = 1;
    if (cnt > 0 && my + cnt == n) sh.final_sum = sv;
    jb = __syncthreads_or(jb);
    if (t == 0) sh.bad |= jb;
    cluster.sync();
    if (rank == 0 && t == 0) {
        int b = 0;
        unsigned long long csum = 0;
        double sum = 0.0;
        for (int r = 0; r < kCC; ++r) {
            ClusterShared* o = cluster.map_shared_rank(&sh, r);
            b |= o->bad;
            csum += o->cta_cbo;
            if (o->has_final) sum = o->final_sum;
        }
        double ml;
        uint32_t fast = 1;
        if (b) {
            fast = 0;
            double sl = 0.0;
            for (uint32_t i = 0; i < n; ++i) sl = __dadd_rn(sl, lcom[i]);
            ml = n ? __ddiv_rn(sl, (double)n) : 0.0;
        } else {
            ml = n ? __ddiv_rn(sum, (double)n) : 0.0;
        }
        double mc;
        if (csum < (1ull << 53)) {
            mc = n ? __ddiv_rn((double)csum, (double)n) : 0.0;
        } else {
            fast = 0;
            double sc = 0.0;
            for (uint32_t i = 0; i < n; ++i) sc = __dadd_rn(sc, cbo ? (double)cbo[i] : 0.0);
            mc = n ? __ddiv_rn(sc, (double)n) : 0.0;
        }
        out->lcom = ml;
        out->cbo = mc;
        out->fast_path_ok = fast;
    }
    cluster.sync();  // CTA 0 read the others' shared memory: keep them resident until here
}

// Serial fallback kernel (n too large for one co-resident tile per CTA).
// The sequential sums literally, by one warp: each 32-element chunk is loaded
// coalesced, then every lane runs the same left-to-right chain over the
// shuffled values (loads and shuffles stay off the dependent add chain).
// Exact for any input; used for small n (faster than the cooperative kernel's
// grid syncs below ~16k classes) and as the fallback.
__global__ void k_thresholds_serial(const double* __restrict__ lcom, const uint32_t* __restrict__ cbo, uint32_t n,
                                    DevThresholds* __restrict__ out) {
    if (blockIdx.x != 0) return;
    const int lane = threadIdx.x & 31;
    double sl = 0.0, sc = 0.0;
    for (uint32_t b = 0; b < n; b += 32) {
        const uint32_t i = b + lane;
        const double v = i < n ? lcom[i] : 0.0;
        const double w = (i < n && cbo) ? (double)cbo[i] : 0.0;
        const uint32_t m = min(32u, n - b);
#pragma unroll 8
        for (uint32_t k = 0; k < m; ++k) {
            sl = __dadd_rn(sl, __shfl_sync(0xffffffffu, v, k));
            sc = __dadd_rn(sc, __shfl_sync(0xffffffffu, w, k));
        }
    }
    if (lane == 0) {
        out->lcom = n ? __ddiv_rn(sl, (double)n) : 0.0;
        out->cbo = n ? __ddiv_rn(sc, (double)n) : 0.0;
        out->fast_path_ok = 0;
    }
}

}  // namespace

constexpr int kMaxDevices = 64;

bool getenv_flag(const char* name) {
    const char* v = std::getenv(name);
    return v && v[0] == '1';
}
constexpr uint32_t kSerialMax = 2048;  // below this one warp's serial chain beats three grid syncs (measured)

size_t thresholds_scratch_bytes(uint32_t n) {
    const size_t tiles = (n + kTile - 1) / kTile;
    return tiles * (3 * sizeof(u128) + kSlot * sizeof(Piece) + sizeof(int)) + 64;
}

cudaError_t launch_thresholds(const double* lcom, const uint32_t* cbo, uint32_t n, DevThresholds* out,
                              void* scratch, size_t scratch_bytes, cudaStream_t st, bool allow_serial) {
    const uint32_t tiles = (n + kTile - 1) / kTile;
    // co-resident CTA bound of the current device (per device: contexts on
    // several GPUs may be driven from several host threads)
    static std::atomic<int> coresident[kMaxDevices];
    int dev = 0;
    cudaGetDevice(&dev);
    int max_coresident = dev < kMaxDevices ? coresident[dev].load(std::memory_order_relaxed) : 0;
    if (max_coresident <= 0) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_thresholds_coop, kTT, 0);
        max_coresident = sms * per_sm;
        if (dev < kMaxDevices) coresident[dev].store(max_coresident, std::memory_order_relaxed);
    }
    if (n == 0 || (allow_serial && n <= kSerialMax)) {
        k_thresholds_serial<<<1, 32, 0, st>>>(lcom, cbo, n, out);
        return cudaGetLastError();
    }
    if (n <= kClusterMax && !getenv_flag("MMGPU_THR_BLOCK")) {  // 8 CTAs of one cluster, values in shared memory
        const uint32_t E = (n + kCC * kBT - 1) / (kCC * kBT);
        const size_t dyn = (sizeof(double) + sizeof(uint32_t)) * kBT * E;
        static std::atomic<size_t> configured[kMaxDevices];
        if (dev < kMaxDevices && configured[dev].load(std::memory_order_relaxed) < dyn) {
            const cudaError_t e = cudaFuncSetAttribute(k_thresholds_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       (int)((sizeof(double) + sizeof(uint32_t)) * kBT * kCPer));
            if (e != cudaSuccess) return e;
            configured[dev].store((sizeof(double) + sizeof(uint32_t)) * kBT * kCPer, std::memory_order_relaxed);
        }
        k_thresholds_cluster<<<kCC, kBT, dyn, st>>>(lcom, cbo, n, out);
        return cudaGetLastError();
    }
    if (n <= kBlockMax) {  // one CTA, no grid syncs
        k_thresholds_block<<<1, kBT, 0, st>>>(lcom, cbo, n, out);
        return cudaGetLastError();
    }
    if (tiles > (uint32_t)max_coresident || scratch_bytes < thresholds_scratch_bytes(n)) {
        k_thresholds_serial<<<1, 32, 0, st>>>(lcom, cbo, n, out);
        return cudaGetLastError();
    }
    char* p = static_cast<char*>(scratch);
    Scratch g;
    g.tile_sum = reinterpret_cast<u128*>(p);
    g.tile_entry = g.tile_sum + tiles;
    g.tile_exit = g.tile_entry + tiles;
    g.pieces = reinterpret_cast<Piece*>(g.tile_exit + tiles);
    g.n_pieces = reinterpret_cast<int*>(g.pieces + (size_t)tiles * kSlot);
    g.cbo_sum = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(g.n_pieces + tiles) + 15) & ~uintptr_t(15));
    g.bad = reinterpret_cast<int*>(g.cbo_sum + 1);
    cudaMemsetAsync(g.cbo_sum, 0, 16, st);
    void* args[] = {(void*)&lcom, (void*)&cbo, (void*)&n, (void*)&g, (void*)&out};
    return cudaLaunchCooperativeKernel((const void*)k_thresholds_coop, dim3(tiles), dim3(kTT), args, 0, st);
}

}  // namespace mmg
