// k_similarity.cu — the sparse similarity table (all_similarities,
// metrics.hpp:39-77; parallel_similarities, parallel.hpp:71-121).
//
// A pair (i, j) shares a property exactly when some call target or accessed
// attribute of i is also one of j's, and |P_i ∩ P_j| counts those shared
// properties (calls and accesses are separate id spaces, lists unique). So
// the row of method i is the multiset ⋃_{t ∈ props(i)} users(t) restricted to
// j > i: its distinct j are the stored pairs, their multiplicities the
// intersections — an A·Aᵀ over the method × property incidence, done sparse:
//   1. inverted indices users_c[t] (callers of t) and users_a[a] (accessors
//      of a) by counting, scan and scatter;
//   2. one warp per row gathers the row's candidate list from the inverted
//      lists (flattened over lanes: one memory round trip per 32 candidates),
//      sorts it in shared memory and run-length encodes it;
//   3. pass 0 stores the row's pair count, a scan gives the row offsets, pass
//      1 writes (i, j, inter / (|P_i| + |P_j| − inter)) in j order — the
//      output is already sorted by (first, second), no global sort.
// Rows too long for a warp's shared-memory buffer (> 4096 candidates or
// > 1024 properties: hub methods, attributes with thousands of users) take
// the huge-row path: one CTA per row gathers the candidates into global
// scratch, a segmented radix sort (CUB) orders each row, one CTA per row
// run-length encodes it — in batches bounded by the scratch, so any row
// length works (all_similarities has no bound, metrics.hpp:67-77).
// The division is the reference's single IEEE division (similarity_if_nonzero,
// metrics.hpp:47-55), so every value is bit-identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cub/device/device_segmented_sort.cuh>

#include "mm_device.cuh"
#include "mm_kernels.h"

namespace mmg {
namespace {

constexpr uint32_t kScanBlock = 1024;

__global__ void k_count_users(const uint32_t* __restrict__ tgt, uint64_t n, uint32_t* __restrict__ cnt) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(cnt + tgt[e], 1u);
}

// exclusive scan, three launches: block scans + block totals, scan of the
// totals (one block), block offsets added back
__global__ void __launch_bounds__(kScanBlock) k_scan_blocks(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                                            uint32_t n, uint32_t* __restrict__ totals) {
    __shared__ uint32_t s_w[32];
    const uint32_t i = blockIdx.x * kScanBlock + threadIdx.x;
    const uint32_t v = i < n ? in[i] : 0u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = s_w[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
            if (lane >= d) w += y;
        }
        s_w[lane] = w;
    }
    __syncthreads();
    const uint32_t incl = x + (warp ? s_w[warp - 1] : 0u);
    if (i < n) out[i] = incl - v;
    if (threadIdx.x == kScanBlock - 1) totals[blockIdx.x] = incl;
}

__global__ void __launch_bounds__(1024) k_scan_totals(uint32_t* __restrict__ totals, uint32_t nb,
                                                      uint32_t* __restrict__ grand) {
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_carry;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nb; b0 += 1024) {
        const uint32_t i = b0 + threadIdx.x;
        const uint32_t v = i < nb ? totals[i] : 0u;
        uint32_t x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (lane == 31) s_w[warp] = x;
        __syncthreads();
        if (warp == 0) {
            uint32_t w = s_w[lane];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += y;
            }
            s_w[lane] = w;
        }
        __syncthreads();
        const uint32_t carry = s_carry;
        const uint32_t incl = x + (warp ? s_w[warp - 1] : 0u);
        if (i < nb) totals[i] = carry + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *grand = s_carry;
}

__global__ void k_scan_add(uint32_t* __restrict__ out, uint32_t n, const uint32_t* __restrict__ totals) {
    const uint32_t i = blockIdx.x * kScanBlock + threadIdx.x;
    if (i < n) out[i] += totals[blockIdx.x];
}

// users[cur[t]++] = q for every edge q -> t (order inside a list is free:
// rows are sorted after the gather)
__global__ void k_fill_users(const uint32_t* __restrict__ off, const uint32_t* __restrict__ tgt, uint32_t M,
                             uint32_t* __restrict__ cur, uint32_t* __restrict__ users) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= M) return;
    for (uint32_t e = off[q]; e < off[q + 1]; ++e) users[atomicAdd(cur + tgt[e], 1u)] = q;
}

__device__ __forceinline__ void warp_sort(uint32_t* buf, uint32_t N, int lane) {
    for (uint32_t k = 2; k <= N; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = lane; i < N; i += 32) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const uint32_t a = buf[i], b = buf[ixj];
                    if ((a > b) == ((i & k) == 0)) { buf[i] = b; buf[ixj] = a; }
                }
            }
            __syncwarp();
        }
}

struct SimArgs {
    DevModel s;
    const uint32_t* uc_off;  // callers of each method (M + 1)
    const uint32_t* uc;
    const uint32_t* ua_off;  // accessors of each attribute (A + 1)
    const uint32_t* ua;
    uint32_t* row_cnt;        // pass 0 output: pairs per row (kNone: row deferred to the wide kernel)
    const uint32_t* row_off;  // pass 1 input: first pair of each row
    mm_similarity* out;
    uint32_t* wide_list;      // rows whose candidate list exceeds the narrow buffer
    uint32_t* n_wide;
    uint32_t* err;            // reserved
    unsigned long long* total;  // pass 0: Σ pairs (u32 row offsets need it < 2^32)
    uint32_t* huge_list;      // rows beyond the wide buffer (huge-row path)
    unsigned long long* huge_tot;  // their candidate counts
    uint32_t* n_huge;
};

// One row: gather its candidates j > i into buf (flattened over the row's
// properties), sort, run-length encode; pass 0 counts, pass 1 writes.
// Returns false when the candidate list exceeds cap.
template <int PASS>
__device__ __forceinline__ bool sim_row(const SimArgs& a, uint32_t i, uint32_t* buf, uint32_t* pre, uint32_t cap,
                                        uint32_t pre_cap, int lane, unsigned long long* total_out = nullptr) {
    const DevModel& s = a.s;
    const uint32_t cb = s.call_off[i], nc = s.call_off[i + 1] - cb;
    const uint32_t ab = s.acc_off[i], na = s.acc_off[i + 1] - ab;
    const uint32_t np = nc + na;
    // user-list sizes of the row's properties, prefix-summed into pre[]
    unsigned long long total = 0;
    for (uint32_t p0 = 0; p0 < np; p0 += 32) {
        const uint32_t p = p0 + lane;
        uint32_t sz = 0;
        if (p < np) {
            if (p < nc) {
                const uint32_t t = s.call_tgt[cb + p];
                sz = a.uc_off[t + 1] - a.uc_off[t];
            } else {
                const uint32_t t = s.acc_tgt[ab + (p - nc)];
                sz = a.ua_off[t + 1] - a.ua_off[t];
            }
        }
        uint32_t x = sz;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += y;
        }
        if (p < np && p < pre_cap) pre[p] = (uint32_t)(total + x - sz);
        total += __shfl_sync(0xffffffffu, x, 31);
    }
    if (total_out) *total_out = total;
    if (total > cap || np > pre_cap) return false;
    __syncwarp();
    // candidates j > i (the row's own id never qualifies)
    uint32_t n = 0;
    for (uint32_t k0 = 0; k0 < total; k0 += 32) {
        const uint32_t k = k0 + lane;
        uint32_t j = kNone;
        if (k < total) {
            uint32_t lo = 0, hi = np;  // last property with pre <= k
            while (lo + 1 < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (pre[mid] <= k) lo = mid;
                else hi = mid;
            }
            const uint32_t r = k - pre[lo];
            j = lo < nc ? a.uc[a.uc_off[s.call_tgt[cb + lo]] + r] : a.ua[a.ua_off[s.acc_tgt[ab + (lo - nc)]] + r];
        }
        const bool keep = k < total && j > i && j != kNone;
        const uint32_t b = __ballot_sync(0xffffffffu, keep);
        if (keep) buf[n + __popc(b & ((1u << lane) - 1))] = j;
        n += __popc(b);
    }
    __syncwarp();
    uint32_t N = 1;
    while (N < n) N <<= 1;
    for (uint32_t k = n + lane; k < N; k += 32) buf[k] = kNone;
    __syncwarp();
    if (N > 1) warp_sort(buf, N, lane);
    // run heads = distinct j; run length = |P_i ∩ P_j|
    uint32_t pairs = 0;
    const uint32_t base = PASS ? a.row_off[i] : 0u;
    for (uint32_t k0 = 0; k0 < n; k0 += 32) {
        const uint32_t k = k0 + lane;
        const bool head = k < n && (k == 0 || buf[k] != buf[k - 1]);
        const uint32_t hb = __ballot_sync(0xffffffffu, head);
        if (PASS && head) {
            const uint32_t j = buf[k];
            uint32_t e = k + 1;
            while (e < n && buf[e] == j) ++e;
            const uint64_t inter = e - k;
            const uint64_t pj = (uint64_t)(s.call_off[j + 1] - s.call_off[j]) + (s.acc_off[j + 1] - s.acc_off[j]);
            const uint64_t uni = (uint64_t)np + pj - inter;
            mm_similarity r;
            r.first = i;
            r.second = j;
            r.value = __ddiv_rn((double)inter, (double)uni);  // similarity_if_nonzero, metrics.hpp:52-53
            a.out[base + pairs + __popc(hb & ((1u << lane) - 1))] = r;
        }
        pairs += __popc(hb);
    }
    if (!PASS && lane == 0) {
        a.row_cnt[i] = pairs;
        if (pairs) atomicAdd(a.total, (unsigned long long)pairs);
    }
    return true;
}

constexpr uint32_t kNarrowCap = 512;   // candidates per row in the narrow kernel (8 warps per block)
constexpr uint32_t kWideCap = 4096;    // wide kernel (2 warps per block)
constexpr uint32_t kWidePre = 1024;    // properties of one method in the wide kernel

template <int PASS>
__global__ void __launch_bounds__(256) k_sim_narrow(SimArgs a) {
    __shared__ uint32_t s_buf[8][kNarrowCap], s_pre[8][kNarrowCap];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t nw = gridDim.x * 8;
    for (uint32_t i = blockIdx.x * 8 + warp; i < a.s.M; i += nw) {
        if (PASS && a.row_cnt[i] == kNone) continue;  // the wide kernel's row
        if (!sim_row<PASS>(a, i, s_buf[warp], s_pre[warp], kNarrowCap, kNarrowCap, lane) && !PASS && lane == 0) {
            a.row_cnt[i] = kNone;
            a.wide_list[atomicAdd(a.n_wide, 1u)] = i;
        }
        __syncwarp();
    }
}

template <int PASS>
__global__ void __launch_bounds__(64) k_sim_wide(SimArgs a) {
    __shared__ uint32_t s_buf[2][kWideCap], s_pre[2][kWidePre];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n = *a.n_wide;
    for (uint32_t w = blockIdx.x * 2 + warp; w < n; w += gridDim.x * 2) {
        const uint32_t i = a.wide_list[w];
        unsigned long long tot = 0;
        if (!sim_row<PASS>(a, i, s_buf[warp], s_pre[warp], kWideCap, kWidePre, lane, &tot)) {
            if (lane == 0 && !PASS) {  // the huge-row path counts (and later writes) this row
                a.row_cnt[i] = 0;
                const uint32_t slot = atomicAdd(a.n_huge, 1u);
                a.huge_list[slot] = i;
                a.huge_tot[slot] = tot;
            }
        }
        __syncwarp();
    }
}

// ---- huge rows: global scratch + segmented sort --------------------------
constexpr int kHugeThreads = 256;

struct HugeArgs {
    DevModel s;
    const uint32_t* uc_off;
    const uint32_t* uc;
    const uint32_t* ua_off;
    const uint32_t* ua;
    const uint32_t* rows;  // batch: the rows
    const uint32_t* seg;   // batch: segment offsets (n_rows + 1)
    uint32_t* keys;        // gather output
    const uint32_t* sorted;  // sorted keys
    uint32_t* row_cnt;
    const uint32_t* row_off;
    mm_similarity* out;
    unsigned long long* total;
};

__device__ __forceinline__ uint32_t blk_excl_scan(uint32_t v, uint32_t* s_w, uint32_t* block_total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
    }
    if (lane == 31) s_w[warp] = x;
    __syncthreads();
    uint32_t pre = 0, all = 0;
    for (int w = 0; w < kHugeThreads / 32; ++w) {
        if (w < warp) pre += s_w[w];
        all += s_w[w];
    }
    __syncthreads();
    *block_total = all;
    return pre + x - v;
}

// One CTA per row: the candidates j (> i, else kNone) of the row's properties,
// in property order, into keys[seg[b] ...]
__global__ void __launch_bounds__(kHugeThreads) k_huge_gather(HugeArgs h) {
    __shared__ uint32_t s_w[kHugeThreads / 32];
    __shared__ uint32_t s_pre[kHugeThreads + 1];
    __shared__ uint32_t s_beg[kHugeThreads];
    const uint32_t b = blockIdx.x, i = h.rows[b];
    const DevModel& s = h.s;
    const uint32_t cb = s.call_off[i], nc = s.call_off[i + 1] - cb;
    const uint32_t ab = s.acc_off[i], np = nc + (s.acc_off[i + 1] - ab);
    uint64_t at = h.seg[b];
    for (uint32_t p0 = 0; p0 < np; p0 += kHugeThreads) {
        const uint32_t p = p0 + threadIdx.x;
        uint32_t sz = 0, beg = 0;
        if (p < np) {
            if (p < nc) {
                const uint32_t t = s.call_tgt[cb + p];
                beg = h.uc_off[t];
                sz = h.uc_off[t + 1] - beg;
            } else {
                const uint32_t t = s.acc_tgt[ab + (p - nc)];
                beg = h.ua_off[t] | 0x80000000u;  // accessor list (the id spaces differ)
                sz = h.ua_off[t + 1] - h.ua_off[t];
            }
        }
        uint32_t tot;
        const uint32_t ex = blk_excl_scan(sz, s_w, &tot);
        s_pre[threadIdx.x] = ex;
        s_beg[threadIdx.x] = beg;
        if (threadIdx.x == 0) s_pre[kHugeThreads] = tot;
        __syncthreads();
        const uint32_t n_here = min((uint32_t)kHugeThreads, np - p0);
        for (uint32_t k = threadIdx.x; k < tot; k += kHugeThreads) {
            uint32_t lo = 0, hi = n_here;  // last property with pre <= k
            while (lo + 1 < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (s_pre[mid] <= k) lo = mid;
                else hi = mid;
            }
            const uint32_t r = k - s_pre[lo], bg = s_beg[lo];
            const uint32_t j = (bg & 0x80000000u) ? h.ua[(bg & 0x7fffffffu) + r] : h.uc[bg + r];
            h.keys[at + k] = j > i ? j : kNone;
        }
        at += tot;
        __syncthreads();
    }
}

// One CTA per row over its sorted candidates: distinct j are the pairs, run
// lengths the intersections. Pass 0 counts, pass 1 writes in j order.
template <int PASS>
__global__ void __launch_bounds__(kHugeThreads) k_huge_rle(HugeArgs h) {
    __shared__ uint32_t s_w[kHugeThreads / 32];
    const uint32_t b = blockIdx.x, i = h.rows[b];
    const uint32_t* key = h.sorted + h.seg[b];
    const uint32_t n = h.seg[b + 1] - h.seg[b];
    const DevModel& s = h.s;
    const uint64_t np = (uint64_t)(s.call_off[i + 1] - s.call_off[i]) + (s.acc_off[i + 1] - s.acc_off[i]);
    uint32_t pairs = 0;
    const uint32_t base = PASS ? h.row_off[i] : 0u;
    for (uint32_t k0 = 0; k0 < n; k0 += kHugeThreads) {
        const uint32_t k = k0 + threadIdx.x;
        const uint32_t j = k < n ? key[k] : kNone;
        const bool head = j != kNone && (k == 0 || key[k - 1] != j);
        uint32_t tot;
        const uint32_t pos = blk_excl_scan(head ? 1u : 0u, s_w, &tot);
        if (PASS && head) {
            uint32_t e = k + 1;
            while (e < n && key[e] == j) ++e;
            const uint64_t inter = e - k;
            const uint64_t pj = (uint64_t)(s.call_off[j + 1] - s.call_off[j]) + (s.acc_off[j + 1] - s.acc_off[j]);
            mm_similarity r;
            r.first = i;
            r.second = j;
            r.value = __ddiv_rn((double)inter, (double)(np + pj - inter));  // metrics.hpp:52-53
            h.out[base + pairs + pos] = r;
        }
        pairs += tot;
    }
    if (!PASS && threadIdx.x == 0) {
        h.row_cnt[i] = pairs;
        if (pairs) atomicAdd(h.total, (unsigned long long)pairs);
    }
}

void scan_exclusive(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* totals, uint32_t* grand,
                    cudaStream_t st) {
    const uint32_t nb = (n + kScanBlock - 1) / kScanBlock;
    if (!nb) {
        cudaMemsetAsync(grand, 0, 4, st);
        return;
    }
    k_scan_blocks<<<nb, kScanBlock, 0, st>>>(in, out, n, totals);
    k_scan_totals<<<1, 1024, 0, st>>>(totals, nb, grand);
    k_scan_add<<<nb, kScanBlock, 0, st>>>(out, n, totals);
}

}  // namespace

cudaError_t launch_similarity_index(const DevModel& s, uint64_t Ec, uint64_t Ea, uint32_t* uc_off, uint32_t* uc,
                                    uint32_t* ua_off, uint32_t* ua, uint32_t* cur, uint32_t* totals,
                                    uint32_t* grand, cudaStream_t st) {
    const uint32_t grid = 148 * 8;
    cudaMemsetAsync(cur, 0, 4ull * (s.M + 1), st);
    if (Ec) k_count_users<<<grid, 256, 0, st>>>(s.call_tgt, Ec, cur);
    scan_exclusive(cur, uc_off, s.M + 1, totals, grand, st);
    cudaMemcpyAsync(cur, uc_off, 4ull * (s.M + 1), cudaMemcpyDeviceToDevice, st);
    if (s.M) k_fill_users<<<(s.M + 255) / 256, 256, 0, st>>>(s.call_off, s.call_tgt, s.M, cur, uc);
    cudaMemsetAsync(cur, 0, 4ull * (s.A + 1), st);
    if (Ea) k_count_users<<<grid, 256, 0, st>>>(s.acc_tgt, Ea, cur);
    scan_exclusive(cur, ua_off, s.A + 1, totals, grand, st);
    cudaMemcpyAsync(cur, ua_off, 4ull * (s.A + 1), cudaMemcpyDeviceToDevice, st);
    if (s.M) k_fill_users<<<(s.M + 255) / 256, 256, 0, st>>>(s.acc_off, s.acc_tgt, s.M, cur, ua);
    return cudaGetLastError();
}

cudaError_t launch_similarity_rows(const DevModel& s, int pass, const uint32_t* uc_off, const uint32_t* uc,
                                   const uint32_t* ua_off, const uint32_t* ua, uint32_t* row_cnt,
                                   const uint32_t* row_off, mm_similarity* out, uint32_t* wide_list, uint32_t* n_wide,
                                   uint32_t* err, unsigned long long* total, uint32_t* huge_list,
                                   unsigned long long* huge_tot, uint32_t* n_huge, cudaStream_t st) {
    if (!s.M) return cudaSuccess;
    SimArgs a{s, uc_off, uc, ua_off, ua, row_cnt, row_off, out, wide_list, n_wide, err, total, huge_list, huge_tot,
              n_huge};
    const uint32_t narrow = std::min<uint32_t>((s.M + 7) / 8, 148 * 16);
    if (pass == 0) {
        k_sim_narrow<0><<<narrow, 256, 0, st>>>(a);
        k_sim_wide<0><<<148 * 4, 64, 0, st>>>(a);
    } else {
        k_sim_narrow<1><<<narrow, 256, 0, st>>>(a);
        k_sim_wide<1><<<148 * 4, 64, 0, st>>>(a);
    }
    return cudaGetLastError();
}

size_t similarity_huge_temp_bytes(uint32_t max_items, uint32_t max_rows) {
    size_t bytes = 0;
    cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)max_items,
                                       (int)max_rows, (const uint32_t*)nullptr, (const uint32_t*)nullptr, 0);
    return bytes;
}

cudaError_t launch_similarity_huge(const DevModel& s, int pass, const uint32_t* uc_off, const uint32_t* uc,
                                   const uint32_t* ua_off, const uint32_t* ua, const uint32_t* rows, uint32_t n_rows,
                                   const uint32_t* seg, uint32_t n_items, uint32_t* keys, uint32_t* sorted,
                                   void* temp, size_t temp_bytes, uint32_t* row_cnt, const uint32_t* row_off,
                                   mm_similarity* out, unsigned long long* total, cudaStream_t st) {
    if (!n_rows) return cudaSuccess;
    HugeArgs h{s, uc_off, uc, ua_off, ua, rows, seg, keys, sorted, row_cnt, row_off, out, total};
    k_huge_gather<<<n_rows, kHugeThreads, 0, st>>>(h);
    size_t tb = temp_bytes;
    cudaError_t e = cub::DeviceSegmentedSort::SortKeys(temp, tb, keys, sorted, (int)n_items, (int)n_rows, seg,
                                                       seg + 1, st);
    if (e != cudaSuccess) return e;
    if (pass == 0) k_huge_rle<0><<<n_rows, kHugeThreads, 0, st>>>(h);
    else k_huge_rle<1><<<n_rows, kHugeThreads, 0, st>>>(h);
    return cudaGetLastError();
}

cudaError_t launch_scan(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* totals, uint32_t* grand,
                        cudaStream_t st) {
    scan_exclusive(in, out, n, totals, grand, st);
    return cudaGetLastError();
}

}  // namespace mmg
