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
// The division is the reference's single IEEE division (similarity_if_nonzero,
// metrics.hpp:47-55), so every value is bit-identical.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

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
    uint32_t* err;            // bit 1: a row beyond the wide buffer
    unsigned long long* total;  // pass 0: Σ pairs (u32 row offsets need it < 2^32)
};

// One row: gather its candidates j > i into buf (flattened over the row's
// properties), sort, run-length encode; pass 0 counts, pass 1 writes.
// Returns false when the candidate list exceeds cap.
template <int PASS>
__device__ __forceinline__ bool sim_row(const SimArgs& a, uint32_t i, uint32_t* buf, uint32_t* pre, uint32_t cap,
                                        uint32_t pre_cap, int lane) {
    const DevModel& s = a.s;
    const uint32_t cb = s.call_off[i], nc = s.call_off[i + 1] - cb;
    const uint32_t ab = s.acc_off[i], na = s.acc_off[i + 1] - ab;
    const uint32_t np = nc + na;
    // user-list sizes of the row's properties, prefix-summed into pre[]
    uint32_t total = 0;
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
        if (p < np && p < pre_cap) pre[p] = total + x - sz;
        total += __shfl_sync(0xffffffffu, x, 31);
    }
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
        if (!sim_row<PASS>(a, i, s_buf[warp], s_pre[warp], kWideCap, kWidePre, lane)) {
            if (lane == 0) {
                atomicOr(a.err, 2u);
                if (!PASS) a.row_cnt[i] = 0;
            }
        }
        __syncwarp();
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
                                   uint32_t* err, unsigned long long* total, cudaStream_t st) {
    if (!s.M) return cudaSuccess;
    SimArgs a{s, uc_off, uc, ua_off, ua, row_cnt, row_off, out, wide_list, n_wide, err, total};
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

cudaError_t launch_scan(const uint32_t* in, uint32_t* out, uint32_t n, uint32_t* totals, uint32_t* grand,
                        cudaStream_t st) {
    scan_exclusive(in, out, n, totals, grand, st);
    return cudaGetLastError();
}

}  // namespace mmg
