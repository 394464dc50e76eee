// k_ck_mma.cu — LCOM-CK of dense classes on the 5th-generation tensor cores.
//
// LCOM-CK needs Q = #pairs (i < j) of members whose own-attribute sets
// intersect (metrics.hpp:135-157). For a class with A ≤ 64 attributes the
// sets are the method pass's u64 masks; with B the M×64 0/1 matrix of those
// masks, |own_i ∩ own_j| = (B·Bᵀ)[i][j], so Q = #{i < j : (B·Bᵀ)[i][j] > 0}.
// The popc path (k_class_large) tests every pair with a 64-bit AND; here one
// elected thread issues `tcgen05.mma.kind::i8` (u8 × u8 → s32, exact) on
// 128×128 tiles of the upper triangle, the accumulator lives in TMEM, and the
// four warps read it back with `tcgen05.ld` and count the nonzero entries.
// Integer counts, so the result is the reference's integer bit for bit.
//
// Shared-memory operand layout (no swizzle, K-major "core matrices" of 8 rows
// × 16 bytes): byte (r, k) sits at (r / 8)·512 + (k / 16)·128 + (r % 8)·16 +
// k % 16 — LBO = 128 B between the K-adjacent core matrices, SBO = 512 B
// between 8-row groups (descriptor fields per cute/arch/mma_sm100_desc.hpp).
#include <cuda_runtime.h>

#include <atomic>

#include <cstdint>

#include "mm_device.cuh"
#include "mm_kernels.h"

namespace mmg {
namespace {

constexpr uint32_t kTile = 128;         // UMMA M = N
constexpr uint32_t kRowBytes = 64;      // K = 64 attributes, one byte each
constexpr uint32_t kSBO = 512;          // bytes between 8-row core-matrix groups
constexpr uint32_t kLBO = 128;          // bytes between K-adjacent core matrices
constexpr uint32_t kTmemCols = 128;     // one 128×128 s32 accumulator

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor, SWIZZLE_NONE, K-major, version 1 (sm_100)
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);            // start address, bits [0,14)
    d |= (uint64_t)((kLBO >> 4) & 0x3FFFu) << 16;       // leading byte offset, bits [16,30)
    d |= (uint64_t)((kSBO >> 4) & 0x3FFFu) << 32;       // stride byte offset, bits [32,46)
    d |= (uint64_t)1 << 46;                              // version, bits [46,48)
    // base offset [49,52) = 0, LBO mode bit 52 = 0, layout type [61,64) = 0 (no swizzle)
    return d;
}

// instruction descriptor, kind::i8: D = s32, A = B = unsigned 8-bit, both
// K-major, N = 128, M = 128
constexpr uint32_t kIdesc = (2u << 4)            // D format s32, bits [4,6)
                          | (0u << 7)            // A format u8, bits [7,10)
                          | (0u << 10)           // B format u8, bits [10,13)
                          | ((kTile >> 3) << 17)  // N >> 3, bits [17,23)
                          | ((kTile >> 4) << 24); // M >> 4, bits [24,29)

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t"
        "}\n" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}

__device__ __forceinline__ void commit_to(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}

// bounded: a commit that never arrives traps (a launch error) instead of hanging the GPU
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t parity) {
    for (uint32_t spin = 0;; ++spin) {
        uint32_t done;
        asm volatile(
            "{\n\t"
            ".reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t"
            "}\n"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
        if (done) return;
        if (spin > (1u << 26)) __trap();
    }
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// one CTA (8 warps) per listed class; dynamic shared memory = M_pad × 64 B.
// Warp w drains TMEM lane quarter w % 4, column half w / 4.
__global__ void __launch_bounds__(256) k_ck_mma(DevModel s, const uint32_t* __restrict__ list,
                                                const uint64_t* __restrict__ own_mask,
                                                uint64_t* __restrict__ ck_out) {
    extern __shared__ __align__(1024) unsigned char opnd[];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_red[8];
    const uint32_t c = list[blockIdx.x];
    const uint32_t mb = s.cls_moff[c];
    const uint32_t M = s.cls_moff[c + 1] - mb;
    const uint32_t T = (M + kTile - 1) / kTile;  // 128-row tiles
    const uint32_t rows = T * kTile;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {  // TMEM: one 128-column accumulator
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    // B (rows × 64 u8 in {0,1}) from the masks, 16 bytes (one core-matrix row) per step
    for (uint32_t q = threadIdx.x; q < rows * 4; q += blockDim.x) {
        const uint32_t r = q >> 2, kc = q & 3;
        const uint32_t bits = r < M ? (uint32_t)(__ldg(own_mask + mb + r) >> (16 * kc)) & 0xFFFFu : 0u;
        uint4 w;
        w.x = ((bits & 0xFu) * 0x00204081u) & 0x01010101u;  // nibble -> 4 bytes of 0/1
        w.y = (((bits >> 4) & 0xFu) * 0x00204081u) & 0x01010101u;
        w.z = (((bits >> 8) & 0xFu) * 0x00204081u) & 0x01010101u;
        w.w = (((bits >> 12) & 0xFu) * 0x00204081u) & 0x01010101u;
        *reinterpret_cast<uint4*>(opnd + (r >> 3) * kSBO + kc * kLBO + (r & 7) * 16) = w;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    const uint32_t base = smem_u32(opnd);
    const uint32_t bar = smem_u32(&s_bar);

    uint32_t q = 0, parity = 0;
    for (uint32_t I = 0; I < T; ++I)
        for (uint32_t J = I; J < T; ++J) {
            if (threadIdx.x == 0) {
                // K = 64 as two K = 32 steps (two core matrices each)
                for (uint32_t k = 0; k < 2; ++k) {
                    const uint64_t da = smem_desc(base + I * (kTile / 8) * kSBO + k * 2 * kLBO);
                    const uint64_t db = smem_desc(base + J * (kTile / 8) * kSBO + k * 2 * kLBO);
                    mma_i8(tmem, da, db, k);
                }
                commit_to(bar);
            }
            wait_parity(bar, parity);
            parity ^= 1u;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // warp w reads accumulator rows 32w..32w+31 (its TMEM lane quarter);
            // off-diagonal tiles have j > i everywhere, so only the last tile's
            // padding columns need a bound
            const uint32_t quarter = warp & 3, half = warp >> 2;
            const uint32_t il = 32 * quarter + lane;  // row inside the tile
            const uint32_t i = I * kTile + il;
            const uint32_t jlim = min(kTile, M - J * kTile);  // valid columns of this tile
            uint32_t qt = 0;
            for (uint32_t c0 = half * (kTile / 2); c0 < (half + 1) * (kTile / 2); c0 += 32) {
                // diagonal tile: columns left of this warp's rows lie below the diagonal
                // (warp-uniform: the chunk is 32 columns, the rows 32 lanes)
                if (I == J && c0 + 32 <= 32 * quarter) continue;
                uint32_t v[32];
                tmem_ld32(tmem + ((32u * quarter) << 16) + c0, v);
                // every entry of the chunk counts: inside the valid columns and, on a
                // diagonal tile, right of all of this warp's rows (warp-uniform)
                if (c0 + 32 <= jlim && (I != J || c0 >= 32 * (quarter + 1))) {
                    // nonzero count as Σ min(v, 1): two IMNMX and one IADD3 per pair of
                    // entries instead of a compare and an add per entry
#pragma unroll
                    for (int t = 0; t < 32; t += 2) {
                        uint32_t a, b;  // (PTX min: kept as IMNMX, not re-derived into compares)
                        asm("min.u32 %0, %1, 1;" : "=r"(a) : "r"(v[t]));
                        asm("min.u32 %0, %1, 1;" : "=r"(b) : "r"(v[t + 1]));
                        qt += a + b;
                    }
                } else {
                    // this lane's valid columns t ∈ [lo, hi): j < jlim and, on a diagonal
                    // tile, j > i; the nonzero pattern as a bit mask (IMNMX + LEA per
                    // entry), counted once
                    const uint32_t lo = (I == J) ? min(max(il + 1, c0) - c0, 32u) : 0u;
                    const uint32_t hi = jlim > c0 ? min(jlim - c0, 32u) : 0u;
                    const uint32_t keep = (hi >= 32 ? 0xffffffffu : ((1u << hi) - 1u)) & ~((lo >= 32) ? 0xffffffffu : ((1u << lo) - 1u));
                    uint32_t nz = 0;
#pragma unroll
                    for (int t = 0; t < 32; ++t) {
                        uint32_t a;
                        asm("min.u32 %0, %1, 1;" : "=r"(a) : "r"(v[t]));
                        nz += a << t;
                    }
                    qt += __popc(nz & keep);
                }
            }
            q += i < M ? qt : 0u;
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncthreads();  // accumulator drained before the next tile overwrites it
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
    const uint32_t wq = __reduce_add_sync(0xffffffffu, q);
    if (lane == 0) s_red[warp] = wq;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t Q = 0;
        for (int w = 0; w < 8; ++w) Q += s_red[w];
        const uint64_t P = (uint64_t)M * (M - 1) / 2 - Q;
        ck_out[c] = P > Q ? P - Q : 0;  // metrics.hpp:147-156
    }
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

}  // namespace

uint32_t ck_mma_smem_bytes(uint32_t max_members) {
    return ((max_members + kTile - 1) / kTile) * kTile * kRowBytes;
}

// The attribute belongs to the function, process-wide, not to a context: a
// later upload of a smaller system (another engine, another thread) must not
// lower it under a launch planned with more. Raised only, never lowered.
cudaError_t set_ck_mma_smem(uint32_t bytes) {
    static std::atomic<int> granted{0};
    int cur = granted.load(std::memory_order_relaxed);
    while ((int)bytes > cur) {
        const cudaError_t e = cudaFuncSetAttribute(k_ck_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        if (e != cudaSuccess) return e;
        if (granted.compare_exchange_weak(cur, (int)bytes, std::memory_order_relaxed)) break;
    }
    return cudaSuccess;
}

void launch_ck_mma(const DevModel& s, const uint32_t* list, uint32_t n, uint32_t smem_bytes,
                   const uint64_t* own_mask, uint64_t* ck, cudaStream_t st) {
    if (!n) return;
    k_ck_mma<<<n, 256, smem_bytes, st>>>(s, list, own_mask, ck);
}

}  // namespace mmg
