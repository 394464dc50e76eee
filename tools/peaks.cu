// peaks.cu — measured integer peaks of this B200 for the roofline of the
// integer / tensor-core kernels ("report the fraction of the
// measured integer / int8-MMA peak" for the dense LCOM-CK configuration).
//
//   int32:  LOP3 + IMAD chains, 8 independent accumulators per thread, every
//           SM full: integer operations per second.
//   i8 MMA: tcgen05.mma.cta_group::1.kind::i8, M = 128, N = 256, K = 32 (u8 ×
//           u8 -> s32), issued back to back by one elected thread per CTA from
//           shared-memory operands into a TMEM accumulator, one CTA per SM:
//           dense int8 tensor operations per second (2 ops per MAC).
//
// Prints one JSON line. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -o tools/_build/peaks tools/peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::printf("{\"error\": \"%s at %s:%d\"}\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

constexpr int kIntIters = 4096;

__global__ void __launch_bounds__(1024) k_int32(uint32_t seed, uint32_t* out) {
    uint32_t a[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = seed ^ (threadIdx.x * 0x9E3779B1u + k);
    const uint32_t m = seed | 1u;
#pragma unroll 4
    for (int i = 0; i < kIntIters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t x;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(x) : "r"(a[k]), "r"(m), "r"(a[(k + 1) & 7]));
            a[k] = x * m + (uint32_t)k;  // IMAD
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) r ^= a[k];
    if (r == 0x12345678u) out[0] = r;  // keep the chains alive
}

// ---- tcgen05 kind::i8 ----
constexpr uint32_t kM = 128, kN = 256, kK = 32;
constexpr uint32_t kSBO = 256;  // 8 rows × 32 B (K = 32 u8: two 16-byte core matrices side by side)
constexpr uint32_t kLBO = 128;
constexpr uint32_t kIdesc = (2u << 4) | ((kN >> 3) << 17) | ((kM >> 4) << 24);  // s32 D, u8 A/B, K-major

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)((kLBO >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((kSBO >> 4) & 0x3FFFu) << 32) | ((uint64_t)1 << 46);
}

__global__ void __launch_bounds__(128) k_mma_i8(uint32_t iters, uint32_t* out) {
    __shared__ __align__(1024) unsigned char A[kM * kK];
    __shared__ __align__(1024) unsigned char B[kN * kK];
    __shared__ uint32_t s_tmem;
    __shared__ __align__(8) uint64_t bar;
    for (uint32_t i = threadIdx.x; i < kM * kK / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(A)[i] = 0x01010101u;
    for (uint32_t i = threadIdx.x; i < kN * kK / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(B)[i] = 0x01010101u;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                     "r"(256u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = s_tmem;
    if (threadIdx.x == 0) {
        const uint64_t da = sdesc(smem_u32(A)), db = sdesc(smem_u32(B));
        for (uint32_t i = 0; i < iters; ++i) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem),
                "l"(da), "l"(db), "r"(kIdesc), "r"(i), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         smem_u32(&bar))
                     : "memory");
    }
    if (threadIdx.x == 0) {
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}\n"
                         : "=r"(done)
                         : "r"(smem_u32(&bar))
                         : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x < 32) {
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (threadIdx.x == 0) out[blockIdx.x] = v;  // K·iters when every product is 1
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256u));
    }
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    uint32_t* out = nullptr;
    CK(cudaMalloc(&out, 4 * 4096));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float ms = 0;
    // int32: 2 ops (LOP3, IMAD) × 8 chains × iterations per thread
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_int32, 1024, 0));
    const int iblocks = sms * per_sm * 4;
    k_int32<<<iblocks, 1024>>>(1u, out);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    k_int32<<<iblocks, 1024>>>(3u, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    CK(cudaEventElapsedTime(&ms, a, b));
    const double int_ops = (double)iblocks * 1024 * kIntIters * 8 * 2;
    const double int_tops = int_ops / (ms * 1e-3) / 1e12;
    // i8 MMA: one CTA per SM, 2·M·N·K ops per instruction
    const uint32_t iters = 20000;
    k_mma_i8<<<sms, 128>>>(1000, out);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a));
    k_mma_i8<<<sms, 128>>>(iters, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms2 = 0;
    CK(cudaEventElapsedTime(&ms2, a, b));
    uint32_t chk = 0;
    CK(cudaMemcpy(&chk, out, 4, cudaMemcpyDeviceToHost));
    const double mma_ops = (double)sms * iters * 2.0 * kM * kN * kK;
    const double i8_tops = mma_ops / (ms2 * 1e-3) / 1e12;
    std::printf("{\"sms\": %d, \"clock_khz\": %d, \"int32_tops\": %.3f, \"int32_ms\": %.3f, \"i8_mma_tops\": %.1f, "
                "\"i8_mma_ms\": %.3f, \"i8_check\": %u, \"i8_check_expected\": %u}\n",
                sms, clk, int_tops, ms, i8_tops, ms2, chk, kK * iters);
    return 0;
}
