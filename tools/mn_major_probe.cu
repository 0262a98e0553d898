// mn_major_probe.cu -- which shared-memory descriptor fields (LBO / SBO) address an MN-major SWIZZLE_NONE
// operand of tcgen05.mma kind::f16 on sm_100a, with the instruction descriptor's transpose bits (15: A,
// 16: B). Fills the operand with small integers (exact fp32 sums) in the layout
//   element (k, mn) at (mn / 8) * 2048 + (k / 8) * 128 + (k % 8) * 16 + (mn % 8) * 2
// (core matrix = 8 K-rows x 8 MN elements, 128 B; K-adjacent core matrices 128 B apart, MN-adjacent 2048 B)
// and tries both (LBO, SBO) assignments; prints which reproduces A . B. Case 1: TS, A (M = 128, K = 16)
// from TMEM, B MN-major (N = 128). Case 2: SS, A MN-major (M = 128, K = 16), B K-major (N = 16).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mn_major_probe tools/mn_major_probe.cu
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int n, uint32_t tA, uint32_t tB) {
    return (1u << 4) | (tA << 15) | (tB << 16) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}
__device__ __forceinline__ float av(int m, int k) { return (float)(((m * 3 + k * 5) % 7) - 3); }
__device__ __forceinline__ float bv(int k, int n) { return (float)(((k * 2 + n * 7) % 5) - 2); }
__device__ __forceinline__ uint32_t mn_off(int k, int mn) { return (mn / 8) * 2048 + (k / 8) * 128 + (k % 8) * 16 + (mn % 8) * 2; }

// mode 0: TS + B MN-major (N = 128); mode 1: SS + A MN-major, B K-major (N = 16). swap: LBO/SBO swapped
__global__ void __launch_bounds__(128, 1) probe(int mode, int swap, float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __half* hs = reinterpret_cast<__half*>(smem);
    for (int i = threadIdx.x; i < 64 * 1024 / 2; i += blockDim.x) hs[i] = __float2half(0.0f);
    __syncthreads();
    // operand tiles: [0, 32K) MN-major tile (B for mode 0, A for mode 1); [32K, ...) K-major B (mode 1)
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) {
        const int k = i / 128, mn = i % 128;
        const float v = mode == 0 ? bv(k, mn) : av(mn, k);
        hs[mn_off(k, mn) / 2] = __float2half(v);
    }
    if (mode == 1) {   // B K-major, N = 16: core (kb, nb) at (kb * 2 + nb) * 128, row n % 8, col k % 8
        for (int i = threadIdx.x; i < 16 * 16; i += blockDim.x) {
            const int n = i / 16, k = i % 16;
            hs[(32768 + ((k / 8) * 2 + n / 8) * 128 + (n % 8) * 16 + (k % 8) * 2) / 2] = __float2half(bv(k, n));
        }
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    // A in TMEM (mode 0): lane m, columns 256..263 = fp16 pairs (k 2j, 2j+1)
    if (mode == 0) {
        const int m = 32 * (warp & 3) + lane;
        uint32_t w[8];
        for (int j = 0; j < 8; ++j) {
            __half2 h = __floats2half2_rn(av(m, 2 * j), av(m, 2 * j + 1));
            w[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                         tmem + 256u + ((uint32_t)(32 * (warp & 3)) << 16)),
                     "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0 && lane == 0) {
        const uint32_t lbo = swap ? 128 : 2048, sbo = swap ? 2048 : 128;
        const uint64_t mnd = sdesc(smem_u32(smem), lbo, sbo);
        if (mode == 0) {
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(tmem + 256u),
                         "l"(mnd), "r"(idesc(128, 0, 1)));
        } else {
            const uint64_t bd = sdesc(smem_u32(smem + 32768), 256, 128);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(mnd), "l"(bd),
                         "r"(idesc(16, 1, 0)));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    if (lane == 0) {
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)));
    }
    __syncwarp();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // D: lane m, columns 0..N-1
    const int m = 32 * (warp & 3) + lane;
    const int N = mode == 0 ? 128 : 16;
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                     : "r"(tmem + (uint32_t)c0 + ((uint32_t)(32 * (warp & 3)) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) out[m * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

static float hav(int m, int k) { return (float)(((m * 3 + k * 5) % 7) - 3); }
static float hbv(int k, int n) { return (float)(((k * 2 + n * 7) % 5) - 2); }

int main() {
    float* d;
    cudaMalloc(&d, 128 * 128 * 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    static float h[128 * 128];
    for (int mode = 0; mode < 2; ++mode) {
        for (int swap = 0; swap < 2; ++swap) {
            cudaMemset(d, 0, 128 * 128 * 4);
            probe<<<1, 128, 64 * 1024>>>(mode, swap, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("mode %d swap %d: %s\n", mode, swap, cudaGetErrorString(e)); return 1; }
            const int N = mode == 0 ? 128 : 16;
            cudaMemcpy(h, d, 128 * N * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int m = 0; m < 128; ++m)
                for (int n = 0; n < N; ++n) {
                    float r = 0;
                    for (int k = 0; k < 16; ++k) r += hav(m, k) * hbv(k, n);
                    bad += h[m * N + n] != r;
                }
            printf("%s, (LBO, SBO) = (%d, %d): %s (%d of %d wrong)\n",
                   mode == 0 ? "TS, B MN-major" : "SS, A MN-major", swap ? 128 : 2048, swap ? 2048 : 128,
                   bad ? "MISMATCH" : "MATCH", bad, 128 * N);
        }
    }
    return 0;
}
