// mma_shapes.cu -- tcgen05.mma kind::f16 issue rate per instruction shape on one SM pass (148 CTAs):
// M = 128, K = 16, N in {16, 32, 64, 128, 256}, A from TMEM (TS) or shared memory (SS), B from shared
// memory (SWIZZLE_NONE K-major). Back-to-back from one thread, accumulate on, one commit at the end.
// Also: alternating N=64 halves into two D regions (the NIF's N-split), and TS N=128 interleaved with
// an SS bias step every 8 MMAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/mma_shapes tools/mma_shapes.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int n, uint32_t ta = 0, uint32_t tb = 0) {
    return (1u << 4) | (ta << 15) | (tb << 16) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
}

// mode: 0 TS single N, 1 SS single N, 2 TS N=64 halves alternating D regions, 3 TS N=128 + SS bias / 8,
// 4 TS with B MN-major (SWIZZLE_NONE, LBO = K stride 128 B, SBO = MN stride 2048 B; transpose-B bit),
// 5 SS with A MN-major (same layout) and B K-major, 6 TS N=128 with a tcgen05.commit after every 9 MMAs
// (the NIF's per-layer commit), 7 as 6 alternating two D regions (two slots), 8 as 7 with each D region's
// MMAs and commits issued by its own warp (does a commit stall only its issuing thread?); 9-12 see below
template <int mode, int n>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    __shared__ __align__(8) uint64_t bar2;
    __shared__ __align__(8) uint64_t bar3;
    __shared__ __align__(8) uint64_t bar4;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(mode == 8 ? 2 : 1));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar3)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar4)), "r"(1 << 20));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tslot;
    unsigned long long t0 = clock64();
    if ((warp == 0 || (mode == 8 && warp == 1)) && lane == 0) {
        const uint32_t b = smem_u32(smem), a_s = smem_u32(smem + 64 * 1024);
        const uint64_t bd = sdesc(b, (uint32_t)(n / 8) * 128, 128);
        const uint64_t ad = sdesc(a_s, 2048, 128);
        for (int it = 0; it < iters; ++it) {
            const uint32_t acc = (it & 7) != 0;
            if (mode == 4) {
                const uint64_t bm = sdesc(b + (uint32_t)(it % 8) * 256, 128, 2048);
                const uint32_t a = tmem + 384u + (uint32_t)(8 * (it % 8));
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(a),
                             "l"(bm), "r"(idesc(n, 0, 1)), "r"(acc));
            } else if (mode == 5) {
                const uint64_t am = sdesc(b + (uint32_t)(it % 8) * 256, 128, 2048);
                const uint64_t bk = sdesc(a_s, 256, 128);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(am),
                             "l"(bk), "r"(idesc(n, 1, 0)), "r"(acc));
            } else if (mode == 8) {
                // two issuing warps, each with its own D region and commit barrier (half the iterations each)
                if ((it & 1) != warp) continue;
                const uint32_t d = tmem + 128u * warp;
                const uint32_t a = tmem + 384u + (uint32_t)(8 * ((it >> 1) % 8));
                const uint32_t acc8 = ((it >> 1) % 9) != 0;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                             "l"(bd), "r"(idesc(n)), "r"(acc8));
                if ((it >> 1) % 9 == 8)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(warp ? &bar3 : &bar2)));
            } else if (mode >= 9 && mode <= 12) {
                // 9: commit/9 with accumulate always on (no D overwrite at a group start); 10: commit/9
                // alternating two barriers; 11: commit/9 onto a barrier whose phase never completes;
                // 12: commit/9 then wait for it (the round trip a dependent epilogue sees)
                const uint32_t a = tmem + 384u + (uint32_t)(8 * (it % 8));
                const uint32_t accx = mode == 9 ? 1u : (uint32_t)((it % 9) != 0);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(a),
                             "l"(bd), "r"(idesc(n)), "r"(accx));
                if (it % 9 == 8) {
                    const uint64_t* cb = mode == 10 ? (((it / 9) & 1) ? &bar3 : &bar2) : (mode == 11 ? &bar4 : &bar2);
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(cb)));
                    if (mode == 12) {
                        const uint32_t par = (uint32_t)((it / 9) & 1);
                        uint32_t ok = 0;
                        while (!ok)
                            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar2)), "r"(par));
                    }
                }
            } else if (mode == 6 || mode == 7) {
                const uint32_t d = mode == 7 ? tmem + 128u * ((it / 9) & 1) : tmem;
                const uint32_t a = tmem + 384u + (uint32_t)(8 * (it % 8));
                const uint32_t acc6 = (it % 9) != 0;
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                             "l"(bd), "r"(idesc(n)), "r"(acc6));
                if (it % 9 == 8)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                        smem_u32(&bar2)));
            } else if (mode == 0 || mode == 2) {
                const uint32_t d = mode == 2 ? tmem + 64u * (it & 1) : tmem;
                const uint32_t a = tmem + 384u + (uint32_t)(8 * ((it >> (mode == 2 ? 1 : 0)) % 8));
                const uint32_t id = idesc(mode == 2 ? 64 : n);
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                             "l"(bd), "r"(id), "r"(acc));
            } else if (mode == 1 || ((it & 7) == 7 && mode == 3)) {
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem), "l"(ad),
                             "l"(bd), "r"(idesc(n)), "r"(acc));
            } else {
                const uint32_t a = tmem + 384u + (uint32_t)(8 * (it % 8));
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(a),
                             "l"(bd), "r"(idesc(n)), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)));
        }
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// commit round trip: one thread issues k TS MMAs (N = 128), commits, waits on the barrier; repeated.
// cycles per round = k * issue interval + the fixed MMA-completion + commit-notify latency
__global__ void __launch_bounds__(128, 1) commit_rtt(int k, int rounds, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
    if (warp == 0 && lane == 0) {
        const uint64_t bd = sdesc(smem_u32(smem), 16 * 128, 128);
        unsigned long long t0 = clock64();
        for (int r = 0; r < rounds; ++r) {
            for (int i = 0; i < k; ++i) {
                const uint32_t a = tmem + 384u + (uint32_t)(8 * (i % 8));
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                             "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem), "r"(a),
                             "l"(bd), "r"(idesc(128)), "r"((uint32_t)(i > 0)));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
            uint32_t ok = 0;
            while (!ok)
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                             "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)), "r"((uint32_t)(r & 1)));
        }
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    unsigned long long* d_out;
    cudaMalloc(&d_out, 148 * 8);
    const char* mname[13] = {"TS", "SS", "TS N64 halves", "TS + SS bias/8", "TS B MN-major", "SS A MN-major",
                            "TS + commit/9", "TS + commit/9, 2 D", "TS + commit/9, 2 issuing warps",
                            "TS + commit/9, acc on", "TS + commit/9, 2 bars", "TS + commit/9, no phase",
                            "TS + commit/9 + wait"};
    struct { int mode, n; void (*k)(int, unsigned long long*); } cases[] = {
        {0, 16, mma_rate<0, 16>}, {0, 32, mma_rate<0, 32>}, {0, 64, mma_rate<0, 64>}, {0, 128, mma_rate<0, 128>},
        {0, 256, mma_rate<0, 256>}, {1, 16, mma_rate<1, 16>}, {1, 64, mma_rate<1, 64>}, {1, 128, mma_rate<1, 128>},
        {1, 256, mma_rate<1, 256>}, {2, 64, mma_rate<2, 64>}, {3, 128, mma_rate<3, 128>},
        {4, 128, mma_rate<4, 128>}, {5, 16, mma_rate<5, 16>}, {6, 128, mma_rate<6, 128>}, {7, 128, mma_rate<7, 128>},
        {8, 128, mma_rate<8, 128>}, {9, 128, mma_rate<9, 128>}, {10, 128, mma_rate<10, 128>},
        {11, 128, mma_rate<11, 128>}, {12, 128, mma_rate<12, 128>}};
    for (auto c : cases) {
        const int iters = 9 * 1024;
        cudaFuncSetAttribute(c.k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        c.k<<<148, 128, 96 * 1024>>>(iters, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long h[148], mx = 0;
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        const int n = c.mode == 2 ? 64 : c.n;
        const double clk = (double)mx / iters;
        printf("%-16s N=%3d: %6.1f clk/MMA  %6.0f FLOP/clk/SM (%.0f%% of 8192)\n", mname[c.mode], n, clk,
               2.0 * 128 * n * 16 / clk, 100.0 * 2.0 * 128 * n * 16 / clk / 8192);
    }
    cudaFuncSetAttribute(commit_rtt, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int grid : {1, 148}) {
        for (int k : {1, 2, 4, 9, 18, 36}) {
            const int rounds = 256;
            commit_rtt<<<grid, 128, 64 * 1024>>>(k, rounds, d_out);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
            unsigned long long h[148], mx = 0;
            cudaMemcpy(h, d_out, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
            for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("commit round trip, grid %3d, %2d MMAs (N=128) per commit: %7.1f clk per round (%.1f per MMA)\n",
                   grid, k, (double)mx / rounds, (double)mx / rounds / k);
        }
    }
    return 0;
}
