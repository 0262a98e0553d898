// tmem_probe.cu -- microbenchmarks of the sm_100a resources the fused NIF kernel depends on:
//   mode 0: tcgen05.ld 32x32b.x32 throughput (TMEM -> registers), W warps per CTA
//   mode 1: tcgen05.mma kind::f16 M=128 N=128 K=16 with A in TMEM (TS), back-to-back, one thread
//   mode 2: both at once (MMA on columns 0-127/256-383, loads from 128-255)
//   mode 3: tcgen05.st 32x32b.x16 throughput
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512, 1) probe(int mode, int iters, unsigned long long* out, uint32_t* sink) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
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
    unsigned long long t0 = clock64();
    uint32_t acc = 0;
    const bool do_ld = (mode == 0 || mode == 2) && warp >= 1;
    const bool do_mma = (mode == 1 || mode == 2) && warp == 0;
    const bool do_st = (mode == 3) && warp >= 1;
    if (do_ld) {
        const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (mode == 2 ? 128u : 0u);
        for (int it = 0; it < iters; ++it) {
            uint32_t v[32];
            const uint32_t a = base + (uint32_t)((it * 32) & (mode == 2 ? 127 : 511));
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
                "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                  "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                  "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                : "r"(a));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= v[j];
        }
    }
    if (do_st) {
        const uint32_t base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
        uint32_t v[16];
        for (int j = 0; j < 16; ++j) v[j] = j + lane;
        for (int it = 0; it < iters; ++it) {
            const uint32_t a = base + (uint32_t)((it * 16) & 511);
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                ::"r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
                : "memory");
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    if (do_mma && lane == 0) {
        const uint32_t idesc = (1u << 4) | (16u << 17) | (8u << 24);
        uint64_t bdesc = (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF) | ((uint64_t)(2048 >> 4) << 16) |
                         ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
        for (int it = 0; it < iters; ++it) {
            const uint32_t d = tmem + (mode == 2 ? 0u : 0u);
            const uint32_t a = tmem + 384u + (uint32_t)(8 * (it % 8));
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a),
                         "l"(bdesc), "r"(idesc), "r"(it & 7));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t ok = 0;
        while (!ok) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(smem_u32(&bar)));
        }
    }
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
    if (acc == 0x12345678u) sink[0] = acc;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    unsigned long long* d_out;
    uint32_t* sink;
    cudaMalloc(&d_out, 148 * 16 * 8);
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    const char* names[4] = {"tcgen05.ld 32x32b.x32 (4 KB/warp)", "tcgen05.mma TS 128x128x16", "ld + mma concurrently",
                            "tcgen05.st 32x32b.x16 (2 KB/warp)"};
    for (int mode = 0; mode < 4; ++mode) {
        for (int warps : {4, 8, 16}) {
            if (mode == 1 && warps != 4) continue;
            const int iters = mode == 1 ? 4096 : 2048;
            int threads = 32 * (warps + 1);
            probe<<<148, threads, 64 * 1024>>>(mode, iters, d_out, sink);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf("mode %d err %s\n", mode, cudaGetErrorString(e)); return 1; }
            unsigned long long h[148 * 16];
            cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
            unsigned long long mx_ld = 0, mma = h[0];
            for (int w = 1; w <= warps; ++w) mx_ld = h[w] > mx_ld ? h[w] : mx_ld;
            if (mode == 0 || mode == 3) {
                double bytes = (double)warps * iters * (mode == 0 ? 4096 : 2048);
                printf("%-36s warps=%2d: %.1f B/clk/SM (cycles %llu)\n", names[mode], warps, bytes / mx_ld, mx_ld);
            } else if (mode == 1) {
                printf("%-36s: %.1f clk per MMA -> %.0f FLOP/clk/SM\n", names[mode], (double)mma / iters,
                       2.0 * 128 * 128 * 16 * iters / mma);
            } else {
                printf("%-36s warps=%2d: ld %.1f B/clk, mma %.1f clk/MMA\n", names[mode], warps,
                       (double)warps * iters * 4096 / mx_ld, (double)mma / iters);
            }
        }
    }
    return 0;
}
