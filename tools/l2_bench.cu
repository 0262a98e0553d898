// l2_bench.cu -- L2 read bandwidth of this B200 ("the L2 peak must be measured"):
// every SM streams a 48 MiB L2-resident buffer with 128-bit loads; best of 10; CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/l2_bench tools/l2_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) rd(const int4* __restrict__ p, size_t n, int reps, int* out) {
    int acc = 0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r)
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
            int4 v = __ldcg(p + i);     // L2 (bypass L1)
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x1234567) out[0] = acc;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    const size_t bytes = 48ull << 20;
    int4* p;
    int* o;
    cudaMalloc(&p, bytes);
    cudaMalloc(&o, 4);
    cudaMemset(p, 1, bytes);
    const size_t n = bytes / 16;
    const int reps = 20;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    rd<<<sms * 4, 512>>>(p, n, 2, o);
    float best = 1e30f;
    for (int it = 0; it < 10; ++it) {
        cudaEventRecord(a);
        rd<<<sms * 4, 512>>>(p, n, reps, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    const double gbs = (double)bytes * reps / (best / 1e3) / 1e9;
    printf("{\"l2_read_gbs\": %.1f, \"buffer_mib\": %zu, \"l2_bytes\": %d, \"sms\": %d}\n", gbs, bytes >> 20, l2, sms);
    return 0;
}
