// mlp_kernel.cu -- the paper's NIF family of the size sweep (
// DESIGN.md reading R23) as a chain of per-layer tcgen05 GEMMs with fused epilogues.
//
// What it computes, per escaped ray (direction d, or (u, v) from the query hook) with throughput beta:
//   gamma = (sin 2 pi B x, cos 2 pi B x) (40 features of x = (u, v)); h_0 = relu(W_0 gamma + b_0);
//   h_l = relu(W_l a_{l-1} + b_l) with a_c = [h_c, gamma] for the concat layer c and a_l = h_l otherwise;
//   yuv = W_L a_{L-1} + b_L; rgb = M_601 yuv; radiance = beta * exp(rgb).
//
// Why layered and not fused: from H = 256 the weights (387 KiB, 14 MiB for H1024 L8) no longer fit one
// SM's shared memory, and for H = 1024 one 128-row tile's activations (128 x 1024 fp16 = 256 KiB) no
// longer fit TMEM or shared memory either -- the regime the paper calls the point "at which current GPUs
// can not operate ... loads weights into SRAM/registers exactly once". On B200 each layer
// is one GEMM over the whole batch of escaped rays: activations stream through L2/HBM in a blocked fp16
// layout, weights stream as K-chunks (or stay resident in shared memory when a layer fits, H <= 256).
//
// GEMM kernel (one persistent CTA per SM, 192 threads):
//   warp 0 producer: cp.async.bulk of 16 KB A chunks (128 rows x 64 K) and BN x 64 B chunks into a
//     STAGES-deep shared-memory ring (mbarrier complete_tx); resident-B mode loads the layer's whole B
//     once.
//   warp 1 MMA: 4 SS tcgen05.mma (M = 128, N = BN, K = 16) per chunk, commit frees the stage; one commit
//     per tile hands the TMEM accumulator (2 buffers x BN columns) to the epilogue.
//   warps 2-5 epilogue (one TMEM lane quarter each): bias + ReLU + fp16 pack, 16-byte stores into the
//     next layer's blocked A layout; the output layer instead applies YUV -> RGB, exp and beta and
//     writes the path's wave slot.
// Blocked layout (A and B alike, SWIZZLE_NONE K-major core matrices): a (R rows x 128 bytes of K) chunk
// is one contiguous block, core matrix (rows 8nb..8nb+7, K bytes 16kb..16kb+15) at ((kb * R/8) + nb) * 128.
// fp16 networks hold 64 K elements per chunk; the fp8 variant ("float8 ... would halve the
// memory ... and increase performance") stores weights and activations as e4m3, 128 K
// elements per chunk, and runs tcgen05.mma kind::f8f6f4 (K = 32 per instruction, the same bytes and
// cycles as an fp16 K = 16 step, i.e. twice the FLOP rate).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "pt_internal.h"
#include "tc_ptx.cuh"

namespace pt {

namespace mlp {

constexpr int kBM = 128;
constexpr int kChunkBytesK = 128;               // bytes of K per chunk row (64 fp16 or 128 fp8 elements)
constexpr int kAChunk = kBM * kChunkBytesK;     // 16 KB
constexpr int kThreads = 192;
constexpr int kSmemBudget = 220 * 1024;
constexpr int kMaxStages = 8;
// barriers: [0..7] full[stage], [8..15] empty[stage], [16..17] acc_full, [18..19] acc_empty, [20] b_res;
// TMEM base address at 21 * 8
constexpr int kBarBytes = 256;

__host__ __device__ constexpr uint32_t idesc(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

struct LayerArgs {
    const uint8_t* A;        // blocked input activations of this row chunk, [m_tiles][KC][16 KB]
    const uint8_t* B;        // blocked weights, [NT][KC][BN * 128]
    const float* bias;       // [NT * BN] fp32, zero padded
    uint8_t* out_act;        // blocked output activations, [m_tiles][out_KC][16 KB] (kEpi 0)
    int KC, NT, N_valid, out_KC;
    int b_res, stages;
    const uint32_t* count;   // device row count (all chunks)
    int row0, rows_cap;      // this chunk: rows [row0, row0 + min(count - row0, rows_cap))
    const float4* esc;       // output layer: queue entries (slot in .w) and throughputs
    const float4* esc_beta;
    float* out_rgb;
};

// address of element column `col` (a multiple of 8) of one row in a blocked activation buffer
__device__ __forceinline__ uint8_t* act_ptr(uint8_t* buf, int out_KC, int tile, int row_in_tile, int col, int esize) {
    const int bc = col * esize;
    const int kc = bc >> 7, kb = (bc & 127) >> 4;
    return buf + ((size_t)tile * out_KC + kc) * kAChunk + ((kb * 16 + (row_in_tile >> 3)) * 128) + (row_in_tile & 7) * 16 +
           (bc & 15);
}
// 8 consecutive columns: 16 B of fp16 or 8 B of e4m3
__device__ __forceinline__ void store_act8(uint8_t* buf, int out_KC, int tile, int row_in_tile, int col, uint4 v) {
    *reinterpret_cast<uint4*>(act_ptr(buf, out_KC, tile, row_in_tile, col, 2)) = v;
}
__device__ __forceinline__ void store_act8_f8(uint8_t* buf, int out_KC, int tile, int row_in_tile, int col, uint2 v) {
    *reinterpret_cast<uint2*>(act_ptr(buf, out_KC, tile, row_in_tile, col, 1)) = v;
}
// two floats -> e4m3x2 (RN, saturating), `lo` in the low byte (the lower column)
__device__ __forceinline__ uint32_t e4m3x2(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}
// relu fused into the conversion (F2FP.SATFINITE.RELU.E4M3)
__device__ __forceinline__ uint32_t e4m3x2_relu(float lo, float hi) {
    uint16_t r;
    asm("cvt.rn.satfinite.relu.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(hi), "f"(lo));
    return r;
}

}  // namespace mlp

// Fourier features of the chunk's rows into a blocked activation buffer: part 0 writes the layer-0
// input (columns 0..39 = [sin_0..19, cos_0..19], 40..63 zero), part 1 the concat columns H-40..H-1 of
// the layer after the concat layer. Rows past the count get the features of (u, v) = (0.5, 0.5).
__global__ void mlp_features_kernel(const float4* __restrict__ esc, const uint32_t* __restrict__ count, int row0,
                                    int rows_cap, int dir_input, const float* __restrict__ freq, uint8_t* out,
                                    int out_KC, int col0, int zero_pad, int fp8) {
    const uint32_t n = *count;
    const int M = (int)min((int64_t)rows_cap, max((int64_t)0, (int64_t)n - row0));
    const int rows = ((M + mlp::kBM - 1) / mlp::kBM) * mlp::kBM;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        float u = 0.5f, v = 0.5f;
        if (r < M) {
            const float4 en = __ldg(esc + row0 + r);
            u = en.x;
            v = en.y;
            if (dir_input) equirect_f32(make_float3(en.x, en.y, en.z), u, v);
        }
        float f[40];
#pragma unroll
        for (int j = 0; j < 20; ++j) {
            const float p = fmaf(__ldg(freq + 2 * j), u, __ldg(freq + 2 * j + 1) * v);
            const float q = p - rintf(p);                 // exact-range turns in [-1/2, 1/2]
            __sincosf(6.28318530717958647692f * q, &f[j], &f[20 + j]);
        }
        const int tile = r / mlp::kBM, rt = r % mlp::kBM;
        if (!fp8) {
#pragma unroll
            for (int g = 0; g < 5; ++g) {
                uint4 w;
                uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                for (int i = 0; i < 4; ++i) wp[i] = pack_half2(f[8 * g + 2 * i], f[8 * g + 2 * i + 1]);
                mlp::store_act8(out, out_KC, tile, rt, col0 + 8 * g, w);
            }
            if (zero_pad) {
#pragma unroll
                for (int g = 5; g < 8; ++g) mlp::store_act8(out, out_KC, tile, rt, col0 + 8 * g, make_uint4(0, 0, 0, 0));
            }
        } else {
#pragma unroll
            for (int g = 0; g < 5; ++g) {
                const uint32_t lo = mlp::e4m3x2(f[8 * g], f[8 * g + 1]) | (mlp::e4m3x2(f[8 * g + 2], f[8 * g + 3]) << 16);
                const uint32_t hi = mlp::e4m3x2(f[8 * g + 4], f[8 * g + 5]) | (mlp::e4m3x2(f[8 * g + 6], f[8 * g + 7]) << 16);
                mlp::store_act8_f8(out, out_KC, tile, rt, col0 + 8 * g, make_uint2(lo, hi));
            }
            if (zero_pad) {
#pragma unroll
                for (int g = 5; g < 16; ++g) mlp::store_act8_f8(out, out_KC, tile, rt, col0 + 8 * g, make_uint2(0, 0));
            }
        }
    }
}

template <int BN, int kEpi, bool kFp8>
__global__ void __launch_bounds__(mlp::kThreads, 1) mlp_layer_kernel(mlp::LayerArgs a) {
    using namespace mlp;
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kBChunk = BN * kChunkBytesK;
    constexpr uint32_t kTmemCols = (2 * BN) < 32 ? 32u : (uint32_t)(2 * BN);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 21 * 8);
    auto bar = [&](int b) { return smem_u32(&bars[b]); };
    const int stage_bytes = kAChunk + (a.b_res ? 0 : kBChunk);
    uint8_t* ring = smem + kBarBytes;                               // stages x (A [, B])
    uint8_t* bres = ring + a.stages * stage_bytes;                  // resident B: KC x kBChunk

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n = *a.count;
    const int M = (int)min((int64_t)a.rows_cap, max((int64_t)0, (int64_t)n - a.row0));
    const int m_tiles = (M + kBM - 1) / kBM;
    const int n_tiles_total = m_tiles * a.NT;
    if (m_tiles == 0) return;

    if (warp == 0 && lane == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(bar(s), 1);
            mbar_init(bar(8 + s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(bar(16 + b), 1);
            mbar_init(bar(18 + b), 4);
        }
        mbar_init(bar(20), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===== producer =====
        if (lane == 0) {
            if (a.b_res) {
                mbar_expect_tx(bar(20), (uint32_t)(a.KC * kBChunk));
                for (int kc = 0; kc < a.KC; ++kc)
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(bres + kc * kBChunk)),
                        "l"(a.B + (size_t)kc * kBChunk), "r"(kBChunk), "r"(bar(20))
                        : "memory");
            }
            int stage = 0;
            uint32_t phase = 0;
            int it = 0;
            for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
                const int mt = t / a.NT, nt = t % a.NT;
                for (int kc = 0; kc < a.KC; ++kc, ++it) {
                    if (it >= a.stages) mbar_wait(bar(8 + stage), phase ^ 1);
                    uint8_t* sa = ring + stage * stage_bytes;
                    mbar_expect_tx(bar(stage), (uint32_t)stage_bytes);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            smem_u32(sa)),
                        "l"(a.A + ((size_t)mt * a.KC + kc) * kAChunk), "r"(kAChunk), "r"(bar(stage))
                        : "memory");
                    if (!a.b_res)
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                smem_u32(sa + kAChunk)),
                            "l"(a.B + ((size_t)nt * a.KC + kc) * kBChunk), "r"(kBChunk), "r"(bar(stage))
                            : "memory");
                    if (++stage == a.stages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer =====
        if (a.b_res) mbar_wait(bar(20), 0);
        int stage = 0;
        uint32_t phase = 0;
        uint32_t acc_phase[2] = {0, 0};
        int local = 0;
        for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++local) {
            const int nt = t % a.NT;
            const int acc = local & 1;
            if (local >= 2) {
                mbar_wait(bar(18 + acc), acc_phase[acc]);       // epilogue drained this accumulator
                acc_phase[acc] ^= 1;
            }
            tc_fence_after();
            const uint32_t dt = tmem + (uint32_t)(acc * BN);
            for (int kc = 0; kc < a.KC; ++kc) {
                mbar_wait(bar(stage), phase);
                tc_fence_after();
                const uint8_t* sa = ring + stage * stage_bytes;
                const uint8_t* sb = a.b_res ? bres + kc * kBChunk : sa + kAChunk;
                (void)nt;
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const uint64_t ad = smem_desc(smem_u32(sa) + k * 2 * 2048, 2048, 128);
                        const uint64_t bd = smem_desc(smem_u32(sb) + k * 2 * (BN / 8) * 128, (BN / 8) * 128, 128);
                        if (kFp8) mma_ss_f8(dt, ad, bd, idesc(BN), (kc | k) != 0);
                        else mma_ss(dt, ad, bd, idesc(BN), (kc | k) != 0);
                    }
                    mma_commit(bar(8 + stage));                  // stage free once these MMAs are done
                }
                __syncwarp();
                if (++stage == a.stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) mma_commit(bar(16 + acc));          // accumulator complete
            __syncwarp();
        }
    } else {
        // ===== epilogue: warps 2-5, TMEM lane quarter warp % 4 =====
        const int q = warp & 3;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        uint32_t acc_phase[2] = {0, 0};
        int local = 0;
        for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++local) {
            const int mt = t / a.NT, nt = t % a.NT;
            const int acc = local & 1;
            mbar_wait(bar(16 + acc), acc_phase[acc]);
            acc_phase[acc] ^= 1;
            tc_fence_after();
            const int rt = 32 * q + lane;                          // row within the tile
            const int row = a.row0 + mt * kBM + rt;
            const bool valid = mt * kBM + rt < M;
            const uint32_t dt = tmem + (uint32_t)(acc * BN) + lane_addr;
            if (kEpi == 0) {
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    const int col = nt * BN + 32 * c;
                    if (col >= a.N_valid) break;
                    uint32_t v[32];
                    TMEM_LD32(dt + 32 * c, v);
                    tmem_wait_ld_dep(v);
                    const float4* bp = reinterpret_cast<const float4*>(a.bias + col);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (col + 8 * g >= a.N_valid) break;
                        const float4 b0 = __ldg(bp + 2 * g), b1 = __ldg(bp + 2 * g + 1);
                        const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                        float h[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) h[i] = __uint_as_float(v[8 * g + i]) + bb[i];
                        if (!kFp8) {
                            uint4 w;
                            uint32_t* wp = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(wp[i]) : "f"(h[2 * i + 1]), "f"(h[2 * i]));
                            store_act8(a.out_act, a.out_KC, mt, rt, col + 8 * g, w);
                        } else {
                            const uint32_t lo = e4m3x2_relu(h[0], h[1]) | (e4m3x2_relu(h[2], h[3]) << 16);
                            const uint32_t hi = e4m3x2_relu(h[4], h[5]) | (e4m3x2_relu(h[6], h[7]) << 16);
                            store_act8_f8(a.out_act, a.out_KC, mt, rt, col + 8 * g, make_uint2(lo, hi));
                        }
                    }
                }
            } else {
                uint32_t v[4];
                tmem_ld4(dt, v);
                tmem_wait_ld_dep4(v);
                if (valid) {
                    const float Y = __uint_as_float(v[0]) + __ldg(a.bias + 0);
                    const float U = __uint_as_float(v[1]) + __ldg(a.bias + 1);
                    const float V = __uint_as_float(v[2]) + __ldg(a.bias + 2);
                    // fixed BT.601 YUV -> RGB colour layer, log space; then exp
                    const float r = fmaf(1.13983f, V, Y);
                    const float gch = fmaf(-0.58060f, V, fmaf(-0.39465f, U, Y));
                    const float bch = fmaf(2.03211f, U, Y);
                    const uint32_t slot = __float_as_uint(__ldg(a.esc + row).w);
                    const float4 beta = __ldg(a.esc_beta + row);
                    a.out_rgb[3 * (size_t)slot + 0] = beta.x * __expf(r);
                    a.out_rgb[3 * (size_t)slot + 1] = beta.y * __expf(gch);
                    a.out_rgb[3 * (size_t)slot + 2] = beta.z * __expf(bch);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(18 + acc));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ---------------------------------------------------------------------------------------------
// Fused variant for H <= 256: one 128-row tile runs through all layers with its activations resident
// in TMEM (A: H/2 columns of fp16 pairs, D: H fp32 columns) and the layers' weights streamed from L2 as
// the same blocked K-chunks through a shared-memory ring -- no activation traffic to HBM at all (the
// layered path moves 4 H bytes per ray per layer). 320 threads: warp 0 producer (bulk copies of weight
// chunks in the order the MMA consumes them), warp 1 MMA issuer (TS MMAs, A from TMEM), warps 2-9 the
// epilogue (bias + ReLU + fp16 into A, the Fourier features into A for layer 0 and the concat columns,
// the YUV -> RGB / exp / beta output).
// ---------------------------------------------------------------------------------------------
namespace mlpf {
constexpr int kMaxLayers = 17;
constexpr int kRing = 6;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
struct FusedArgs {
    const uint8_t* W[kMaxLayers];      // blocked weights of layer l, one N tile: [KC][BN * 128 B]
    const float* bias[kMaxLayers];
    int KC[kMaxLayers], BN[kMaxLayers], N[kMaxLayers];
    int L, c;
    const float* freq;
    const float4* esc;
    const float4* esc_beta;
    const uint32_t* count;
    float* out;
    int dir_input;
};
}  // namespace mlpf

template <int kH>
constexpr int fused_ctas_per_sm() { return kH == 64 ? 3 : kH == 128 ? 2 : 1; }

// kFp8: e4m3 weights, features and activations (reading R24), tcgen05 kind::f8f6f4 with A in TMEM:
// a 128-B K-chunk is 128 elements and 4 MMAs of K = 32, so the MMA schedule and A column offsets are
// those of fp16 (whose 128-B chunk is 64 elements, 4 MMAs of K = 16); A holds 4 activations per column.
template <int kH, bool kFp8>
__global__ void __launch_bounds__(mlpf::kThreads, fused_ctas_per_sm<kH>()) mlp_fused_kernel(mlpf::FusedArgs a) {
    using namespace mlpf;
    constexpr int kStage = kH * 128;                         // bytes of the widest weight chunk
    constexpr uint32_t kTmemCols = kH == 256 ? 512u : (kH == 128 ? 256u : 128u);
    constexpr uint32_t kDCol = 0, kACol = kH;                // D: kH fp32 columns; A: kH / 2 (fp8: kH / 4) columns
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);     // [0..5] full, [6..11] empty, [12] d_full, [13] a_ready
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 120);
    uint8_t* ring = smem + 1024;
    float* sbias = reinterpret_cast<float*>(ring + kRing * kStage);   // [layer][kH]: the epilogue's biases
    auto bar = [&](int b) { return smem_u32(&bars[b]); };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n_rows = *a.count;
    const uint32_t n_tiles = (n_rows + mlp::kBM - 1) / mlp::kBM;
    if (blockIdx.x >= n_tiles) return;
    for (int l = 0; l <= a.L; ++l)
        for (int i = threadIdx.x; i < a.BN[l]; i += blockDim.x) sbias[l * kH + i] = __ldg(a.bias[l] + i);
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < kRing; ++s) {
            mbar_init(bar(s), 1);
            mbar_init(bar(kRing + s), 1);
        }
        mbar_init(bar(12), 1);
        mbar_init(bar(13), kEpiWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0, it = 0;
            uint32_t phase = 0;
            for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
                for (int l = 0; l <= a.L; ++l) {
                    const uint32_t bytes = (uint32_t)a.BN[l] * 128u;
                    for (int kc = 0; kc < a.KC[l]; ++kc, ++it) {
                        if (it >= kRing) mbar_wait(bar(kRing + stage), phase ^ 1);
                        mbar_expect_tx(bar(stage), bytes);
                        asm volatile(
                            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                smem_u32(ring + stage * kStage)),
                            "l"(a.W[l] + (size_t)kc * bytes), "r"(bytes), "r"(bar(stage))
                            : "memory");
                        if (++stage == kRing) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        int stage = 0;
        uint32_t phase = 0, a_phase = 0;
        for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            for (int l = 0; l <= a.L; ++l) {
                mbar_wait(bar(13), a_phase);                  // this layer's A written (and D read out)
                a_phase ^= 1;
                tc_fence_after();
                const int bn = a.BN[l];
                const uint32_t id = mlp::idesc(bn);
                const uint32_t lbo = (uint32_t)(bn / 8) * 128u;
                for (int kc = 0; kc < a.KC[l]; ++kc) {
                    mbar_wait(bar(stage), phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t sb = smem_u32(ring + stage * kStage);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                        {
                            const uint32_t at = tmem + kACol + (uint32_t)(32 * kc + 8 * k);
                            const uint64_t bd = smem_desc(sb + k * 2 * lbo, lbo, 128);
                            if (kFp8) mma_ts_f8(tmem + kDCol, at, bd, id, (kc | k) != 0);
                            else mma_ts(tmem + kDCol, at, bd, id, (kc | k) != 0);
                        }
                        mma_commit(bar(kRing + stage));
                    }
                    __syncwarp();
                    if (++stage == kRing) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (elect_one()) mma_commit(bar(12));
                __syncwarp();
            }
        }
    } else {
        // ===== epilogue: warps 2-9; two per TMEM lane quarter (half 0 / 1 split the column work) =====
        const int e = warp - 2;
        const int half = e >> 2;
        const int q = warp & 3;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        const uint32_t A = tmem + kACol + lane_addr, D = tmem + kDCol + lane_addr;
        uint32_t d_phase = 0;
        // Fourier features of this row into A element columns col0 .. col0 + 39: half 0 the 20 sines,
        // half 1 the 20 cosines; `pad` also zeroes element columns 40..63 (layer-0 input)
        auto write_features = [&](float u, float v, int col0, bool pad) {
            float f[20];
#pragma unroll
            for (int fj = 0; fj < 20; ++fj) {
                const float p = fmaf(__ldg(a.freq + 2 * fj), u, __ldg(a.freq + 2 * fj + 1) * v);
                const float r = p - rintf(p);
                f[fj] = half == 0 ? __sinf(6.28318530717958647692f * r) : __cosf(6.28318530717958647692f * r);
            }
            if (!kFp8) {
                uint32_t w[10];
#pragma unroll
                for (int j = 0; j < 10; ++j) w[j] = pack_half2(f[2 * j], f[2 * j + 1]);
                const uint32_t c0 = A + (uint32_t)(col0 / 2 + 10 * half);
                tmem_st8(c0, w);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(c0 + 8), "r"(w[8]), "r"(w[9])
                             : "memory");
                if (pad && half == 1) {
                    const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                    tmem_st8(A + 20, z);
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(A + 28), "r"(0u)
                                 : "memory");
                }
            } else {
                uint32_t w[5];
#pragma unroll
                for (int j = 0; j < 5; ++j)
                    w[j] = mlp::e4m3x2(f[4 * j], f[4 * j + 1]) | (mlp::e4m3x2(f[4 * j + 2], f[4 * j + 3]) << 16);
                const uint32_t c0 = A + (uint32_t)(col0 / 4 + 5 * half);
                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(c0), "r"(w[0]), "r"(w[1]),
                             "r"(w[2]), "r"(w[3])
                             : "memory");
                asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(c0 + 4), "r"(w[4]) : "memory");
                if (pad && half == 1) {                     // elements 40..127 (K = 128) = A columns 10..31
                    const uint32_t z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
                    TMEM_ST16(A + 10, z);
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(A + 26), "r"(0u)
                                 : "memory");
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%1};" ::"r"(A + 30), "r"(0u) : "memory");
                }
            }
        };
        if (kFp8 && kH == 64 && half == 0) {
            // e4m3 K-chunks are 128 wide: A columns 16..31 (elements 64..127, zero weights) stay 0, not NaN
            const uint32_t z[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
            TMEM_ST16(A + 16, z);
        }
        float4 en_next = make_float4(0.5f, 0.5f, 0.0f, 0.0f), beta_next = en_next;
        {
            const uint32_t r0 = blockIdx.x * mlp::kBM + 32 * q + lane;
            if (r0 < n_rows) {
                en_next = __ldg(a.esc + r0);
                beta_next = __ldg(a.esc_beta + r0);
            }
        }
        for (uint32_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
            const uint32_t row = t * mlp::kBM + 32 * q + lane;
            const bool valid = row < n_rows;
            // this tile's queue entry was loaded one tile ahead (off the tile's critical path)
            const float4 en = en_next, beta = beta_next;
            {
                const uint32_t tn = t + gridDim.x, rn = tn * mlp::kBM + 32 * q + lane;
                if (tn < n_tiles && rn < n_rows) {
                    en_next = __ldg(a.esc + rn);
                    beta_next = __ldg(a.esc_beta + rn);
                }
            }
            float u = 0.5f, v = 0.5f;
            if (valid) {
                u = en.x;
                v = en.y;
                if (a.dir_input) equirect_f32(make_float3(en.x, en.y, en.z), u, v);
            }
            write_features(u, v, 0, true);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(13));
            for (int l = 0; l <= a.L; ++l) {
                mbar_wait(bar(12), d_phase);
                d_phase ^= 1;
                tc_fence_after();
                if (l < a.L) {
                    const int N = a.N[l];
                    const float* bias = sbias + l * kH;
                    for (int j = half; 32 * j < N; j += 2) {
                        uint32_t vv[32];
                        TMEM_LD32(D + 32 * j, vv);
                        tmem_wait_ld_dep(vv);
                        uint32_t pk[16];
                        const float4* bp = reinterpret_cast<const float4*>(bias + 32 * j);   // shared memory
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            const float4 b4 = bp[g];
                            const float x0 = __uint_as_float(vv[4 * g]) + b4.x, x1 = __uint_as_float(vv[4 * g + 1]) + b4.y;
                            const float x2 = __uint_as_float(vv[4 * g + 2]) + b4.z, x3 = __uint_as_float(vv[4 * g + 3]) + b4.w;
                            if (!kFp8) {
                                asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(pk[2 * g]) : "f"(x1), "f"(x0));
                                asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(pk[2 * g + 1]) : "f"(x3), "f"(x2));
                            } else {
                                pk[g] = mlp::e4m3x2_relu(x0, x1) | (mlp::e4m3x2_relu(x2, x3) << 16);
                            }
                        }
                        if (!kFp8) {
                            if (32 * j + 32 <= N) {
                                TMEM_ST16(A + 16 * j, pk);
                            } else {
                                // the concat layer's last chunk: 24 valid columns (H - 40 = 24 mod 32)
                                tmem_st8(A + 16 * j, pk);
                                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(A + 16 * j + 8),
                                             "r"(pk[8]), "r"(pk[9]), "r"(pk[10]), "r"(pk[11])
                                             : "memory");
                            }
                        } else {
                            if (32 * j + 32 <= N) {
                                tmem_st8(A + 8 * j, pk);
                            } else {
                                // 24 valid columns = 6 A columns of 4 e4m3
                                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(A + 8 * j),
                                             "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3])
                                             : "memory");
                                asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(A + 8 * j + 4),
                                             "r"(pk[4]), "r"(pk[5])
                                             : "memory");
                            }
                        }
                    }
                    if (l == a.c) write_features(u, v, kH - 40, false);   // the concat skip
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar(13));
                } else {
                    // output layer: YUV (D columns 0..2) + bias -> fixed BT.601 -> RGB -> exp -> beta
                    if (half == 0) {
                        uint32_t y[4];
                        tmem_ld4(D, y);
                        tmem_wait_ld_dep4(y);
                        if (valid) {
                            const float Y = __uint_as_float(y[0]) + sbias[l * kH + 0];
                            const float U = __uint_as_float(y[1]) + sbias[l * kH + 1];
                            const float V = __uint_as_float(y[2]) + sbias[l * kH + 2];
                            const float r = fmaf(1.13983f, V, Y);
                            const float gch = fmaf(-0.58060f, V, fmaf(-0.39465f, U, Y));
                            const float bch = fmaf(2.03211f, U, Y);
                            const uint32_t slot = __float_as_uint(en.w);
                            a.out[3 * (size_t)slot + 0] = beta.x * __expf(r);
                            a.out[3 * (size_t)slot + 1] = beta.y * __expf(gch);
                            a.out[3 * (size_t)slot + 2] = beta.z * __expf(bch);
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ---------------------------------------------------------------------------------------------
// Host side: weight re-layout at load, launch sequence per row chunk
// ---------------------------------------------------------------------------------------------
namespace {

int pick_bn(int n_valid) { return n_valid <= 16 ? 16 : n_valid <= 64 ? 64 : n_valid <= 128 ? 128 : 256; }

}  // namespace

// shared with the paper-NIF kernel's fp8 image (nif_kernel.cu): one e4m3 rounding of the weights
float half_to_float(uint16_t h) {
    const int e = (h >> 10) & 31, m = h & 1023;
    float v = e == 0 ? std::ldexp((float)m, -24) : std::ldexp((float)(m | 1024), e - 25);
    return (h & 0x8000) ? -v : v;
}

// fp32 -> OCP e4m3 (1-4-3, bias 7, no infinities, max 448), round to nearest even, saturating: the
// conversion cvt.rn.satfinite.e4m3x2.f32 does on the device
uint8_t float_to_e4m3(float x) {
    const uint8_t sign = std::signbit(x) ? 0x80 : 0;
    double a = std::fabs((double)x);
    if (!(a > 0.0)) return sign;
    if (a >= 448.0) return sign | 0x7E;                   // 448 = 1.75 * 2^8
    int e;
    std::frexp(a, &e);                                     // a = f * 2^e, f in [0.5, 1)
    int ex = std::max(e - 1, -6);                          // subnormals share the exponent of 2^-6
    const double q = std::ldexp(1.0, ex - 3);              // quantum
    double m = a / q;                                      // in [0, 16)
    double r = std::nearbyint(m);                          // ties to even (default rounding mode)
    if (r >= 16.0) { r = 8.0; ex += 1; }
    if (ex > 8 || (ex == 8 && r > 14.0)) return sign | 0x7E;
    if (r < 8.0) return sign | (uint8_t)r;                 // subnormal (ex == -6)
    return sign | (uint8_t)(((ex + 7) << 3) | ((int)r - 8));
}


int mlp_concat_layer(int L) {
    int c = 0;
    for (int l = 1; 2 * l < L; l += 2) c = l;
    return c;
}

int64_t mlp_blob_halves(int H, int L) {
    const int c = mlp_concat_layer(L);
    int64_t n = 40;
    for (int l = 0; l <= L; ++l) {
        const int64_t fin = l == 0 ? 40 : H, fout = l == L ? 3 : (l == c ? H - 40 : H);
        n += fin * fout + fout;
    }
    return n;
}

// Build the blocked device weights of every layer (K padded to 64, N padded to BN, zeros elsewhere).
int mlp_load(pt_nif* nif, int H, int L, const uint16_t* blob, int fp8, std::string* msg) {
    const int c = mlp_concat_layer(L);
    nif->mlp_H = H;
    nif->mlp_L = L;
    nif->mlp_c = c;
    nif->mlp_fp8 = fp8 ? 1 : 0;
    const int esize = fp8 ? 1 : 2, chunk_k = 128 / esize;
    int64_t off = 0;
    std::vector<float> freq(40);
    for (int i = 0; i < 40; ++i) freq[i] = half_to_float(blob[off++]);
    if (cudaMalloc(&nif->mlp_freq, sizeof(float) * 40) != cudaSuccess ||
        cudaMemcpy(nif->mlp_freq, freq.data(), sizeof(float) * 40, cudaMemcpyHostToDevice) != cudaSuccess) {
        *msg = "mlp: frequency upload failed";
        return PT_ERR_CUDA;
    }
    for (int l = 0; l <= L; ++l) {
        MlpLayer ly;
        const int fin = l == 0 ? 40 : H, fout = l == L ? 3 : (l == c ? H - 40 : H);
        ly.K = ((fin + chunk_k - 1) / chunk_k) * chunk_k;
        ly.N_valid = fout;
        ly.BN = pick_bn(fout);
        ly.NT = (fout + ly.BN - 1) / ly.BN;
        const int KC = ly.K / chunk_k;
        std::vector<uint8_t> img((size_t)ly.NT * KC * ly.BN * 128, 0);
        const uint16_t* W = blob + off;
        off += (int64_t)fin * fout;
        const uint16_t* b = blob + off;
        off += fout;
        for (int nrow = 0; nrow < fout; ++nrow) {
            const int nt = nrow / ly.BN, nn = nrow % ly.BN, nb = nn >> 3, r = nn & 7;
            for (int k = 0; k < fin; ++k) {
                const int bc = k * esize, kc = bc >> 7, kb = (bc & 127) >> 4, cc = bc & 15;
                const size_t o = ((size_t)nt * KC + kc) * ly.BN * 128 + (size_t)((kb * (ly.BN / 8) + nb) * 128) + r * 16 + cc;
                const uint16_t w = W[(int64_t)nrow * fin + k];
                if (fp8) img[o] = float_to_e4m3(half_to_float(w));
                else std::memcpy(&img[o], &w, 2);
            }
        }
        std::vector<float> bias((size_t)ly.NT * ly.BN, 0.0f);
        for (int i = 0; i < fout; ++i) bias[i] = half_to_float(b[i]);
        if (cudaMalloc(&ly.d_w, img.size()) != cudaSuccess ||
            cudaMemcpy(ly.d_w, img.data(), img.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
            cudaMalloc(&ly.d_bias, sizeof(float) * bias.size()) != cudaSuccess ||
            cudaMemcpy(ly.d_bias, bias.data(), sizeof(float) * bias.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
            *msg = "mlp: weight upload failed";
            nif->mlp_layers.push_back(ly);
            return PT_ERR_OOM;
        }
        nif->mlp_layers.push_back(ly);
    }
    return PT_OK;
}

void mlp_free(pt_nif* nif) {
    for (auto& ly : nif->mlp_layers) {
        cudaFree(ly.d_w);
        cudaFree(ly.d_bias);
    }
    nif->mlp_layers.clear();
    cudaFree(nif->mlp_freq);
    cudaFree(nif->mlp_act[0]);
    cudaFree(nif->mlp_act[1]);
    if (nif->mlp_last_use) cudaEventDestroy(nif->mlp_last_use);
    nif->mlp_last_use = nullptr;
    nif->mlp_freq = nullptr;
    nif->mlp_act[0] = nif->mlp_act[1] = nullptr;
}

template <int BN, int kEpi, bool kFp8>
static cudaError_t launch_layer_t(const mlp::LayerArgs& a, int grid, int smem, cudaStream_t st) {
    cudaError_t e = ensure_dyn_smem((const void*)mlp_layer_kernel<BN, kEpi, kFp8>, std::max(smem, mlp::kSmemBudget + mlp::kBarBytes));
    if (e != cudaSuccess) return e;
    mlp_layer_kernel<BN, kEpi, kFp8><<<grid, mlp::kThreads, smem, st>>>(a);
    return cudaGetLastError();
}

template <bool kFp8>
static cudaError_t launch_layer_bn(int bn, int epi, const mlp::LayerArgs& a, int grid, int smem, cudaStream_t st) {
    if (epi == 1) return launch_layer_t<16, 1, kFp8>(a, grid, smem, st);
    switch (bn) {
        case 64: return launch_layer_t<64, 0, kFp8>(a, grid, smem, st);
        case 128: return launch_layer_t<128, 0, kFp8>(a, grid, smem, st);
        case 256: return launch_layer_t<256, 0, kFp8>(a, grid, smem, st);
        default: return launch_layer_t<16, 0, kFp8>(a, grid, smem, st);
    }
}

static cudaError_t launch_layer(const MlpLayer& ly, int epi, int fp8, mlp::LayerArgs a, cudaStream_t st) {
    using namespace mlp;
    const int KC = ly.K / (fp8 ? 128 : 64);
    const int bchunk = ly.BN * 128;
    const bool res = ly.NT == 1 && (int64_t)KC * bchunk <= 128 * 1024;
    const int stage_bytes = kAChunk + (res ? 0 : bchunk);
    const int avail = kSmemBudget - (res ? KC * bchunk : 0);
    a.KC = KC;
    a.NT = ly.NT;
    a.N_valid = ly.N_valid;
    a.B = (const uint8_t*)ly.d_w;
    a.bias = ly.d_bias;
    a.b_res = res ? 1 : 0;
    a.stages = std::min(kMaxStages, avail / stage_bytes);
    const int smem = kBarBytes + a.stages * stage_bytes + (res ? KC * bchunk : 0);
    const int64_t tiles = (int64_t)((a.rows_cap + kBM - 1) / kBM) * ly.NT;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms()));
    return fp8 ? launch_layer_bn<true>(ly.BN, epi, a, grid, smem, st) : launch_layer_bn<false>(ly.BN, epi, a, grid, smem, st);
}

// Row chunks of up to kChunkRows rows; every chunk launch reads the device row count and exits when
// the chunk is empty, so the host never synchronises on the count.
constexpr int kChunkRows = 1 << 20;

template <int kH, bool kFp8>
static cudaError_t launch_fused_t(const mlpf::FusedArgs& fa, int grid, cudaStream_t st) {
    const int smem = 1024 + mlpf::kRing * kH * 128 + mlpf::kMaxLayers * kH * 4;   // + the bias table
    cudaError_t e = ensure_dyn_smem((const void*)mlp_fused_kernel<kH, kFp8>, smem);
    if (e != cudaSuccess) return e;
    mlp_fused_kernel<kH, kFp8><<<grid * fused_ctas_per_sm<kH>(), mlpf::kThreads, smem, st>>>(fa);
    return cudaGetLastError();
}

// The fused path serves H = 64, 128, 256 in fp16 and fp8 (PT_MLP_LAYERED=1 forces the layered path, for tests)
static bool use_fused(const pt_nif* nif) {
    const char* env = std::getenv("PT_MLP_LAYERED");
    const bool layered = env && env[0] == '1';
    return !layered && (nif->mlp_H == 64 || nif->mlp_H == 128 || nif->mlp_H == 256) &&
           nif->mlp_L + 1 <= mlpf::kMaxLayers;
}

cudaError_t launch_mlp(pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count, int64_t max_rows,
                       float* out, int dir_input, cudaStream_t st) {
    using namespace mlp;
    const int H = nif->mlp_H, L = nif->mlp_L, c = nif->mlp_c, fp8 = nif->mlp_fp8;
    if (use_fused(nif)) {
        mlpf::FusedArgs fa{};
        for (int l = 0; l <= L; ++l) {
            const MlpLayer& ly = nif->mlp_layers[l];
            fa.W[l] = (const uint8_t*)ly.d_w;
            fa.bias[l] = ly.d_bias;
            fa.KC[l] = ly.K / (fp8 ? 128 : 64);
            fa.BN[l] = ly.BN;
            fa.N[l] = ly.N_valid;
        }
        fa.L = L;
        fa.c = c;
        fa.freq = nif->mlp_freq;
        fa.esc = esc;
        fa.esc_beta = esc_beta;
        fa.count = count;
        fa.out = out;
        fa.dir_input = dir_input;
        const int64_t tiles = (max_rows + kBM - 1) / kBM;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms()));   // x CTAs per SM
        if (fp8)
            return H == 256 ? launch_fused_t<256, true>(fa, grid, st)
                            : H == 128 ? launch_fused_t<128, true>(fa, grid, st) : launch_fused_t<64, true>(fa, grid, st);
        return H == 256 ? launch_fused_t<256, false>(fa, grid, st)
                        : H == 128 ? launch_fused_t<128, false>(fa, grid, st) : launch_fused_t<64, false>(fa, grid, st);
    }
    const int kc_of_H = (H * (fp8 ? 1 : 2) + 127) / 128;          // K chunks of an H-wide activation row
    const int cap = (int)std::min<int64_t>(kChunkRows, ((max_rows + kBM - 1) / kBM) * kBM);
    const int64_t need = (int64_t)((cap + kBM - 1) / kBM) * kAChunk * kc_of_H;
    // the activation buffers are per-handle scratch: serialise their (re)allocation and order this use
    // after the previous one, which may run on another stream
    std::lock_guard<std::mutex> lk(nif->mlp_mu);
    if (!nif->mlp_last_use) {
        cudaError_t e = cudaEventCreateWithFlags(&nif->mlp_last_use, cudaEventDisableTiming);
        if (e != cudaSuccess) return e;
    } else {
        cudaError_t e = cudaStreamWaitEvent(st, nif->mlp_last_use, 0);
        if (e != cudaSuccess) return e;
    }
    struct RecordOnExit {
        cudaEvent_t ev;
        cudaStream_t st;
        ~RecordOnExit() { cudaEventRecord(ev, st); }
    } record_on_exit{nif->mlp_last_use, st};
    if (need > nif->mlp_act_bytes) {
        cudaEventSynchronize(nif->mlp_last_use);   // no earlier use may still read the old buffers
        cudaStreamSynchronize(st);
        cudaFree(nif->mlp_act[0]);
        cudaFree(nif->mlp_act[1]);
        nif->mlp_act[0] = nif->mlp_act[1] = nullptr;
        nif->mlp_act_bytes = 0;
        cudaError_t e = cudaMalloc(&nif->mlp_act[0], need);
        if (e == cudaSuccess) e = cudaMalloc(&nif->mlp_act[1], need);
        // K padding columns (fp8 H = 64: 64..127) are never written and must read as zeros
        if (e == cudaSuccess) e = cudaMemsetAsync(nif->mlp_act[0], 0, need, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(nif->mlp_act[1], 0, need, st);
        if (e != cudaSuccess) return e;
        nif->mlp_act_bytes = need;
    }
    uint8_t* buf[2] = {(uint8_t*)nif->mlp_act[0], (uint8_t*)nif->mlp_act[1]};
    for (int64_t r0 = 0; r0 < max_rows; r0 += cap) {
        const int fgrid = std::max(1, std::min(num_sms() * 4, (cap + 255) / 256));
        // layer-0 input; the concat columns of layer c + 1 too when that buffer is not read before
        mlp_features_kernel<<<fgrid, 256, 0, st>>>(esc, count, (int)r0, cap, dir_input, nif->mlp_freq, buf[0], 1, 0, 1,
                                                   fp8);
        for (int l = 0; l <= L; ++l) {
            if (l == c) {
                mlp_features_kernel<<<fgrid, 256, 0, st>>>(esc, count, (int)r0, cap, dir_input, nif->mlp_freq,
                                                           buf[(c + 1) & 1], kc_of_H, H - 40, 0, fp8);
            }
            LayerArgs a{};
            a.A = buf[l & 1];
            a.out_act = buf[(l + 1) & 1];
            a.out_KC = kc_of_H;
            a.count = count;
            a.row0 = (int)r0;
            a.rows_cap = cap;
            a.esc = esc;
            a.esc_beta = esc_beta;
            a.out_rgb = out;
            cudaError_t e = launch_layer(nif->mlp_layers[l], l == L ? 1 : 0, fp8, a, st);
            if (e != cudaSuccess) return e;
        }
    }
    return cudaGetLastError();
}

}  // namespace pt
