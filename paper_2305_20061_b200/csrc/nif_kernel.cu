// nif_kernel.cu -- the paper's own HDR-NIF (PT_NIF_FOURIER_RELU) fused on sm_100a tensor cores
// (tcgen05 + TMEM); the SIREN NIF of the hot path is siren_kernel.cu.
//
// What it computes (reading R4): for every escaped ray with equirect (u, v)
// and throughput beta: Fourier features (sin, cos)(2 pi B (u, v)) (F = 20 frequencies) -> 4 ReLU layers
// of width 128 with the features concatenated again after the second (layer 1 has 88 units) -> linear
// (Y, U, V) -> fixed BT.601 YUV -> RGB -> exp; radiance = beta * exp(rgb).
// One persistent CTA per SM keeps the fp16 weight set resident in shared memory (one bulk TMA copy);
// each layer of a 128-ray tile is a chain of tcgen05.mma kind::f16 (M = 128, K = 16 steps) with fp32
// accumulators in TMEM and the fp16 activations written back to TMEM as the next layer's A operand.
// Biases ride in the MMA as an extra K step against a constant-1 column in shared memory. Two tiles are
// in flight per CTA; each layer is issued as two column halves with their own commit barriers so the
// low-half epilogue overlaps the high-half MMAs. The feature columns stay in A buffer 0 (columns
// 44..63) for the concat skip, so A is double-buffered per slot.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "pt_internal.h"
#include "tc_ptx.cuh"

namespace pt {

namespace nif {

constexpr int kHid = 128;
constexpr int kTileM = 128;
constexpr int kOnesBytes = 128 * 16 * 2;
// The paper's own NIF (kind 1: Fourier features + ReLU + concat skip + YUV->RGB, reading R4):
//   B0: N=128, K=48 (+16 bias) -- K' 0..7 zero, K' 8+2j / 9+2j = weights of sin_j / cos_j
//   B1: N=96 (88 used), K=128 (+16); B2: N=128, K = [h1 (88), (sin_j, cos_j) interleaved (40)] (+16)
//   B3: N=128, K=128 (+16); B4: N=16 (3 used: Y, U, V), K=128 (+16); frequencies as fp32 [20][2]
constexpr int kFrOffB0 = 0;
constexpr int kFrOffB1 = kFrOffB0 + 128 * 64 * 2;
constexpr int kFrOffB2 = kFrOffB1 + 96 * 144 * 2;
constexpr int kFrOffB3 = kFrOffB2 + 128 * 144 * 2;
constexpr int kFrOffB4 = kFrOffB3 + 128 * 144 * 2;
constexpr int kFrOffOnes = kFrOffB4 + 16 * 144 * 2;
constexpr int kFrOffFreq = kFrOffOnes + kOnesBytes;
constexpr int kFrImageBytes = kFrOffFreq + 20 * 2 * 4;   // 126,624
constexpr int kBarBytes = 80;   // [0] weights, [1..4] a_ready[slot][half], [5..8] d_full[slot][half]; TMEM at +72
constexpr int kSmemBytes = kFrImageBytes + kBarBytes + 128;

constexpr int kNumEpiWarps = 16;                   // 4 per TMEM lane quarter, 32 columns each
constexpr int kEpiArrivals = kNumEpiWarps;         // arrivals per a_ready phase
constexpr int kFirstEpiWarp = 4;
constexpr int kThreads = 32 * (kFirstEpiWarp + kNumEpiWarps);   // 640

// TMEM columns (512 allocated): slot s: D at 256 s (128 fp32 columns), then two 64-column fp16 A
// buffers (layer l reads buffer l % 2 while its epilogue writes buffer (l+1) % 2, so no epilogue write
// can race an MMA still reading A). The layer-1 input (K=16) is the first 8 columns of buffer 0.
// The bias K step reads its A operand (a constant-1 column) from shared memory instead of TMEM.
constexpr uint32_t kTmemCols = 512;
__host__ __device__ constexpr uint32_t d_col(int s) { return 256u * s; }
__host__ __device__ constexpr uint32_t a_col(int s, int buf) { return 256u * s + 128u + 64u * buf; }

// instruction descriptor: D f32, A/B f16, K-major both, M=128, N given
__host__ __device__ constexpr uint32_t idesc(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

inline void put_core(std::vector<uint8_t>& img, int base, int N, int n, int k, uint16_t v) {
    const int nb = n >> 3, r = n & 7, kb = k >> 3, c = k & 7;
    const int off = base + ((kb * (N / 8)) + nb) * 128 + r * 16 + c * 2;
    std::memcpy(&img[off], &v, 2);
}

}  // namespace nif

// The paper's NIF (blob: B[20][2], then W[out][in], b[out] of the 5 layers) -> kind-1 smem image.
void nif_build_smem_image_fr(const uint16_t* blob, std::vector<uint8_t>* image) {
    using namespace nif;
    std::vector<uint8_t>& img = *image;
    img.assign(kFrImageBytes, 0);
    size_t off = 0;
    float freq[40];
    for (int i = 0; i < 40; ++i) {
        const uint16_t h = blob[off++];
        const int e = (h >> 10) & 31, m = h & 1023;
        double v = e == 0 ? std::ldexp((double)m, -24) : std::ldexp((double)(m | 1024), e - 25);
        freq[i] = (float)((h & 0x8000) ? -v : v);
    }
    std::memcpy(&img[kFrOffFreq], freq, sizeof(freq));
    // layer 0: W0 [128][40] (inputs sin_0..19, cos_0..19), b0
    const uint16_t* W0 = blob + off; off += 128 * 40;
    const uint16_t* b0 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        for (int j = 0; j < 20; ++j) {
            put_core(img, kFrOffB0, 128, n, 8 + 2 * j, W0[n * 40 + j]);
            put_core(img, kFrOffB0, 128, n, 9 + 2 * j, W0[n * 40 + 20 + j]);
        }
        put_core(img, kFrOffB0, 128, n, 48, b0[n]);
    }
    // layer 1: W1 [88][128], b1 -> N padded to 96
    const uint16_t* W1 = blob + off; off += 88 * 128;
    const uint16_t* b1 = blob + off; off += 88;
    for (int n = 0; n < 88; ++n) {
        for (int k = 0; k < 128; ++k) put_core(img, kFrOffB1, 96, n, k, W1[n * 128 + k]);
        put_core(img, kFrOffB1, 96, n, 128, b1[n]);
    }
    // layer 2: W2 [128][128] over [h1 (88), sin (20), cos (20)] -> Fourier inputs interleaved
    const uint16_t* W2 = blob + off; off += 128 * 128;
    const uint16_t* b2 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        for (int k = 0; k < 88; ++k) put_core(img, kFrOffB2, 128, n, k, W2[n * 128 + k]);
        for (int j = 0; j < 20; ++j) {
            put_core(img, kFrOffB2, 128, n, 88 + 2 * j, W2[n * 128 + 88 + j]);
            put_core(img, kFrOffB2, 128, n, 89 + 2 * j, W2[n * 128 + 108 + j]);
        }
        put_core(img, kFrOffB2, 128, n, 128, b2[n]);
    }
    // layer 3
    const uint16_t* W3 = blob + off; off += 128 * 128;
    const uint16_t* b3 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        for (int k = 0; k < 128; ++k) put_core(img, kFrOffB3, 128, n, k, W3[n * 128 + k]);
        put_core(img, kFrOffB3, 128, n, 128, b3[n]);
    }
    // layer 4: W4 [3][128] -> N padded to 16
    const uint16_t* W4 = blob + off; off += 3 * 128;
    const uint16_t* b4 = blob + off; off += 3;
    for (int n = 0; n < 3; ++n) {
        for (int k = 0; k < 128; ++k) put_core(img, kFrOffB4, 16, n, k, W4[n * 128 + k]);
        put_core(img, kFrOffB4, 16, n, 128, b4[n]);
    }
    for (int m = 0; m < 128; ++m) put_core(img, kFrOffOnes, 128, m, 0, 0x3C00);
}

// ---------------------------------------------------------------------------------------------
// The fused kernel
// ---------------------------------------------------------------------------------------------
// Per-layer MMA layout: B tile base, K-direction core-matrix stride (LBO = N/8 * 128 B), N of the low and
// high column halves.
struct LayerDesc {
    uint32_t base, lbo;
    int n_lo, n_hi;
};
__device__ __forceinline__ LayerDesc layer_desc(int layer) {
    using namespace nif;
    if (layer == 1) return {(uint32_t)kFrOffB1, 1536u, 64, 32};
    if (layer == 2) return {(uint32_t)kFrOffB2, 2048u, 64, 64};
    if (layer == 3) return {(uint32_t)kFrOffB3, 2048u, 64, 64};
    return {(uint32_t)kFrOffB4, 256u, 16, 0};
}

template <bool kDebug>
__global__ void __launch_bounds__(nif::kThreads, 1)
    nif_fr_kernel(const uint8_t* __restrict__ g_image, const float4* __restrict__ esc,
                     const float4* __restrict__ esc_beta, const uint32_t* __restrict__ count, float* __restrict__ out,
                     float* __restrict__ dbg, int dir_input) {
    using namespace nif;
    constexpr int kImg = kFrImageBytes;
    constexpr uint32_t kOnesOff = kFrOffOnes;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* image = smem;
    // [0] weights, [1..4] a_ready[slot][column half], [5..8] d_full[slot][column half]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kFrImageBytes);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kFrImageBytes + 72);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t n_rows = *count;
    const uint32_t n_tiles = (n_rows + kTileM - 1) / kTileM;
    const uint32_t bar_w = smem_u32(&bars[0]);

    if (warp == 1 && lane == 0) {
        mbar_init(bar_w, 1);
        for (int b = 1; b < 5; ++b) mbar_init(smem_u32(&bars[b]), kEpiArrivals / 2);
        for (int b = 5; b < 9; ++b) mbar_init(smem_u32(&bars[b]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 1 && lane == 0 && blockIdx.x < n_tiles) {
        // stage the whole weight image once (bulk TMA copy, complete_tx on bar_w)
        mbar_expect_tx(bar_w, (uint32_t)kImg);
        constexpr int kChunk = 16384;
        for (int off = 0; off < kImg; off += kChunk) {
            const int bytes = (kImg - off) < kChunk ? (kImg - off) : kChunk;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(image + off)),
                "l"(g_image + off), "r"(bytes), "r"(bar_w)
                : "memory");
        }
    }

    if (warp == 0) {
        if (blockIdx.x < n_tiles) {
            // ===== MMA issuer: warp 0 walks the schedule, one elected lane issues =====
            // Layer l reads A buffer l % 2. Each layer runs as two column halves with their own commit
            // barrier; the low half's K steps 0-3 (A columns 0-31, written by the low-half epilogue
            // warps) start before the high half of A is ready.
            mbar_wait(bar_w, 0);
            const uint32_t img = smem_u32(image);
            const uint64_t ones = smem_desc(img + kOnesOff, 2048, 128);
            uint32_t a_phase[2] = {0, 0};
            for (uint32_t i = 0;; i += 2) {
                const uint32_t t0 = blockIdx.x + i * gridDim.x;
                if (t0 >= n_tiles) break;
                const int nslots = (t0 + gridDim.x < n_tiles) ? 2 : 1;
                for (int layer = 0; layer < 5; ++layer) {
                    for (int s = 0; s < nslots; ++s) {
                        const uint32_t bar_alo = smem_u32(&bars[1 + 2 * s]), bar_ahi = smem_u32(&bars[2 + 2 * s]);
                        const uint32_t bar_lo = smem_u32(&bars[5 + 2 * s]), bar_hi = smem_u32(&bars[6 + 2 * s]);
                        const uint32_t dt = tmem + d_col(s);
                        const uint32_t at = tmem + a_col(s, layer & 1);
                        mbar_wait(bar_alo, a_phase[s]);
                        tc_fence_after();
                        if (layer == 0) {
                            mbar_wait(bar_ahi, a_phase[s]);
                            tc_fence_after();
                            if (elect_one()) {
                                // Fourier features in A columns 40..63 (K' 0..47) + bias step
#pragma unroll
                                for (int half = 0; half < 2; ++half) {
                                    const uint32_t b0 = img + kFrOffB0 + 1024 * half;
#pragma unroll
                                    for (int k = 0; k < 3; ++k)
                                        mma_ts(dt + 64 * half, at + 40 + 8 * k, smem_desc(b0 + k * 2 * 2048, 2048, 128),
                                               idesc(64), k > 0);
                                    mma_ss(dt + 64 * half, ones, smem_desc(b0 + 6 * 2048, 2048, 128), idesc(64), 1);
                                    mma_commit(half ? bar_hi : bar_lo);
                                }
                            }
                        } else {
                            const LayerDesc L = layer_desc(layer);
                            const uint32_t base = img + L.base, lbo = L.lbo;
                            const uint32_t id_lo = idesc(L.n_lo);
                            if (elect_one()) {
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    mma_ts(dt, at + 8 * k, smem_desc(base + k * 2 * lbo, lbo, 128), id_lo, k > 0);
                            }
                            __syncwarp();
                            mbar_wait(bar_ahi, a_phase[s]);
                            tc_fence_after();
                            if (elect_one()) {
#pragma unroll
                                for (int k = 4; k < 8; ++k)
                                    mma_ts(dt, at + 8 * k, smem_desc(base + k * 2 * lbo, lbo, 128), id_lo, 1);
                                mma_ss(dt, ones, smem_desc(base + 16 * lbo, lbo, 128), id_lo, 1);   // + bias
                                mma_commit(bar_lo);
                                if (L.n_hi > 0) {
                                    const uint32_t id_hi = idesc(L.n_hi);
#pragma unroll
                                    for (int k = 0; k < 8; ++k)
                                        mma_ts(dt + 64, at + 8 * k, smem_desc(base + 1024 + k * 2 * lbo, lbo, 128), id_hi,
                                               k > 0);
                                    mma_ss(dt + 64, ones, smem_desc(base + 1024 + 16 * lbo, lbo, 128), id_hi, 1);
                                }
                                mma_commit(bar_hi);
                            }
                        }
                        a_phase[s] ^= 1;
                        __syncwarp();
                    }
                }
            }
        }
    } else if (warp >= kFirstEpiWarp) {
        // ===== epilogue warps =====
        // All 16 epilogue warps work on one (slot, layer) at a time, in the MMA's issue order, so the
        // tensor core runs the other slot's layer while this one's activations are computed. Warp w
        // owns TMEM lane quarter w % 4 (hardware rule) and the 32-column block cb of the 128 columns.
        const int e = warp - kFirstEpiWarp;
        const int cb = e >> 2;                        // column block 0..3
        const int q = warp & 3;                       // TMEM lane quarter
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        const float* freq = reinterpret_cast<const float*>(image + kFrOffFreq);
        uint32_t d_phase[2] = {0, 0};
        float4 ent[2] = {make_float4(0.5f, 0.5f, 0.0f, 0.0f), make_float4(0.5f, 0.5f, 0.0f, 0.0f)};
        auto row_of = [&](uint32_t tile) { return tile * kTileM + 32 * q + lane; };
        auto write_a0 = [&](int s, float4 en) {
            const uint32_t a0 = tmem + a_col(s, 0) + lane_addr;
            {
                // Fourier features (sin_j, cos_j) of 2 pi B_j.(u, v) into A column 44 + j; the four warps
                // of a lane quarter split the 20 frequencies (4 / 8 / 8) and zero columns 40..43
                auto feat = [&](int j) {
                    const float p = fmaf(freq[2 * j], en.x, freq[2 * j + 1] * en.y);
                    const float r = p - rintf(p);                  // exact-range turns in [-1/2, 1/2]
                    float sn, cs;
                    __sincosf(6.28318530717958647692f * r, &sn, &cs);
                    return pack_half2(sn, cs);
                };
                uint32_t v[8];
                if (cb == 0) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = feat(j);
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a0 + 44), "r"(v[0]),
                                 "r"(v[1]), "r"(v[2]), "r"(v[3])
                                 : "memory");
                } else if (cb == 3) {
                    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%1,%1,%1};" ::"r"(a0 + 40), "r"(0u)
                                 : "memory");
                } else {
                    const int j0 = cb == 1 ? 4 : 12;
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = feat(j0 + j);
                    tmem_st8(a0 + 44 + j0, v);
                }
            }
        };
        // queue entry -> (u, v, -, slot): the render queues escape directions (d.xyz, slot) and the
        // query hook (u, v, 0, slot)
        auto load_ent = [&](uint32_t tile) {
            const uint32_t row = row_of(tile);
            float4 en = (tile < n_tiles && row < n_rows) ? __ldg(esc + row) : make_float4(0.5f, 0.5f, 0.0f, 0.0f);
            if (dir_input && tile < n_tiles && row < n_rows)
                equirect_f32(make_float3(en.x, en.y, en.z), en.x, en.y);
            return en;
        };
        // prologue: layer-1 inputs of the first tile pair (the frequencies are part of the weight image)
        if (blockIdx.x < n_tiles) mbar_wait(bar_w, 0);
        for (int s = 0; s < 2; ++s) {
            const uint32_t tile = blockIdx.x + s * gridDim.x;
            ent[s] = load_ent(tile);
            if (tile < n_tiles) write_a0(s, ent[s]);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
            if (blockIdx.x < n_tiles) mbar_arrive(smem_u32(&bars[1 + (cb >> 1)]));
            if (blockIdx.x + gridDim.x < n_tiles) mbar_arrive(smem_u32(&bars[3 + (cb >> 1)]));
        }
        for (uint32_t i = 0;; i += 2) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = (t0 + gridDim.x < n_tiles) ? 2 : 1;
            // prefetch: this pair's throughputs (cb == 0) and the next pair's queue entries
            float4 beta[2] = {make_float4(0, 0, 0, 0), make_float4(0, 0, 0, 0)};
            float4 ent_next[2] = {ent[0], ent[1]};
            for (int s = 0; s < nslots; ++s) {
                const uint32_t tile = t0 + s * gridDim.x;
                const uint32_t row = row_of(tile);
                if (cb == 0 && row < n_rows) beta[s] = __ldg(esc_beta + row);
                ent_next[s] = load_ent(tile + 2 * gridDim.x);
            }
            for (int layer = 0; layer < 5; ++layer) {
                for (int s = 0; s < nslots; ++s) {
                    const uint32_t tile = t0 + s * gridDim.x;
                    const uint32_t row = row_of(tile);
                    const bool valid = row < n_rows;
                    const uint32_t dt = tmem + d_col(s) + lane_addr;
                    const uint32_t at = tmem + a_col(s, (layer + 1) & 1) + lane_addr;   // next layer's A
                    const uint32_t dph = d_phase[s];
                    d_phase[s] ^= 1;
                    mbar_wait(smem_u32(&bars[5 + 2 * s + (cb >> 1)]), dph);
                    tc_fence_after();
                    bool arrive = true;
                    if (layer < 4) {
                        // hidden layer: D (fp32) -> ReLU -> fp16 -> A (this warp's 32 columns). Layer 1:
                        // only D columns 0..87 are units (A columns 0..43); A columns 44..63 keep the
                        // Fourier features for the concat skip.
                        const int col = 32 * cb;
                        const bool skip = layer == 1 && cb == 3;
                        if (!skip) {
                            uint32_t v[32];
                            TMEM_LD32(dt + col, v);
                            tmem_wait_ld_dep(v);
                            if (kDebug && valid) {
                                for (int j = 0; j < 32; ++j)
                                    dbg[((size_t)layer * n_rows + row) * kHid + col + j] = __uint_as_float(v[j]);
                            }
                            uint32_t p[16];
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                p[j] = relu_pack(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
                            if (layer == 1 && cb == 2) {
                                tmem_st8(at + 32, p);        // units 64..79
                                asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(at + 40),
                                             "r"(p[8]), "r"(p[9]), "r"(p[10]), "r"(p[11])
                                             : "memory");   // units 80..87
                            } else {
                                TMEM_ST16(at + col / 2, p);
                            }
                        }
                    } else {
                        // output layer: y = D[:, 0:3]; radiance = beta * exp(y); then the layer-1
                        // input of this slot's next tile (if any) into the A region
                        const uint32_t next = tile + 2 * gridDim.x;
                        if (cb == 0) {
                            uint32_t v[4];
                            tmem_ld4(dt, v);
                            tmem_wait_ld_dep4(v);
                            if (valid) {
                                const uint32_t slot = __float_as_uint(ent[s].w);
                                float y0 = __uint_as_float(v[0]), y1 = __uint_as_float(v[1]), y2 = __uint_as_float(v[2]);
                                if (kDebug) {
                                    dbg[((size_t)4 * n_rows + row) * kHid + 0] = y0;
                                    dbg[((size_t)4 * n_rows + row) * kHid + 1] = y1;
                                    dbg[((size_t)4 * n_rows + row) * kHid + 2] = y2;
                                }
                                {
                                    // fixed BT.601 YUV -> RGB colour layer, log space
                                    const float Y = y0, U = y1, V = y2;
                                    y0 = fmaf(1.13983f, V, Y);
                                    y1 = fmaf(-0.58060f, V, fmaf(-0.39465f, U, Y));
                                    y2 = fmaf(2.03211f, U, Y);
                                }
                                out[3 * (size_t)slot + 0] = beta[s].x * __expf(y0);
                                out[3 * (size_t)slot + 1] = beta[s].y * __expf(y1);
                                out[3 * (size_t)slot + 2] = beta[s].z * __expf(y2);
                            }
                        }
                        ent[s] = ent_next[s];
                        if (next < n_tiles) write_a0(s, ent[s]);
                        arrive = next < n_tiles;
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0 && arrive) mbar_arrive(smem_u32(&bars[1 + 2 * s + (cb >> 1)]));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev & 63;
}

int num_sms() {
    static std::atomic<int> n[64];
    const int dev = current_device();
    int v = n[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        n[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

cudaError_t ensure_dyn_smem(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> done;   // (device, kernel) -> bytes configured
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(mu);
    int& have = done[{dev, kernel}];
    if (have >= bytes) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

// ---------------------------------------------------------------------------------------------
// The paper's NIF on the SIREN kernel's schedule (round 2, PT_NIF_FR3): three 128-ray tiles in flight,
// layer groups rotating over two accumulator regions, two 8-warp epilogue teams (team t = region t), one
// MMA issuer per region with single-waiter barriers, full-N layers (one commit per layer). Layers:
//   stage 0 (L0): the tile's 40 Fourier features from shared memory (SS, K' = 48) + bias -> 128 units
//   stage 1 (L1): 128 -> 96 (88 used) TS + bias; its epilogue writes relu(h1) (88) and features 0..3
//                 (sin/cos, the K step that straddles the concat boundary) into A
//   stage 2 (L2): concat skip: 6 TS K steps (h1 + features 0..3) + 2 SS K steps (features 4..19 read
//                 from the feature tile) + bias -> 128
//   stage 3 (L3): 128 -> 128 TS + bias
//   output  (L4): 128 -> 16 (Y, U, V used) TS + bias into O(s), issued with the slot's next L0; the
//                 slot's 4 output warps apply BT.601 YUV -> RGB, exp, beta.
// The producer warps compute the features (equirect of the queued direction, then sin/cos of
// 2 pi B.(u, v) in turns) into the slot's feature tile, which stays live until L2 of the tile is done.
// ---------------------------------------------------------------------------------------------
#ifndef PT_NIF_FR3
#define PT_NIF_FR3 1
#endif
namespace fr3 {
using nif::kFrImageBytes;
constexpr int kTileM = 128;
constexpr int kSlots = 3;
constexpr int kDRegions = 2;
constexpr int kIssuers = 2;
constexpr int kTeamWarps = 8;
constexpr int kNumEpiWarps = 16;
// four producer warps (one per SM sub-partition): 40 sin/cos per row are the producers' work, and two
// warps measured too slow to keep three tiles in flight (6.4 G inferences/s)
constexpr int kProducerWarp0 = 2;
#ifndef PT_FR3_DIAG
#define PT_FR3_DIAG 0   // diagnostic builds only: 1 = producers skip the sin/cos
#endif
#ifndef PT_FR3_PRODUCERS
#define PT_FR3_PRODUCERS 4
#endif
constexpr int kProducerWarps = PT_FR3_PRODUCERS;
constexpr int kProducerThreads = 32 * kProducerWarps;
constexpr int kFirstEpiWarp = kProducerWarp0 + kProducerWarps;   // 6
constexpr int kThreads = 32 * (kFirstEpiWarp + kNumEpiWarps);     // 704
constexpr int kFtBytes = 128 * 48 * 2;                          // feature tile: 128 rows x K' 48 (fp16)
// feature tiles per slot: 2 = double-buffered by round parity, so the producers can stage a slot's next
// tile before the current one's concat layer (L2) has read its features
#ifndef PT_FR3_FT_BUFS
#define PT_FR3_FT_BUFS 2
#endif
constexpr int kFtBufs = PT_FR3_FT_BUFS;
constexpr int kNumFt = kSlots * kFtBufs;
constexpr int kOffBars = ((kFrImageBytes + 1023) / 1024) * 1024;
constexpr int kNumBars = 1 + (1 + kIssuers) * kSlots + 2 * kNumFt + 2 * kDRegions;
constexpr int kOffTmemSlot = kOffBars + 8 * kNumBars;
constexpr int kOffFt = ((kOffTmemSlot + 16 + 1023) / 1024) * 1024;
constexpr int kSmemBytes = kOffFt + kNumFt * kFtBytes;
__host__ __device__ constexpr int ft_buf(int s, uint32_t i) {   // slot s in the round starting at i (i += kSlots)
    return s + kSlots * (int)((i / kSlots) % kFtBufs);
}
enum {
    kBarW = 0,
    kBarAReady = 1,   // a_ready(s, consumer p) at kBarAReady + kIssuers s + p
    kBarFtFull = kBarAReady + kIssuers * kSlots,   // per feature tile (kNumFt)
    kBarFtEmpty = kBarFtFull + kNumFt,
    kBarOFull = kBarFtEmpty + kNumFt,
    kBarDFull = kBarOFull + kSlots,
    kBarDEmpty = kBarDFull + kDRegions
};
constexpr uint32_t kTmemCols = 512;
__host__ __device__ constexpr uint32_t a_col(int s) { return 64u * s; }
__host__ __device__ constexpr uint32_t o_col(int s) { return 192u + 16u * s; }
__host__ __device__ constexpr uint32_t d_col(int j) { return 256u + 128u * j; }
__device__ __forceinline__ int slots_in_round(uint32_t t0, uint32_t n_tiles) {
    int n = 1;
    while (n < kSlots && t0 + (uint32_t)n * gridDim.x < n_tiles) ++n;
    return n;
}
// fp8 image (reading R24: e4m3 weights, features and activations; fp32 biases): K-major 8-bit core
// matrices (8 rows x 16 B = 16 K elements), K = 32 per tcgen05.mma kind::f8f6f4. L0's K' order is the
// feature tile's: [g_8 .. g_39, g_0 .. g_7, 0 x 24] (g = sin_0..19, cos_0..19), so the concat layer's
// last K step reads g_8..39 straight from the tile and g_0..7 ride in A after h1.
constexpr int k8OffB0 = 0;                              // N = 128, K' = 64
constexpr int k8OffB1 = k8OffB0 + 128 * 64;             // N = 96 (88 used), K = 128
constexpr int k8OffB2 = k8OffB1 + 96 * 128;             // N = 128, K = [h1 (88), g (40)]
constexpr int k8OffB3 = k8OffB2 + 128 * 128;
constexpr int k8OffB4 = k8OffB3 + 128 * 128;            // N = 16 (3 used), K = 128
constexpr int k8OffBias = k8OffB4 + 16 * 128;           // fp32: b0[128] b1[96] b2[128] b3[128] b4[16]
constexpr int k8OffFreq = k8OffBias + 496 * 4;          // fp32 [20][2]
constexpr int k8ImageBytes = k8OffFreq + 40 * 4;
__host__ __device__ constexpr int k8bias(int l) {       // float offset of layer l's bias
    return l == 0 ? 0 : l == 1 ? 128 : l == 2 ? 224 : l == 3 ? 352 : 480;
}
constexpr int k8FtBytes = 128 * 64;                     // feature tile: 128 rows x K' 64 (e4m3)
}  // namespace fr3

// The paper's NIF -> the fp8 image of nif_fr3_kernel<kFp8 = true>
void nif_build_smem_image_fr8(const uint16_t* blob, std::vector<uint8_t>* image) {
    using namespace fr3;
    std::vector<uint8_t>& img = *image;
    img.assign(k8ImageBytes, 0);
    auto put8 = [&](int base, int N, int n, int k, uint8_t v) {
        img[base + ((k >> 4) * (N / 8) + (n >> 3)) * 128 + (n & 7) * 16 + (k & 15)] = v;
    };
    auto q8 = [&](uint16_t h) { return float_to_e4m3(half_to_float(h)); };
    float* bias = reinterpret_cast<float*>(&img[k8OffBias]);
    float* freq = reinterpret_cast<float*>(&img[k8OffFreq]);
    size_t off = 0;
    for (int i = 0; i < 40; ++i) freq[i] = half_to_float(blob[off++]);
    // L0: W0 [128][40] over g = (sin_0..19, cos_0..19); K' k < 32 -> g_{k+8}, 32 <= k < 40 -> g_{k-32}
    const uint16_t* W0 = blob + off; off += 128 * 40;
    const uint16_t* b0 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        for (int k = 0; k < 40; ++k) put8(k8OffB0, 128, n, k, q8(W0[n * 40 + (k < 32 ? k + 8 : k - 32)]));
        bias[k8bias(0) + n] = half_to_float(b0[n]);
    }
    const uint16_t* W1 = blob + off; off += 88 * 128;
    const uint16_t* b1 = blob + off; off += 88;
    for (int n = 0; n < 88; ++n) {
        for (int k = 0; k < 128; ++k) put8(k8OffB1, 96, n, k, q8(W1[n * 128 + k]));
        bias[k8bias(1) + n] = half_to_float(b1[n]);
    }
    const uint16_t* W2 = blob + off; off += 128 * 128;
    const uint16_t* b2 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        for (int k = 0; k < 128; ++k) put8(k8OffB2, 128, n, k, q8(W2[n * 128 + k]));   // [h1, g] in order
        bias[k8bias(2) + n] = half_to_float(b2[n]);
    }
    const uint16_t* W3 = blob + off; off += 128 * 128;
    const uint16_t* b3 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        for (int k = 0; k < 128; ++k) put8(k8OffB3, 128, n, k, q8(W3[n * 128 + k]));
        bias[k8bias(3) + n] = half_to_float(b3[n]);
    }
    const uint16_t* W4 = blob + off; off += 3 * 128;
    const uint16_t* b4 = blob + off; off += 3;
    for (int n = 0; n < 3; ++n) {
        for (int k = 0; k < 128; ++k) put8(k8OffB4, 16, n, k, q8(W4[n * 128 + k]));
        bias[k8bias(4) + n] = half_to_float(b4[n]);
    }
}

__device__ __forceinline__ uint32_t fr8_pack(float a, float b, float c, float d) {
    uint16_t lo, hi;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
    return (uint32_t)lo | ((uint32_t)hi << 16);
}
__device__ __forceinline__ uint32_t fr8_pack_relu(float a, float b, float c, float d) {
    uint16_t lo, hi;
    asm("cvt.rn.satfinite.relu.e4m3x2.f32 %0, %1, %2;" : "=h"(lo) : "f"(b), "f"(a));
    asm("cvt.rn.satfinite.relu.e4m3x2.f32 %0, %1, %2;" : "=h"(hi) : "f"(d), "f"(c));
    return (uint32_t)lo | ((uint32_t)hi << 16);
}

template <bool kDebug, bool kFp8>
__global__ void __launch_bounds__(fr3::kThreads, 1)
    nif_fr3_kernel(const uint8_t* __restrict__ g_image, const float4* __restrict__ esc,
                   const float4* __restrict__ esc_beta, const uint32_t* __restrict__ count, float* __restrict__ out,
                   float* __restrict__ dbg, int dir_input) {
    using namespace fr3;
    using nif::idesc;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBars);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffTmemSlot);
    auto bar = [&](int b) { return smem_u32(&bars[b]); };
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    pdl_trigger();

    if (warp == 1 && lane == 0) {
        mbar_init(bar(kBarW), 1);
        for (int s = 0; s < kSlots; ++s) {
            for (int p = 0; p < kIssuers; ++p) mbar_init(bar(kBarAReady + kIssuers * s + p), kTeamWarps);
            mbar_init(bar(kBarOFull + s), 1);
        }
        for (int b = 0; b < kNumFt; ++b) {
            mbar_init(bar(kBarFtFull + b), kProducerThreads);
            mbar_init(bar(kBarFtEmpty + b), 1);
        }
        for (int j = 0; j < kDRegions; ++j) {
            mbar_init(bar(kBarDFull + j), 1);
            mbar_init(bar(kBarDEmpty + j), kTeamWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    constexpr int kImg = kFp8 ? k8ImageBytes : kFrImageBytes;
    constexpr int kFt = kFp8 ? k8FtBytes : kFtBytes;
    if (warp == 1 && lane == 0) {
        mbar_expect_tx(bar(kBarW), (uint32_t)kImg);
        constexpr int kChunk = 16384;
        for (int off = 0; off < kImg; off += kChunk) {
            const int bytes = (kImg - off) < kChunk ? (kImg - off) : kChunk;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(smem + off)),
                "l"(g_image + off), "r"(bytes), "r"(bar(kBarW))
                : "memory");
        }
    }

    pdl_wait();
    const uint32_t n_rows = *count;
    const uint32_t n_tiles = (n_rows + kTileM - 1) / kTileM;

    if (warp < kIssuers) {
        // ===== MMA issuers: warp j issues the layer groups of D region j =====
        const uint32_t me = (uint32_t)warp;
        if (blockIdx.x < n_tiles) {
            mbar_wait(bar(kBarW), 0);
            const uint32_t img = smem_u32(smem);
            const uint64_t ones = smem_desc(img + nif::kFrOffOnes, 2048, 128);
            uint32_t a_phase = 0, f_phase = 0, e_phase = 0, pend = 0, out_by_me = 0;
            uint32_t g = 0;
            auto issue_out = [&](int s) {
                mbar_wait(bar(kBarAReady + kIssuers * s + (int)me), (a_phase >> s) & 1u);
                a_phase ^= 1u << s;
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t at = tmem + a_col(s);
                    if (kFp8) {
                        const uint32_t base = img + k8OffB4;   // b4 is added by the output warps
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            mma_ts_f8(tmem + o_col(s), at + 8 * k, smem_desc(base + k * 2 * 256, 256, 128), idesc(16), k > 0);
                    } else {
                        const uint32_t base = img + nif::kFrOffB4;
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            mma_ts(tmem + o_col(s), at + 8 * k, smem_desc(base + k * 2 * 256, 256, 128), idesc(16), k > 0);
                        mma_ss(tmem + o_col(s), ones, smem_desc(base + 16 * 256, 256, 128), idesc(16), 1);   // + bias
                    }
                    mma_commit(bar(kBarOFull + s));
                }
                __syncwarp();
            };
            for (uint32_t i = 0;; i += kSlots) {
                const uint32_t t0 = blockIdx.x + i * gridDim.x;
                if (t0 >= n_tiles) break;
                const int nslots = slots_in_round(t0, n_tiles);
                for (int stage = 0; stage < 4; ++stage) {
                    for (int s = 0; s < nslots; ++s, ++g) {
                        const int j = (int)(g & 1u);
                        if (stage == 3) {
                            const bool mine_out = ((g + (uint32_t)nslots) & 1u) == me;
                            out_by_me = mine_out ? (out_by_me | 1u << s) : (out_by_me & ~(1u << s));
                        }
                        if (stage == 0) pend |= 1u << s;
                        if ((uint32_t)j != me) continue;
                        if (stage == 0) {
                            if (i > 0) issue_out(s);
                            const int fb = ft_buf(s, i);
                            mbar_wait(bar(kBarFtFull + fb), (f_phase >> fb) & 1u);   // features staged
                            f_phase ^= 1u << fb;
                        } else {
                            mbar_wait(bar(kBarAReady + kIssuers * s + (int)me), (a_phase >> s) & 1u);
                            a_phase ^= 1u << s;
                        }
                        if (g >= (uint32_t)kDRegions) {
                            mbar_wait(bar(kBarDEmpty + j), (e_phase >> j) & 1u);
                            e_phase ^= 1u << j;
                        }
                        tc_fence_after();
                        const uint32_t dt = tmem + d_col(j);
                        const uint32_t ft = smem_u32(smem + kOffFt + ft_buf(s, i) * kFt);
                        if (kFp8 && elect_one()) {
                            // e4m3, K = 32 per MMA, no bias steps (the epilogue adds the fp32 biases)
                            const uint32_t at = tmem + a_col(s);
                            if (stage == 0) {
#pragma unroll
                                for (int k = 0; k < 2; ++k)
                                    mma_ss_f8(dt, smem_desc(ft + k * 2 * 2048, 2048, 128),
                                              smem_desc(img + k8OffB0 + k * 2 * 2048, 2048, 128), idesc(128), k > 0);
                            } else if (stage == 1) {
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    mma_ts_f8(dt, at + 8 * k, smem_desc(img + k8OffB1 + k * 2 * 1536, 1536, 128), idesc(96),
                                              k > 0);
                            } else if (stage == 2) {
#pragma unroll
                                for (int k = 0; k < 3; ++k)   // h1 (88) and g_0..7 from A
                                    mma_ts_f8(dt, at + 8 * k, smem_desc(img + k8OffB2 + k * 2 * 2048, 2048, 128), idesc(128),
                                              k > 0);
                                mma_ss_f8(dt, smem_desc(ft, 2048, 128), smem_desc(img + k8OffB2 + 3 * 2 * 2048, 2048, 128),
                                          idesc(128), 1);     // g_8..39: feature-tile K' 0..31
                            } else {
#pragma unroll
                                for (int k = 0; k < 4; ++k)
                                    mma_ts_f8(dt, at + 8 * k, smem_desc(img + k8OffB3 + k * 2 * 2048, 2048, 128), idesc(128),
                                              k > 0);
                            }
                            mma_commit(bar(kBarDFull + j));
                            if (stage == 2) mma_commit(bar(kBarFtEmpty + ft_buf(s, i)));
                        } else if (!kFp8 && elect_one()) {
                            const uint32_t at = tmem + a_col(s);
                            if (stage == 0) {
                                const uint32_t b0 = img + nif::kFrOffB0;
#pragma unroll
                                for (int k = 0; k < 3; ++k)
                                    mma_ss(dt, smem_desc(ft + k * 2 * 2048, 2048, 128),
                                           smem_desc(b0 + k * 2 * 2048, 2048, 128), idesc(128), k > 0);
                                mma_ss(dt, ones, smem_desc(b0 + 6 * 2048, 2048, 128), idesc(128), 1);
                            } else if (stage == 1) {
                                const uint32_t b1 = img + nif::kFrOffB1;
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                    mma_ts(dt, at + 8 * k, smem_desc(b1 + k * 2 * 1536, 1536, 128), idesc(96), k > 0);
                                mma_ss(dt, ones, smem_desc(b1 + 16 * 1536, 1536, 128), idesc(96), 1);
                            } else if (stage == 2) {
                                const uint32_t b2 = img + nif::kFrOffB2;
#pragma unroll
                                for (int k = 0; k < 6; ++k)
                                    mma_ts(dt, at + 8 * k, smem_desc(b2 + k * 2 * 2048, 2048, 128), idesc(128), k > 0);
#pragma unroll
                                for (int k = 6; k < 8; ++k)   // features 4..19: feature-tile K' 16..47
                                    mma_ss(dt, smem_desc(ft + (2 * k - 10) * 2048, 2048, 128),
                                           smem_desc(b2 + k * 2 * 2048, 2048, 128), idesc(128), 1);
                                mma_ss(dt, ones, smem_desc(b2 + 16 * 2048, 2048, 128), idesc(128), 1);
                            } else {
                                const uint32_t b3 = img + nif::kFrOffB3;
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                    mma_ts(dt, at + 8 * k, smem_desc(b3 + k * 2 * 2048, 2048, 128), idesc(128), k > 0);
                                mma_ss(dt, ones, smem_desc(b3 + 16 * 2048, 2048, 128), idesc(128), 1);
                            }
                            mma_commit(bar(kBarDFull + j));
                            if (stage == 2) mma_commit(bar(kBarFtEmpty + ft_buf(s, i)));   // feature tile free after L2
                        }
                        __syncwarp();
                    }
                }
            }
            for (int s = 0; s < kSlots; ++s)
                if ((pend >> s) & (out_by_me >> s) & 1u) issue_out(s);
        }
    } else if (warp >= kProducerWarp0 && warp < kFirstEpiWarp) {
        // ===== producers: the Fourier features of each tile into the slot's feature tile =====
        // row m, K' block kb (8 fp16) at kb * 2048 + 16 m; K' 0..7 zero, K' 8 + 2j / 9 + 2j = sin_j / cos_j
        const int p = threadIdx.x - 32 * kProducerWarp0;
        uint8_t* fts = smem + kOffFt;
        for (int m = p; m < kNumFt * 128; m += kProducerThreads) {
            // the K blocks no feature lands in: fp16 K' 0..7; fp8 K' 40..47 (second half of block 2), 48..63
            uint8_t* t = fts + (m >> 7) * kFt + 16 * (m & 127);
            if (kFp8) {
                *reinterpret_cast<uint4*>(t + 2 * 2048) = make_uint4(0, 0, 0, 0);
                *reinterpret_cast<uint4*>(t + 3 * 2048) = make_uint4(0, 0, 0, 0);
            } else {
                *reinterpret_cast<uint4*>(t) = make_uint4(0, 0, 0, 0);
            }
        }
        if (blockIdx.x < n_tiles) mbar_wait(bar(kBarW), 0);   // the frequencies are in the image
        const float* freq = reinterpret_cast<const float*>(smem + (kFp8 ? k8OffFreq : nif::kFrOffFreq));
        uint32_t e_phase = 0, filled = 0;
        // one row per producer thread: its queue entry for each slot's next tile is loaded a round ahead,
        // so the global-load latency overlaps the waits instead of each tile's production
        static_assert(kProducerThreads == 128, "one row per producer thread");
        auto load_row = [&](uint32_t tile) {
            const uint32_t row = tile * kTileM + (uint32_t)p;
            return (tile < n_tiles && row < n_rows) ? __ldg(esc + row) : make_float4(0.5f, 0.5f, 0.0f, 0.0f);
        };
        float4 en_pf[kSlots];
#pragma unroll
        for (int s = 0; s < kSlots; ++s) en_pf[s] = load_row(blockIdx.x + s * gridDim.x);
        for (uint32_t i = 0;; i += kSlots) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = slots_in_round(t0, n_tiles);
#pragma unroll
            for (int s = 0; s < kSlots; ++s) {
                if (s >= nslots) break;
                const uint32_t tile = t0 + s * gridDim.x;
                const int fb = ft_buf(s, i);
                if ((filled >> fb) & 1u) {
                    mbar_wait(bar(kBarFtEmpty + fb), (e_phase >> fb) & 1u);
                    e_phase ^= 1u << fb;
                }
                filled |= 1u << fb;
                const float4 en = en_pf[s];
                en_pf[s] = load_row(tile + kSlots * gridDim.x);
                {
                    const int m = p;
                    const uint32_t row = tile * kTileM + m;
                    float u = 0.5f, v = 0.5f;
                    if (row < n_rows) {
                        u = en.x;
                        v = en.y;
                        if (dir_input) equirect_f32(make_float3(en.x, en.y, en.z), u, v);
                    }
                    uint8_t* base = fts + fb * kFt + 16 * m;
                    if (kFp8) {
                        // g = (sin_0..19, cos_0..19) in e4m3; tile row = [g_8 .. g_39 | g_0 .. g_7 | 0]
                        float g[40];
#pragma unroll
                        for (int jj = 0; jj < 20; ++jj) {
                            const float pp = fmaf(freq[2 * jj], u, freq[2 * jj + 1] * v);
                            const float r = pp - rintf(pp);
                            __sincosf(6.28318530717958647692f * r, &g[jj], &g[20 + jj]);
                        }
                        uint32_t w[10];
#pragma unroll
                        for (int t = 0; t < 8; ++t) w[t] = fr8_pack(g[8 + 4 * t], g[9 + 4 * t], g[10 + 4 * t], g[11 + 4 * t]);
                        w[8] = fr8_pack(g[0], g[1], g[2], g[3]);
                        w[9] = fr8_pack(g[4], g[5], g[6], g[7]);
                        *reinterpret_cast<uint4*>(base) = make_uint4(w[0], w[1], w[2], w[3]);
                        *reinterpret_cast<uint4*>(base + 2048) = make_uint4(w[4], w[5], w[6], w[7]);
                        *reinterpret_cast<uint2*>(base + 2 * 2048) = make_uint2(w[8], w[9]);
                    } else {
                        uint32_t f[20];
#pragma unroll
                        for (int jj = 0; jj < 20; ++jj) {
                            const float pp = fmaf(freq[2 * jj], u, freq[2 * jj + 1] * v);
                            const float r = pp - rintf(pp);                  // exact-range turns in [-1/2, 1/2]
                            float sn, cs;
                            if (PT_FR3_DIAG == 1) { sn = r; cs = pp; }   // diagnostic: no sin/cos (wrong results)
                            else __sincosf(6.28318530717958647692f * r, &sn, &cs);
                            f[jj] = pack_half2(sn, cs);
                        }
#pragma unroll
                        for (int kb = 1; kb < 6; ++kb)
                            *reinterpret_cast<uint4*>(base + kb * 2048) =
                                make_uint4(f[4 * kb - 4], f[4 * kb - 3], f[4 * kb - 2], f[4 * kb - 1]);
                    }
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
                mbar_arrive(bar(kBarFtFull + fb));
            }
        }
    } else if (warp >= kFirstEpiWarp) {
        // ===== epilogue teams (see the SIREN kernel): team t runs the groups of D region t =====
        const int e = warp - kFirstEpiWarp;
        const int team = e >> 3;
        const int h = (e >> 2) & 1;
        const int q = warp & 3;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        const int my_slot = 2 * h + team;
        const bool out_warp = my_slot < kSlots;
        uint32_t d_phase = 0, o_phase = 0;
        float4 beta = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        uint32_t oslot = 0, prow = 0;
        bool ovalid = false, pend = false;
        auto output = [&](uint32_t dbg_row) {
            mbar_wait(bar(kBarOFull + my_slot), o_phase);
            o_phase ^= 1;
            tc_fence_after();
            uint32_t v[4];
            tmem_ld4(tmem + o_col(my_slot) + lane_addr, v);
            tmem_wait_ld_dep4(v);
            if (ovalid) {
                float y0 = __uint_as_float(v[0]), y1 = __uint_as_float(v[1]), y2 = __uint_as_float(v[2]);
                if (kFp8) {
                    const float* b4 = reinterpret_cast<const float*>(smem + k8OffBias) + k8bias(4);
                    y0 += b4[0];
                    y1 += b4[1];
                    y2 += b4[2];
                }
                if (kDebug) {
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 0] = y0;
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 1] = y1;
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 2] = y2;
                }
                // fixed BT.601 YUV -> RGB colour layer, log space
                const float Y = y0, U = y1, V = y2;
                y0 = fmaf(1.13983f, V, Y);
                y1 = fmaf(-0.58060f, V, fmaf(-0.39465f, U, Y));
                y2 = fmaf(2.03211f, U, Y);
                out[3 * (size_t)oslot + 0] = beta.x * __expf(y0);
                out[3 * (size_t)oslot + 1] = beta.y * __expf(y1);
                out[3 * (size_t)oslot + 2] = beta.z * __expf(y2);
            }
        };
        const uint32_t dreg = tmem + d_col(team) + lane_addr + 64u * (uint32_t)h;
        const int m_row = 32 * q + lane;   // this thread's row of the tile
        uint32_t g = 0;
        for (uint32_t i = 0;; i += kSlots) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = slots_in_round(t0, n_tiles);
            for (int stage = 0; stage < 4; ++stage) {
                for (int s = 0; s < nslots; ++s, ++g) {
                    if ((int)(g & 1u) != team) continue;
                    const uint32_t tile = t0 + s * gridDim.x;
                    const uint32_t row = tile * kTileM + m_row;
                    const bool valid = row < n_rows;
                    mbar_wait(bar(kBarDFull + team), d_phase);
                    d_phase ^= 1;
                    tc_fence_after();
                    const uint32_t areg = tmem + a_col(s) + lane_addr + (kFp8 ? 16u : 32u) * (uint32_t)h;
                    // L1 has 96 columns: the high half loads only its first 32 (units 64..87 + padding)
                    const int nchunk = (stage == 1 && h == 1) ? 1 : 2;
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if (c >= nchunk) break;
                        uint32_t v[32];
                        uint32_t pk[16];
                        TMEM_LD32(dreg + 32u * (uint32_t)c, v);
                        tmem_wait_ld_dep(v);
                        if (c == nchunk - 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(bar(kBarDEmpty + team));
                        }
                        if (kDebug && valid)
                            for (int k = 0; k < 32; ++k)
                                dbg[((size_t)stage * n_rows + row) * 128 + 64 * h + 32 * c + k] = __uint_as_float(v[k]);
                        if (kFp8) {
                            // + the layer's fp32 bias, ReLU, e4m3 (4 per A column)
                            const float4* bp = reinterpret_cast<const float4*>(smem + k8OffBias) +
                                               (k8bias(stage) + 64 * h + 32 * c) / 4;
#pragma unroll
                            for (int t = 0; t < 8; ++t) {
                                const float4 b = bp[t];
                                const float2 x01 = __fadd2_rn(make_float2(__uint_as_float(v[4 * t]), __uint_as_float(v[4 * t + 1])),
                                                              make_float2(b.x, b.y));
                                const float2 x23 = __fadd2_rn(make_float2(__uint_as_float(v[4 * t + 2]), __uint_as_float(v[4 * t + 3])),
                                                              make_float2(b.z, b.w));
                                pk[t] = fr8_pack_relu(x01.x, x01.y, x23.x, x23.y);
                            }
                            if (stage == 1 && h == 1) {
                                // units 64..87 -> A columns 16..21; g_0..7 (feature-tile K' 32..39) -> 22..23
                                const uint2 fw = *reinterpret_cast<const uint2*>(smem + kOffFt + ft_buf(s, i) * kFt + 2 * 2048 + 16 * m_row);
                                pk[6] = fw.x;
                                pk[7] = fw.y;
                            }
                            tmem_st8(areg + 8u * (uint32_t)c, pk);
                            continue;
                        }
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            pk[k] = relu_pack(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                        if (stage == 1 && h == 1) {
                            // units 64..87 -> A columns 32..43; features 0..3 (feature-tile K' 8..15, the K
                            // step straddling the concat boundary) -> A columns 44..47
                            const uint4 fw = *reinterpret_cast<const uint4*>(smem + kOffFt + ft_buf(s, i) * kFt + 2048 + 16 * m_row);
                            pk[12] = fw.x;
                            pk[13] = fw.y;
                            pk[14] = fw.z;
                            pk[15] = fw.w;
                        }
                        TMEM_ST16(areg + 16u * (uint32_t)c, pk);
                    }
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar(kBarAReady + kIssuers * s + (int)((g + (uint32_t)nslots) & 1u)));
                    if (stage == 0 && s == my_slot && pend) output(prow);
                    if (stage == 2 && s == my_slot) {
                        ovalid = valid;
                        prow = row;
                        if (valid) {
                            beta = __ldg(esc_beta + row);
                            oslot = __float_as_uint(__ldg(esc + row).w);
                        }
                        pend = true;
                    }
                }
            }
        }
        if (out_warp && pend) output(prow);
    }
    if (warp == 1 && lane == 0 && blockIdx.x >= n_tiles) mbar_wait(bar(kBarW), 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

template <bool kDebug, bool kFp8 = false>
static cudaError_t nif_fr3_launch_t(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                                    int grid, float* out, float* dbg, int dir_input, cudaStream_t st) {
    cudaError_t e = ensure_dyn_smem((const void*)nif_fr3_kernel<kDebug, kFp8>, fr3::kSmemBytes);
    if (e != cudaSuccess) return e;
    return launch_pdl(nif_fr3_kernel<kDebug, kFp8>, dim3(grid), dim3(fr3::kThreads), fr3::kSmemBytes, st,
                      (const uint8_t*)nif->d_smem_image, esc, esc_beta, count, out, dbg, dir_input);
}

template <bool kDebug>
static cudaError_t nif_fr_launch_t(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                                   int grid, float* out, float* dbg, int dir_input, cudaStream_t st) {
    using namespace nif;
    cudaError_t e = ensure_dyn_smem((const void*)nif_fr_kernel<kDebug>, kSmemBytes);
    if (e != cudaSuccess) return e;
    nif_fr_kernel<kDebug><<<grid, kThreads, kSmemBytes, st>>>((const uint8_t*)nif->d_smem_image, esc, esc_beta, count,
                                                               out, dbg, dir_input);
    return cudaGetLastError();
}

cudaError_t launch_siren(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count, int grid,
                         float* out, float* dbg, int dir_input, cudaStream_t st);

// one persistent CTA per SM (or per tile when there are fewer tiles); the row count is read on device
static cudaError_t nif_launch_impl(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                                   int64_t max_rows, float* out, float* dbg, int dir_input, cudaStream_t st) {
    int64_t tiles = (max_rows + 127) / 128;
    int grid = num_sms();
    if (tiles < grid) grid = (int)(tiles > 0 ? tiles : 1);
    if (nif->kind == PT_NIF_FR_FAMILY) {
        if (dbg) return cudaErrorNotSupported;
        // (128, 4) fp16 = the paper's network: the three-tile kernel (unless the tests force the layered path)
        const char* env = std::getenv("PT_MLP_LAYERED");
        if (PT_NIF_FR3 && nif->d_smem_image && !(env && env[0] == '1'))
            return nif->mlp_fp8 ? nif_fr3_launch_t<false, true>(nif, esc, esc_beta, count, grid, out, nullptr, dir_input, st)
                                : nif_fr3_launch_t<false, false>(nif, esc, esc_beta, count, grid, out, nullptr, dir_input, st);
        return launch_mlp(const_cast<pt_nif*>(nif), esc, esc_beta, count, max_rows, out, dir_input, st);
    }
    if (nif->kind == PT_NIF_FOURIER_RELU) {
        if (PT_NIF_FR3)
            return dbg ? nif_fr3_launch_t<true>(nif, esc, esc_beta, count, grid, out, dbg, dir_input, st)
                       : nif_fr3_launch_t<false>(nif, esc, esc_beta, count, grid, out, dbg, dir_input, st);
        return dbg ? nif_fr_launch_t<true>(nif, esc, esc_beta, count, grid, out, dbg, dir_input, st)
                   : nif_fr_launch_t<false>(nif, esc, esc_beta, count, grid, out, dbg, dir_input, st);
    }
    return launch_siren(nif, esc, esc_beta, count, grid, out, dbg, dir_input, st);
}

cudaError_t launch_nif(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                       int64_t max_rows, float* out, int dir_input, cudaStream_t st) {
    return nif_launch_impl(nif, esc, esc_beta, count, max_rows, out, nullptr, dir_input, st);
}

cudaError_t launch_nif_debug(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                             int64_t rows, float* out, float* dbg, cudaStream_t st) {
    return nif_launch_impl(nif, esc, esc_beta, count, rows, out, dbg, 0, st);
}

}  // namespace pt
