// siren_kernel.cu -- fused SIREN HDR-NIF inference on sm_100a tensor cores (tcgen05 + TMEM), step S5.
//
// What it computes (BASELINE.json SIREN; readings R1-R3, R14, R15):
//   for every escaped ray (direction d, or (u, v) from the query hook) with throughput beta:
//     (u, v) = equirect(d); x0 = (2u-1, 2v-1); h1 = sin(W1' x0 + b1'); h_{k+1} = sin(W'_{k+1} h_k + b'_{k+1})
//     (k = 1..3); y = W5 h4 + b5; radiance = beta * exp(y)   (written to the path's own wave slot)
//
// Design: the layers are computed TRANSPOSED, D^T = W . H^T. One persistent CTA per SM
// holds the four sine layers' weights in TMEM as the A operand (lanes = output features; loaded once per
// CTA from the shared-memory image) and two 128-ray tiles ("slots") in flight:
//   * Layer 1 (2 -> 128): one TS MMA, K = 16, B = a K-major shared-memory tile staged by two producer
//     warps (equirect, hi/lo split of x0, constant-1 column against b1 in A).
//   * Layers 2-4 (128 -> 128): 8 TS MMAs, M = N = 128, K = 16 each; B = the previous layer's fp16
//     activations, an MN-major shared-memory tile (rays contiguous) that the epilogue writes with 16-byte
//     st.shared -- so the epilogue reads TMEM (D) but never writes it. The bias is one register per
//     epilogue thread (thread = output feature), folded into the sine's range reduction.
//   * Layer 5 (128 -> 3): 8 SS MMAs with N = 16: A = the layer-4 activations reinterpreted as an MN-major
//     A operand (M = rays), B = W5 (K-major); D = the slot's own output columns O (lanes = rays); b5 is
//     added by the output warps. Issued together with layer 1 of the slot's next tile.
// TMEM (512 columns): weights W1^T at 0 (8 columns), W2^T..W4^T at 8, 72, 136 (64 each); O(s) at 208 + 16 s;
// D(s) at 256 + 128 s (lanes = features, columns = rays). D and the activation tile are single-buffered
// per slot: each layer's epilogue starts after the layer's commit, i.e. after the MMA finished reading
// the activation tile it overwrites.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <vector>

#include "pt_internal.h"
#include "tc_ptx.cuh"

namespace pt {

namespace siren {

constexpr int kTileM = 128;
// shared-memory weight image (built by nif_build_smem_image):
//   W1^T rows: 128 x 16 fp16 (w_x, w_y, w_x, w_y, b1, 0 ...), 32 B each          at kOffW1
//   W2^T..W4^T rows: 128 x 128 fp16 per layer, row stride 272 B (16-B padding: conflict-free 16-B loads)
//   b2..b4: 3 x 128 fp32                                                         at kOffBias
//   W5 as the K-major B operand of layer 5 (N = 16 padded, K = 128; core matrix (nb, kb) = rows 8nb..8nb+7
//   x k 8kb..8kb+7, 128 B at (kb * 2 + nb) * 128), then b5 (3 fp32)                at kOffW5, kOffB5
constexpr int kRowStride = 272;
constexpr int kOffW1 = 0;
constexpr int kOffWH = kOffW1 + 128 * 32;
constexpr int kWHBytes = 128 * kRowStride;
constexpr int kOffBias = kOffWH + 3 * kWHBytes;
constexpr int kOffW5 = kOffBias + 3 * 128 * 4;
constexpr int kW5Bytes = 16 * 128 * 2;
constexpr int kOffB5 = kOffW5 + kW5Bytes;
constexpr int kImageBytes = ((kOffB5 + 16 + 127) / 128) * 128;
// after the image: barriers, staged layer-1 tiles (2 slots, K-major, 4 KiB), activation tiles (2 slots,
// MN-major: element (feature k, ray r) at (r / 8) * 2048 + k * 16 + (r % 8) * 2, 32 KiB)
constexpr int kOffBars = kImageBytes;
constexpr int kOffA0 = ((kOffBars + 128 + 1023) / 1024) * 1024;
constexpr int kA0Bytes = 128 * 16 * 2;
constexpr int kOffH = kOffA0 + 2 * kA0Bytes;
constexpr int kHBytes = 128 * 128 * 2;
constexpr int kSmemBytes = kOffH + 2 * kHBytes;
// MN-major operand strides: core matrices adjacent in MN are 2048 B apart, adjacent in K 128 B. For an
// MN-major SWIZZLE_NONE operand the descriptor's LBO field holds the K stride and SBO the MN stride
// (measured: tools/mn_major_probe.cu, profiles/round2/mn_major_probe.txt)
constexpr uint32_t kMnStrideMN = 2048, kMnStrideK = 128;

constexpr int kNumEpiWarps = 16;                // 4 per TMEM lane quarter, 32 columns (rays) each
constexpr int kFirstEpiWarp = 4;
constexpr int kProducerWarp0 = 2;               // warps 2-3 stage the layer-1 inputs
constexpr int kProducerThreads = 64;
constexpr int kThreads = 32 * (kFirstEpiWarp + kNumEpiWarps);   // 640
// barriers: [0] weights (bulk copies), [1..2] a_ready[slot] (16 epilogue warps: the next layer's activation
// tile written), [3..4] d_full[slot] (commit of layers 1-4), [5..6] a0_full[slot] (64 producer threads),
// [7..8] a0_empty[slot] (commit), [9..10] o_full[slot] (commit of layer 5), [11] w_tmem (16 epilogue warps:
// the weights are in TMEM); TMEM base address at +120. (O(s) needs no "free" barrier: the output warps
// read it before they arrive on a_ready(s) for the next tile's layer 4, which the issuer waits for before
// it issues that tile's layer 5.)
#ifndef PT_NIF_DIAG
#define PT_NIF_DIAG 0   // diagnostic builds only (wrong results): 1 = no activation store, 2 = no sine
#endif
enum { kBarW = 0, kBarAReady = 1, kBarDFull = 3, kBarA0Full = 5, kBarA0Empty = 7, kBarOFull = 9, kBarWTmem = 11 };

constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColW1 = 0, kColWH = 8;   // + 64 l for hidden layer l = 0..2
__host__ __device__ constexpr uint32_t o_col(int s) { return 208u + 16u * s; }
__host__ __device__ constexpr uint32_t d_col(int s) { return 256u + 128u * s; }

// instruction descriptor: D f32, A/B f16, M = 128, N given; transpose bits 15 (A MN-major), 16 (B MN-major)
__host__ __device__ constexpr uint32_t idesc(int n, uint32_t ta = 0, uint32_t tb = 0) {
    return (1u << 4) | (ta << 15) | (tb << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

}  // namespace siren

int64_t nif_smem_image_bytes() { return siren::kImageBytes; }

// Re-lay the fp16 SIREN blob (layer l: W_l[out][in] then b_l[out]) into the kernel's shared-memory image.
void nif_build_smem_image(const uint16_t* blob, std::vector<uint8_t>* image) {
    using namespace siren;
    std::vector<uint8_t>& img = *image;
    img.assign(kImageBytes, 0);
    size_t off = 0;
    auto put16 = [&](int at, uint16_t v) { std::memcpy(&img[at], &v, 2); };
    // layer 1: W1 [128][2], b1 [128] -> row n = (W n0, W n1, W n0, W n1, b n, 0 ...) against the staged B
    // row (x_hi, y_hi, x_lo, y_lo, 1, 0 ...)
    const uint16_t* W1 = blob + off; off += 128 * 2;
    const uint16_t* b1 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        const int r = kOffW1 + 32 * n;
        put16(r + 0, W1[2 * n + 0]);
        put16(r + 2, W1[2 * n + 1]);
        put16(r + 4, W1[2 * n + 0]);
        put16(r + 6, W1[2 * n + 1]);
        put16(r + 8, b1[n]);
    }
    // layers 2-4: rows W[n][0..127] (the A operand rows, TMEM lane n), biases as fp32
    for (int l = 0; l < 3; ++l) {
        const uint16_t* W = blob + off; off += 128 * 128;
        const uint16_t* b = blob + off; off += 128;
        for (int n = 0; n < 128; ++n) {
            std::memcpy(&img[kOffWH + l * kWHBytes + n * kRowStride], &W[n * 128], 256);
            const __half_raw hr{b[n]};
            const float bf = __half2float(__half(hr));
            std::memcpy(&img[kOffBias + (l * 128 + n) * 4], &bf, 4);
        }
    }
    // layer 5: W5 [3][128] -> K-major B operand, N padded to 16; b5 as fp32
    const uint16_t* W5 = blob + off; off += 3 * 128;
    const uint16_t* b5 = blob + off; off += 3;
    for (int n = 0; n < 3; ++n) {
        for (int k = 0; k < 128; ++k)
            put16(kOffW5 + ((k >> 3) * 2 + (n >> 3)) * 128 + (n & 7) * 16 + (k & 7) * 2, W5[n * 128 + k]);
        const __half_raw hr{b5[n]};
        const float bf = __half2float(__half(hr));
        std::memcpy(&img[kOffB5 + 4 * n], &bf, 4);
    }
}

#ifdef PT_NIF_TRACE
// timing trace of CTA 0 (variant builds only): [role][record][2] clock64 stamps
__device__ unsigned long long g_nif_trace[3 * 4096 * 2];
#define NIF_TRACE(role, rec, k)                                                                           \
    do {                                                                                                  \
        if (blockIdx.x == 0 && (rec) < 4096) g_nif_trace[((role) * 4096 + (rec)) * 2 + (k)] = clock64(); \
    } while (0)
#else
#define NIF_TRACE(role, rec, k) \
    do {                        \
    } while (0)
#endif

// sine of 32 accumulator columns of one feature (rays 32 cb .. 32 cb + 31) with the feature's bias,
// packed to fp16 pairs of consecutive rays: the SFU takes sfu_pair() pairs, the FMA pipe the others
// (fp32 quarter-period reduction with the bias folded in, fp16x2 odd polynomial)
__device__ __forceinline__ void sine_bias_half(const uint32_t* v, int h, float bias, float bias_q, uint32_t* p) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const int j = 8 * h + jj;
        const float a = __uint_as_float(v[2 * jj]), b = __uint_as_float(v[2 * jj + 1]);
        if (sfu_pair(j)) {
            const float2 x = __fadd2_rn(make_float2(a, b), make_float2(bias, bias));
            p[jj] = pack_half2(__sinf(x.x), __sinf(x.y));
        } else {
            p[jj] = sin2_poly_q(a, b, bias_q);
        }
    }
}

template <bool kDebug>
__global__ void __launch_bounds__(siren::kThreads, 1)
    siren_kernel(const uint8_t* __restrict__ g_image, const float4* __restrict__ esc,
                 const float4* __restrict__ esc_beta, const uint32_t* __restrict__ count, float* __restrict__ out,
                 float* __restrict__ dbg, int dir_input) {
    using namespace siren;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kOffBars);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + kOffBars + 120);
    auto bar = [&](int b) { return smem_u32(&bars[b]); };

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    pdl_trigger();

    if (warp == 1 && lane == 0) {
        mbar_init(bar(kBarW), 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(bar(kBarAReady + s), kNumEpiWarps);
            mbar_init(bar(kBarDFull + s), 1);
            mbar_init(bar(kBarA0Full + s), kProducerThreads);
            mbar_init(bar(kBarA0Empty + s), 1);
            mbar_init(bar(kBarOFull + s), 1);
        }
        mbar_init(bar(kBarWTmem), kNumEpiWarps);
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

    if (warp == 1 && lane == 0) {
        // stage the whole weight image once (bulk TMA copies, complete_tx on the weight barrier); the
        // image is the NIF's own, so this runs before the wait on the previous kernel of the wave
        mbar_expect_tx(bar(kBarW), (uint32_t)kImageBytes);
        constexpr int kChunk = 16384;
        for (int off = 0; off < kImageBytes; off += kChunk) {
            const int bytes = (kImageBytes - off) < kChunk ? (kImageBytes - off) : kChunk;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(smem + off)),
                "l"(g_image + off), "r"(bytes), "r"(bar(kBarW))
                : "memory");
        }
    }

    pdl_wait();                       // the escaped queue and its count are complete and visible
    const uint32_t n_rows = *count;
    const uint32_t n_tiles = (n_rows + kTileM - 1) / kTileM;

    if (warp == 0) {
        // ===== MMA issuer: warp 0 walks the schedule, one elected lane issues =====
        if (blockIdx.x < n_tiles) {
            mbar_wait(bar(kBarW), 0);
            mbar_wait(bar(kBarWTmem), 0);     // weights are in TMEM
            const uint32_t img = smem_u32(smem);
            const uint32_t hbase = smem_u32(smem + kOffH);
            uint32_t a_phase[2] = {0, 0}, f_phase[2] = {0, 0};
            bool pend[2] = {false, false};   // a tile of this slot still needs its output layer
            int rec = 0;
            // layer 5 of the slot's previous tile (after its layer-4 epilogue): O(s) = H4 W5^T
            auto issue_out = [&](int s) {
                mbar_wait(bar(kBarAReady + s), a_phase[s]);
                a_phase[s] ^= 1;
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t h = hbase + s * kHBytes;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        mma_ss(tmem + o_col(s), smem_desc(h + k * 2 * kMnStrideK, kMnStrideK, kMnStrideMN),
                               smem_desc(img + kOffW5 + k * 2 * 256, 256, 128), idesc(16, 1, 0), k > 0);
                    mma_commit(bar(kBarOFull + s));
                }
                __syncwarp();
            };
            for (uint32_t i = 0;; i += 2) {
                const uint32_t t0 = blockIdx.x + i * gridDim.x;
                if (t0 >= n_tiles) break;
                const int nslots = (t0 + gridDim.x < n_tiles) ? 2 : 1;
                for (int stage = 0; stage < 4; ++stage) {
                    for (int s = 0; s < nslots; ++s, ++rec) {
                        if (stage == 0) {
                            if (pend[s]) issue_out(s);                   // previous tile's output layer
                            mbar_wait(bar(kBarA0Full + s), f_phase[s]);  // layer-1 inputs staged
                            f_phase[s] ^= 1;
                        } else {
                            mbar_wait(bar(kBarAReady + s), a_phase[s]);  // this layer's activations written
                            a_phase[s] ^= 1;
                        }
                        if (lane == 0) NIF_TRACE(0, rec, 0);
                        tc_fence_after();
                        const uint32_t dt = tmem + d_col(s);
                        if (elect_one()) {
                            if (stage == 0) {
                                const uint64_t x0 = smem_desc(smem_u32(smem + kOffA0 + s * kA0Bytes), 2048, 128);
                                mma_ts(dt, tmem + kColW1, x0, idesc(128), 0);
                                mma_commit(bar(kBarDFull + s));
                                mma_commit(bar(kBarA0Empty + s));   // staging tile free once layer 1 is done
                            } else {
                                const uint32_t h = hbase + s * kHBytes;
                                const uint32_t wa = tmem + kColWH + 64u * (stage - 1);
#pragma unroll
                                for (int k = 0; k < 8; ++k)
                                    mma_ts(dt, wa + 8 * k, smem_desc(h + k * 2 * kMnStrideK, kMnStrideK, kMnStrideMN),
                                           idesc(128, 0, 1), k > 0);
                                mma_commit(bar(kBarDFull + s));
                            }
                        }
                        __syncwarp();
                        if (stage == 0) pend[s] = true;
                        if (lane == 0) NIF_TRACE(0, rec, 1);
                    }
                }
            }
            for (int s = 0; s < 2; ++s)
                if (pend[s]) issue_out(s);                           // the last tiles' output layers
        }
    } else if (warp == kProducerWarp0 || warp == kProducerWarp0 + 1) {
        // ===== producers: layer-1 inputs of every tile, staged one tile ahead per slot =====
        // queue entry -> (u, v) (equirect of the escape direction for the render queue, reading R14)
        // -> x0 = (2u-1, 2v-1) split into fp16 hi + lo (reading R15), constant-1 bias column; the tile is
        // the K-major B operand of layer 1 (row = ray).
        const int p = threadIdx.x - 32 * kProducerWarp0;
        uint8_t* a0s = smem + kOffA0;
        for (int i = p; i < 2 * kA0Bytes / 16; i += kProducerThreads)
            *reinterpret_cast<uint4*>(a0s + 16 * i) = make_uint4(0, 0, 0, 0);
        uint32_t e_phase[2] = {0, 0};
        uint32_t fills[2] = {0, 0};
        for (uint32_t i = 0;; i += 2) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = (t0 + gridDim.x < n_tiles) ? 2 : 1;
            for (int s = 0; s < nslots; ++s) {
                const uint32_t tile = t0 + s * gridDim.x;
                if (fills[s]++ > 0) {
                    mbar_wait(bar(kBarA0Empty + s), e_phase[s]);
                    e_phase[s] ^= 1;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = p + 64 * h;
                    const uint32_t row = tile * kTileM + m;
                    float u = 0.5f, v = 0.5f;
                    if (row < n_rows) {
                        const float4 en = __ldg(esc + row);
                        u = en.x;
                        v = en.y;
                        if (dir_input) equirect_f32(make_float3(en.x, en.y, en.z), u, v);
                    }
                    const float x = 2.0f * u - 1.0f, y = 2.0f * v - 1.0f;
                    const __half xh = __float2half_rn(x), yh = __float2half_rn(y);
                    const __half xl = __float2half_rn(x - __half2float(xh)), yl = __float2half_rn(y - __half2float(yh));
                    // K-major core-matrix layout of rows m (K 0..7 only; K 8..15 stay zero)
                    *reinterpret_cast<uint4*>(a0s + s * kA0Bytes + 16 * m) = make_uint4(
                        (uint32_t)__half_as_ushort(xh) | ((uint32_t)__half_as_ushort(yh) << 16),
                        (uint32_t)__half_as_ushort(xl) | ((uint32_t)__half_as_ushort(yl) << 16), 0x00003C00u, 0u);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
                mbar_arrive(bar(kBarA0Full + s));
            }
        }
    } else if (warp >= kFirstEpiWarp) {
        // ===== epilogue warps =====
        // All 16 work on one (slot, layer) at a time, in the MMA's issue order. Warp w owns TMEM lane
        // quarter q = w % 4 (hardware rule), i.e. output features 32 q .. 32 q + 31 (thread = feature f),
        // and the 32-ray column block cb of the tile.
        const int e = warp - kFirstEpiWarp;
        const int cb = e >> 2;
        const int q = warp & 3;
        const int f = 32 * q + lane;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        mbar_wait(bar(kBarW), 0);
        // weights -> TMEM (A operand rows: lane f): block 0 loads W1^T, blocks 1-3 one hidden layer each
        if (cb == 0) {
            const uint4 w0 = *reinterpret_cast<const uint4*>(smem + kOffW1 + 32 * f);
            const uint32_t w[8] = {w0.x, w0.y, w0.z, w0.w, 0u, 0u, 0u, 0u};
            tmem_st8(tmem + kColW1 + lane_addr, w);
        } else {
            const uint8_t* row = smem + kOffWH + (cb - 1) * kWHBytes + f * kRowStride;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t w[16];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint4 x = *reinterpret_cast<const uint4*>(row + 64 * c + 16 * j);
                    w[4 * j] = x.x; w[4 * j + 1] = x.y; w[4 * j + 2] = x.z; w[4 * j + 3] = x.w;
                }
                TMEM_ST16(tmem + kColWH + 64u * (cb - 1) + 16u * c + lane_addr, w);
            }
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar(kBarWTmem));
        // this thread's biases (layers 2-4; layer 1's rides in the MMA) and their quarter-period forms
        constexpr float kInv2Pi = 0.15915494309189535f;
        const float bias1 = *reinterpret_cast<const float*>(smem + kOffBias + (0 * 128 + f) * 4);
        const float bias2 = *reinterpret_cast<const float*>(smem + kOffBias + (1 * 128 + f) * 4);
        const float bias3 = *reinterpret_cast<const float*>(smem + kOffBias + (2 * 128 + f) * 4);
        // (selected per stage without a dynamically indexed array: no local memory)
        auto bias_of = [&](int stage) { return stage == 0 ? 0.0f : stage == 1 ? bias1 : stage == 2 ? bias2 : bias3; };
        float b5[3] = {0.0f, 0.0f, 0.0f};
        if (cb == 0) {
#pragma unroll
            for (int n = 0; n < 3; ++n) b5[n] = *reinterpret_cast<const float*>(smem + kOffB5 + 4 * n);
        }
        uint32_t d_phase[2] = {0, 0}, o_phase[2] = {0, 0};
        // the output rows of each slot's previous tile (cb == 0 warps, thread = ray 32 q + lane)
        float4 beta[2] = {make_float4(0, 0, 0, 0), make_float4(0, 0, 0, 0)};
        uint32_t oslot[2] = {0, 0};
        bool ovalid[2] = {false, false}, pend[2] = {false, false};
        uint32_t prow[2] = {0, 0};
        // layer 5 of the slot's previous tile: y = O[ray, 0:3] + b5; radiance = beta * exp(y)
        auto output = [&](int s, uint32_t dbg_row) {
            mbar_wait(bar(kBarOFull + s), o_phase[s]);
            o_phase[s] ^= 1;
            tc_fence_after();
            uint32_t v[4];
            tmem_ld4(tmem + o_col(s) + lane_addr, v);
            tmem_wait_ld_dep4(v);
            if (ovalid[s]) {
                const float y0 = __uint_as_float(v[0]) + b5[0], y1 = __uint_as_float(v[1]) + b5[1],
                            y2 = __uint_as_float(v[2]) + b5[2];
                if (kDebug) {
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 0] = y0;
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 1] = y1;
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 2] = y2;
                }
                out[3 * (size_t)oslot[s] + 0] = beta[s].x * __expf(y0);
                out[3 * (size_t)oslot[s] + 1] = beta[s].y * __expf(y1);
                out[3 * (size_t)oslot[s] + 2] = beta[s].z * __expf(y2);
            }
        };
        uint8_t* hrow = smem + kOffH + f * 16;   // this feature's 16-B row inside each 8-ray core matrix
        int rec = 0;
        for (uint32_t i = 0;; i += 2) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = (t0 + gridDim.x < n_tiles) ? 2 : 1;
            for (int stage = 0; stage < 4; ++stage) {
                for (int s = 0; s < nslots; ++s, ++rec) {
                    const uint32_t tile = t0 + s * gridDim.x;
                    mbar_wait(bar(kBarDFull + s), d_phase[s]);
                    d_phase[s] ^= 1;
                    const int trole = (warp == kFirstEpiWarp) ? 1 : (warp == kFirstEpiWarp + kNumEpiWarps - 1 ? 2 : -1);
                    if (trole > 0 && lane == 0) NIF_TRACE(trole, rec, 0);
                    tc_fence_after();
                    uint32_t v[32];
                    uint32_t pk[16];
                    const float bs = bias_of(stage), bq = fmaf(bs, kInv2Pi, 0.25f);
                    if (kDebug) {
                        TMEM_LD32(tmem + d_col(s) + lane_addr + 32 * cb, v);
                        tmem_wait_ld_dep(v);
                        for (int j = 0; j < 32; ++j) {
                            const uint32_t r = tile * kTileM + 32 * cb + j;
                            if (r < n_rows) dbg[((size_t)stage * n_rows + r) * 128 + f] = __uint_as_float(v[j]) + bs;
                        }
                        sine_bias_half(v, 0, bs, bq, pk);
                        sine_bias_half(v + 16, 1, bs, bq, pk + 8);
                    } else if (PT_NIF_DIAG == 2) {
                        TMEM_LD32(tmem + d_col(s) + lane_addr + 32 * cb, v);
                        tmem_wait_ld_dep(v);
#pragma unroll
                        for (int j = 0; j < 16; ++j) pk[j] = v[2 * j] ^ v[2 * j + 1];
                    } else {
                        // D (fp32) -> sin(. + b) -> fp16: the second 16 rays load while the first are computed
                        TMEM_LD16(tmem + d_col(s) + lane_addr + 32 * cb, v);
                        tmem_wait_ld_dep16(v);
                        TMEM_LD16(tmem + d_col(s) + lane_addr + 32 * cb + 16, v + 16);
                        sine_bias_half(v, 0, bs, bq, pk);
                        tmem_wait_ld_dep16(v + 16);
                        sine_bias_half(v + 16, 1, bs, bq, pk + 8);
                    }
                    // -> the slot's activation tile (B of the next layer): rays 32 cb + 8 j .. + 7 of feature f
                    // are one 16-B core-matrix row; a warp's 32 features are 512 contiguous bytes per store
                    if (PT_NIF_DIAG != 1) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            *reinterpret_cast<uint4*>(hrow + s * kHBytes + (4 * cb + j) * kMnStrideMN) =
                                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
                    } else if (pk[0] == 0x7FFF7FFFu && pk[15] == 0x7FFF7FFFu) {   // diagnostic: keep pk live
                        out[0] = 0.0f;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
                    tc_fence_before();
                    __syncwarp();
                    if (trole > 0 && lane == 0) NIF_TRACE(trole, rec, 1);
                    if (lane == 0) mbar_arrive(bar(kBarAReady + s));
                    // O(prev) was committed with this layer 1: read it once this warp's share of the next
                    // layer's input is handed over, off the MMA's critical path
                    if (cb == 0 && stage == 0 && pend[s]) output(s, prow[s]);
                    if (cb == 0 && stage == 1) {
                        // this tile's output rows (after the previous tile's output was written)
                        const uint32_t row = tile * kTileM + 32 * q + lane;
                        ovalid[s] = row < n_rows;
                        prow[s] = row;
                        if (row < n_rows) {
                            beta[s] = __ldg(esc_beta + row);
                            oslot[s] = __float_as_uint(__ldg(esc + row).w);
                        }
                    }
                    if (stage == 0) pend[s] = true;
                }
            }
            rec += nslots;   // (trace records of the MMA's layer-5 steps)
        }
        if (cb == 0)
            for (int s = 0; s < 2; ++s)
                if (pend[s]) output(s, prow[s]);   // the last tiles' output layers
    }
    // a CTA without tiles still owns the weight copies in flight into its shared memory
    if (warp == 1 && lane == 0 && blockIdx.x >= n_tiles) mbar_wait(bar(kBarW), 0);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

template <bool kDebug>
static cudaError_t siren_launch_t(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                                  int grid, float* out, float* dbg, int dir_input, cudaStream_t st) {
    cudaError_t e = ensure_dyn_smem((const void*)siren_kernel<kDebug>, siren::kSmemBytes);
    if (e != cudaSuccess) return e;
    return launch_pdl(siren_kernel<kDebug>, dim3(grid), dim3(siren::kThreads), siren::kSmemBytes, st,
                      (const uint8_t*)nif->d_smem_image, esc, esc_beta, count, out, dbg, dir_input);
}

cudaError_t launch_siren(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count, int grid,
                         float* out, float* dbg, int dir_input, cudaStream_t st) {
    return dbg ? siren_launch_t<true>(nif, esc, esc_beta, count, grid, out, dbg, dir_input, st)
               : siren_launch_t<false>(nif, esc, esc_beta, count, grid, out, dbg, dir_input, st);
}

}  // namespace pt

#ifdef PT_NIF_TRACE
extern "C" __attribute__((visibility("default"))) int pt_debug_nif_trace(unsigned long long* host_out) {
    return (int)cudaMemcpyFromSymbol(host_out, pt::g_nif_trace, sizeof(pt::g_nif_trace));
}
#endif
