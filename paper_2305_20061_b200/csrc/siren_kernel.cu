// siren_kernel.cu -- fused SIREN HDR-NIF inference on sm_100a tensor cores (tcgen05 + TMEM), step S5.
//
// What it computes (BASELINE.json SIREN; readings R1-R3, R14, R15):
//   for every escaped ray (direction d, or (u, v) from the query hook) with throughput beta:
//     (u, v) = equirect(d); x0 = (2u-1, 2v-1); h1 = sin(W1' x0 + b1'); h_{k+1} = sin(W'_{k+1} h_k + b'_{k+1})
//     (k = 1..3); y = W5 h4 + b5; radiance = beta * exp(y)   (written to the path's own wave slot)
//
// Design. One persistent CTA per SM keeps the weights resident in shared memory
// (one bulk TMA copy per CTA). Two 128-ray tiles ("slots") are in flight: the tensor core runs one
// slot's layer while 16 epilogue warps apply the sine to the other slot's accumulator.
//   * Layer 1 (2 -> 128): one SS MMA, K = 16, A = a shared-memory tile staged by two producer warps
//     (equirect, hi/lo split of x0, constant-1 bias column), so no epilogue work is spent on inputs.
//   * Layers 2-4 (128 -> 128): 9 TS MMAs, M = N = 128, K = 16 each; A = the previous layer's fp16
//     activations in TMEM, the 9th K step reads a constant-1 TMEM column against the bias row of B.
//     Whole-N MMAs (tools/mma_shapes.cu: N = 64 from TMEM costs 57 of N = 128's 64 cycles) and no
//     TMEM/SMEM A switch inside a layer (~50 cycles each).
//   * Layer 5 (128 -> 3): 8 TS MMAs with N = 16 into the slot's own output columns O (b5 is added by the
//     output warps). It is issued together with layer 1 of the slot's next tile (one commit group), so
//     the tensor pipe never holds an output layer in front of the MMA the epilogue needs next; the 4
//     warps owning TMEM lane quarters at column block 0 read O(prev tile) during the next tile's first
//     sine stage (exp, beta, store). (On the FMA pipe inside the layer-4 epilogue it lengthened the
//     epilogue, the bottleneck, by ~700 cycles per tile: tools/nif_trace.py.)
// TMEM (512 columns): slot s: D at 256 s (128 fp32 columns), A at 256 s + 128 (64 columns of fp16
// pairs + the constant K block 64..71), O at 256 s + 208 (16 columns). A is single-buffered: each
// layer's epilogue starts after the layer's one commit, i.e. after the MMA finished reading A.
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
// shared-memory image (K-major SWIZZLE_NONE core-matrix tiles: core matrix (nb, kb) = rows 8nb..8nb+7
// x k 8kb..8kb+7, 128 B, at ((kb * N/8) + nb) * 128)
constexpr int kB1Bytes = 128 * 16 * 2;          // layer 1: N = 128, K = 16 (x_hi, y_hi, x_lo, y_lo, bias)
constexpr int kBHBytes = 128 * 144 * 2;         // layers 2-4: N = 128, K = 128 + bias step
constexpr int kOffBH = kB1Bytes;
constexpr int kOffB5 = kOffBH + 3 * kBHBytes;   // layer 5: N = 16 (3 used), K = 128 + bias step
constexpr int kB5Bytes = 16 * 144 * 2;
constexpr int kImageBytes = kOffB5 + kB5Bytes;  // 119,296
// after the image: barriers, staged layer-1 A tiles (2 slots)
constexpr int kOffBars = kImageBytes;
constexpr int kOffA0 = ((kOffBars + 128 + 1023) / 1024) * 1024;
constexpr int kA0Bytes = 128 * 16 * 2;
constexpr int kSmemBytes = kOffA0 + 2 * kA0Bytes;

constexpr int kNumEpiWarps = 16;                // 4 per TMEM lane quarter, 32 columns each
constexpr int kFirstEpiWarp = 4;
constexpr int kProducerWarp0 = 2;               // warps 2-3 stage the layer-1 inputs
constexpr int kProducerThreads = 64;
constexpr int kThreads = 32 * (kFirstEpiWarp + kNumEpiWarps);   // 640
// barriers: [0] weights, [1..2] a_ready[slot] (16 epilogue warps: next layer's A written), [3..4] d_full[slot]
// (commit of layers 1-4), [5..6] a0_full[slot] (64 producer threads), [7..8] a0_empty[slot] (commit),
// [9..10] o_full[slot] (commit of layer 5); TMEM base address at +120. (O(s) needs no "free" barrier:
// the output warps read it before they arrive on a_ready(s) for the next tile's layer 4, which the
// issuer waits for before it issues that tile's layer 5.)
#ifndef PT_NIF_DIAG
#define PT_NIF_DIAG 0   // diagnostic builds only (wrong results): 1 = no TMEM store of A, 2 = no sine,
                        // 3 = no epilogue TMEM traffic (neither the accumulator load nor the A store)
#endif
#ifndef PT_NIF_DEFER_ST
#define PT_NIF_DEFER_ST 0   // measured slower (5.96 vs 7.25 G inferences/s, profiles/round2/nif_defer.log)
#endif
#ifndef PT_NIF_OUT_EARLY
#define PT_NIF_OUT_EARLY 0
#endif
enum { kBarW = 0, kBarAReady = 1, kBarDFull = 3, kBarA0Full = 5, kBarA0Empty = 7, kBarOFull = 9 };

constexpr uint32_t kTmemCols = 512;
__host__ __device__ constexpr uint32_t d_col(int s) { return 256u * s; }
__host__ __device__ constexpr uint32_t a_col(int s) { return 256u * s + 128u; }
__host__ __device__ constexpr uint32_t o_col(int s) { return 256u * s + 208u; }

// instruction descriptor: D f32, A/B f16, K-major both, M = 128, N given
__host__ __device__ constexpr uint32_t idesc(int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

inline void put_core(std::vector<uint8_t>& img, int base, int N, int n, int k, uint16_t v) {
    const int nb = n >> 3, r = n & 7, kb = k >> 3, c = k & 7;
    const int off = base + ((kb * (N / 8)) + nb) * 128 + r * 16 + c * 2;
    std::memcpy(&img[off], &v, 2);
}

}  // namespace siren

int64_t nif_smem_image_bytes() { return siren::kImageBytes; }

// Re-lay the fp16 SIREN blob (layer l: W_l[out][in] then b_l[out]) into the kernel's shared-memory image.
void nif_build_smem_image(const uint16_t* blob, std::vector<uint8_t>* image) {
    using namespace siren;
    std::vector<uint8_t>& img = *image;
    img.assign(kImageBytes, 0);
    size_t off = 0;
    // layer 1: W1 [128][2], b1 [128] -> B1 row n = (W n0, W n1, W n0, W n1, b n, 0 ...) against the
    // staged A row (x_hi, y_hi, x_lo, y_lo, 1, 0 ...)
    const uint16_t* W1 = blob + off; off += 128 * 2;
    const uint16_t* b1 = blob + off; off += 128;
    for (int n = 0; n < 128; ++n) {
        put_core(img, 0, 128, n, 0, W1[2 * n + 0]);
        put_core(img, 0, 128, n, 1, W1[2 * n + 1]);
        put_core(img, 0, 128, n, 2, W1[2 * n + 0]);
        put_core(img, 0, 128, n, 3, W1[2 * n + 1]);
        put_core(img, 0, 128, n, 4, b1[n]);
    }
    // layers 2-4: W [128][128] + bias at k = 128 (against the constant-1 TMEM column)
    for (int l = 0; l < 3; ++l) {
        const uint16_t* W = blob + off; off += 128 * 128;
        const uint16_t* b = blob + off; off += 128;
        const int base = kOffBH + l * kBHBytes;
        for (int n = 0; n < 128; ++n) {
            // 8 consecutive k of one row are one 16-byte core-matrix row
            for (int kb = 0; kb < 16; ++kb)
                std::memcpy(&img[base + ((kb * 16) + (n >> 3)) * 128 + (n & 7) * 16], &W[n * 128 + 8 * kb], 16);
            put_core(img, base, 128, n, 128, b[n]);
        }
    }
    // layer 5: W5 [3][128], b5 [3] -> N padded to 16
    const uint16_t* W5 = blob + off; off += 3 * 128;
    const uint16_t* b5 = blob + off; off += 3;
    for (int n = 0; n < 3; ++n) {
        for (int k = 0; k < 128; ++k) put_core(img, kOffB5, 16, n, k, W5[n * 128 + k]);
        put_core(img, kOffB5, 16, n, 128, b5[n]);
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
            const uint32_t img = smem_u32(smem);
            uint32_t a_phase[2] = {0, 0}, f_phase[2] = {0, 0};
            bool pend[2] = {false, false};   // a tile of this slot still needs its output layer
            int rec = 0;
            // layer 5 of the slot's previous tile: after its layer-4 epilogue (a_ready), into O(s)
            auto issue_out = [&](int s) {
                mbar_wait(bar(kBarAReady + s), a_phase[s]);
                a_phase[s] ^= 1;
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t base = img + kOffB5;
                    const uint32_t at = tmem + a_col(s);
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        mma_ts(tmem + o_col(s), at + 8 * k, smem_desc(base + k * 2 * 256, 256, 128), idesc(16), k > 0);
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
                            mbar_wait(bar(kBarAReady + s), a_phase[s]);  // this layer's A written
                            a_phase[s] ^= 1;
                        }
                        if (lane == 0) NIF_TRACE(0, rec, 0);
                        tc_fence_after();
                        const uint32_t dt = tmem + d_col(s);
                        if (elect_one()) {
                            if (stage == 0) {
                                const uint64_t a0 = smem_desc(smem_u32(smem + kOffA0 + s * kA0Bytes), 2048, 128);
                                mma_ss(dt, a0, smem_desc(img, 2048, 128), idesc(128), 0);
                                mma_commit(bar(kBarDFull + s));
                                mma_commit(bar(kBarA0Empty + s));   // staging tile free once layer 1 is done
                            } else {
                                const uint32_t base = img + kOffBH + (stage - 1) * kBHBytes;
                                const uint32_t at = tmem + a_col(s);
#pragma unroll
                                for (int k = 0; k < 9; ++k)
                                    mma_ts(dt, at + 8 * k, smem_desc(base + k * 2 * 2048, 2048, 128), idesc(128), k > 0);
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
        // -> x0 = (2u-1, 2v-1) split into fp16 hi + lo (reading R15), constant-1 bias column.
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
        // quarter w % 4 (hardware rule) and the 32-column block cb of the 128 columns.
        const int e = warp - kFirstEpiWarp;
        const int cb = e >> 2;
        const int q = warp & 3;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        // constant-1 K block (A columns 64..71 = fp16 (1, 0, ... 0) per row) of both slots' A buffers
        if (cb == 0) {
            const uint32_t one[8] = {0x00003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            tmem_st8(tmem + a_col(0) + 64 + lane_addr, one);
            tmem_st8(tmem + a_col(1) + 64 + lane_addr, one);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        // b5 (fp16 in the image's bias step of B5: row n, k = 128), added by the output warps once the
        // weight image has landed (the bulk copies complete on kBarW)
        float b5[3] = {0.0f, 0.0f, 0.0f};
        if (cb == 0) {
            mbar_wait(bar(kBarW), 0);
#pragma unroll
            for (int n = 0; n < 3; ++n)
                b5[n] = __half2float(*reinterpret_cast<const __half*>(smem + kOffB5 + (16 * 2) * 128 + n * 16));
        }
        uint32_t d_phase[2] = {0, 0}, o_phase[2] = {0, 0};
        // the output rows of each slot's previous tile (cb == 0 warps): slot id, throughput, validity
        float4 beta[2] = {make_float4(0, 0, 0, 0), make_float4(0, 0, 0, 0)};
        uint32_t oslot[2] = {0, 0};
        bool ovalid[2] = {false, false}, pend[2] = {false, false};
        // layer 5 of the slot's previous tile: y = O[:, 0:3] + b5; radiance = beta * exp(y)
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
        uint32_t prow[2] = {0, 0};
        // PT_NIF_DEFER_ST: a stage's TMEM store of A is completed (wait::st, fence, a_ready arrive) only
        // after the next stage's accumulator load is issued, so the store latency overlaps it; a pending
        // output read of the slot (cb == 0, layer 1) follows the hand-over
        int held = -1;                 // slot whose A store is still to be completed and signalled
        bool held_out = false;         // ... and whose previous tile's output is to be read after it
        auto hand_over = [&]() {
            if (held < 0) return;
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(bar(kBarAReady + held));
            if (held_out) output(held, prow[held]);
            held = -1;
            held_out = false;
        };
        int rec = 0;
        for (uint32_t i = 0;; i += 2) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = (t0 + gridDim.x < n_tiles) ? 2 : 1;
            for (int stage = 0; stage < 4; ++stage) {
                for (int s = 0; s < nslots; ++s, ++rec) {
                    const uint32_t tile = t0 + s * gridDim.x;
                    const uint32_t row = tile * kTileM + 32 * q + lane;
                    const bool valid = row < n_rows;
                    // complete the held hand-over now unless this stage's accumulator is already there
                    if (held >= 0 && !mbar_try(bar(kBarDFull + s), d_phase[s])) hand_over();
                    mbar_wait(bar(kBarDFull + s), d_phase[s]);
                    d_phase[s] ^= 1;
                    const int trole = (warp == kFirstEpiWarp) ? 1 : (warp == kFirstEpiWarp + kNumEpiWarps - 1 ? 2 : -1);
                    if (trole > 0 && lane == 0) NIF_TRACE(trole, rec, 0);
                    tc_fence_after();
                    uint32_t v[32];
                    uint32_t pk[16];
                    if (kDebug) {
                        TMEM_LD32(tmem + d_col(s) + lane_addr + 32 * cb, v);
                        tmem_wait_ld_dep(v);
                        if (valid)
                            for (int j = 0; j < 32; ++j)
                                dbg[((size_t)stage * n_rows + row) * 128 + 32 * cb + j] = __uint_as_float(v[j]);
                        sine_half(v, 0, pk);
                        sine_half(v + 16, 1, pk + 8);
                    } else if (PT_NIF_DIAG == 4) {
                        // diagnostic (wrong results): the epilogue only hands over (MMA + hand-off latency)
#pragma unroll
                        for (int j = 0; j < 16; ++j) pk[j] = (uint32_t)(j + lane);
                    } else if (PT_NIF_DIAG == 3) {
                        // diagnostic (wrong results): no TMEM traffic at all -- the sine on registers only
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = __float_as_uint((float)(j + lane) * 0.01f);
                        sine_half(v, 0, pk);
                        sine_half(v + 16, 1, pk + 8);
                    } else if (PT_NIF_DIAG == 2) {
                        // diagnostic (wrong results): TMEM round trip without the sine
                        TMEM_LD32(tmem + d_col(s) + lane_addr + 32 * cb, v);
                        tmem_wait_ld_dep(v);
#pragma unroll
                        for (int j = 0; j < 16; ++j) pk[j] = v[2 * j] ^ v[2 * j + 1];
                    } else {
                        // D (fp32) -> sin -> fp16: the second 16 columns load while the first are computed
                        TMEM_LD16(tmem + d_col(s) + lane_addr + 32 * cb, v);
                        hand_over();   // (the previous stage's, if held)
                        tmem_wait_ld_dep16(v);
                        TMEM_LD16(tmem + d_col(s) + lane_addr + 32 * cb + 16, v + 16);
                        sine_half(v, 0, pk);
                        tmem_wait_ld_dep16(v + 16);
                        sine_half(v + 16, 1, pk + 8);
                    }
#if PT_NIF_OUT_EARLY
                    if (cb == 0 && stage == 0 && pend[s]) output(s, prow[s]);   // O(prev) committed with layer 1
#endif
                    {
                        // -> A of the next layer (this warp's 32 columns)
                        if (PT_NIF_DIAG != 1 && PT_NIF_DIAG != 3 && PT_NIF_DIAG != 4) {
                            TMEM_ST16(tmem + a_col(s) + lane_addr + 16 * cb, pk);
                        } else if (pk[0] == 0x7FFF7FFFu && pk[15] == 0x7FFF7FFFu) {   // diagnostic: keep pk live
                            out[0] = 0.0f;
                        }
                    }
                    if (trole > 0 && lane == 0) NIF_TRACE(trole, rec, 1);
                    held = s;
                    // O(prev) was committed with this layer 1: read it once this warp's share of the next
                    // layer's A is handed over, off the MMA's critical path
                    held_out = !PT_NIF_OUT_EARLY && cb == 0 && stage == 0 && pend[s];
                    if (!PT_NIF_DEFER_ST || kDebug || PT_NIF_DIAG) hand_over();
                    if (cb == 0 && stage == 1) {
                        // this tile's output rows (after the previous tile's output was written)
                        ovalid[s] = valid;
                        prow[s] = row;
                        if (valid) {
                            beta[s] = __ldg(esc_beta + row);
                            oslot[s] = __float_as_uint(__ldg(esc + row).w);
                        }
                    }
                    if (stage == 0) pend[s] = true;
                }
            }
        }
        hand_over();
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
