// siren_kernel.cu -- fused SIREN HDR-NIF inference on sm_100a tensor cores (tcgen05 + TMEM), step S5.
//
// What it computes (BASELINE.json SIREN; readings R1-R3, R14, R15):
//   for every escaped ray (direction d, or (u, v) from the query hook) with throughput beta:
//     (u, v) = equirect(d); x0 = (2u-1, 2v-1); h1 = sin(W1' x0 + b1'); h_{k+1} = sin(W'_{k+1} h_k + b'_{k+1})
//     (k = 1..3); y = W5 h4 + b5; radiance = beta * exp(y)   (written to the path's own wave slot)
//
// Design. One persistent CTA per SM keeps the weights resident in shared memory
// (one bulk TMA copy per CTA). kSlots (3) 128-ray tiles ("slots") are in flight: the tensor core runs
// one slot's layer while an 8-warp epilogue team applies the sine to another slot's accumulator. A
// 9-MMA layer group takes ~880 cycles from issue to a visible commit (tools/mma_shapes.cu commit round
// trip: ~240 fixed + ~71 per MMA) against 576 cycles of tensor work, and each slot's chain then adds its
// sine epilogue, so with two slots the tensor pipe idled about half the time; three slots cover more
// of it. Accumulators are not owned by slots: layer groups rotate over two D regions in issue order,
// team t runs the groups of region t, and a warp frees the region (d_empty) as soon as its 64 columns
// are in registers, before the sine.
//   * Layer 1 (2 -> 128): one SS MMA, K = 16, A = a shared-memory tile staged by two producer warps
//     (equirect, hi/lo split of x0, constant-1 bias column), so no epilogue work is spent on inputs.
//   * Layers 2-4 (128 -> 128): 9 TS MMAs, M = N = 128, K = 16 each; A = the previous layer's fp16
//     activations in TMEM, the 9th K step reads a constant-1 TMEM column against the bias row of B.
//     Whole-N MMAs (tools/mma_shapes.cu: N = 64 from TMEM costs 57 of N = 128's 64 cycles) and no
//     TMEM/SMEM A switch inside a layer (~50 cycles each).
//   * Layer 5 (128 -> 3): 8 TS MMAs with N = 16 into the slot's own output columns O (b5 is added by the
//     output warps). It is issued together with layer 1 of the slot's next tile (one commit group), so
//     the tensor pipe never holds an output layer in front of the MMA the epilogue needs next; the slot's
//     4 output warps (team s % 2, column half s / 2, one per TMEM lane quarter) read O(prev tile) after
//     handing over the next tile's layer-1 epilogue (exp, beta, store). (On the FMA pipe inside the
//     layer-4 epilogue it lengthened the epilogue by ~700 cycles per tile in round 1.)
// TMEM (512 columns): A(s) at 64 s (64 columns of fp16 pairs), O(s) at 192 + 16 s (16 columns), the
// constant-1 K block shared by all slots at 240 (8 columns), D regions at 256 and 384 (128 fp32 columns
// each). A is single-buffered: each layer's epilogue starts after the layer's one commit, i.e. after
// the MMA finished reading A.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>
#include <vector>

#include "pt_internal.h"
// SFU share of the sine (tc_ptx.cuh): 10 of 16 column pairs on MUFU.SIN measured best with the team
// epilogue (8.31 vs 8.04 G inferences/s at 9, 8.27 at 11; profiles/round2/nif_slots.log)
#ifndef PT_NIF_MUFU_PAIRS
#define PT_NIF_MUFU_PAIRS 10
#endif
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
#ifndef PT_NIF_SLOTS
#define PT_NIF_SLOTS 3
#endif
constexpr int kSlots = PT_NIF_SLOTS;            // tiles in flight (2 or 3: TMEM layout below)
static_assert(kSlots == 2 || kSlots == 3, "TMEM holds at most three slots");
constexpr int kDRegions = 2;
// after the image: barriers, the TMEM base address, staged layer-1 A tiles (one per slot)
constexpr int kOffBars = kImageBytes;
// MMA issuers: warp j issues the layer groups of D region j (kIssuers = 2) or warp 0 all of them. A
// tcgen05.mma the tensor pipe cannot take yet stalls its warp's SM sub-partition, which slowed that
// sub-partition's epilogue warps by ~250 cycles per layer with one issuer (tools/nif_trace.py); two
// issuers halve it. Every barrier an issuer waits on has that issuer as its only waiter, so each
// waiter sees every phase in order (a_ready is per slot and per consuming issuer).
#ifndef PT_NIF_ISSUERS
#define PT_NIF_ISSUERS 2
#endif
constexpr int kIssuers = PT_NIF_ISSUERS;
static_assert(kIssuers == 1 || kIssuers == 2 || kIssuers == 4, "1, 2 or 4 issuer warps");
// issuer k issues the groups g with g % kIssuers == k; d_empty and a_ready are addressed to the issuer
// that consumes them (group g's release to the issuer of g + 2, its A to the issuer of g + nslots). Four
// issuers (704 threads, an 80-register cap with spills) measured 9.74 vs 7.50 ms per step in the render.
constexpr int kNumBars = 1 + (3 + kIssuers) * kSlots + kDRegions + kIssuers;
constexpr int kOffTmemSlot = kOffBars + 8 * kNumBars;
constexpr int kOffA0 = ((kOffTmemSlot + 16 + 1023) / 1024) * 1024;
constexpr int kA0Bytes = 128 * 16 * 2;
constexpr int kSmemBytes = kOffA0 + kSlots * kA0Bytes;

// Epilogue: two teams of 8 warps (2 per TMEM lane quarter, 64 columns each). Team t owns D region t,
// i.e. every other layer group, so one team applies the sine while the other waits for its next
// accumulator and the SM sub-partitions stay busy (with all 16 warps on every group, they all idled
// together between groups and the slowest warp of each group gated the next; tools/nif_trace.py).
constexpr int kNumEpiWarps = 16;
constexpr int kTeamWarps = 8;
constexpr int kProducerWarp0 = kIssuers > 2 ? kIssuers : 2;   // two warps stage the layer-1 inputs
constexpr int kFirstEpiWarp = kProducerWarp0 + 2;
constexpr int kProducerThreads = 64;
constexpr int kThreads = 32 * (kFirstEpiWarp + kNumEpiWarps);   // 640
// barriers: weights; per slot a_ready (the 8 warps of the team that ran the layer: next layer's A
// written), a0_full (64 producer threads), a0_empty (commit), o_full (commit of layer 5); per D region
// d_full (commit of a layer 1-4 group) and d_empty (the region's team: the accumulator is in registers).
// (O(s) needs no "free" barrier: the output warps read it before they arrive on a_ready(s) for the
// next tile's layer 2, and layer 5 of that tile is issued after its layer-4 epilogue.)
#ifndef PT_NIF_ISSUE_SLEEP
#define PT_NIF_ISSUE_SLEEP 0   // ns the issuing lane sleeps after MMAs 3 and 6 of a layer (A/B knob)
#endif
#ifndef PT_NIF_DIAG
#define PT_NIF_DIAG 0   // diagnostic builds only (wrong results): 1 = no TMEM store of A, 2 = no sine,
                        // 3 = no epilogue TMEM traffic (neither the accumulator load nor the A store),
                        // 4 = hand-off only, 5 = no output layer work (exp, stores, throughput loads),
                        // 6 = no equirect in the producers (the queue's direction read as (u, v))
#endif
enum {
    kBarW = 0,
    kBarAReady = 1,
    kBarA0Full = kBarAReady + kIssuers * kSlots,   // a_ready(s, consumer p) at kBarAReady + kIssuers s + p
    kBarA0Empty = kBarA0Full + kSlots,
    kBarOFull = kBarA0Empty + kSlots,
    kBarDFull = kBarOFull + kSlots,
    kBarDEmpty = kBarDFull + kDRegions
};

constexpr uint32_t kTmemCols = 512;
__host__ __device__ constexpr uint32_t a_col(int s) { return 64u * s; }
__host__ __device__ constexpr uint32_t o_col(int s) { return 192u + 16u * s; }
constexpr uint32_t kConstCol = 240u;
__host__ __device__ constexpr uint32_t d_col(int j) { return 256u + 128u * j; }

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
// timing trace of CTA 0 (variant builds only): [role][record][4] clock64 stamps. Issuer (role 0):
// 3 group start, 2 slot input ready, 0 D region free, 1 issued. Epilogue warp e (role 1 + e):
// 0 accumulator committed, 2 accumulator in registers (D released), 1 A stored, 3 A handed over
__device__ unsigned long long g_nif_trace[17 * 4096 * 4];
#define NIF_TRACE(role, rec, k)                                                                           \
    do {                                                                                                  \
        if (blockIdx.x == 0 && (rec) < 4096) g_nif_trace[((role) * 4096 + (rec)) * 4 + (k)] = clock64(); \
    } while (0)
#else
#define NIF_TRACE(role, rec, k) \
    do {                        \
    } while (0)
#endif

// slots of the round starting at tile t0 (tiles t0 + s * gridDim.x, s < kSlots, that exist)
__device__ __forceinline__ int slots_in_round(uint32_t t0, uint32_t n_tiles) {
    int n = 1;
    while (n < siren::kSlots && t0 + (uint32_t)n * gridDim.x < n_tiles) ++n;
    return n;
}

template <bool kDebug>
__global__ void __launch_bounds__(siren::kThreads, 1)
    siren_kernel(const uint8_t* __restrict__ g_image, const float4* __restrict__ esc,
                 const float4* __restrict__ esc_beta, const uint32_t* __restrict__ count, float* __restrict__ out,
                 float* __restrict__ dbg, int dir_input) {
    using namespace siren;
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
            mbar_init(bar(kBarA0Full + s), kProducerThreads);
            mbar_init(bar(kBarA0Empty + s), 1);
            mbar_init(bar(kBarOFull + s), 1);
        }
        for (int j = 0; j < kDRegions; ++j) {
            mbar_init(bar(kBarDFull + j), 1);
        }
        for (int j = 0; j < kIssuers; ++j) {
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

    if (warp < kIssuers) {
        // ===== MMA issuers: each walks the whole schedule and issues (one elected lane) its groups =====
        const uint32_t me = (uint32_t)warp;
        if (blockIdx.x < n_tiles) {
            mbar_wait(bar(kBarW), 0);
            const uint32_t img = smem_u32(smem);
            // per-slot / per-region barrier phases and flags as bit masks (bit s), so the dynamic slot
            // index needs no local-memory array
            uint32_t a_phase = 0, f_phase = 0, e_phase = 0;
            uint32_t pend = 0;               // bit s: a tile of slot s still needs its output layer
            uint32_t out_by_me = 0;          // bit s: that output layer is this warp's to issue
            int rec = 0;
            uint32_t g = 0;                  // layer 1-4 groups (D region g % 2)
            // layer 5 of the slot's previous tile: after its layer-4 epilogue (a_ready), into O(s)
            auto issue_out = [&](int s) {
                mbar_wait(bar(kBarAReady + kIssuers * s + (int)me), (a_phase >> s) & 1u);
                a_phase ^= 1u << s;
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
            for (uint32_t i = 0;; i += kSlots) {
                const uint32_t t0 = blockIdx.x + i * gridDim.x;
                if (t0 >= n_tiles) break;
                const int nslots = slots_in_round(t0, n_tiles);
                for (int stage = 0; stage < 4; ++stage) {
                    for (int s = 0; s < nslots; ++s, ++rec, ++g) {
                        const int j = (int)(g & 1u);
                        // the consumer of this group's epilogue is group g + nslots (the slot's next layer,
                        // or for stage 3 the output layer issued with the slot's next layer 1)
                        if (stage == 3) {
                            const bool mine_out = ((g + (uint32_t)nslots) % (uint32_t)kIssuers) == me;
                            out_by_me = mine_out ? (out_by_me | 1u << s) : (out_by_me & ~(1u << s));
                        }
                        if (stage == 0) pend |= 1u << s;
                        if (g % (uint32_t)kIssuers != me) continue;
                        if (lane == 0) NIF_TRACE(0, rec, 3);
                        if (stage == 0) {
                            if (i > 0) issue_out(s);                               // previous tile's output layer
                            mbar_wait(bar(kBarA0Full + s), (f_phase >> s) & 1u);  // layer-1 inputs staged
                            f_phase ^= 1u << s;
                        } else {
                            mbar_wait(bar(kBarAReady + kIssuers * s + (int)me), (a_phase >> s) & 1u);  // A written
                            a_phase ^= 1u << s;
                        }
                        if (lane == 0) NIF_TRACE(0, rec, 2);
                        if (g >= (uint32_t)kDRegions) {
                            mbar_wait(bar(kBarDEmpty + (int)me), e_phase & 1u);  // D region's last group loaded
                            e_phase ^= 1u;
                        }
                        if (lane == 0) NIF_TRACE(0, rec, 0);
                        tc_fence_after();
                        const uint32_t dt = tmem + d_col(j);
                        if (elect_one()) {
                            if (stage == 0) {
                                const uint64_t a0 = smem_desc(smem_u32(smem + kOffA0 + s * kA0Bytes), 2048, 128);
                                mma_ss(dt, a0, smem_desc(img, 2048, 128), idesc(128), 0);
                                mma_commit(bar(kBarDFull + j));
                                mma_commit(bar(kBarA0Empty + s));   // staging tile free once layer 1 is done
                            } else {
                                const uint32_t base = img + kOffBH + (stage - 1) * kBHBytes;
                                const uint32_t at = tmem + a_col(s);
#pragma unroll
                                for (int k = 0; k < 9; ++k) {
                                    mma_ts(dt, k < 8 ? at + 8 * k : tmem + kConstCol, smem_desc(base + k * 2 * 2048, 2048, 128),
                                           idesc(128), k > 0);
                                    if (PT_NIF_ISSUE_SLEEP > 0 && (k == 2 || k == 5)) __nanosleep(PT_NIF_ISSUE_SLEEP);
                                }
                                mma_commit(bar(kBarDFull + j));
                            }
                        }
                        __syncwarp();
                        if (lane == 0) NIF_TRACE(0, rec, 1);
                    }
                }
            }
            for (int s = 0; s < kSlots; ++s)                          // the last tiles' output layers
                if ((pend >> s) & (out_by_me >> s) & 1u) issue_out(s);
        }
    } else if (warp == kProducerWarp0 || warp == kProducerWarp0 + 1) {
        // ===== producers: layer-1 inputs of every tile, staged one tile ahead per slot =====
        // queue entry -> (u, v) (equirect of the escape direction for the render queue, reading R14)
        // -> x0 = (2u-1, 2v-1) split into fp16 hi + lo (reading R15), constant-1 bias column.
        const int p = threadIdx.x - 32 * kProducerWarp0;
        uint8_t* a0s = smem + kOffA0;
        for (int i = p; i < kSlots * kA0Bytes / 16; i += kProducerThreads)
            *reinterpret_cast<uint4*>(a0s + 16 * i) = make_uint4(0, 0, 0, 0);
        uint32_t e_phase = 0, filled = 0;   // bit s
        for (uint32_t i = 0;; i += kSlots) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = slots_in_round(t0, n_tiles);
            for (int s = 0; s < nslots; ++s) {
                const uint32_t tile = t0 + s * gridDim.x;
                if ((filled >> s) & 1u) {
                    mbar_wait(bar(kBarA0Empty + s), (e_phase >> s) & 1u);
                    e_phase ^= 1u << s;
                }
                filled |= 1u << s;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int m = p + 64 * h;
                    const uint32_t row = tile * kTileM + m;
                    float u = 0.5f, v = 0.5f;
                    if (row < n_rows) {
                        const float4 en = __ldg(esc + row);
                        u = en.x;
                        v = en.y;
                        if (dir_input && PT_NIF_DIAG != 6) equirect_f32(make_float3(en.x, en.y, en.z), u, v);
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
        // ===== epilogue warps: team t = D region t = the groups g with g % 2 == t, in issue order =====
        // Warp e of a team owns TMEM lane quarter warp % 4 (hardware rule) and the 64-column half h.
        const int e = warp - kFirstEpiWarp;
        const int team = e >> 3;
        const int h = (e >> 2) & 1;
        const int q = warp & 3;
        const uint32_t lane_addr = (uint32_t)(32 * q) << 16;
        // the constant-1 K block (fp16 (1, 0, ... 0) per row) every layer's 9th K step reads
        if (team == 0 && h == 0) {
            const uint32_t one[8] = {0x00003C00u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
            tmem_st8(tmem + kConstCol + lane_addr, one);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        // Output duty: slot s's output layer (O(s) -> exp -> store) is read by the warps (team s % 2,
        // half s / 2) after the layer-1 epilogue of the slot's next tile -- stage k of slot s is group
        // 4 kSlots r + kSlots k + s, run by team (kSlots k + s) % 2, so stages 0 and 2 of slot s belong to
        // team s % 2: the rows' throughput and queue slot are loaded at stage 2 for the output at the next
        // tile's stage 0.
        const int my_slot = 2 * h + team;            // the slot this warp outputs (if < kSlots)
        const bool out_warp = my_slot < kSlots;
        float b5[3] = {0.0f, 0.0f, 0.0f};
        if (out_warp) {
            mbar_wait(bar(kBarW), 0);
#pragma unroll
            for (int n = 0; n < 3; ++n)
                b5[n] = __half2float(*reinterpret_cast<const __half*>(smem + kOffB5 + (16 * 2) * 128 + n * 16));
        }
        uint32_t d_phase = 0, o_phase = 0;
        float4 beta = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        uint32_t oslot = 0, prow = 0;
        bool ovalid = false, pend = false;
        // layer 5 of the owned slot's previous tile: y = O[:, 0:3] + b5; radiance = beta * exp(y)
        auto output = [&](uint32_t dbg_row) {
            mbar_wait(bar(kBarOFull + my_slot), o_phase);
            o_phase ^= 1;
            tc_fence_after();
            uint32_t v[4];
            tmem_ld4(tmem + o_col(my_slot) + lane_addr, v);
            tmem_wait_ld_dep4(v);
            if (ovalid) {
                const float y0 = __uint_as_float(v[0]) + b5[0], y1 = __uint_as_float(v[1]) + b5[1],
                            y2 = __uint_as_float(v[2]) + b5[2];
                if (kDebug) {
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 0] = y0;
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 1] = y1;
                    dbg[((size_t)4 * n_rows + dbg_row) * 128 + 2] = y2;
                }
                out[3 * (size_t)oslot + 0] = beta.x * __expf(y0);
                out[3 * (size_t)oslot + 1] = beta.y * __expf(y1);
                out[3 * (size_t)oslot + 2] = beta.z * __expf(y2);
            }
        };
        const uint32_t dreg = tmem + d_col(team) + lane_addr + 64u * (uint32_t)h;
        int rec = 0;
        uint32_t g = 0;
        for (uint32_t i = 0;; i += kSlots) {
            const uint32_t t0 = blockIdx.x + i * gridDim.x;
            if (t0 >= n_tiles) break;
            const int nslots = slots_in_round(t0, n_tiles);
            for (int stage = 0; stage < 4; ++stage) {
                for (int s = 0; s < nslots; ++s, ++rec, ++g) {
                    if ((int)(g & 1u) != team) continue;
                    const uint32_t tile = t0 + s * gridDim.x;
                    const uint32_t row = tile * kTileM + 32 * q + lane;
                    const bool valid = row < n_rows;
                    mbar_wait(bar(kBarDFull + team), d_phase);
                    d_phase ^= 1;
                    if (lane == 0) NIF_TRACE(1 + e, rec, 0);
                    tc_fence_after();
                    const uint32_t areg = tmem + a_col(s) + lane_addr + 32u * (uint32_t)h;
                    // two 32-column chunks: D (fp32) -> registers (the region is released after the
                    // second load) -> sin -> fp16 pairs -> A of the next layer
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t v[32];
                        uint32_t pk[16];
                        if (PT_NIF_DIAG == 3 || PT_NIF_DIAG == 4) {
                            // diagnostic (wrong results): no accumulator load
#pragma unroll
                            for (int k = 0; k < 32; ++k) v[k] = __float_as_uint((float)(k + lane) * 0.01f);
                        } else {
                            TMEM_LD32(dreg + 32u * (uint32_t)c, v);
                            tmem_wait_ld_dep(v);
                        }
                        if (c == 1) {
                            tc_fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive(bar(kBarDEmpty + (int)((g + 2u) % (uint32_t)kIssuers)));
                            if (lane == 0) NIF_TRACE(1 + e, rec, 2);
                        }
                        if (kDebug && valid)
                            for (int k = 0; k < 32; ++k)
                                dbg[((size_t)stage * n_rows + row) * 128 + 64 * h + 32 * c + k] = __uint_as_float(v[k]);
                        if (PT_NIF_DIAG == 2 || PT_NIF_DIAG == 4) {
#pragma unroll
                            for (int k = 0; k < 16; ++k) pk[k] = v[2 * k] ^ v[2 * k + 1];
                        } else {
                            sine_half(v, 0, pk);
                            sine_half(v + 16, 1, pk + 8);
                        }
                        if (PT_NIF_DIAG != 1 && PT_NIF_DIAG != 3 && PT_NIF_DIAG != 4) {
                            TMEM_ST16(areg + 16u * (uint32_t)c, pk);
                        } else if (pk[0] == 0x7FFF7FFFu && pk[15] == 0x7FFF7FFFu) {   // diagnostic: keep pk live
                            out[0] = 0.0f;
                        }
                    }
                    if (lane == 0) NIF_TRACE(1 + e, rec, 1);
                    tmem_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar(kBarAReady + kIssuers * s + (int)((g + (uint32_t)nslots) % (uint32_t)kIssuers)));
                    // O(prev) was committed with this layer 1: read it once this warp's share of the next
                    // layer's A is handed over, off the MMA's critical path
                    if (PT_NIF_DIAG != 5 && stage == 0 && s == my_slot && pend) output(prow);
                    if (lane == 0) NIF_TRACE(1 + e, rec, 3);
                    if (PT_NIF_DIAG != 5 && stage == 2 && s == my_slot) {
                        // this tile's output rows (after the previous tile's output was written)
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
        if (PT_NIF_DIAG != 5 && out_warp && pend) output(prow);   // the last tile's output layer of the owned slot
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
