// tc_ptx.cuh -- sm_100a PTX wrappers shared by the fused NIF kernels (siren_kernel.cu, nif_kernel.cu):
// mbarrier, elect, tcgen05 fences / MMA / commit / TMEM ld-st, the hybrid SFU + fp16x2-polynomial sine
// epilogue, the equirect map of escape directions and the ReLU pack. Device code of libpt_b200 only.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

namespace pt {

// ---------------------------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase)
        : "memory");
    return ok != 0;
}
// try_wait with a suspend-time hint: the waiting warp is parked by the hardware until the phase
// completes (or ~1 ms passes) instead of spinning, so waiting warps (the MMA issuer, producers, idle
// epilogue warps) do not steal issue slots from the epilogue warps sharing their SM sub-partition
__device__ __forceinline__ bool mbar_try_sleep(uint32_t bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(phase), "r"(1000000u)
        : "memory");
    return ok != 0;
}
// bounded wait: a protocol bug traps (kernel error) instead of hanging the GPU. PT_MBAR_SPIN=1 polls
// without the suspend hint (A/B measurement of the wake-up latency)
#ifndef PT_MBAR_SPIN
#define PT_MBAR_SPIN 0
#endif
// PT_MBAR_BACKOFF: 0 = check the trap deadline every retry; 1 = every 64th retry (the retry loop of the
// warps that wait issues fewer instructions next to the epilogue warps that work); 2 = as 1 plus a
// __nanosleep(PT_MBAR_NS) between retries
#ifndef PT_MBAR_BACKOFF
#define PT_MBAR_BACKOFF 1
#endif
#ifndef PT_MBAR_NS
#define PT_MBAR_NS 32
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    if (mbar_try(bar, phase)) return;
    const long long t0 = clock64();
    uint32_t n = 0;
    while (!(PT_MBAR_SPIN ? mbar_try(bar, phase) : mbar_try_sleep(bar, phase))) {
        if (PT_MBAR_BACKOFF == 2) __nanosleep(PT_MBAR_NS);
        if (PT_MBAR_BACKOFF == 0 || (++n & 63u) == 0u) {
            if (clock64() - t0 > 4000000000ll) __trap();
        }
    }
}

__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // SWIZZLE_NONE K-major canonical layout; version bits [46,48) = 1 (sm_100)
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(id), "r"(acc)
        : "memory");
}
// e4m3 A and B (kind::f8f6f4, K = 32 per instruction); the instruction descriptor's A/B format fields
// are 0 for both f16 and e4m3, so idesc() serves both kinds
__device__ __forceinline__ void mma_ss_f8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}"
        ::"r"(d_tmem), "l"(a_desc), "l"(b_desc), "r"(id), "r"(acc)
        : "memory");
}
// e4m3 A from TMEM (4 per column), e4m3 B from shared memory (kind::f8f6f4, K = 32)
__device__ __forceinline__ void mma_ts_f8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}"
        ::"r"(d_tmem), "r"(a_tmem), "l"(b_desc), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

#define TMEM_LD32(taddr, v)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
        "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                              \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),          \
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),    \
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),  \
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])   \
        : "r"(taddr))

#define TMEM_ST16(taddr, v)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"   \
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),      \
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])              \
        : "memory")

#define TMEM_LD16(taddr, v)                                                                                    \
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
                 : "=r"((v)[0]), "=r"((v)[1]), "=r"((v)[2]), "=r"((v)[3]), "=r"((v)[4]), "=r"((v)[5]),         \
                   "=r"((v)[6]), "=r"((v)[7]), "=r"((v)[8]), "=r"((v)[9]), "=r"((v)[10]), "=r"((v)[11]),        \
                   "=r"((v)[12]), "=r"((v)[13]), "=r"((v)[14]), "=r"((v)[15])                                   \
                 : "r"(taddr))
// wait for all prior tcgen05.ld of this thread, pinning the 16 registers of one of them
__device__ __forceinline__ void tmem_wait_ld_dep16(uint32_t* v) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                   "+r"(v[15])
                 :
                 : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t* v) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
    const __half2 h = __floats2half2_rn(lo, hi);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// wait for all prior tcgen05.ld of this thread; the register operands pin later uses of v after it
__device__ __forceinline__ void tmem_wait_ld_dep(uint32_t* v) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),
                   "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),
                   "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                   "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),
                   "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
                 :
                 : "memory");
}

__device__ __forceinline__ void tmem_wait_ld_dep4(uint32_t* v) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]) : : "memory");
}

// Sine epilogue, split between two pipes: the SFU (MUFU.SIN, 16 lanes/clk/SM) and
// the FMA pipe, where sin runs as an fp16x2 odd polynomial after an fp32 quarter-period reduction
// w = |frac(x/2pi + 1/4)| - 1/4, sin(x) = sin(2 pi w), |w| <= 1/4 (max abs error 1.1e-3 in fp16).
#ifndef PT_NIF_MUFU_PAIRS
#define PT_NIF_MUFU_PAIRS 9   // of the 16 column pairs of a 32-column chunk, on the SFU
#endif
__device__ __forceinline__ uint32_t sin2_poly(float a, float b) {
    // packed fp32x2 range reduction (FFMA2/FADD2, sm_100), then an fp16x2 odd polynomial
    constexpr float kInv2Pi = 0.15915494309189535f;
    constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23: x + magic - magic = rint(x)
    const float2 sv = __ffma2_rn(make_float2(a, b), make_float2(kInv2Pi, kInv2Pi), make_float2(0.25f, 0.25f));
    const float2 tv = __fadd2_rn(sv, make_float2(kMagic, kMagic));
    const float2 kv = __fadd2_rn(tv, make_float2(-kMagic, -kMagic));
    const float2 uv = __fadd2_rn(sv, make_float2(-kv.x, -kv.y));
    const float2 wv = __fadd2_rn(make_float2(fabsf(uv.x), fabsf(uv.y)), make_float2(-0.25f, -0.25f));
    const __half2 w = __floats2half2_rn(wv.x, wv.y);
    const __half2 w2 = __hmul2(w, w);
    const __half2 c1 = __halves2half2(__ushort_as_half(0x4648), __ushort_as_half(0x4648));   //  6.28125
    const __half2 c3 = __halves2half2(__ushort_as_half(0xD123), __ushort_as_half(0xD123));   // -41.09375
    const __half2 c5 = __halves2half2(__ushort_as_half(0x5499), __ushort_as_half(0x5499));   //  73.5625
    __half2 p = __hfma2(w2, c5, c3);
    p = __hfma2(p, w2, c1);
    const __half2 r = __hmul2(p, w);
    return *reinterpret_cast<const uint32_t*>(&r);
}
// as sin2_poly with the layer's bias folded into the reduction: q = 1/4 + b/(2 pi), sin(x + b) per lane
__device__ __forceinline__ uint32_t sin2_poly_q(float a, float b, float q) {
    constexpr float kInv2Pi = 0.15915494309189535f;
    constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23: x + magic - magic = rint(x)
    const float2 sv = __ffma2_rn(make_float2(a, b), make_float2(kInv2Pi, kInv2Pi), make_float2(q, q));
    const float2 tv = __fadd2_rn(sv, make_float2(kMagic, kMagic));
    const float2 kv = __fadd2_rn(tv, make_float2(-kMagic, -kMagic));
    const float2 uv = __fadd2_rn(sv, make_float2(-kv.x, -kv.y));
    const float2 wv = __fadd2_rn(make_float2(fabsf(uv.x), fabsf(uv.y)), make_float2(-0.25f, -0.25f));
    const __half2 w = __floats2half2_rn(wv.x, wv.y);
    const __half2 w2 = __hmul2(w, w);
    const __half2 c1 = __halves2half2(__ushort_as_half(0x4648), __ushort_as_half(0x4648));   //  6.28125
    const __half2 c3 = __halves2half2(__ushort_as_half(0xD123), __ushort_as_half(0xD123));   // -41.09375
    const __half2 c5 = __halves2half2(__ushort_as_half(0x5499), __ushort_as_half(0x5499));   //  73.5625
    __half2 p = __hfma2(w2, c5, c3);
    p = __hfma2(p, w2, c1);
    const __half2 r = __hmul2(p, w);
    return *reinterpret_cast<const uint32_t*>(&r);
}
// half of a 32-column chunk (pairs 8 h .. 8 h + 7), loaded while the other half is computed; the SFU
// pairs are the even ones plus pair 1 (9 of 16 at the default), so both halves carry a similar SFU share
__device__ __forceinline__ bool sfu_pair(int j) {
    return PT_NIF_MUFU_PAIRS >= 16 || (j % 2 == 0 ? j / 2 < PT_NIF_MUFU_PAIRS : (j - 1) / 2 + 8 < PT_NIF_MUFU_PAIRS);
}
__device__ __forceinline__ void sine_half(const uint32_t* v, int h, uint32_t* p) {
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) {
        const int j = 8 * h + jj;
        const float a = __uint_as_float(v[2 * jj]), b = __uint_as_float(v[2 * jj + 1]);
        p[jj] = sfu_pair(j) ? pack_half2(__sinf(a), __sinf(b)) : sin2_poly(a, b);
    }
}
__device__ __forceinline__ void sine_chunk(const uint32_t* v, uint32_t* p) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float a = __uint_as_float(v[2 * j]), b = __uint_as_float(v[2 * j + 1]);
        p[j] = j < PT_NIF_MUFU_PAIRS ? pack_half2(__sinf(a), __sinf(b)) : sin2_poly(a, b);
    }
}


// atan2 on the FMA pipe: octant reduction to a = min/max in [0, 1], a degree-15 odd polynomial (8
// coefficients fitted for minimax error on [0, 1]: 3.7e-8 in exact arithmetic, <= 1.6e-7 rad evaluated in
// fp32; tools/equirect_check.cu measures the whole map against fp64), then the octant's reflections; atan2(+-0, x < 0) = +-pi like atan2f. (y, x) = (0, 0) is the
// caller's case.
__device__ __forceinline__ float atan2_poly(float y, float x) {
    const float ax = fabsf(x), ay = fabsf(y);
    const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
    const float a = mx > 0.0f ? __fdividef(mn, mx) : 0.0f;   // 2 ulp: adds <= 2.4e-7 rad
    const float s = a * a;
    float p = -0.004054564982652664f;
    p = fmaf(p, s, 0.021862955763936043f);
    p = fmaf(p, s, -0.055912334471940994f);
    p = fmaf(p, s, 0.0964219868183136f);
    p = fmaf(p, s, -0.1390863060951233f);
    p = fmaf(p, s, 0.19946566224098206f);
    p = fmaf(p, s, -0.33329859375953674f);
    p = fmaf(p, s, 0.9999993443489075f);
    float r = p * a;
    if (ay > ax) r = 1.57079637f - r;
    if (x < 0.0f) r = 3.14159274f - r;
    return copysignf(r, y);
}

// Equirect map of an escaped direction (S4 -> S5; moved here from the trace kernel so the divergent
// atan2/acos run once per queued ray in the NIF prologue instead of in the traversal warps).
// v = acos(d.y / |d|) / pi is evaluated as atan2(|(d.x, d.z)|, d.y) / pi: the same angle, well conditioned
// at the poles (acos of a rounded cosine near +-1 loses ~sqrt(eps) there), and both angles go through
// atan2_poly (the producer warps' share of the NIF's issue slots).
__device__ __forceinline__ void equirect_f32(float3 d, float& u, float& v) {
    // SPEC.md:438 convention (reading R14): u = 0.5 + atan2(d.x, -d.z)/2pi wrapped to [0,1); v = acos(d.y)/pi
    float uu;
    if (d.x == 0.0f && d.z == 0.0f) uu = 0.5f;
    else {
        uu = 0.5f + atan2_poly(d.x, -d.z) * (0.5f / CUDART_PI_F);
        if (uu >= 1.0f) uu -= 1.0f;
    }
    const float h = sqrtf(d.x * d.x + d.z * d.z);
    u = uu;
    v = (h == 0.0f && d.y == 0.0f) ? 0.5f : atan2_poly(h, d.y) * (1.0f / CUDART_PI_F);
}

// ReLU epilogue of the paper's NIF: relu + fp16x2 pack in one cvt per pair
__device__ __forceinline__ uint32_t relu_pack(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

}  // namespace pt
