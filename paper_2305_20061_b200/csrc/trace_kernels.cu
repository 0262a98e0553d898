// trace_kernels.cu -- wavefront path-tracing kernels for sm_100a: raygen, traverse, shade (scatter +
// Russian roulette + warp-aggregated compaction of alive and escaped paths), accumulate.
//
// Method (PAPER.md = /root/reference/PAPER.md line): no light sampling, contributions from emitters
// hit by chance and from escaped rays; escaped rays are queued for the batched HDR-NIF
// ("we need to run inference on large batches of ray queries"); Russian roulette from
// depth 3 with survival proportional to throughput. Wide compressed BVH with
// conservative fp16 child boxes. Readings R1-R22 in DESIGN.md.
//
// Exactness contract with the fp64 oracle: camera rays are computed with
// explicitly rounded fp32 intrinsics (no contraction), primitive tests run in fp64 with explicitly
// rounded intrinsics in the oracle's operation order, so primary hits are bit-identical.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>

#include "pt_internal.h"

namespace pt {

// ---------------------------------------------------------------------------------------------
// Philox-4x32-10 (Salmon et al. SC'11), counter (pixel, sample, slot, stream), key = seed (R13)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox10(uint4 c, uint2 k) {
#pragma unroll
    for (int i = 0; i < 10; ++i) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}
__device__ __forceinline__ float u01f(uint32_t x) { return (float)(x >> 8) * 0x1p-24f; }  // exact

// ---------------------------------------------------------------------------------------------
// Camera (fp32, explicitly rounded, reading R22)
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ float3 cam_dir(const Cam32& k, int W, int H, int x, int y, float xi0, float xi1) {
    const float px = __fadd_rn((float)x, xi0);
    const float py = __fadd_rn((float)y, xi1);
    const float sx = __fsub_rn(__fdiv_rn(__fmul_rn(2.0f, px), (float)W), 1.0f);
    const float sy = __fsub_rn(1.0f, __fdiv_rn(__fmul_rn(2.0f, py), (float)H));
    const float cx = __fmul_rn(sx, k.ta);
    const float cy = __fmul_rn(sy, k.t);
    float v[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) v[a] = __fadd_rn(__fadd_rn(k.f[a], __fmul_rn(cx, k.r[a])), __fmul_rn(cy, k.u[a]));
    const float l2 = __fadd_rn(__fadd_rn(__fmul_rn(v[0], v[0]), __fmul_rn(v[1], v[1])), __fmul_rn(v[2], v[2]));
    const float l = __fsqrt_rn(l2);
    return make_float3(__fdiv_rn(v[0], l), __fdiv_rn(v[1], l), __fdiv_rn(v[2], l));
}

// ---------------------------------------------------------------------------------------------
// Primitive tests. Decisions are exactly those of the fp64 oracle (watertight: Woop/Benthin/Wald
// 2013): a conservative fp32 pre-test rejects only triangles whose edge functions have
// mixed signs by more than a proven fp32 error bound; every remaining candidate is decided in fp64
// with explicitly rounded intrinsics in the oracle's operation order (R22).
// ---------------------------------------------------------------------------------------------
// Kept compact (14 registers) because it is live through the whole traversal under the path kernels'
// 72-register cap; the shear matrix of the certified pre-test is rebuilt inside each triangle test.
// PT_RAY_LOCAL=1: the origin and the slab reciprocals also live in the local-memory record (two 16-B
// loads per node visit instead of registers the 72-register cap spills anyway)
#ifndef PT_RAY_LOCAL
#define PT_RAY_LOCAL 0   // measured slower (2.72 vs 2.78 G samples/s on config 3, profiles/round2/raylocal.log)
#endif
constexpr int kColdBytes = PT_RAY_LOCAL ? 64 : 32;
struct RayT {
#if !PT_RAY_LOCAL
    float o[3], inv[3];         // slab test
#endif
    uint32_t kbits;             // kx | ky << 2 | kz << 4 | negmask << 8 (bit a: d[a] has its sign bit set)
    uint32_t cold;              // local-memory address of (Sx, Sy, rz, |d[kz]|) (d.x, d.y, d.z, 0) [(o, 0)
                                // (inv, 0)]: spilled by hand, not by ptxas
};
__device__ __forceinline__ float4 ldl4(uint32_t a) {
    float4 v;
    asm volatile("ld.local.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void stl4(uint32_t a, float4 v) {
    asm volatile("st.local.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float4 ray_shear_consts(const RayT& r) { return ldl4(r.cold); }   // Sx, Sy, rz, |d[kz]|
__device__ __forceinline__ float3 ray_o(const RayT& r) {
#if PT_RAY_LOCAL
    const float4 v = ldl4(r.cold + 32);
    return make_float3(v.x, v.y, v.z);
#else
    return make_float3(r.o[0], r.o[1], r.o[2]);
#endif
}
__device__ __forceinline__ float3 ray_inv(const RayT& r) {
#if PT_RAY_LOCAL
    const float4 v = ldl4(r.cold + 48);
    return make_float3(v.x, v.y, v.z);
#else
    return make_float3(r.inv[0], r.inv[1], r.inv[2]);
#endif
}
__device__ __forceinline__ float3 ray_dir(const RayT& r) {
    const float4 v = ldl4(r.cold + 16);
    return make_float3(v.x, v.y, v.z);
}
__device__ __forceinline__ int ray_kx(const RayT& r) { return (int)(r.kbits & 3u); }
__device__ __forceinline__ int ray_ky(const RayT& r) { return (int)((r.kbits >> 2) & 3u); }
__device__ __forceinline__ int ray_kz(const RayT& r) { return (int)((r.kbits >> 4) & 3u); }
// fp32 shear as a matrix over the world axes a, so a vertex is sheared with packed FFMA2s instead of
// permutation selects: (Ax, Ay) = sum_a mxy[a] (v - o)_a with mxy[a] = ((e_kx - Sx e_kz)_a,
// (e_ky - Sy e_kz)_a), Az = sum_a mz[a] (v - o)_a with mz = Sz e_kz
struct Shear32 {
    float2 mxy[3];
    float mz[3];
};
__device__ __forceinline__ Shear32 shear_matrix(const RayT& r, float4 sc) {
    uint32_t kb = r.kbits;
    asm volatile("" : "+r"(kb));   // rebuilt per test: keep the compiler from hoisting it into registers
    const int kx = (int)(kb & 3u), ky = (int)((kb >> 2) & 3u), kz = (int)((kb >> 4) & 3u);
    Shear32 m;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        m.mxy[a] = make_float2(a == kx ? 1.0f : (a == kz ? -sc.x : 0.0f), a == ky ? 1.0f : (a == kz ? -sc.y : 0.0f));
        m.mz[a] = a == kz ? sc.z : 0.0f;
    }
    return m;
}

// 32-B read-only global load (LDG.E.ENL2.256), p 32-B aligned
__device__ __forceinline__ void ldg256(const uint4* p, uint4& a, uint4& b) {
    asm("ld.global.nc.v8.u32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w)
        : "l"(p));
}

__device__ __forceinline__ float self3(float3 v, int k) { return k == 0 ? v.x : (k == 1 ? v.y : v.z); }

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// n / d for n < 2^31, quotient < 2^20, with inv = fl(1 / d): the fp32 estimate is within one of the
// quotient (relative error < 2^-22), then one exact correction each way; r = n - q d
__device__ __forceinline__ uint32_t udiv_exact(uint32_t n, uint32_t d, float inv, uint32_t& r) {
    uint32_t q = __float2uint_rz(__uint2float_rn(n) * inv);
    int32_t rr = (int32_t)(n - q * d);
    if (rr < 0) {
        --q;
        rr += (int32_t)d;
    } else if (rr >= (int32_t)d) {
        ++q;
        rr -= (int32_t)d;
    }
    r = (uint32_t)rr;
    return q;
}

__device__ __forceinline__ void ray_prepare(float3 o, float3 d, RayT& r, uint32_t cold) {
    int kz = 0;
    if (fabsf(d.y) > fabsf(d.x)) kz = 1;
    if (fabsf(d.z) > fabsf(self3(d, kz))) kz = 2;
    int kx = kz + 1; if (kx == 3) kx = 0;
    int ky = kx + 1; if (ky == 3) ky = 0;
    const float dkz = self3(d, kz);
    if (dkz < 0.0f) { int t = kx; kx = ky; ky = t; }
    // fp32 shear for the pre-test only (its error bound tolerates the reciprocal-multiply form);
    // the fp64 shear of the exact test is recomputed by each (rare) fp64 test: caching it would keep
    // six more registers live through the whole traversal
    const float rz = __frcp_rn(dkz);
    r.cold = cold;
    stl4(cold, make_float4(self3(d, kx) * rz, self3(d, ky) * rz, rz, fabsf(dkz)));
    stl4(cold + 16, make_float4(d.x, d.y, d.z, 0.0f));
    // slab reciprocals: the SFU approximation (<= 1 ulp); the slab bound below allows for its rounding
#if PT_RAY_LOCAL
    stl4(cold + 32, make_float4(o.x, o.y, o.z, 0.0f));
    stl4(cold + 48, make_float4(rcp_approx(d.x), rcp_approx(d.y), rcp_approx(d.z), 0.0f));
#else
    r.o[0] = o.x; r.o[1] = o.y; r.o[2] = o.z;
    r.inv[0] = rcp_approx(d.x); r.inv[1] = rcp_approx(d.y); r.inv[2] = rcp_approx(d.z);
#endif
    const uint32_t negmask = (signbit(d.x) ? 1u : 0u) | (signbit(d.y) ? 2u : 0u) | (signbit(d.z) ? 4u : 0u);
    r.kbits = (uint32_t)kx | ((uint32_t)ky << 2) | ((uint32_t)kz << 4) | (negmask << 8);
}

// fp64 shear constants, exactly the oracle's divisions
struct Shear64 {
    double Sx, Sy, Sz;
};
__device__ __forceinline__ Shear64 shear64(const RayT& r) {
    const float3 d = ray_dir(r);
    const double dkz64 = (double)self3(d, ray_kz(r));
    return {__ddiv_rn((double)self3(d, ray_kx(r)), dkz64), __ddiv_rn((double)self3(d, ray_ky(r)), dkz64), __ddiv_rn(1.0, dkz64)};
}

// Shear one vertex into the ray's frame: D = v - o (world axes, one rounding each), then the products
// with the 0/1/-S entries of the shear rows; at most two roundings per sheared coordinate (the -S
// product and the sum), the same single-rounding Sz D[kz] for Az as the permuted form.
__device__ __forceinline__ void shear_vertex(float3 ro, const Shear32& m, float3 v, float& x, float& y, float& z) {
    const float2 dxy = __fadd2_rn(make_float2(v.x, v.y), make_float2(-ro.x, -ro.y));
    const float dz = v.z - ro.z;
    float2 a = __fmul2_rn(m.mxy[0], make_float2(dxy.x, dxy.x));
    a = __ffma2_rn(m.mxy[1], make_float2(dxy.y, dxy.y), a);
    a = __ffma2_rn(m.mxy[2], make_float2(dz, dz), a);
    x = a.x;
    y = a.y;
    z = fmaf(m.mz[2], dz, fmaf(m.mz[1], dxy.y, m.mz[0] * dxy.x));
}

// Certified fp32 watertight test. Returns 0 if the exact (hence the fp64 oracle's) test certainly
// misses, 1 if it certainly hits with t in [t - dt, t + dt], t - dt > 0, and 2 if undecided (near an
// edge or t ~ 0): then the fp64 test decides. Error bounds: with eps = 2^-24,
// mX >= max|A[kx]| + |Sx| max|A[kz]| (over the 3 vertices; computed as max|Ax| + 2|Sx| max|A[kz]|) and
// likewise mY, the sheared coordinates carry |dAx| <= eX = 5 eps mX, |dAy| <= eY = 5 eps mY (two
// roundings, the D = v - o rounding and the fp32 S). First a uniform bound on the edge functions,
// |dU| <= 23 eps mX mY (we use 26); if that leaves the signs undecided (ray origins far from small
// triangles: mX mY >> |U|), per-edge bounds that scale with the sheared coordinates themselves,
//   |dU| <= eX (|By| + |Cy|) + eY (|Bx| + |Cx|) + eps (|U| + |Cy Bx|) + 50 eps^2 mX mY
// (U = Cx By - Cy Bx; likewise V, W), plus 2^-44 mX mY for the fp64 oracle's own rounding, times 1.125.
// Then |dT| <= (eU + eV + eW) mZ + 18 eps maxE mZ, |ddet| <= eU + eV + eW + 6 eps maxE, mZ >= max|Az|.
__device__ __forceinline__ int tri_test32(const RayT& r, float3 v0, float3 v1, float3 v2, float& t, float& dt) {
    constexpr float eps = 0x1p-24f;
    float Ax, Ay, Az, Bx, By, Bz, Cx, Cy, Cz;
    const float4 sc = ray_shear_consts(r);
    const Shear32 m = shear_matrix(r, sc);
    const float3 ro = ray_o(r);
    shear_vertex(ro, m, v0, Ax, Ay, Az);
    shear_vertex(ro, m, v1, Bx, By, Bz);
    shear_vertex(ro, m, v2, Cx, Cy, Cz);
    const float CyBx = Cy * Bx, AyCx = Ay * Cx, ByAx = By * Ax;
    const float U = fmaf(Cx, By, -CyBx);
    const float V = fmaf(Ax, Cy, -AyCx);
    const float W = fmaf(Bx, Ay, -ByAx);
    const float mZ = (1.0f + 2.0f * eps) * fmaxf(fabsf(Az), fmaxf(fabsf(Bz), fabsf(Cz)));   // >= max|Sz A[kz]|
    const float mz2 = (1.0f + 4.0f * eps) * mZ * sc.w;                                        // >= max|A[kz]|
    const float mX = fmaf(2.0f * fabsf(sc.x), mz2, fmaxf(fabsf(Ax), fmaxf(fabsf(Bx), fabsf(Cx))));
    const float mY = fmaf(2.0f * fabsf(sc.y), mz2, fmaxf(fabsf(Ay), fmaxf(fabsf(By), fabsf(Cy))));
    float eU = (26.0f * eps) * mX * mY, eV = eU, eW = eU;
    bool neg = U < -eU || V < -eV || W < -eW;
    bool pos = U > eU || V > eV || W > eW;
    if (neg && pos) return 0;
    bool certain = (U > eU && V > eV && W > eW) || (U < -eU && V < -eV && W < -eW);
    if (!certain) {
        const float eX = (5.0f * eps) * mX, eY = (5.0f * eps) * mY;
        const float tail = (50.0f * eps * eps + 0x1p-44f) * mX * mY;
        const float aAx = fabsf(Ax), aAy = fabsf(Ay), aBx = fabsf(Bx), aBy = fabsf(By), aCx = fabsf(Cx), aCy = fabsf(Cy);
        eU = 1.125f * (eX * (aBy + aCy) + eY * (aBx + aCx) + eps * (fabsf(U) + fabsf(CyBx)) + tail);
        eV = 1.125f * (eX * (aCy + aAy) + eY * (aCx + aAx) + eps * (fabsf(V) + fabsf(AyCx)) + tail);
        eW = 1.125f * (eX * (aAy + aBy) + eY * (aAx + aBx) + eps * (fabsf(W) + fabsf(ByAx)) + tail);
        neg = U < -eU || V < -eV || W < -eW;
        pos = U > eU || V > eV || W > eW;
        if (neg && pos) return 0;
        certain = (U > eU && V > eV && W > eW) || (U < -eU && V < -eV && W < -eW);
        if (!certain) return 2;
    }
    const float det = U + V + W;
    const float T = fmaf(W, Cz, fmaf(V, Bz, U * Az));
    const float maxE = fmaxf(fabsf(U), fmaxf(fabsf(V), fabsf(W)));
    const float eSum = eU + eV + eW;
    const float dT = eSum * mZ + (18.0f * eps) * maxE * mZ;
    const float dDet = eSum + (6.0f * eps) * maxE;
    const float adet = fabsf(det);
    if (adet <= 2.0f * dDet) return 2;
    // t = T / det via rcp.approx (max error 1 ulp) and one rounded product: |t - T/det| <= 3 eps |t|
    // (bounded with 6 eps); the bound's own quotient carries the same relative error, inside the 1.25
    t = T * rcp_approx(det);
    dt = 1.25f * ((dT + fabsf(t) * dDet) * rcp_approx(adet - dDet) + (6.0f * eps) * fabsf(t));
    if (!(dt < CUDART_INF_F)) return 2;          // subnormal det (flushed by rcp.approx.ftz) or overflow
    if (t + dt <= 0.0f) return 0;
    if (t - dt <= 0.0f) return 2;
    return 1;
}

// fp64 watertight test in the oracle's operation order; true and t if hit with t > 0
__device__ __forceinline__ bool tri_test64(RayT& r, float3 v0, float3 v1, float3 v2, double& t_out) {
    const Shear64 sh = shear64(r);
    const float3 o32 = ray_o(r);
    const int kx = ray_kx(r), ky = ray_ky(r), kz = ray_kz(r);
    const double ox = self3(o32, kx), oy = self3(o32, ky), oz = self3(o32, kz);
    const double A0 = __dsub_rn((double)self3(v0, kx), ox);
    const double A1 = __dsub_rn((double)self3(v0, ky), oy);
    const double A2 = __dsub_rn((double)self3(v0, kz), oz);
    const double B0 = __dsub_rn((double)self3(v1, kx), ox);
    const double B1 = __dsub_rn((double)self3(v1, ky), oy);
    const double B2 = __dsub_rn((double)self3(v1, kz), oz);
    const double C0 = __dsub_rn((double)self3(v2, kx), ox);
    const double C1 = __dsub_rn((double)self3(v2, ky), oy);
    const double C2 = __dsub_rn((double)self3(v2, kz), oz);
    const double Ax = __dsub_rn(A0, __dmul_rn(sh.Sx, A2));
    const double Ay = __dsub_rn(A1, __dmul_rn(sh.Sy, A2));
    const double Bx = __dsub_rn(B0, __dmul_rn(sh.Sx, B2));
    const double By = __dsub_rn(B1, __dmul_rn(sh.Sy, B2));
    const double Cx = __dsub_rn(C0, __dmul_rn(sh.Sx, C2));
    const double Cy = __dsub_rn(C1, __dmul_rn(sh.Sy, C2));
    const double U = __dsub_rn(__dmul_rn(Cx, By), __dmul_rn(Cy, Bx));
    const double V = __dsub_rn(__dmul_rn(Ax, Cy), __dmul_rn(Ay, Cx));
    const double Wt = __dsub_rn(__dmul_rn(Bx, Ay), __dmul_rn(By, Ax));
    if ((U < 0.0 || V < 0.0 || Wt < 0.0) && (U > 0.0 || V > 0.0 || Wt > 0.0)) return false;
    const double det = __dadd_rn(__dadd_rn(U, V), Wt);
    if (det == 0.0) return false;
    const double Az = __dmul_rn(sh.Sz, A2);
    const double Bz = __dmul_rn(sh.Sz, B2);
    const double Cz = __dmul_rn(sh.Sz, C2);
    const double T = __dadd_rn(__dadd_rn(__dmul_rn(U, Az), __dmul_rn(V, Bz)), __dmul_rn(Wt, Cz));
    if (det < 0.0 && T >= 0.0) return false;
    if (det > 0.0 && T <= 0.0) return false;
    t_out = __ddiv_rn(T, det);
    return true;
}

__device__ __forceinline__ bool sph_test64(RayT& r, float3 c, float rad, double& t_out) {
    const float3 dd = ray_dir(r);
    const double d0 = dd.x, d1 = dd.y, d2 = dd.z;
    const float3 ro = ray_o(r);
    const double oc0 = __dsub_rn((double)ro.x, (double)c.x);
    const double oc1 = __dsub_rn((double)ro.y, (double)c.y);
    const double oc2 = __dsub_rn((double)ro.z, (double)c.z);
    const double a = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
    const double b = __dadd_rn(__dadd_rn(__dmul_rn(oc0, d0), __dmul_rn(oc1, d1)), __dmul_rn(oc2, d2));
    const double cc = __dsub_rn(__dadd_rn(__dadd_rn(__dmul_rn(oc0, oc0), __dmul_rn(oc1, oc1)), __dmul_rn(oc2, oc2)),
                                __dmul_rn((double)rad, (double)rad));
    const double disc = __dsub_rn(__dmul_rn(b, b), __dmul_rn(a, cc));
    if (disc < 0.0) return false;
    const double sq = __dsqrt_rn(disc);
    const double t0 = __ddiv_rn(__dsub_rn(-b, sq), a);
    const double t1 = __ddiv_rn(__dadd_rn(-b, sq), a);
    if (t0 > 0.0) { t_out = t0; return true; }
    if (t1 > 0.0) { t_out = t1; return true; }
    return false;
}

// Certified fp32 ray/sphere test (same contract as tri_test32): with a = d.d, q = |oc|^2 + r^2 the
// discriminant carries |d disc| <= 24 eps a q (we use 32), b <= 5 eps |oc||d|, and the roots inherit
// |dt| <= (db + d sqrt(disc)) / a + 5 eps |t|. Grazing rays and roots near 0 defer to fp64.
__device__ __forceinline__ int sph_test32(const RayT& r, float3 c, float rad, float& t, float& dt) {
    constexpr float eps = 0x1p-24f;
    const float3 ro = ray_o(r);
    const float ox = ro.x - c.x, oy = ro.y - c.y, oz = ro.z - c.z;
    const float3 dd = ray_dir(r);
    const float a = fmaf(dd.x, dd.x, fmaf(dd.y, dd.y, dd.z * dd.z));
    const float b = fmaf(ox, dd.x, fmaf(oy, dd.y, oz * dd.z));
    const float oc2 = fmaf(ox, ox, fmaf(oy, oy, oz * oz));
    const float cc = oc2 - rad * rad;
    const float disc = fmaf(b, b, -a * cc);
    const float q = oc2 + rad * rad;
    const float ddisc = (32.0f * eps) * a * q;
    if (disc < -ddisc) return 0;
    if (disc <= ddisc) return 2;
    const float sq = sqrtf(disc);
    const float dsq = ddisc / (sqrtf(disc - ddisc) + sq) + 2.0f * eps * sq;
    const float db = (5.0f * eps) * sqrtf(oc2 * a);
    const float ia = 1.0f / a;
    const float t0 = (-b - sq) * ia, t1 = (-b + sq) * ia;
    const float e0 = (db + dsq) * ia + (5.0f * eps) * fabsf(t0);
    const float e1 = (db + dsq) * ia + (5.0f * eps) * fabsf(t1);
    if (t0 - e0 > 0.0f) { t = t0; dt = 1.25f * e0; return 1; }
    if (t0 + e0 > 0.0f) return 2;                 // smaller root near 0: undecided
    if (t1 - e1 > 0.0f) { t = t1; dt = 1.25f * e1; return 1; }
    if (t1 + e1 > 0.0f) return 2;
    return 0;
}

// ---------------------------------------------------------------------------------------------
// Wide-BVH closest hit: (t, id) lexicographic minimum over all primitives (reading R11)
// ---------------------------------------------------------------------------------------------
// Best hit so far. Decided exactly like the fp64 oracle, but carried as a certified fp32 interval
// [tlo, thi] until a near-tie forces the exact fp64 t (exact == true).
#ifdef PT_TAIL_TRACE
// tail-analysis build (tools/tail_trace.py): globaltimer at each warp's exit, [kernel][warp]
__device__ unsigned long long g_tail[2][1 << 14];
__device__ __forceinline__ void tail_stamp(int k) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if ((threadIdx.x & 31) == 0 && w < (1 << 14)) g_tail[k][w] = t;
}
#define TAIL_STAMP(k) tail_stamp(k)
#else
#define TAIL_STAMP(k) do { } while (0)
#endif
#ifdef PT_COUNT
// counting build (tools/trace_count.py): node visits, box tests, primitive tests, fp64 tests, rays
__device__ unsigned long long g_trav_count[8];
#define TCOUNT(i, v) atomicAdd(&g_trav_count[i], (unsigned long long)(v))
#else
#define TCOUNT(i, v) do { } while (0)
#endif

struct Hit {
    double t;
    float tlo, thi;
    int32_t prim;
    uint32_t unit;
    bool exact;
};

__device__ __forceinline__ float half_bits_to_float(uint32_t h) {
    return __half2float(__ushort_as_half((unsigned short)(h & 0x7FFFu)));
}

__device__ __forceinline__ float cull_bound(const Hit& best) {
    // fp32 upper bound of the best t with margin for the slab rounding
    return best.prim < 0 ? CUDART_INF_F : __fmul_ru(best.thi, 1.0000005f);
}

// exact fp64 test of the primitive stored at `unit`
__device__ __forceinline__ bool exact_test(const uint4* __restrict__ pool, uint32_t unit, RayT& r, double& t) {
    const uint4 u0 = __ldg(pool + unit);
    const uint4 u1 = __ldg(pool + unit + 1);
    const float3 p0 = make_float3(__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z));
    if (u0.w & kSphereFlag) return sph_test64(r, p0, __uint_as_float(u1.x), t);
    const uint4 u2 = __ldg(pool + unit + 2);
    return tri_test64(r, p0, make_float3(__uint_as_float(u1.x), __uint_as_float(u1.y), __uint_as_float(u1.z)),
                      make_float3(__uint_as_float(u2.x), __uint_as_float(u2.y), __uint_as_float(u2.z)), t);
}

__device__ __forceinline__ void test_prim(const uint4* __restrict__ pool, uint32_t unit, RayT& r, Hit& best) {
    const uint4 u0 = __ldg(pool + unit);
    const uint4 u1 = __ldg(pool + unit + 1);
    const uint32_t idw = u0.w;
    const int32_t id = (int32_t)(idw & ~kSphereFlag);
    const float3 p0 = make_float3(__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z));
    double t64 = 0.0;
    float t32 = 0.0f, dt = 0.0f;
    bool exact;
    TCOUNT(2, 1);
    if (idw & kSphereFlag) {
        const int c = sph_test32(r, p0, __uint_as_float(u1.x), t32, dt);
        if (c == 0) return;
        if (c == 2) {
            if (!sph_test64(r, p0, __uint_as_float(u1.x), t64)) return;
            exact = true;
        } else {
            exact = false;
        }
    } else {
        const uint4 u2 = __ldg(pool + unit + 2);
        const float3 p1 = make_float3(__uint_as_float(u1.x), __uint_as_float(u1.y), __uint_as_float(u1.z));
        const float3 p2 = make_float3(__uint_as_float(u2.x), __uint_as_float(u2.y), __uint_as_float(u2.z));
        const int c = tri_test32(r, p0, p1, p2, t32, dt);
        if (c == 0) return;
        if (c == 2) {
            TCOUNT(3, 1);
            if (!tri_test64(r, p0, p1, p2, t64)) return;
            exact = true;
        } else {
            exact = false;
        }
    }
    const float tlo = exact ? __double2float_rd(t64) : t32 - dt;
    const float thi = exact ? __double2float_ru(t64) : t32 + dt;
    if (best.prim >= 0) {
        if (tlo > best.thi) return;                 // certainly farther
        if (!(thi < best.tlo)) {                    // not certainly closer: decide exactly, as the oracle
            if (!exact) {
                if (!exact_test(pool, unit, r, t64)) return;
                exact = true;
            }
            if (!best.exact) {
                double tb;
                exact_test(pool, best.unit, r, tb);
                best.t = tb;
                best.tlo = __double2float_rd(tb);
                best.thi = __double2float_ru(tb);
                best.exact = true;
            }
            if (!(t64 < best.t || (t64 == best.t && id < best.prim))) return;
        }
    }
    best.prim = id;
    best.unit = unit;
    best.exact = exact;
    best.t = exact ? t64 : (double)t32;
    best.tlo = exact ? __double2float_rd(t64) : tlo;
    best.thi = exact ? __double2float_ru(t64) : thi;
}

// child order at an interior node: 5 = full sorting network; 3 = nearest first, the other three only
// partially ordered (A/B knob: the closest hit does not depend on the visit order, ties break on (t, id))
#ifndef PT_CHILD_SORT
#define PT_CHILD_SORT 5
#endif
__device__ __forceinline__ void cswap(float& ta, uint32_t& oa, float& tb, uint32_t& ob) {
    if (tb < ta) {
        const float t = ta; ta = tb; tb = t;
        const uint32_t o = oa; oa = ob; ob = o;
    }
}

// Traversal entries (stack, current node, postponed leaf): one word per child,
//   interior node: its unit index (< 2^28);  leaf: unit index of its first primitive | (3 count) << 28,
//   i.e. the child's size nibble itself (one IMAD to form);  kNoEntry: nothing.
constexpr uint32_t kNoEntry = 0xFFFFFFFFu;
__device__ __forceinline__ bool is_node(uint32_t e) { return e < (1u << 28); }
__device__ __forceinline__ bool is_leaf(uint32_t e) { return e - (1u << 28) < 0xE0000000u; }   // nibble 1..14

// Closest-hit traversal, resumable: the state of one lane's traversal (the ray, the current entry, the
// postponed leaf, the stack pointer and the best hit) lives in a Trav, its stack and cold ray data in
// local memory the caller owns. closest_hit() runs it to completion; the path kernel interleaves it with
// the shading of lanes whose traversal has finished (dynamic replacement, Aila & Laine 2009).
struct Trav {
    RayT r;
    uint32_t cur, leaf;
    float cur_t, leaf_t;
    int sp;
    Hit best;
    bool tracing;
};

__device__ __forceinline__ void stk_push(uint32_t stk, int& sp, uint32_t e, float t) {
    asm volatile("st.local.v2.u32 [%0], {%1, %2};" ::"r"(stk + 8u * (uint32_t)sp), "r"(e), "r"(__float_as_uint(t))
                 : "memory");
    ++sp;
}
__device__ __forceinline__ uint2 stk_top(uint32_t stk, int sp) {
    uint2 v;
    asm volatile("ld.local.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(stk + 8u * (uint32_t)sp));
    return v;
}

// cold: local address of 32 B (the ray's spilled constants); stk: local address of kStackSize 8-B entries
__device__ __forceinline__ void trav_begin(Trav& t, const TraceParams& tp, float3 o, float3 d, uint32_t cold) {
    t.best = Hit{CUDART_INF, CUDART_INF_F, CUDART_INF_F, -1, 0u, true};
    ray_prepare(o, d, t.r, cold);
    t.cur = 0;
    t.cur_t = -CUDART_INF_F;
    t.leaf = kNoEntry;
    t.leaf_t = 0.0f;
    t.sp = 0;
    t.tracing = !tp.empty;
    TCOUNT(4, 1);
}

// One round of the while-while loop with postponed leaves (Aila & Laine 2009): interior nodes are visited
// until every tracing lane of the warp holds a leaf (or has finished), then the lanes test their leaves'
// primitives together, so the primitive test runs warp-convergent. Box culling uses the best hit at the
// time an entry is popped or visited; it only drops boxes entered strictly beyond a conservative bound of
// the best t (reading R11), so the visiting order never changes the result. Clears t.tracing when the
// traversal is complete.
__device__ __forceinline__ void trav_round(const TraceParams& tp, Trav& t, uint32_t stk) {
    // PBRT-v3's robust t_far * (1 + 2 gamma_3), with gamma_5: the approximate reciprocal adds up to
    // two more roundings' worth of relative error to each slab distance
    constexpr float kGrow = 1.0f + 2.0f * (5.0f * 0x1p-24f) / (1.0f - 5.0f * 0x1p-24f);   // 1 + 2 gamma_5
    const uint4* __restrict__ pool = tp.pool;
    RayT& r = t.r;
    // per-axis fp16x2 half swap so that t.x is always the near slab plane and t.y the far one
    uint32_t swz[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) swz[a] = ((r.kbits >> (8 + a)) & 1u) ? 0x1032u : 0x3210u;
    auto pop = [&](float tcull) -> uint32_t {
        while (t.sp > 0) {
            --t.sp;
            const uint2 v = stk_top(stk, t.sp);
            if (__uint_as_float(v.y) <= tcull) {
                t.cur_t = __uint_as_float(v.y);
                return v.x;
            }
        }
        return kNoEntry;
    };
    // ---- phase 1: interior nodes --------------------------------------------------------------------
    while (is_node(t.cur)) {
        const float tcull0 = cull_bound(t.best);
        if (t.cur_t > tcull0) {          // entered beyond the best hit found since it was pushed
            t.cur = pop(tcull0);
        } else {
            TCOUNT(0, 1);
            uint4 h, q0, q1, q2;
            ldg256(pool + t.cur, h, q0);               // a node is 64 B, 64-B aligned: two 32-B loads
            ldg256(pool + t.cur + 2, q1, q2);
            const uint32_t w[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
            const float O[3] = {__uint_as_float(h.x), __uint_as_float(h.y), __uint_as_float(h.z)};
            const float3 ro3 = ray_o(r), ri3 = ray_inv(r);
            const float ro[3] = {ro3.x, ro3.y, ro3.z}, ri[3] = {ri3.x, ri3.y, ri3.z};
            // child sizes in units (nibbles: 0 none, 4 interior, 3 * count leaf), see pt_internal.h
            const uint32_t meta = (h.x & 15u) | ((h.y & 15u) << 4) | ((h.z & 15u) << 8) | ((h.w >> 28) << 12);
            uint32_t off = h.w & 0x0FFFFFFFu;
            // per-child results in registers (static indices only: no local-memory arrays)
            float ctn[4];
            uint32_t cent[4];
#pragma unroll
            for (int ci = 0; ci < 4; ++ci) {
                const uint32_t nib = (meta >> (4 * ci)) & 15u;
                const bool valid = nib != 0u;
                const bool lf = nib != (uint32_t)kNodeUnits;
                float tn = 0.0f, tf = CUDART_INF_F;
#pragma unroll
                for (int a = 0; a < 3; ++a) {
                    // (near, far) bounds of this axis: exact fp16 -> fp32, then the same rn ops as the
                    // builder's check (the half swap only reorders the two lanes)
                    const uint32_t ws = __byte_perm(w[3 * ci + a], 0u, swz[a]);
                    const float2 lh = __half22float2(*reinterpret_cast<const __half2*>(&ws));
                    const float2 b = __fadd2_rn(make_float2(O[a], O[a]), lh);
                    const float2 tt = __fmul2_rn(__fadd2_rn(b, make_float2(-ro[a], -ro[a])),
                                                 make_float2(ri[a], ri[a]));
                    tn = fmaxf(tn, tt.x);
                    tf = fminf(tf, tt.y);
                }
                tf = tf * kGrow;
                const bool hit = valid && tn <= tf && tn <= tcull0;
                ctn[ci] = hit ? tn : CUDART_INF_F;
                cent[ci] = off + ((lf ? nib : 0u) << 28);
                off += nib;
            }
            // sort the children by entry distance (network of 5 compare-swaps), push all but the
            // nearest (farthest first), descend into the nearest
            cswap(ctn[0], cent[0], ctn[1], cent[1]);
            cswap(ctn[2], cent[2], ctn[3], cent[3]);
            cswap(ctn[0], cent[0], ctn[2], cent[2]);
            if (PT_CHILD_SORT == 5) {
                cswap(ctn[1], cent[1], ctn[3], cent[3]);
                cswap(ctn[1], cent[1], ctn[2], cent[2]);
            }
            // (non-hit children carry +inf; the bound may be +inf, so test finiteness explicitly)
#pragma unroll
            for (int ci = 3; ci >= 1; --ci)
                if (ctn[ci] < CUDART_INF_F) stk_push(stk, t.sp, cent[ci], ctn[ci]);
            if (ctn[0] < CUDART_INF_F) {
                t.cur = cent[0];
                t.cur_t = ctn[0];
            } else {
                t.cur = pop(tcull0);
            }
        }
        // postpone the first leaf reached and keep traversing until the whole warp holds one
        if (is_leaf(t.cur) && t.leaf == kNoEntry) {
            t.leaf = t.cur;
            t.leaf_t = t.cur_t;
            t.cur = pop(cull_bound(t.best));
        }
        if (!__any_sync(__activemask(), t.leaf == kNoEntry)) break;
    }
    // ---- phase 2: primitives of the postponed leaf (and of leaves met next) -------------------------
    while (t.leaf != kNoEntry) {
        if (t.leaf_t <= cull_bound(t.best)) {
            const uint32_t cnt = ((t.leaf >> 28) * 86u) >> 8;   // nibble / 3
            uint32_t unit = t.leaf & 0x0FFFFFFFu;
            for (uint32_t k = 0; k < cnt; ++k, unit += kPrimUnits) test_prim(pool, unit, r, t.best);
        }
        t.leaf = kNoEntry;
        if (is_leaf(t.cur)) {
            t.leaf = t.cur;
            t.leaf_t = t.cur_t;
            t.cur = pop(cull_bound(t.best));
        }
    }
    if (t.cur == kNoEntry) {
        t.tracing = false;
        // the fp32 sphere t can lose ~1e-5 (disc cancellation): refine the winner's t in fp64 so the
        // spawn point stays well inside the 1e-4 self-intersection offset (reading R10)
        if (t.best.prim >= 0 && !t.best.exact && t.best.prim >= (int32_t)tp.n_tris) {
            double t64;
            if (exact_test(pool, t.best.unit, r, t64)) t.best.t = t64;
        }
    }
}

__device__ Hit closest_hit(const TraceParams& tp, float3 o, float3 d) {
    float4 cold[kColdBytes / 16];                   // local memory: written and read only through ld/st.local asm
    uint2 stk[kStackSize];            // local memory: through ld/st.local asm
    Trav t;
    trav_begin(t, tp, o, d, (uint32_t)__cvta_generic_to_local(cold));
    const uint32_t stk_a = (uint32_t)__cvta_generic_to_local(stk);
    while (t.tracing) trav_round(tp, t, stk_a);
    return t.best;
}

// ---------------------------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------------------------

// Geometric normal and material of the hit primitive, from its record in the BVH pool (just read by the
// traversal): triangle n_g = normalize((v1 - v0) x (v2 - v0)), sphere n_g = (P - c) / r.
// The shading path and the Table-3 AOV hook (pt_trace_primary_aov) share this code.
__device__ __forceinline__ void hit_normal(const uint4* __restrict__ pool, uint32_t unit, float3 P, float3& ng,
                                           uint32_t& mi) {
    const uint4 u0 = __ldg(pool + unit), u1 = __ldg(pool + unit + 1);
    if (!(u0.w & kSphereFlag)) {
        const uint4 u2 = __ldg(pool + unit + 2);
        const float3 v0 = make_float3(__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z));
        const float3 e1 = make_float3(__uint_as_float(u1.x) - v0.x, __uint_as_float(u1.y) - v0.y,
                                      __uint_as_float(u1.z) - v0.z);
        const float3 e2 = make_float3(__uint_as_float(u2.x) - v0.x, __uint_as_float(u2.y) - v0.y,
                                      __uint_as_float(u2.z) - v0.z);
        ng = make_float3(e1.y * e2.z - e1.z * e2.y, e1.z * e2.x - e1.x * e2.z, e1.x * e2.y - e1.y * e2.x);
        const float il = rsqrtf(ng.x * ng.x + ng.y * ng.y + ng.z * ng.z);
        ng = make_float3(ng.x * il, ng.y * il, ng.z * il);
        mi = u1.w;
    } else {
        const float ir = 1.0f / __uint_as_float(u1.x);
        ng = make_float3((P.x - __uint_as_float(u0.x)) * ir, (P.y - __uint_as_float(u0.y)) * ir,
                         (P.z - __uint_as_float(u0.z)) * ir);
        mi = u1.y;
    }
}

// fp32 barycentrics (b1, b2) = (V, W) / det of the watertight test's sheared edge functions (the AOV hook)
__device__ __forceinline__ float2 tri_bary32(float3 o, float3 d, float3 v0, float3 v1, float3 v2) {
    int kz = 0;
    if (fabsf(d.y) > fabsf(d.x)) kz = 1;
    if (fabsf(d.z) > fabsf(self3(d, kz))) kz = 2;
    int kx = kz + 1; if (kx == 3) kx = 0;
    int ky = kx + 1; if (ky == 3) ky = 0;
    if (self3(d, kz) < 0.0f) { const int t = kx; kx = ky; ky = t; }
    const float Sx = self3(d, kx) / self3(d, kz), Sy = self3(d, ky) / self3(d, kz);
    auto sh = [&](float3 v, float& x, float& y) {
        const float3 q = make_float3(v.x - o.x, v.y - o.y, v.z - o.z);
        x = self3(q, kx) - Sx * self3(q, kz);
        y = self3(q, ky) - Sy * self3(q, kz);
    };
    float Ax, Ay, Bx, By, Cx, Cy;
    sh(v0, Ax, Ay);
    sh(v1, Bx, By);
    sh(v2, Cx, Cy);
    const float U = Cx * By - Cy * Bx, V = Ax * Cy - Ay * Cx, W = Bx * Ay - By * Ax;
    const float det = U + V + W;
    return det != 0.0f ? make_float2(V / det, W / det) : make_float2(0.0f, 0.0f);
}

struct ShadeArgs {
    TraceParams tp;
    Cam32 cam;
    int W, H, first_sample, depth, max_depth;
    float inv_np, inv_w;        // 1 / np, 1 / W for udiv_exact
    int np;                     // pixels of the rendered row range (W x rows)
    uint32_t p0;                // its first pixel (row0 W): slot i = (pixel p0 + i % np, sample first + i / np)
    uint32_t tiles_x;           // > 0: the first bounce visits the slots in 8 x 4 pixel tiles (W % 8 == 0, rows % 4 == 0)
    float inv_tiles_x;
    uint32_t g_log2;            // PT_TILE_ORDER 2: a warp = 2^g_log2 samples x (32 >> g_log2) consecutive pixels
    uint32_t npg;               // ... pixel groups (np / (32 >> g_log2)); 0: not in use
    float inv_npg;
    uint32_t k_wave;            // samples of the wave; with npg != 0 the wave buffer is pixel-major:
                                // radiance of slot (pixel p, sample s) at index p * k_wave + s
    uint2 key;
    const uint32_t* counters;   // the wave's counters (pt_internal.h kCounters layout)
    uint32_t n_slots;           // paths of the wave
    uint32_t* work;             // fetch counter of the kernel
    uint32_t* alive_count;      // paths alive after the first bounce (its output queue length)
    uint32_t* esc_count;        // escaped-queue length
    uint32_t* seg_count;        // traced segments
    int use_nif;
    float3 env;
    // path state after the first bounce, in queue order: (o.xyz, slot), (d.xyz, beta.x), (beta.y, beta.z)
    float4* qA;
    float4* qB;
    float2* qC;
    float4* esc;
    float4* esc_beta;
    float* wave_buf;
};

// One segment of one path: closest hit over the wide BVH (S2), then emission, BSDF sampling and
// Russian roulette (S3). `depth` counts this segment (reading R7).
struct SegOut {
    bool alive, escaped, done;
    float3 o, d, beta, L;
    int32_t prim;     // the segment's hit (-1 escape); read only by the path-record debug kernel
    uint32_t flags;   // kSegReflect: dielectric chose reflection; kSegRRKill: roulette ended the path
};
constexpr uint32_t kSegReflect = 1u, kSegRRKill = 2u;

// Emission, BSDF sampling and Russian roulette of one segment whose closest hit is hh (S3).
__device__ __forceinline__ void shade_hit(const ShadeArgs& a, int depth, uint32_t slot, float3 o, float3 d,
                                          float3 bt, const Hit& hh, SegOut& r) {
    const int np = a.np;
    r.alive = false;
    r.escaped = false;
    r.done = true;
    r.L = make_float3(0, 0, 0);
    r.beta = bt;
    r.d = d;
    r.o = o;
    const int32_t prim = hh.prim;
    r.prim = prim;
    r.flags = 0u;
    if (prim < 0) {                                   // escaped: environment light
        if (a.use_nif) {
            // queued by direction; the NIF kernel maps it to equirect (u, v) (S4 -> S5)
            r.escaped = true;
            r.done = false;
        } else {
            r.L = make_float3(bt.x * a.env.x, bt.y * a.env.y, bt.z * a.env.z);
        }
        return;
    }
    const float t = (float)hh.t;
    const float3 P = make_float3(fmaf(t, d.x, o.x), fmaf(t, d.y, o.y), fmaf(t, d.z, o.z));
    float3 ng;
    uint32_t mi;
    hit_normal(a.tp.pool, hh.unit, P, ng, mi);
    const DevMaterial m = a.tp.mats[mi];
    const float cosd = d.x * ng.x + d.y * ng.y + d.z * ng.z;
    if (m.kind == PT_EMISSIVE) {
        if (cosd < 0.0f) r.L = make_float3(bt.x * m.emission[0], bt.y * m.emission[1], bt.z * m.emission[2]);
        return;
    }
    if (depth >= a.max_depth) return;                 // capped: no further segment, no env (reading R7)
    uint32_t pu;
    const int s = a.first_sample + (int)udiv_exact(slot, (uint32_t)np, a.inv_np, pu);
    const int p = (int)(a.p0 + pu);
    const uint4 rr = philox10(make_uint4((uint32_t)p, (uint32_t)s, (uint32_t)depth, 0u), a.key);
    const float xi0 = u01f(rr.x), xi1 = u01f(rr.y), xi2 = u01f(rr.z), xi3 = u01f(rr.w);
    const bool entering = cosd < 0.0f;
    const float3 n = entering ? ng : make_float3(-ng.x, -ng.y, -ng.z);
    float side = 1.0f;
    float3 wi;
    if (m.kind == PT_LAMBERT) {
        // cosine-weighted hemisphere, ONB of Duff et al. 2017 (reading R9)
        const float sg = copysignf(1.0f, n.z);
        const float aa = -rcp_approx(sg + n.z);           // |sg + n.z| in [1, 2]
        const float bb = n.x * n.y * aa;
        const float3 t1 = make_float3(1.0f + sg * n.x * n.x * aa, sg * bb, -sg * n.x);
        const float3 t2 = make_float3(bb, sg + n.y * n.y * aa, -n.y);
        float sphi, cphi;
        sincospif(2.0f * xi1, &sphi, &cphi);   // sin/cos(2 pi xi1), cheap exact-argument reduction
        const float rho = sqrtf(xi0), c3 = sqrtf(1.0f - xi0);
        const float c1 = rho * cphi, c2 = rho * sphi;
        wi = make_float3(c1 * t1.x + c2 * t2.x + c3 * n.x, c1 * t1.y + c2 * t2.y + c3 * n.y,
                         c1 * t1.z + c2 * t2.z + c3 * n.z);
        bt = make_float3(bt.x * m.albedo[0], bt.y * m.albedo[1], bt.z * m.albedo[2]);
    } else if (m.kind == PT_MIRROR) {
        const float dn = d.x * n.x + d.y * n.y + d.z * n.z;
        wi = make_float3(d.x - 2.0f * dn * n.x, d.y - 2.0f * dn * n.y, d.z - 2.0f * dn * n.z);
        bt = make_float3(bt.x * m.albedo[0], bt.y * m.albedo[1], bt.z * m.albedo[2]);
    } else {
        // dielectric, Schlick Fresnel, TIR -> F = 1 (reading R9)
        const float eta = entering ? 1.0f / m.ior : m.ior;
        const float cosi = -(d.x * n.x + d.y * n.y + d.z * n.z);
        const float sin2t = eta * eta * (1.0f - cosi * cosi);
        float F = 1.0f, cost = 0.0f;
        if (sin2t <= 1.0f) {
            cost = sqrtf(1.0f - sin2t);
            const float c = entering ? cosi : cost;
            float r0 = (1.0f - m.ior) / (1.0f + m.ior);
            r0 = r0 * r0;
            const float mm = 1.0f - c;
            F = r0 + (1.0f - r0) * (mm * mm * mm * mm * mm);
        }
        if (xi2 < F) {
            r.flags |= kSegReflect;
            wi = make_float3(d.x + 2.0f * cosi * n.x, d.y + 2.0f * cosi * n.y, d.z + 2.0f * cosi * n.z);
        } else {
            const float k = eta * cosi - cost;
            wi = make_float3(eta * d.x + k * n.x, eta * d.y + k * n.y, eta * d.z + k * n.z);
            side = -1.0f;
        }
    }
    const float il = rsqrtf(wi.x * wi.x + wi.y * wi.y + wi.z * wi.z);
    wi = make_float3(wi.x * il, wi.y * il, wi.z * il);
    // spawn with normal offset on the side wi leaves to (reading R10)
    const float pm = fmaxf(1.0f, fmaxf(fabsf(P.x), fmaxf(fabsf(P.y), fabsf(P.z))));
    const float eps = 1e-4f * pm * side;
    r.o = make_float3(P.x + eps * n.x, P.y + eps * n.y, P.z + eps * n.z);
    r.d = wi;
    r.alive = true;
    r.done = false;
    // Russian roulette from depth 3, q = min(1, max beta) (reading R8)
    if (depth >= 3) {
        const float q = fminf(1.0f, fmaxf(bt.x, fmaxf(bt.y, bt.z)));
        if (xi3 >= q) {
            r.flags |= kSegRRKill;
            r.alive = false;
            r.done = true;
            return;
        }
        const float iq = __frcp_rn(q);            // beta / q as one reciprocal and three products
        bt = make_float3(bt.x * iq, bt.y * iq, bt.z * iq);
    }
    r.beta = bt;
}

// One segment of one path: closest hit over the wide BVH (S2), then shade_hit (S3).
__device__ __forceinline__ void shade_segment(const ShadeArgs& a, int depth, uint32_t slot, float3 o, float3 d,
                                              float3 bt, SegOut& r) {
    const Hit hh = closest_hit(a.tp, o, d);
    shade_hit(a, depth, slot, o, d, bt, hh, r);
}

// The first bounce's visiting order: work index w -> slot, 32 consecutive w = one 8 x 4 pixel tile of one
// sample (PT_TILE_W x 32 / PT_TILE_W; config 3: 2.60 -> 2.78 G samples/s, profiles/round2/tile_order.log)
// sample (row-major tiles), so a warp's camera rays form a compact bundle (when the row range tiles
// evenly; otherwise the identity). Slots keep their meaning (pixel-major), so nothing downstream changes.
#ifndef PT_TILE_W
#define PT_TILE_W 8              // tile width in pixels (height 32 / PT_TILE_W)
#endif
constexpr uint32_t kTileW = PT_TILE_W, kTileH = 32 / PT_TILE_W;
__device__ __forceinline__ uint32_t tile_slot(const ShadeArgs& a, uint32_t w) {
    if (a.npg != 0u) {
        // 32 consecutive work indices = 2^g samples of (32 >> g) consecutive pixels (nearly the same
        // camera ray: coherent traversal); consecutive warps walk the pixels, then the sample groups
        uint32_t pg;
        const uint32_t sg = udiv_exact(w >> 5, a.npg, a.inv_npg, pg);
        const uint32_t k = w & 31u;
        const uint32_t pix = (pg << (5u - a.g_log2)) + (k >> a.g_log2);
        const uint32_t smp = (sg << a.g_log2) + (k & ((1u << a.g_log2) - 1u));
        return smp * (uint32_t)a.np + pix;
    }
    if (a.tiles_x == 0u) return w;
    uint32_t q, tx;
    const uint32_t s = udiv_exact(w, (uint32_t)a.np, a.inv_np, q);
    const uint32_t t = q >> 5, k = q & 31u;
    const uint32_t ty = udiv_exact(t, a.tiles_x, a.inv_tiles_x, tx);
    return s * (uint32_t)a.np + (kTileH * ty + k / kTileW) * (uint32_t)a.W + kTileW * tx + (k % kTileW);
}

// The camera ray of wave slot i = (pixel p0 + i % np, sample first + i / np) (S1, reading R22)
__device__ __forceinline__ float3 camera_ray(const ShadeArgs& a, uint32_t i) {
    uint32_t pu, px;
    const int sm = a.first_sample + (int)udiv_exact(i, (uint32_t)a.np, a.inv_np, pu);
    const int p = (int)(a.p0 + pu);
    const uint32_t py = udiv_exact((uint32_t)p, (uint32_t)a.W, a.inv_w, px);
    const uint4 r = philox10(make_uint4((uint32_t)p, (uint32_t)sm, 0u, 0u), a.key);
    return cam_dir(a.cam, a.W, a.H, (int)px, (int)py, u01f(r.x), u01f(r.y));
}

#ifndef PT_TRACE_WAKE
#define PT_TRACE_WAKE 12
#endif
#ifndef PT_REPLACE_MIN_DEPTH
#define PT_REPLACE_MIN_DEPTH 6   // BVH depth (4-wide levels) from which the replacement kernel runs
#endif
#ifndef PT_TILE_ORDER
#define PT_TILE_ORDER 2          // first-bounce warps: 2 = a pixel's samples together (sample_group_log2),
                                 // else 8 x 4 pixel tiles of one sample (1), or linear (0)
#endif
#ifndef PT_TS_MINB
#define PT_TS_MINB 7   // min resident blocks per SM for the path kernels: 72-register cap; tools/ts_tune.sh
#endif

// Index of a slot's radiance in the wave buffer (and the NIF's output row): the slot itself
// (sample-major), or pixel-major p * k + s when the first bounce runs a pixel's samples in one warp, so
// the radiance stores of those lanes (and the NIF's, whose queue follows the same order) are contiguous
__device__ __forceinline__ uint32_t buf_index(const ShadeArgs& a, uint32_t slot) {
    if (a.npg == 0u) return slot;
    uint32_t p;
    const uint32_t sm = udiv_exact(slot, (uint32_t)a.np, a.inv_np, p);
    return p * a.k_wave + sm;
}

__device__ __forceinline__ void write_radiance(const ShadeArgs& a, const SegOut& r, uint32_t slot) {
    if (r.done) {
        const uint32_t b = buf_index(a, slot);
        a.wave_buf[3 * (size_t)b + 0] = r.L.x;
        a.wave_buf[3 * (size_t)b + 1] = r.L.y;
        a.wave_buf[3 * (size_t)b + 2] = r.L.z;
    }
}

// Bounce 1 (S1 raygen + S2-S4): whole warps of 32 consecutive slots, so the primary rays stay coherent;
// the camera rays are computed here (no raygen pass), survivors are compacted into the path queue
// with warp-aggregated appends, escapes into the NIF queue.
#ifndef PT_FB_MINB
#define PT_FB_MINB PT_TS_MINB   // the first bounce's own register cap (tools/ts_tune.sh)
#endif
__global__ void __launch_bounds__(128, PT_FB_MINB) first_bounce_kernel(ShadeArgs a) {
    pdl_trigger();                    // all CTAs resident (grid = resident capacity): let path_kernel queue
    const uint32_t n = a.n_slots;
    const int lane = threadIdx.x & 31;
    uint32_t segs = 0;
    const uint32_t lt = (1u << lane) - 1u;
    // (work, alive) word: one 64-bit atomic per iteration reserves this chunk's survivors in the path
    // queue and fetches the next chunk of 32 slots
    unsigned long long* const ww = reinterpret_cast<unsigned long long*>(a.work);
    unsigned long long wo = 0;
    if (lane == 0) wo = atomicAdd(ww, 32ull);
    uint32_t base = (uint32_t)__shfl_sync(0xFFFFFFFFu, wo, 0);
    while (base < n) {
        const uint32_t w = base + (uint32_t)lane;
        const uint32_t i = w < n ? tile_slot(a, w) : w;
        SegOut r;
        r.alive = r.escaped = false;
        if (w < n) {
            ++segs;
            const float3 eye = make_float3(a.cam.eye[0], a.cam.eye[1], a.cam.eye[2]);
            shade_segment(a, 1, i, eye, camera_ray(a, i), make_float3(1.0f, 1.0f, 1.0f), r);
            write_radiance(a, r, i);
        }
        const uint32_t ma = __ballot_sync(0xFFFFFFFFu, r.alive), me = __ballot_sync(0xFFFFFFFFu, r.escaped);
        if (lane == 0) wo = atomicAdd(ww, 32ull | ((unsigned long long)__popc(ma) << 32));
        wo = __shfl_sync(0xFFFFFFFFu, wo, 0);
        if (r.alive) {
            const uint32_t pos = (uint32_t)(wo >> 32) + (uint32_t)__popc(ma & lt);
            a.qA[pos] = make_float4(r.o.x, r.o.y, r.o.z, __uint_as_float(i));
            a.qB[pos] = make_float4(r.d.x, r.d.y, r.d.z, r.beta.x);
            a.qC[pos] = make_float2(r.beta.y, r.beta.z);
        }
        if (me != 0u) {                   // camera rays that miss everything: rare inside a scene
            uint32_t eb = 0;
            if (lane == 0) eb = atomicAdd(a.esc_count, (uint32_t)__popc(me));
            eb = __shfl_sync(0xFFFFFFFFu, eb, 0);
            if (r.escaped) {
                const uint32_t pos = eb + (uint32_t)__popc(me & lt);
                a.esc[pos] = make_float4(r.d.x, r.d.y, r.d.z, __uint_as_float(buf_index(a, i)));
                a.esc_beta[pos] = make_float4(r.beta.x, r.beta.y, r.beta.z, 0.0f);
            }
        }
        base = (uint32_t)wo;
    }
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) segs += __shfl_xor_sync(0xFFFFFFFFu, segs, k);
    if (lane == 0) atomicAdd(a.seg_count, segs);
    TAIL_STAMP(0);
}

// Bounces 2.. (persistent): every lane carries one path from the first bounce's queue to its end,
// and a lane whose path ends refills from the queue (one 64-bit atomic per warp iteration for all of the
// warp's free lanes), so the warps stay full without a launch, a barrier or a state round trip through
// HBM per bounce. Per-path results do not depend on the schedule: the RNG is keyed by (pixel, sample,
// depth) and every path writes only its own slot.
// kReplace (deep BVHs, launch_paths): traversal with dynamic replacement (Aila & Laine 2009) -- a lane's
// traversal state survives across rounds, and the warp interrupts its traversal rounds as soon as
// PT_TRACE_WAKE lanes are waiting (traversal finished, or no path while the queue still has some) to
// shade those segments and start the next ones, so lanes with short traversals do not idle behind the
// warp's longest one. Without it every warp iteration runs one whole closest-hit per lane (cheaper where
// traversals are short: configs 0-2).
template <bool kReplace>
__global__ void __launch_bounds__(128, PT_TS_MINB) path_kernel(ShadeArgs a) {
    pdl_wait();                       // first_bounce complete: its queue and counters are visible
    pdl_trigger();
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    // (escaped count, paths taken) word; the alive queue's length is final once first_bounce is done
    unsigned long long* const qw = reinterpret_cast<unsigned long long*>(a.esc_count);
    const int n_alive = (int)*a.alive_count;
    bool have = false, dry = false;
    uint32_t slot = 0;
    int depth = 0;
    float3 bt = make_float3(1, 1, 1);
    uint32_t segs = 0;
    if constexpr (kReplace) {
        float4 cold[kColdBytes / 16];                   // local memory (ld/st.local asm): the ray's spilled constants
        uint2 stk[kStackSize];            // local memory: the traversal stack
        const uint32_t cold_a = (uint32_t)__cvta_generic_to_local(cold);
        const uint32_t stk_a = (uint32_t)__cvta_generic_to_local(stk);
        Trav tv;
        tv.tracing = false;
        // lanes without a path take queue entries r0 - 1 - (rank among them) while those are >= 0
        auto refill = [&](unsigned long long old, uint32_t mneed) {
            if (!have) {
                const int idx = n_alive - 1 - (int)(uint32_t)(old >> 32) - __popc(mneed & lt);
                if (idx >= 0) {
                    const float4 qa = __ldg(a.qA + idx), qb = __ldg(a.qB + idx);
                    const float2 qc = __ldg(a.qC + idx);
                    slot = __float_as_uint(qa.w);
                    bt = make_float3(qb.w, qc.x, qc.y);
                    depth = 2;
                    have = true;
                    trav_begin(tv, a.tp, make_float3(qa.x, qa.y, qa.z), make_float3(qb.x, qb.y, qb.z), cold_a);
                }
            }
            if (__any_sync(0xFFFFFFFFu, !have)) dry = true;   // the queue ran out (taken only grows)
        };
        {
            unsigned long long old = 0;
            if (lane == 0) old = atomicAdd(qw, 32ull << 32);
            refill(__shfl_sync(0xFFFFFFFFu, old, 0), 0xFFFFFFFFu);
        }
        for (;;) {
            // traversal rounds until enough lanes wait (or none traces)
            for (;;) {
                const uint32_t tr = __ballot_sync(0xFFFFFFFFu, tv.tracing);
                const uint32_t wake = __ballot_sync(0xFFFFFFFFu, have ? !tv.tracing : !dry);
                if (tr == 0u || __popc(wake) >= PT_TRACE_WAKE) break;
                if (tv.tracing) trav_round(a.tp, tv, stk_a);
            }
            SegOut r;
            r.escaped = false;
            if (have && !tv.tracing) {
                ++segs;
                shade_hit(a, depth, slot, ray_o(tv.r), ray_dir(tv.r), bt, tv.best, r);
                write_radiance(a, r, slot);
                if (r.alive) {
                    bt = r.beta;
                    ++depth;
                    trav_begin(tv, a.tp, r.o, r.d, cold_a);
                } else {
                    have = false;
                }
            }
            // one 64-bit atomic per warp iteration: append this iteration's escapes (low word) and take
            // new paths for the free lanes (high word) while the queue has some
            const uint32_t me = __ballot_sync(0xFFFFFFFFu, r.escaped);
            const uint32_t mneed = dry ? 0u : __ballot_sync(0xFFFFFFFFu, !have);
            if ((me | mneed) != 0u) {
                const int leader = __ffs(me | mneed) - 1;
                unsigned long long old = 0;
                if (lane == leader)
                    old = atomicAdd(qw, ((unsigned long long)__popc(mneed) << 32) + (unsigned long long)__popc(me));
                old = __shfl_sync(0xFFFFFFFFu, old, leader);
                if (r.escaped) {
                    const uint32_t pos = (uint32_t)old + (uint32_t)__popc(me & lt);
                    a.esc[pos] = make_float4(r.d.x, r.d.y, r.d.z, __uint_as_float(buf_index(a, slot)));
                    a.esc_beta[pos] = make_float4(r.beta.x, r.beta.y, r.beta.z, 0.0f);
                }
                if (mneed) refill(old, mneed);
            }
            if (!__any_sync(0xFFFFFFFFu, have)) break;
        }
    } else {
        float3 o = make_float3(0, 0, 0), d = make_float3(0, 0, 1);
        auto refill = [&](unsigned long long old, uint32_t mneed) {
            if (!have) {
                const int idx = n_alive - 1 - (int)(uint32_t)(old >> 32) - __popc(mneed & lt);
                if (idx >= 0) {
                    const float4 qa = __ldg(a.qA + idx), qb = __ldg(a.qB + idx);
                    const float2 qc = __ldg(a.qC + idx);
                    o = make_float3(qa.x, qa.y, qa.z);
                    slot = __float_as_uint(qa.w);
                    d = make_float3(qb.x, qb.y, qb.z);
                    bt = make_float3(qb.w, qc.x, qc.y);
                    depth = 2;
                    have = true;
                }
            }
        };
        {
            unsigned long long old = 0;
            if (lane == 0) old = atomicAdd(qw, 32ull << 32);
            refill(__shfl_sync(0xFFFFFFFFu, old, 0), 0xFFFFFFFFu);
        }
        for (;;) {
            if (!__any_sync(0xFFFFFFFFu, have)) break;
            SegOut r;
            r.escaped = false;
            if (have) {
                ++segs;
                shade_segment(a, depth, slot, o, d, bt, r);
                write_radiance(a, r, slot);
                if (r.alive) {
                    o = r.o;
                    d = r.d;
                    bt = r.beta;
                    ++depth;
                } else {
                    have = false;
                }
            }
            const uint32_t me = __ballot_sync(0xFFFFFFFFu, r.escaped);
            const uint32_t mneed = __ballot_sync(0xFFFFFFFFu, !have);
            if ((me | mneed) != 0u) {
                const int leader = __ffs(me | mneed) - 1;
                unsigned long long old = 0;
                if (lane == leader)
                    old = atomicAdd(qw, ((unsigned long long)__popc(mneed) << 32) + (unsigned long long)__popc(me));
                old = __shfl_sync(0xFFFFFFFFu, old, leader);
                if (r.escaped) {
                    const uint32_t pos = (uint32_t)old + (uint32_t)__popc(me & lt);
                    a.esc[pos] = make_float4(r.d.x, r.d.y, r.d.z, __uint_as_float(buf_index(a, slot)));
                    a.esc_beta[pos] = make_float4(r.beta.x, r.beta.y, r.beta.z, 0.0f);
                }
                refill(old, mneed);
            }
        }
    }
#pragma unroll
    for (int k = 16; k > 0; k >>= 1) segs += __shfl_xor_sync(0xFFFFFFFFu, segs, k);
    if (lane == 0) atomicAdd(a.seg_count, segs);
    TAIL_STAMP(1);
}

// S6: fb += the wave's per-slot radiance, summed over its k samples in sample order (deterministic); one
// thread also folds the wave's counters into the scene's statistics (paths, segments, escaped)
__global__ void accumulate_kernel(const float* __restrict__ wave_buf, int n_elems, int k, int pixel_major,
                                  float* __restrict__ fb, const uint32_t* __restrict__ counters,
                                  unsigned long long* __restrict__ stats, uint32_t paths) {
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0 && stats) {
        stats[0] += paths;
        stats[1] += counters[kCounterSeg];
        stats[2] += counters[kCounterEsc];
    }
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n_elems; e += gridDim.x * blockDim.x) {
        float s = fb[e];
        if (pixel_major) {
            const int p = e / 3, c = e - 3 * p;
            const float* w = wave_buf + (size_t)3 * k * p + c;
            for (int j = 0; j < k; ++j) s += __ldg(w + 3 * j);                         // fixed sample order
        } else {
            for (int j = 0; j < k; ++j) s += __ldg(wave_buf + (size_t)j * n_elems + e);   // fixed sample order
        }
        fb[e] = s;
    }
}

// Pixel-major wave buffer (PT_TILE_ORDER 2, k % 4 == 0): one thread per pixel reads its 3 k contiguous
// floats as float4s and adds them per component in sample order (the same fixed order as the
// sample-major path, so frames are bit-identical for any wave split)
__global__ void accumulate_pm_kernel(const float4* __restrict__ wave_buf, int np, int k, float* __restrict__ fb,
                                     const uint32_t* __restrict__ counters, unsigned long long* __restrict__ stats,
                                     uint32_t paths) {
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0 && stats) {
        stats[0] += paths;
        stats[1] += counters[kCounterSeg];
        stats[2] += counters[kCounterEsc];
    }
    const int n4 = 3 * k / 4;   // float4s per pixel
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        float acc[3] = {fb[3 * p + 0], fb[3 * p + 1], fb[3 * p + 2]};
        const float4* w = wave_buf + (size_t)p * n4;
        int c = 0;   // component of the next float
        for (int q = 0; q < n4; ++q) {
            const float4 v = __ldg(w + q);
            acc[c] += v.x; c = c == 2 ? 0 : c + 1;
            acc[c] += v.y; c = c == 2 ? 0 : c + 1;
            acc[c] += v.z; c = c == 2 ? 0 : c + 1;
            acc[c] += v.w; c = c == 2 ? 0 : c + 1;
        }
        fb[3 * p + 0] = acc[0];
        fb[3 * p + 1] = acc[1];
        fb[3 * p + 2] = acc[2];
    }
}

__global__ void __launch_bounds__(128, PT_TS_MINB) primary_kernel(TraceParams tp, Cam32 cam, int W, int H, int sample, uint2 key, int32_t* prim,
                               float* tout) {
    const int np = W * H;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        const uint4 r = philox10(make_uint4((uint32_t)p, (uint32_t)sample, 0u, 0u), key);
        const float3 d = cam_dir(cam, W, H, p % W, p / W, u01f(r.x), u01f(r.y));
        const Hit h = closest_hit(tp, make_float3(cam.eye[0], cam.eye[1], cam.eye[2]), d);
        prim[p] = h.prim;
        tout[p] = (float)h.t;
    }
}

// Table-3 AOVs of the primary hits: the kernel's own hit point (P = o + t d as the
// shading computes it), geometric normal (hit_normal, the shading code) and fp32 barycentrics
__global__ void __launch_bounds__(128, PT_TS_MINB) primary_aov_kernel(TraceParams tp, Cam32 cam, int W, int H, int sample,
                                                                      uint2 key, int32_t* prim, float* tout, float* pos,
                                                                      float* nrm, float* bary2) {
    const int np = W * H;
    for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < np; p += gridDim.x * blockDim.x) {
        const uint4 r = philox10(make_uint4((uint32_t)p, (uint32_t)sample, 0u, 0u), key);
        const float3 d = cam_dir(cam, W, H, p % W, p / W, u01f(r.x), u01f(r.y));
        const float3 o = make_float3(cam.eye[0], cam.eye[1], cam.eye[2]);
        const Hit h = closest_hit(tp, o, d);
        prim[p] = h.prim;
        tout[p] = (float)h.t;
        float3 P = make_float3(0, 0, 0), ng = make_float3(0, 0, 0);
        float2 b = make_float2(0, 0);
        if (h.prim >= 0) {
            const float t = (float)h.t;
            P = make_float3(fmaf(t, d.x, o.x), fmaf(t, d.y, o.y), fmaf(t, d.z, o.z));
            uint32_t mi;
            hit_normal(tp.pool, h.unit, P, ng, mi);
            const uint4 u0 = __ldg(tp.pool + h.unit);
            if (!(u0.w & kSphereFlag)) {
                const uint4 u1 = __ldg(tp.pool + h.unit + 1), u2 = __ldg(tp.pool + h.unit + 2);
                b = tri_bary32(o, d, make_float3(__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z)),
                               make_float3(__uint_as_float(u1.x), __uint_as_float(u1.y), __uint_as_float(u1.z)),
                               make_float3(__uint_as_float(u2.x), __uint_as_float(u2.y), __uint_as_float(u2.z)));
            }
        }
        pos[3 * p + 0] = P.x; pos[3 * p + 1] = P.y; pos[3 * p + 2] = P.z;
        nrm[3 * p + 0] = ng.x; nrm[3 * p + 1] = ng.y; nrm[3 * p + 2] = ng.z;
        bary2[2 * p + 0] = b.x; bary2[2 * p + 1] = b.y;
    }
}

__global__ void __launch_bounds__(128, PT_TS_MINB) trace_rays_kernel(TraceParams tp, const float* o, const float* d, int64_t n, int32_t* prim, float* tout) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Hit h = closest_hit(tp, make_float3(o[3 * i], o[3 * i + 1], o[3 * i + 2]),
                                  make_float3(d[3 * i], d[3 * i + 1], d[3 * i + 2]));
        prim[i] = h.prim;
        tout[i] = (float)h.t;
    }
}

// Debug (first-divergence classifier, tests only): one thread per path (listed pixel, sample), the render
// kernels' own shade_segment per segment; records per segment the hit primitive and the decision flags,
// the escape direction and the path radiance (constant environment; with a NIF only the direction).
__global__ void __launch_bounds__(128) path_record_kernel(ShadeArgs a, const int32_t* pix, int n_pix, int n_s,
                                                          int32_t* prims, uint32_t* flags, float* esc_dir, float* Lout) {
    const int n = n_pix * n_s;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int p = pix[i / n_s], sj = i % n_s;
        const uint32_t slot = (uint32_t)sj * (uint32_t)a.np + (uint32_t)p;   // first_sample = s0, p0 = 0
        float3 o = make_float3(a.cam.eye[0], a.cam.eye[1], a.cam.eye[2]), d = camera_ray(a, slot);
        float3 bt = make_float3(1.0f, 1.0f, 1.0f), L = make_float3(0, 0, 0), ed = make_float3(0, 0, 0);
        for (int k = 0; k < a.max_depth; ++k) {
            prims[(size_t)i * a.max_depth + k] = -2;
            flags[(size_t)i * a.max_depth + k] = 0u;
        }
        for (int depth = 1; depth <= a.max_depth; ++depth) {
            SegOut r;
            shade_segment(a, depth, slot, o, d, bt, r);
            prims[(size_t)i * a.max_depth + depth - 1] = r.prim;
            flags[(size_t)i * a.max_depth + depth - 1] = r.flags;
            L = make_float3(L.x + r.L.x, L.y + r.L.y, L.z + r.L.z);
            if (r.escaped) ed = r.d;
            if (!r.alive) break;
            o = r.o;
            d = r.d;
            bt = r.beta;
        }
        esc_dir[3 * i + 0] = ed.x; esc_dir[3 * i + 1] = ed.y; esc_dir[3 * i + 2] = ed.z;
        Lout[3 * i + 0] = L.x; Lout[3 * i + 1] = L.y; Lout[3 * i + 2] = L.z;
    }
}

__global__ void scale_kernel(float* fb, int64_t n, float s) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        fb[i] *= s;
}

__global__ void pack_queries_kernel(const float* uv, int64_t n, float4* esc, float4* esc_beta, uint32_t* count) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        esc[i] = make_float4(uv[2 * i], uv[2 * i + 1], 0.0f, __uint_as_float((uint32_t)i));
        esc_beta[i] = make_float4(1.0f, 1.0f, 1.0f, 0.0f);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *count = (uint32_t)n;
}

// ---------------------------------------------------------------------------------------------
// Launchers: persistent-style grids sized to the SM count (Guideline 11); counts read on device.
// ---------------------------------------------------------------------------------------------
static int grid_for(int64_t n, int block, int per_sm) {
    int64_t g = (n + block - 1) / block;
    int64_t cap = (int64_t)num_sms() * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// persistent grids: exactly the resident block count (one wave), so no SM idles behind a partial wave
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PT_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

template <typename K>
static int resident_grid(K kernel, int block) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0);
    return num_sms() * (per_sm > 0 ? per_sm : 1);
}

// resident grids of the two path kernels, per device (occupancy and SM count are per-device properties)
static int3 path_grids() {
    static std::atomic<int> g1[64], g2[64], g3[64];
    const int dev = current_device();
    int a = g1[dev].load(std::memory_order_relaxed), b = g2[dev].load(std::memory_order_relaxed),
        c = g3[dev].load(std::memory_order_relaxed);
    if (a <= 0 || b <= 0 || c <= 0) {
        a = resident_grid(first_bounce_kernel, 128);
        b = resident_grid(path_kernel<false>, 128);
        c = resident_grid(path_kernel<true>, 128);
        g1[dev].store(a, std::memory_order_relaxed);
        g2[dev].store(b, std::memory_order_relaxed);
        g3[dev].store(c, std::memory_order_relaxed);
    }
    return make_int3(a, b, c);
}

// PT_TILE_ORDER 2: a first-bounce warp takes 2^g samples of 32 / 2^g consecutive pixels, the largest
// g <= 5 with 2^g dividing the wave's samples k and 32 / 2^g dividing np; -1 (8 x 4 tiles of one
// sample, or linear order) when only g = 0 fits
int sample_group_log2(int np, int k) {
    if (PT_TILE_ORDER != 2) return -1;
    for (int g = 5; g >= 1; --g)
        if (k % (1 << g) == 0 && np % (32 >> g) == 0) return g;
    return -1;
}

void launch_paths(const TraceParams& tp, const Cam32& cam, int W, int H, int p0, int np, int first_sample, int n_slots,
                  int max_depth, uint64_t seed, int use_nif, float3 env, Workspace& ws, cudaStream_t st) {
    ShadeArgs a;
    a.n_slots = (uint32_t)n_slots;
    a.tp = tp;
    a.cam = cam;
    a.W = W; a.H = H; a.first_sample = first_sample; a.depth = 1; a.max_depth = max_depth;
    a.np = np;
    a.p0 = (uint32_t)p0;
    a.inv_np = 1.0f / (float)np;
    a.tiles_x = (PT_TILE_ORDER && W % kTileW == 0 && (np / W) % kTileH == 0) ? (uint32_t)(W / kTileW) : 0u;
    a.inv_tiles_x = a.tiles_x ? 1.0f / (float)a.tiles_x : 0.0f;
    a.k_wave = (uint32_t)(n_slots / np);
    const int g = sample_group_log2(np, n_slots / np);
    a.g_log2 = g > 0 ? (uint32_t)g : 0u;
    a.npg = g > 0 ? (uint32_t)(np / (32 >> g)) : 0u;
    a.inv_npg = g > 0 ? 1.0f / (float)a.npg : 0.0f;
    a.inv_w = 1.0f / (float)W;
    a.key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    a.counters = ws.counters;
    a.alive_count = ws.counters + kCounterAlive;
    a.esc_count = ws.counters + kCounterEsc;
    a.seg_count = ws.counters + kCounterSeg;
    a.use_nif = use_nif; a.env = env;
    a.qA = ws.rayA[0]; a.qB = ws.rayB[0]; a.qC = ws.rayC[0];
    a.esc = ws.esc; a.esc_beta = ws.esc_beta; a.wave_buf = ws.wave_buf;
    const int3 grids = path_grids();
    a.work = ws.counters + kCounterWork;
    // (the first bounce's camera rays stay in whole coherent warps: replacement there measured slower,
    // 2.48 vs 2.58 G samples/s on config 3, profiles/round2/fb_replace.log)
    const bool replace = tp.bvh_depth >= PT_REPLACE_MIN_DEPTH;
    first_bounce_kernel<<<grids.x, 128, 0, st>>>(a);
    if (max_depth > 1) {
        if (replace) launch_pdl(path_kernel<true>, dim3(grids.z), dim3(128), 0, st, a);
        else launch_pdl(path_kernel<false>, dim3(grids.y), dim3(128), 0, st, a);
    }
}

int path_launches(int max_depth) { return max_depth > 1 ? 2 : 1; }

void launch_accumulate(const float* wave_buf, int n_pix, int k, float* fb, const uint32_t* counters,
                       unsigned long long* stats, uint32_t paths, cudaStream_t st) {
    const int n = 3 * n_pix;
    const int pixel_major = sample_group_log2(n_pix, k) > 0 ? 1 : 0;   // the layout launch_paths used
    if (pixel_major && k % 4 == 0) {
        launch_pdl(accumulate_pm_kernel, dim3(grid_for(n_pix, 256, 8)), dim3(256), 0, st,
                   reinterpret_cast<const float4*>(wave_buf), n_pix, k, fb, counters, stats, paths);
        return;
    }
    launch_pdl(accumulate_kernel, dim3(grid_for(n, 256, 8)), dim3(256), 0, st, wave_buf, n, k, pixel_major, fb,
               counters, stats, paths);
}

void launch_primary(const TraceParams& tp, const Cam32& cam, int W, int H, int sample, uint64_t seed, int32_t* prim,
                    float* t, cudaStream_t st) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    primary_kernel<<<grid_for((int64_t)W * H, 128, PT_TS_MINB), 128, 0, st>>>(tp, cam, W, H, sample, key, prim, t);
}

void launch_primary_aov(const TraceParams& tp, const Cam32& cam, int W, int H, int sample, uint64_t seed, int32_t* prim,
                        float* t, float* pos, float* nrm, float* bary2, cudaStream_t st) {
    const uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    primary_aov_kernel<<<grid_for((int64_t)W * H, 128, PT_TS_MINB), 128, 0, st>>>(tp, cam, W, H, sample, key, prim, t,
                                                                                   pos, nrm, bary2);
}

void launch_trace_rays(const TraceParams& tp, const float* o, const float* d, int64_t n, int32_t* prim, float* t,
                       cudaStream_t st) {
    trace_rays_kernel<<<grid_for(n, 128, PT_TS_MINB), 128, 0, st>>>(tp, o, d, n, prim, t);
}

void launch_path_record(const TraceParams& tp, const Cam32& cam, int W, int H, int s0, int n_s, int max_depth,
                        uint64_t seed, int use_nif, float3 env, const int32_t* pix, int n_pix, int32_t* prims,
                        uint32_t* flags, float* esc_dir, float* L, cudaStream_t st) {
    ShadeArgs a = {};
    a.tp = tp;
    a.cam = cam;
    a.W = W; a.H = H; a.first_sample = s0; a.depth = 1; a.max_depth = max_depth;
    a.np = W * H;
    a.p0 = 0;
    a.inv_np = 1.0f / (float)((int64_t)W * H);
    a.inv_w = 1.0f / (float)W;
    a.key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
    a.use_nif = use_nif;
    a.env = env;
    path_record_kernel<<<grid_for((int64_t)n_pix * n_s, 128, 4), 128, 0, st>>>(a, pix, n_pix, n_s, prims, flags, esc_dir, L);
}

void launch_scale(float* fb, int64_t n, float s, cudaStream_t st) {
    scale_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(fb, n, s);
}

void launch_pack_queries(const float* uv, int64_t n, float4* esc, float4* esc_beta, uint32_t* count, cudaStream_t st) {
    pack_queries_kernel<<<grid_for(n, 256, 4), 256, 0, st>>>(uv, n, esc, esc_beta, count);
}

}  // namespace pt

#ifdef PT_COUNT
extern "C" __attribute__((visibility("default"))) int pt_debug_trav_counts(unsigned long long* host, int reset) {
    cudaMemcpyFromSymbol(host, pt::g_trav_count, sizeof(pt::g_trav_count));
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(pt::g_trav_count, z, sizeof(z));
    }
    return 0;
}
#endif

namespace pt {
// traversal counters of the counting build (pt_get_stats): reset at the start of a render, read after it
bool trav_counts(int64_t* visits, int64_t* prim_tests, int64_t* fp64) {
#ifdef PT_COUNT
    unsigned long long h[8];
    if (cudaMemcpyFromSymbol(h, g_trav_count, sizeof(h)) != cudaSuccess) return false;
    *visits = (int64_t)h[0];
    *prim_tests = (int64_t)h[2];
    *fp64 = (int64_t)h[3];
    return true;
#else
    (void)visits; (void)prim_tests; (void)fp64;
    return false;
#endif
}
void trav_counts_reset() {
#ifdef PT_COUNT
    unsigned long long z[8] = {0};
    cudaMemcpyToSymbol(g_trav_count, z, sizeof(z));
#endif
}
}  // namespace pt

#ifdef PT_TAIL_TRACE
extern "C" __attribute__((visibility("default"))) int pt_debug_tail(unsigned long long* host) {
    return cudaMemcpyFromSymbol(host, pt::g_tail, sizeof(pt::g_tail)) == cudaSuccess ? 0 : -1;
}
#endif
