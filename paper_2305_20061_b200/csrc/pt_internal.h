// pt_internal.h -- private declarations of libpt_b200 (CUDA path). Not shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "pt.h"

namespace pt {

// ---------------------------------------------------------------------------------------------
// Wide BVH, device layout:
//   a pool of 16-byte units (< 2^28 of them). An interior node is 4 units (64 B, 64-B aligned):
//     unit 0: float O.x, O.y, O.z (node origin, <= the box min, fp32), uint32 base | nib3 << 28
//     units 1-3: 4 child boxes x 12 B: words (lo.x|hi.x) (lo.y|hi.y) (lo.z|hi.z), f16 offsets from O,
//                lo rounded down / hi rounded up so fp32(O + lo) <= exact lo, fp32(O + hi) >= exact hi
//                (the paper's "round-to-nearest-not-lower", made exact for the decode).
//   Child metadata: nibble c = child c's size in units (0 none, 4 interior, 3 * count leaf); nibbles 0-2
//   are the low 4 mantissa bits of O.x, O.y, O.z (the origin is chosen so), nibble 3 the top of word 3.
//   A child block holds the node's children contiguously (first child implicit at `base`, like the
//   paper's "first child is implicitly stored next"): interior children first (4 units
//   each), then the leaves' primitives inline, 3 units (48 B) per primitive:
//     triangle: (v0.xyz, id) (v1.xyz, material) (v2.xyz, 0); sphere: (c.xyz, id | SPHERE_FLAG) (r, material, 0, 0) (0)
//   (shading reads the hit primitive's vertices and material from here: no separate vertex arrays)
// ---------------------------------------------------------------------------------------------
constexpr uint32_t kSphereFlag = 0x80000000u;
constexpr int kNodeUnits = 4;
constexpr int kPrimUnits = 3;
constexpr int kMaxLeafPrims = 4;
constexpr int kStackSize = 64;

struct DevMaterial {        // 32 B, same field order as pt_material
    uint32_t kind;
    float albedo[3];
    float emission[3];
    float ior;
};

struct HostBvh {
    std::unique_ptr<uint4[]> pool;  // 16-B units
    int64_t units = 0;
    int64_t n_nodes = 0, n_leaves = 0, max_depth = 0;
    bool empty = true;
};

// Builds the 4-wide compressed BVH; returns PT_OK or PT_ERR_DOMAIN with msg filled.
int build_wide_bvh(const pt_triangle* tris, int64_t n_tris, const pt_sphere* sph, int64_t n_sph, HostBvh* out,
                   std::string* msg);
// f16 helpers of the conservative quantiser (exposed for tests of the host builder)
uint16_t f16_round_down(double x);
uint16_t f16_round_up(double x);
double f16_value(uint16_t h);

struct Workspace {
    int64_t capacity = 0;      // path slots
    // live-path state in queue order, double buffered (in/out of each bounce):
    float4* rayA[2] = {nullptr, nullptr};   // (o.xyz, slot bits) -- [0]: the first bounce's survivors
    float4* rayB[2] = {nullptr, nullptr};   // (d.xyz, beta.x)
    float2* rayC[2] = {nullptr, nullptr};   // (beta.y, beta.z)
    float4* esc = nullptr;     // [cap] escaped-ray queue: (d.xyz, slot bits); the NIF maps d to (u, v)
    float4* esc_beta = nullptr;// [cap] escaped-ray throughput
    float* wave_buf = nullptr; // [cap][3] radiance per slot, written exactly once per path
    uint32_t* counters = nullptr;  // [kCounters]
    int64_t fb_capacity = 0;
    float* fb = nullptr;       // scratch framebuffer for pt_render (host-output path)
    cudaStream_t own_stream = nullptr;      // the device's host-path stream (not owned)
    unsigned long long* d_stats = nullptr;  // [paths, segments, escaped, -] accumulated per call
};
struct TimedLaunch {
    int cls;
    cudaEvent_t a, b;
};
// device counters of one wave (uint32 words): [128] = escaped paths (the NIF's row count), [129] = error
// flags, [130] / [131] = work-fetch counters of the first-bounce and path kernels, [132] = traced
// segments, [133] = paths alive after the first bounce
constexpr int kCounters = 192;
// Two 8-byte words, each advanced by one 64-bit atomic per warp iteration:
//   [128] escaped-queue length | [129] paths taken from the alive queue by the path kernel
//   [130] first-bounce work (slots fetched) | [131] alive-queue length (paths alive after bounce 1)
constexpr int kCounterEsc = 128;
constexpr int kCounterTaken = 129;
constexpr int kCounterWork = 130;
constexpr int kCounterAlive = 131;
constexpr int kCounterSeg = 132;   // traced segments of the wave

}  // namespace pt

struct pt_scene {
    int device = 0;
    int64_t n_tris = 0, n_sph = 0;
    int32_t n_mats = 0;
    pt_camera cam{};
    void* d_alloc = nullptr;          // the scene's single device allocation (all arrays below)
    size_t d_alloc_bytes = 0;
    uint4* d_pool = nullptr;          // wide BVH + inline primitives
    int64_t pool_units = 0;
    bool empty = true;
    pt::DevMaterial* d_mats = nullptr;
    int64_t bvh_nodes = 0, bvh_leaves = 0, bvh_depth = 0;
    std::mutex mu;                    // guards ws + stats
    pt::Workspace ws;
    pt_stats stats{};
    bool profiling = false;
    std::vector<pt::TimedLaunch> pending;   // launch timers awaiting pt_get_stats
};

// one layer of the layered paper-NIF family (mlp_kernel.cu): blocked fp16 weights, fp32 bias
struct MlpLayer {
    int K = 0, N_valid = 0, BN = 0, NT = 0;
    void* d_w = nullptr;
    float* d_bias = nullptr;
};

struct pt_nif {
    int device = 0;
    int kind = PT_NIF_SIREN;
    void* d_smem_image = nullptr;     // pre-laid-out shared-memory image of the fused kernel (+ raw blob)
    size_t d_alloc_bytes = 0;
    int64_t smem_bytes = 0;
    // PT_NIF_FR_FAMILY (layered GEMM path)
    int mlp_H = 0, mlp_L = 0, mlp_c = 0, mlp_fp8 = 0;
    float* mlp_freq = nullptr;        // B [20][2] fp32
    std::vector<MlpLayer> mlp_layers;
    void* mlp_act[2] = {nullptr, nullptr};   // blocked activation ping-pong buffers (lazily sized)
    int64_t mlp_act_bytes = 0;
    // the layered path's activation buffers are per-handle scratch: mlp_mu guards their (re)allocation
    // and every use is ordered after the previous one by mlp_last_use (recorded on the using stream)
    std::mutex mlp_mu;
    cudaEvent_t mlp_last_use = nullptr;
};

namespace pt {

// camera constants in fp32 (host computes in fp64, rounds once; reading R22)
struct Cam32 {
    float f[3], r[3], u[3], eye[3];
    float ta, t;
};
Cam32 make_cam32(const pt_camera& c, int W, int H);

struct TraceParams {
    const uint4* pool;
    int empty;
    const DevMaterial* mats;
    int64_t n_tris;
    int bvh_depth;       // 4-wide levels (chooses the path kernel variant)
};

// kernel launchers (trace_kernels.cu)
// one wave: slots i in [0, n_slots) = (pixel p0 + i % np, sample first_sample + i / np); np = the pixels of
// the rendered row range (p0 = row0 W)
void launch_paths(const TraceParams& tp, const Cam32& cam, int W, int H, int p0, int np, int first_sample, int n_slots,
                  int max_depth, uint64_t seed, int use_nif, float3 env, Workspace& ws, cudaStream_t st);
int path_launches(int max_depth);   // kernels launch_paths launches per wave
void launch_accumulate(const float* wave_buf, int n_pix, int k, float* fb, const uint32_t* counters,
                       unsigned long long* stats, uint32_t paths, cudaStream_t st);
void launch_primary(const TraceParams& tp, const Cam32& cam, int W, int H, int sample, uint64_t seed,
                    int32_t* prim, float* t, cudaStream_t st);
void launch_primary_aov(const TraceParams& tp, const Cam32& cam, int W, int H, int sample, uint64_t seed, int32_t* prim,
                        float* t, float* pos, float* nrm, float* bary2, cudaStream_t st);
void launch_trace_rays(const TraceParams& tp, const float* o, const float* d, int64_t n, int32_t* prim, float* t,
                       cudaStream_t st);
void launch_scale(float* fb, int64_t n, float s, cudaStream_t st);
void launch_path_record(const TraceParams& tp, const Cam32& cam, int W, int H, int s0, int n_s, int max_depth,
                        uint64_t seed, int use_nif, float3 env, const int32_t* pix, int n_pix, int32_t* prims,
                        uint32_t* flags, float* esc_dir, float* L, cudaStream_t st);
void launch_pack_queries(const float* uv, int64_t n, float4* esc, float4* esc_beta, uint32_t* count,
                         cudaStream_t st);

// NIF (nif_kernel.cu)
int64_t nif_smem_image_bytes();
// counting build (-DPT_COUNT) traversal counters: false / no-op in the product build
bool trav_counts(int64_t* visits, int64_t* prim_tests, int64_t* fp64);
void trav_counts_reset();
void nif_build_smem_image(const uint16_t* blob, std::vector<uint8_t>* image);
void nif_build_smem_image_fr(const uint16_t* blob, std::vector<uint8_t>* image);
void nif_build_smem_image_fr8(const uint16_t* blob, std::vector<uint8_t>* image);   // e4m3 variant (R24)
float half_to_float(uint16_t h);
uint8_t float_to_e4m3(float x);   // OCP e4m3, RN, saturating (cvt.rn.satfinite.e4m3x2.f32 on the host)
cudaError_t launch_nif(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                       int64_t max_rows, float* out, int dir_input, cudaStream_t st);
int num_sms();   // SM count of the current device (cached per device)
int current_device();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (device, kernel): the attribute is per device
cudaError_t ensure_dyn_smem(const void* kernel, int bytes);
// the paper's NIF family (mlp_kernel.cu)
int mlp_concat_layer(int L);
int64_t mlp_blob_halves(int H, int L);
int mlp_load(pt_nif* nif, int H, int L, const uint16_t* blob, int fp8, std::string* msg);
void mlp_free(pt_nif* nif);
cudaError_t launch_mlp(pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count, int64_t max_rows,
                       float* out, int dir_input, cudaStream_t st);

// Programmatic dependent launch along the wave's kernel chain (first_bounce -> path -> siren ->
// accumulate): a kernel launched with launch_pdl may be scheduled while its predecessor drains (the
// predecessor calls pdl_trigger() once all its CTAs are resident); it runs its input-independent prologue
// (barrier init, TMEM alloc, weight copies) and calls pdl_wait() before touching the predecessor's
// outputs (griddepcontrol.wait: the predecessor has completed and its memory is visible). Both are
// no-ops for a normal launch. PT_NO_PDL=1 launches normally (A/B measurement).
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace pt
