/*
 * pt.h -- C-ABI of the B200-native neural path tracer (libpt_b200.so).
 *
 * The calls follow the paper's statement of the problem as BASELINE.json's north_star phrases it:
 *   pt_scene_create(tris, spheres, materials), pt_nif_load(weights),
 *   pt_render(width, height, spp, max_depth, seed) -> float RGB framebuffer.
 * Method: Monte Carlo path tracing with no light sampling; contributions only from emitters hit by
 * chance and from escaped rays, whose radiance is the HDR neural environment light queried at the
 * equirectangular (u,v) of the escape direction (Sec. 3.1, 3.2, 3.3).
 * Citations are /root/reference/PAPER.md line numbers; DESIGN.md lists every reading taken where
 * the paper is silent (camera, materials, RNG, depth semantics ...).
 *
 * Conventions (all entry points):
 *   - return 0 (PT_OK) on success, a negative PT_ERR_* code otherwise; pt_last_error() returns a
 *     thread-local message for the last failing call. No C++ exception crosses this boundary.
 *   - inputs are COPIED: the caller keeps ownership of every host array it passes.
 *   - handles (pt_scene*, pt_nif*) are library-owned, immutable after creation, freed by *_destroy,
 *     and bound to the CUDA device that was current when they were created.
 *   - "d_" pointers are DEVICE pointers owned by the caller; "stream" is a cudaStream_t (NULL = the
 *     legacy default stream). Calls taking a stream are asynchronous with respect to the host unless
 *     stated otherwise; host-pointer calls synchronise before returning.
 *   - concurrent calls on DISTINCT scene handles are safe; calls sharing a scene handle serialise on
 *     that handle's workspace lock.
 *   - there is no CPU fallback: without an sm_100 device every compute call returns PT_ERR_CUDA.
 */
#ifndef PT_H
#define PT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define PT_API __attribute__((visibility("default")))
#else
#define PT_API
#endif

#define PT_OK 0
#define PT_ERR_INVALID_ARG (-1) /* null pointer, size < 0, W/H/spp/max_depth < 1, material out of range */
#define PT_ERR_DOMAIN (-2)      /* non-finite vertex/radius, or a node extent beyond the fp16 range */
#define PT_ERR_FORMAT (-3)      /* NIF blob of the wrong size */
#define PT_ERR_CUDA (-4)        /* CUDA runtime error or no sm_100 device */
#define PT_ERR_OOM (-5)         /* device or host allocation failed */

/* Material kinds. The paper is silent on materials beyond "emissive objects" and shows caustics
   (PAPER.md:78, 221); reading R9 fixes Lambertian / mirror / Schlick dielectric. */
#define PT_LAMBERT 0u
#define PT_MIRROR 1u
#define PT_DIELECTRIC 2u
#define PT_EMISSIVE 3u /* one-sided (front = side the geometric normal points to), no scattering */

/* Triangle, 40 B. Geometric normal = normalize((v1 - v0) x (v2 - v0)). Primitive ids: triangles
   0..n_tris-1 in input order, then spheres n_tris..n_tris+n_spheres-1 (reading R18). */
typedef struct { float v0[3], v1[3], v2[3]; uint32_t material; } pt_triangle;
/* Sphere, 20 B (radius > 0). */
typedef struct { float center[3]; float radius; uint32_t material; } pt_sphere;
/* Material, 32 B. albedo used by LAMBERT/MIRROR, emission by EMISSIVE, ior by DIELECTRIC. */
typedef struct { uint32_t kind; float albedo[3]; float emission[3]; float ior; } pt_material;
/* Pinhole camera, 40 B (reading R5). Row 0 of the image is the top. */
typedef struct { float eye[3], look_at[3], up[3]; float vfov_deg; } pt_camera;

typedef struct pt_scene pt_scene;
typedef struct pt_nif pt_nif;

/* Upload a scene and build its wide (4-ary) BVH with conservatively quantised fp16 child boxes --
   the paper's "round-to-nearest-not-lower" f16 extents widened to a 4-wide node (PAPER.md:101-103,
   Sec. 3.1.4). Host arrays: tris[n_tris], spheres[n_spheres], mats[n_mats], *cam. n_tris and
   n_spheres may be 0 (an empty scene is legal: the furnace case). Every decoded child box is
   verified at build time to contain its subtree's exact fp32 bounds.
   Errors: INVALID_ARG, DOMAIN (non-finite input, a child box beyond the fp16 offset range, or a BVH
   larger than 2^28 16-byte units = 4 GiB), CUDA, OOM. */
PT_API int pt_scene_create(const pt_triangle* tris, int64_t n_tris, const pt_sphere* spheres, int64_t n_spheres,
                    const pt_material* mats, int32_t n_mats, const pt_camera* cam, pt_scene** out);
PT_API int pt_scene_destroy(pt_scene* scene);

/* Load the HDR-NIF (Sec. 3.2; BASELINE.json: SIREN 2->128->128->128->128->3, w0 = 30
   folded into layers 1-4). fp16_blob: n_halves = 50,307 IEEE binary16 values, layer l = 1..5:
   W_l row-major [out][in] then b_l[out]. The network maps x0 = (2u-1, 2v-1) to log-RGB y; the
   environment radiance is exp(y). The weights are re-laid-out once into the shared-memory image of
   the fused kernel (tcgen05 K-major operand tiles) and kept resident on the device.
   Errors: INVALID_ARG, FORMAT (n_halves != 50307), CUDA, OOM. */
PT_API int pt_nif_load(const uint16_t* fp16_blob, int64_t n_halves, pt_nif** out);

/* NIF kinds for pt_nif_load_ex. PT_NIF_SIREN: as pt_nif_load. PT_NIF_FOURIER_RELU: the paper's own
   HDR-NIF (Sec. 3.2; reading R4): Fourier features gamma = (sin 2 pi B x,
   cos 2 pi B x) of x = (u, v) with B [20][2], dense ReLU layers 40->128->88 (+ concat of gamma)->128->128,
   linear 128->3 (YUV, log space), fixed BT.601 YUV->RGB matrix, exp. fp16_blob: n_halves = 50,051 =
   B (40) then W_l [out][in], b_l [out] for the 5 layers. Errors as pt_nif_load. */
#define PT_NIF_SIREN 0
#define PT_NIF_FOURIER_RELU 1
#define PT_NIF_FR_FAMILY 2 /* created by pt_nif_load_family only */
PT_API int pt_nif_load_ex(int32_t kind, const uint16_t* fp16_blob, int64_t n_halves, pt_nif** out);

/* The paper's NIF family of its size sweep ("hidden size H (128) and number of dense-relu
   layers L (4) can be varied"; Fig. nrf-vs-blender H64 L2 / H256 L4 / H1024 L8, PAPER.md:225-227;
   DESIGN.md reading R23): the PT_NIF_FOURIER_RELU architecture with width `hidden` and `layers` dense
   ReLU layers; layer c = the largest odd index below layers/2 (0 if none) outputs hidden - 40 units and
   is concatenated with the 40 Fourier features. fp16_blob: B (40) then W_l [out][in], b_l [out] for the
   layers + 1 layers (n_halves = 40 + sum of fan_out * (fan_in + 1)). Evaluated, for hidden in {64, 128, 256}
   (fp16 or fp8), by one fused kernel (activations resident in TMEM, weights streamed from L2 chunk by chunk),
   otherwise as one tcgen05 GEMM per layer over the whole batch; the environment variable
   PT_MLP_LAYERED=1, read at each inference, forces the per-layer path (for tests). hidden: a multiple of
   64 in [64, 1024]; layers in [1, 16].
   Errors: INVALID_ARG (hidden/layers out of range), FORMAT (n_halves), DOMAIN (non-finite), CUDA, OOM. */
PT_API int pt_nif_load_family(int32_t hidden, int32_t layers, const uint16_t* fp16_blob, int64_t n_halves,
                              pt_nif** out);

/* As pt_nif_load_family with a storage/compute precision: PT_NIF_FP16 (as above) or PT_NIF_FP8 (SURVEY
   8f #4; "float8 ... would halve the memory required for weights and increase performance"):
   weights are rounded once from the fp16 blob to OCP e4m3 (round to nearest even, saturating at 448),
   the Fourier features and every hidden activation are rounded to e4m3 before the next layer, products
   accumulate in fp32 (tcgen05 kind::f8f6f4), biases and the output stay fp32.
   Errors: as pt_nif_load_family; INVALID_ARG for an unknown precision. */
#define PT_NIF_FP16 0
#define PT_NIF_FP8 1
PT_API int pt_nif_load_family_ex(int32_t hidden, int32_t layers, int32_t precision, const uint16_t* fp16_blob,
                                 int64_t n_halves, pt_nif** out);
PT_API int pt_nif_destroy(pt_nif* nif);

/* Render a full frame. env: nif != NULL -> HDR-NIF environment; nif == NULL -> constant env_rgb
   (env_rgb may then not be NULL). out_rgb: HOST buffer of width*height*3 floats, row-major [H][W][3],
   receiving the mean over spp samples. max_depth counts traced segments (reading R7); Russian
   roulette from depth 3. seed keys the Philox-4x32-10 streams (reading R13).
   Synchronous. out_rgb may be pageable or page-locked memory (page-locked makes the read-back a
   direct DMA, ~46 GB/s on the bench box). Errors: INVALID_ARG, CUDA, OOM. */
PT_API int pt_render(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width, int32_t height,
              int32_t spp, int32_t max_depth, uint64_t seed, float* out_rgb);

/* pt_render enqueued on `stream` (a cudaStream_t; NULL = the legacy default stream) without waiting:
   the frame, its scaling and the copy into out_rgb are ordered on the stream, and out_rgb holds the
   frame once the stream reaches that point (cudaStreamSynchronize / an event). out_rgb should be
   page-locked host memory (cudaHostAlloc or registered; pageable memory makes the copy synchronous).
   The caller keeps scene, nif and out_rgb alive until then; calls on one scene handle are ordered only
   when they use the same stream (the scene's framebuffer is reused). Successive frames on two streams
   (with two scene handles) overlap one frame's read-back with the next frame's kernels.
   Errors: INVALID_ARG, CUDA, OOM (launch errors; execution errors surface at the next synchronisation). */
PT_API int pt_render_async(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width,
                           int32_t height, int32_t spp, int32_t max_depth, uint64_t seed, float* out_rgb,
                           void* stream);

/* Multi-GPU / framework path: ADD the per-pixel SUM over samples [first_sample, first_sample +
   n_samples) into the caller-owned DEVICE buffer d_accum[width*height*3] (fp32, row-major [H][W][3]).
   wave_samples (k >= 1, or 0 = automatic: up to 2^28 paths, 108 B of device scratch each) bounds how
   many consecutive samples share one wavefront wave (k * width * height paths in flight). Results are bit-identical for any partition of the
   sample range that keeps wave boundaries, and independent of k up to fp32 summation order.
   Asynchronous on `stream`. Errors: INVALID_ARG, CUDA, OOM. */
PT_API int pt_render_samples(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width,
                      int32_t height, int32_t first_sample, int32_t n_samples, int32_t max_depth, uint64_t seed,
                      int32_t wave_samples, float* d_accum, void* stream);

/* As pt_render_samples for the rows [row0, row1) of the frame only (0 <= row0 < row1 <= height): ADD the
   per-pixel sums over samples [first_sample, first_sample + n_samples) of those rows into d_accum (the
   FULL-frame buffer, [height][width][3]; other rows are not touched). Every path uses the same Philox
   counters (pixel index in the full frame, sample, depth) as a full-frame render, so any partition of the
   (sample, row) range sums to the full-frame result up to fp32 summation order: the multi-GPU split for
   more GPUs than samples (reading R19). Asynchronous. Errors: INVALID_ARG, CUDA, OOM. */
PT_API int pt_render_rows(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width,
                          int32_t height, int32_t row0, int32_t row1, int32_t first_sample, int32_t n_samples,
                          int32_t max_depth, uint64_t seed, int32_t wave_samples, float* d_accum, void* stream);

/* Test/bench hook: closest hits of the camera rays of one sample (raygen + traversal only).
   d_prim[width*height] int32 (-1 = miss), d_t[width*height] float (t of the hit, +inf on miss).
   Asynchronous. Errors: INVALID_ARG, CUDA, OOM. */
PT_API int pt_trace_primary(const pt_scene* scene, int32_t width, int32_t height, uint64_t seed, int32_t sample,
                     int32_t* d_prim, float* d_t, void* stream);

/* Test/report hook: the precision AOVs of PAPER.md:169-188 (Sec. 4.2, Table 3 "normals and primary
   hit-points") for the camera rays of one sample, as the render kernels compute them: d_prim, d_t as
   pt_trace_primary; d_pos[width*height][3] the hit point P = o + t d (fp32, the shading's formula);
   d_normal[width*height][3] the geometric normal the shading uses (triangle: normalize((v1 - v0) x
   (v2 - v0)); sphere: (P - c) / r); d_bary2[width*height][2] the barycentrics (b1, b2) of a triangle
   hit (P = (1 - b1 - b2) v0 + b1 v1 + b2 v2, fp32 watertight edge functions; 0 for spheres). Misses
   write prim -1 and zeros. All buffers are caller-owned device memory. Asynchronous.
   Errors: INVALID_ARG, CUDA. */
PT_API int pt_trace_primary_aov(const pt_scene* scene, int32_t width, int32_t height, uint64_t seed, int32_t sample,
                                int32_t* d_prim, float* d_t, float* d_pos, float* d_normal, float* d_bary2,
                                void* stream);

/* Test/bench hook: closest hits of arbitrary rays. d_o, d_d: [n][3] float device arrays; writes
   d_prim[n] (-1 = miss) and d_t[n]. Asynchronous. */
PT_API int pt_trace_rays(const pt_scene* scene, const float* d_o, const float* d_d, int64_t n, int32_t* d_prim,
                  float* d_t, void* stream);

/* Test/bench hook: the fused NIF kernel on arbitrary queries. d_uv: [n][2] float (u, v in [0,1]);
   d_rgb: [n][3] float receives exp(y) (environment radiance). Asynchronous. */
PT_API int pt_nif_infer(const pt_nif* nif, const float* d_uv, int64_t n, float* d_rgb, void* stream);

/* Statistics of the last pt_render / pt_render_samples on this scene handle (counts are exact;
   kernel times are CUDA-event times summed over launches and are filled only while profiling is on).
   node_visits, prim_tests, fp64_rechecks (interior-node visits, primitive tests, primitive tests decided
   by the fp64 fallback; PAPER.md:103 / SURVEY 8(b)) are filled only by the counting build of the library
   (-DPT_COUNT, tools/trace_count.py: process-wide counters of the last render); -1 otherwise, since
   counting costs an atomic per visit. */
typedef struct {
    int64_t paths, segments, escaped, waves, launches;
    double t_raygen_ms, t_traverse_ms, t_shade_ms, t_nif_ms, t_accum_ms;
    int64_t nif_launches, traverse_launches;
    int64_t node_visits, prim_tests, fp64_rechecks;
} pt_stats;
PT_API int pt_get_stats(const pt_scene* scene, pt_stats* out);

/* Profiling on/off for a scene handle (CUDA events around every kernel; off by default). */
PT_API int pt_set_profiling(pt_scene* scene, int32_t enabled);

/* Thread-local message describing the last non-zero return code ("" if none). Never NULL. */
PT_API const char* pt_last_error(void);

/* Library version string, e.g. "pt_b200 0.1 sm_100a". */
PT_API const char* pt_version(void);

#ifdef __cplusplus
}
#endif

#endif /* PT_H */
