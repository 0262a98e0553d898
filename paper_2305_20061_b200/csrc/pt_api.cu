// pt_api.cu -- C-ABI of libpt_b200 (include/pt.h) and the wavefront render loop.
//
// Per wave of k consecutive samples x all pixels (SURVEY.md 8a "Wave"):
//   raygen -> for depth 1..max_depth { traverse -> shade (scatter, RR, compaction) } -> NIF -> accumulate.
// All queue lengths live in device counters, so the host never synchronises inside a wave; kernels
// size their grids to the SM count and read their work counts on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pt_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CU(expr)                                                                                   \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) {                                                                   \
            return fail(_e == cudaErrorMemoryAllocation ? PT_ERR_OOM : PT_ERR_CUDA,                \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                       \
        }                                                                                          \
    } while (0)

int check_device() {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return fail(PT_ERR_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    int major = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) return fail(PT_ERR_CUDA, "libpt_b200 requires an sm_100 (B200) device");
    return PT_OK;
}

bool finite3(const float* v) { return std::isfinite(v[0]) && std::isfinite(v[1]) && std::isfinite(v[2]); }

// Path-state buffers (the large per-wave arrays) are pooled per device and shared by all scene handles:
// re-creating a scene does not reallocate ~0.5 GB of wave state. Reuse across streams is ordered by
// an event recorded after each render's last use (the next user's stream waits on it).
struct PathPool {
    std::mutex mu;
    int64_t capacity = 0;
    float4* rayA[2] = {nullptr, nullptr};
    float4* rayB[2] = {nullptr, nullptr};
    float2* rayC[2] = {nullptr, nullptr};
    float4* esc = nullptr;
    float4* esc_beta = nullptr;
    float* wave_buf = nullptr;
    cudaEvent_t last_use = nullptr;
    cudaStream_t host_stream = nullptr;   // stream of the host-buffer entry point pt_render (all scenes)
};

// Device blocks of destroyed scene / NIF handles are kept per device and size class (powers of two)
// and handed to the next handle: creating and destroying a handle per frame (the end-to-end path)
// then costs a host-to-device copy, not a cudaMalloc / cudaFree pair. A block returns to the cache
// only after the device is idle (the same guarantee cudaFree gives).
struct BlockCache {
    std::mutex mu;
    std::vector<std::pair<size_t, void*>> free_blocks;   // (class bytes, pointer)
    size_t cached = 0;
};
constexpr size_t kBlockCacheMax = 512ull << 20;

BlockCache& block_cache(int dev) {
    static BlockCache caches[64];
    return caches[dev & 63];
}

size_t block_class(size_t bytes) {
    size_t c = 256;
    while (c < bytes) c <<= 1;
    return c;
}

cudaError_t cache_alloc(int dev, size_t bytes, void** out) {
    const size_t c = block_class(bytes);
    BlockCache& bc = block_cache(dev);
    {
        std::lock_guard<std::mutex> lk(bc.mu);
        for (size_t i = 0; i < bc.free_blocks.size(); ++i) {
            if (bc.free_blocks[i].first == c) {
                *out = bc.free_blocks[i].second;
                bc.free_blocks.erase(bc.free_blocks.begin() + i);
                bc.cached -= c;
                return cudaSuccess;
            }
        }
    }
    return cudaMalloc(out, c);
}

void cache_free(int dev, void* p, size_t bytes) {
    if (!p) return;
    const size_t c = block_class(bytes);
    cudaDeviceSynchronize();   // no stream may still read the block
    BlockCache& bc = block_cache(dev);
    std::lock_guard<std::mutex> lk(bc.mu);
    if (bc.cached + c > kBlockCacheMax) {
        cudaFree(p);
        return;
    }
    bc.free_blocks.emplace_back(c, p);
    bc.cached += c;
}

// Host-to-device uploads of handle data (scene, NIF image) go through one pinned staging buffer per
// device and an async copy on a private stream: a pageable cudaMemcpy stages through the driver and took
// ~2x as long for the 119 KB NIF image. Uploads above kStagingMax fall back to cudaMemcpy.
struct Staging {
    std::mutex mu;
    void* host = nullptr;
    size_t cap = 0;
    cudaStream_t stream = nullptr;
};
constexpr size_t kStagingMax = 64ull << 20;

cudaError_t upload(int dev, void* d_dst, const void* h_src, size_t bytes) {
    if (bytes > kStagingMax) return cudaMemcpy(d_dst, h_src, bytes, cudaMemcpyHostToDevice);
    static Staging stagings[64];
    Staging& st = stagings[dev & 63];
    std::lock_guard<std::mutex> lk(st.mu);
    cudaError_t e = cudaSuccess;
    if (!st.stream) e = cudaStreamCreateWithFlags(&st.stream, cudaStreamNonBlocking);
    if (e == cudaSuccess && st.cap < bytes) {
        if (st.host) cudaFreeHost(st.host);
        st.host = nullptr;
        st.cap = 0;
        const size_t cap = std::max<size_t>(bytes, 1ull << 20);
        e = cudaHostAlloc(&st.host, cap, cudaHostAllocDefault);
        if (e == cudaSuccess) st.cap = cap;
    }
    if (e != cudaSuccess) return cudaMemcpy(d_dst, h_src, bytes, cudaMemcpyHostToDevice);
    std::memcpy(st.host, h_src, bytes);
    e = cudaMemcpyAsync(d_dst, st.host, bytes, cudaMemcpyHostToDevice, st.stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st.stream);   // the staging buffer is reused next call
    return e;
}

PathPool& path_pool(int dev) {
    static PathPool pools[64];
    return pools[dev & 63];
}

int ensure_pool(PathPool& pp, int64_t cap) {
    if (!pp.last_use) CU(cudaEventCreateWithFlags(&pp.last_use, cudaEventDisableTiming));
    if (cap <= pp.capacity) return PT_OK;
    CU(cudaEventSynchronize(pp.last_use));           // no render may still use the old buffers
    for (int b = 0; b < 2; ++b) {
        cudaFree(pp.rayA[b]); cudaFree(pp.rayB[b]); cudaFree(pp.rayC[b]);
        pp.rayA[b] = pp.rayB[b] = nullptr;
        pp.rayC[b] = nullptr;
    }
    cudaFree(pp.esc); cudaFree(pp.esc_beta); cudaFree(pp.wave_buf);
    pp.esc = pp.esc_beta = nullptr;
    pp.wave_buf = nullptr;
    pp.capacity = 0;
    CU(cudaMalloc(&pp.rayA[0], sizeof(float4) * cap));
    CU(cudaMalloc(&pp.rayB[0], sizeof(float4) * cap));
    CU(cudaMalloc(&pp.rayC[0], sizeof(float2) * cap));
    CU(cudaMalloc(&pp.esc, sizeof(float4) * cap));
    CU(cudaMalloc(&pp.esc_beta, sizeof(float4) * cap));
    CU(cudaMalloc(&pp.wave_buf, sizeof(float) * 3 * cap));
    pp.capacity = cap;
    return PT_OK;
}

void free_ws(pt::Workspace& ws) {
    cudaFree(ws.fb);
    ws = pt::Workspace();
}

// the scene's counters and stats live in its single device allocation (pt_scene_create); the
// host-path stream is per device, created once
int ensure_ws(pt_scene* sc) {
    if (!sc->ws.own_stream) {
        PathPool& pp = path_pool(sc->device);
        std::lock_guard<std::mutex> lk(pp.mu);
        if (!pp.host_stream) CU(cudaStreamCreateWithFlags(&pp.host_stream, cudaStreamNonBlocking));
        sc->ws.own_stream = pp.host_stream;
    }
    return PT_OK;
}

pt::TraceParams trace_params(const pt_scene* sc) {
    pt::TraceParams tp;
    tp.pool = sc->d_pool;
    tp.empty = sc->empty ? 1 : 0;
    tp.mats = sc->d_mats;
    tp.n_tris = sc->n_tris;
    tp.bvh_depth = (int)sc->bvh_depth;
    return tp;
}

// kernel-class timers for profiling (CUDA events on the launching stream)
enum { T_RAYGEN, T_TRAVERSE, T_SHADE, T_NIF, T_ACCUM, T_N };

struct Timer {
    bool on;
    cudaStream_t st;
    std::vector<pt::TimedLaunch>* rec;
    void begin(int, cudaEvent_t* a) {
        if (!on) return;
        cudaEventCreate(a);
        cudaEventRecord(*a, st);
    }
    void end(int cls, cudaEvent_t a) {
        if (!on) return;
        cudaEvent_t b;
        cudaEventCreate(&b);
        cudaEventRecord(b, st);
        rec->push_back({cls, a, b});
    }
};

// sum the pending launch timers into stats (synchronises on the recorded events)
void collect_timers(pt_scene* sc) {
    for (auto& r : sc->pending) {
        float ms = 0.0f;
        cudaEventSynchronize(r.b);
        cudaEventElapsedTime(&ms, r.a, r.b);
        double* dst = r.cls == T_RAYGEN ? &sc->stats.t_raygen_ms
                    : r.cls == T_TRAVERSE ? &sc->stats.t_traverse_ms
                    : r.cls == T_SHADE ? &sc->stats.t_shade_ms
                    : r.cls == T_NIF ? &sc->stats.t_nif_ms : &sc->stats.t_accum_ms;
        *dst += ms;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    sc->pending.clear();
}



int render_samples_impl(pt_scene* sc, const pt_nif* nif, const float* env_rgb, int W, int H, int row0, int row1,
                        int first_sample, int n_samples, int max_depth, uint64_t seed, int wave_samples, float* d_accum,
                        cudaStream_t st) {
    if (W < 1 || H < 1 || n_samples < 1 || max_depth < 1 || first_sample < 0)
        return fail(PT_ERR_INVALID_ARG, "width, height, n_samples, max_depth must be >= 1");
    if (row0 < 0 || row1 > H || row0 >= row1) return fail(PT_ERR_INVALID_ARG, "rows must satisfy 0 <= row0 < row1 <= height");
    if (max_depth > 60) return fail(PT_ERR_INVALID_ARG, "max_depth too large (<= 60)");
    if (!nif && !env_rgb) return fail(PT_ERR_INVALID_ARG, "env_rgb must be given when nif is NULL");
    if (!d_accum) return fail(PT_ERR_INVALID_ARG, "d_accum is NULL");
    if ((int64_t)W * H > (1ll << 31) / 2) return fail(PT_ERR_INVALID_ARG, "frame too large");
    const int64_t np = (int64_t)W * (row1 - row0);   // pixels rendered
    const int64_t p0 = (int64_t)W * row0;
    pt::trav_counts_reset();                          // counting build only (pt_get_stats)
    int64_t k = wave_samples;
    // automatic wave: up to 2^28 paths (29 GB of wave state; one wave per frame up to that size): fewer
    // wave tails and NIF launches, and the first bounce's sample groups reach 32 samples per pixel
    // (config 3: 2.19 -> 2.34 G samples/s from 8 to 66 M paths per wave, profiles/round2/wave_k_c3.log;
    // config 4: 2.66 -> 2.86 G from 66 to 265 M, profiles/round2/wavek.log)
    if (k <= 0) k = std::max<int64_t>(1, std::min<int64_t>(n_samples, (int64_t)(1 << 28) / np));
    k = std::min<int64_t>(k, n_samples);
    while (k > 1 && k * np > (1ll << 31)) --k;
    int rc = ensure_ws(sc);
    if (rc) return rc;
    PathPool& pp = path_pool(sc->device);
    std::lock_guard<std::mutex> pool_lock(pp.mu);
    rc = ensure_pool(pp, k * np);
    if (rc) return rc;
    CU(cudaStreamWaitEvent(st, pp.last_use, 0));   // previous user of the pooled buffers is done
    // from here on work may be enqueued on st: record the pool's last use on every exit path, so the
    // next user waits for whatever this call enqueued even when it returns an error
    struct RecordOnExit {
        cudaEvent_t ev;
        cudaStream_t st;
        ~RecordOnExit() { cudaEventRecord(ev, st); }
    } record_on_exit{pp.last_use, st};
    pt::Workspace& ws = sc->ws;
    for (int b = 0; b < 2; ++b) {
        ws.rayA[b] = pp.rayA[b];
        ws.rayB[b] = pp.rayB[b];
        ws.rayC[b] = pp.rayC[b];
    }
    ws.esc = pp.esc;
    ws.esc_beta = pp.esc_beta;
    ws.wave_buf = pp.wave_buf;
    ws.capacity = pp.capacity;
    unsigned long long* d_stats = ws.d_stats;
    CU(cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * 4, st));
    const pt::Cam32 cam = pt::make_cam32(sc->cam, W, H);
    const pt::TraceParams tp = trace_params(sc);
    const float3 env = env_rgb ? make_float3(env_rgb[0], env_rgb[1], env_rgb[2]) : make_float3(0, 0, 0);
    const int use_nif = nif ? 1 : 0;
    collect_timers(sc);                  // drop timers of a previous call
    Timer tm{sc->profiling, st, &sc->pending};
    pt_stats stats{};
    for (int64_t w0 = first_sample; w0 < (int64_t)first_sample + n_samples; w0 += k) {
        const int64_t kk = std::min<int64_t>(k, (int64_t)first_sample + n_samples - w0);
        const int64_t slots = kk * np;
        CU(cudaMemsetAsync(ws.counters, 0, sizeof(uint32_t) * pt::kCounters, st));
        cudaEvent_t e0;
        tm.begin(T_TRAVERSE, &e0);
        pt::launch_paths(tp, cam, W, H, (int)p0, (int)np, (int)w0, (int)slots, max_depth, seed, use_nif, env, ws, st);
        tm.end(T_TRAVERSE, e0);
        stats.launches += pt::path_launches(max_depth);
        stats.traverse_launches += pt::path_launches(max_depth);
        if (use_nif) {
            tm.begin(T_NIF, &e0);
            cudaError_t e = pt::launch_nif(nif, ws.esc, ws.esc_beta, ws.counters + pt::kCounterEsc, slots, ws.wave_buf, 1, st);
            tm.end(T_NIF, e0);
            if (e != cudaSuccess) return fail(PT_ERR_CUDA, std::string("nif launch: ") + cudaGetErrorString(e));
            stats.launches += 1;
            stats.nif_launches += 1;
        }
        tm.begin(T_ACCUM, &e0);
        pt::launch_accumulate(ws.wave_buf, (int)np, (int)kk, d_accum + 3 * p0, ws.counters, d_stats, (uint32_t)slots, st);
        tm.end(T_ACCUM, e0);
        stats.launches += 1;   // accumulate (with the wave statistics)
        stats.waves += 1;
    }
    CU(cudaGetLastError());
    sc->stats = stats;   // kernel times and paths/segments/escaped are resolved by pt_get_stats
    return PT_OK;
}

}  // namespace

namespace pt {

Cam32 make_cam32(const pt_camera& c, int W, int H) {
    // fp64 on the host, rounded once to fp32 (reading R22)
    double f[3], r[3], u[3];
    for (int a = 0; a < 3; ++a) f[a] = (double)c.look_at[a] - (double)c.eye[a];
    const double lf = std::sqrt((f[0] * f[0] + f[1] * f[1]) + f[2] * f[2]);
    for (int a = 0; a < 3; ++a) f[a] /= lf;
    const double up[3] = {c.up[0], c.up[1], c.up[2]};
    r[0] = f[1] * up[2] - f[2] * up[1];
    r[1] = f[2] * up[0] - f[0] * up[2];
    r[2] = f[0] * up[1] - f[1] * up[0];
    const double lr = std::sqrt((r[0] * r[0] + r[1] * r[1]) + r[2] * r[2]);
    for (int a = 0; a < 3; ++a) r[a] /= lr;
    u[0] = r[1] * f[2] - r[2] * f[1];
    u[1] = r[2] * f[0] - r[0] * f[2];
    u[2] = r[0] * f[1] - r[1] * f[0];
    const double t = std::tan(0.5 * (double)c.vfov_deg * 3.14159265358979323846 / 180.0);
    Cam32 k;
    for (int a = 0; a < 3; ++a) {
        k.f[a] = (float)f[a];
        k.r[a] = (float)r[a];
        k.u[a] = (float)u[a];
        k.eye[a] = c.eye[a];
    }
    k.ta = (float)(t * ((double)W / (double)H));
    k.t = (float)t;
    return k;
}

cudaError_t launch_nif_debug(const pt_nif* nif, const float4* esc, const float4* esc_beta, const uint32_t* count,
                             int64_t rows, float* out, float* dbg, cudaStream_t st);

}  // namespace pt

extern "C" {

const char* pt_last_error(void) { return g_err.c_str(); }
const char* pt_version(void) { return "pt_b200 0.1 sm_100a"; }

int pt_scene_create(const pt_triangle* tris, int64_t n_tris, const pt_sphere* spheres, int64_t n_spheres,
                    const pt_material* mats, int32_t n_mats, const pt_camera* cam, pt_scene** out) {
    if (!out || !cam || n_tris < 0 || n_spheres < 0 || n_mats < 0) return fail(PT_ERR_INVALID_ARG, "bad argument");
    if ((n_tris > 0 && !tris) || (n_spheres > 0 && !spheres) || (n_mats > 0 && !mats))
        return fail(PT_ERR_INVALID_ARG, "null array with positive count");
    if (n_tris + n_spheres >= (1ll << 31) - 1) return fail(PT_ERR_INVALID_ARG, "too many primitives");
    *out = nullptr;
    for (int64_t i = 0; i < n_tris; ++i) {
        if (!finite3(tris[i].v0) || !finite3(tris[i].v1) || !finite3(tris[i].v2))
            return fail(PT_ERR_DOMAIN, "non-finite triangle vertex");
        if (tris[i].material >= (uint32_t)n_mats) return fail(PT_ERR_INVALID_ARG, "triangle material out of range");
    }
    for (int64_t i = 0; i < n_spheres; ++i) {
        if (!finite3(spheres[i].center) || !std::isfinite(spheres[i].radius) || !(spheres[i].radius > 0.0f))
            return fail(PT_ERR_DOMAIN, "non-finite sphere or radius <= 0");
        if (spheres[i].material >= (uint32_t)n_mats) return fail(PT_ERR_INVALID_ARG, "sphere material out of range");
    }
    for (int32_t i = 0; i < n_mats; ++i)
        if (mats[i].kind > PT_EMISSIVE) return fail(PT_ERR_INVALID_ARG, "unknown material kind");
    int rc = check_device();
    if (rc) return rc;
    pt::HostBvh bvh;
    std::string msg;
    rc = pt::build_wide_bvh(tris, n_tris, spheres, n_spheres, &bvh, &msg);
    if (rc) return fail(rc, msg);
    pt_scene* sc = new pt_scene();
    cudaGetDevice(&sc->device);
    sc->n_tris = n_tris;
    sc->n_sph = n_spheres;
    sc->n_mats = n_mats;
    sc->cam = *cam;
    sc->empty = bvh.empty;
    sc->bvh_nodes = bvh.n_nodes;
    sc->bvh_leaves = bvh.n_leaves;
    sc->bvh_depth = bvh.max_depth;
    auto cleanup = [&](int code, const std::string& m) {
        pt_scene_destroy(sc);
        return fail(code, m);
    };
#define CUS(expr)                                                                                        \
    do {                                                                                                 \
        cudaError_t _e = (expr);                                                                         \
        if (_e != cudaSuccess)                                                                           \
            return cleanup(_e == cudaErrorMemoryAllocation ? PT_ERR_OOM : PT_ERR_CUDA, cudaGetErrorString(_e)); \
    } while (0)
    // one device allocation for everything the scene owns: materials, the wave's counters and stats
    // (256-B aligned, uploaded from one small zeroed host block), then the BVH pool with its inline
    // primitives (uploaded straight from the builder's buffer; shading reads the hit primitive there)
    sc->pool_units = bvh.units;
    static_assert(sizeof(pt::DevMaterial) == sizeof(pt_material), "material layout");
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    const size_t b_mat = al(sizeof(pt_material) * n_mats), b_cnt = al(sizeof(uint32_t) * pt::kCounters),
                 b_st = al(sizeof(unsigned long long) * 4);
    const size_t b_small = b_mat + b_cnt + b_st;
    const size_t b_pool = sizeof(uint4) * (size_t)sc->pool_units;
    const size_t total = b_small + b_pool;
    std::vector<uint8_t> host(b_small, 0);
    const size_t o_mat = 0, o_cnt = b_mat, o_st = b_mat + b_cnt;
    if (n_mats > 0) std::memcpy(&host[o_mat], mats, sizeof(pt_material) * n_mats);
    sc->d_alloc_bytes = total;
    CUS(cache_alloc(sc->device, total, &sc->d_alloc));
    uint8_t* base = static_cast<uint8_t*>(sc->d_alloc);
    CUS(upload(sc->device, base, host.data(), b_small));
    if (b_pool > 0) CUS(upload(sc->device, base + b_small, bvh.pool.get(), b_pool));
    sc->d_pool = sc->pool_units > 0 ? reinterpret_cast<uint4*>(base + b_small) : nullptr;
    sc->d_mats = n_mats > 0 ? reinterpret_cast<pt::DevMaterial*>(base + o_mat) : nullptr;
    sc->ws.counters = reinterpret_cast<uint32_t*>(base + o_cnt);
    sc->ws.d_stats = reinterpret_cast<unsigned long long*>(base + o_st);
#undef CUS
    *out = sc;
    return PT_OK;
}

int pt_scene_destroy(pt_scene* sc) {
    if (!sc) return PT_OK;
    {
        std::lock_guard<std::mutex> lk(sc->mu);
        collect_timers(sc);
        cache_free(sc->device, sc->d_alloc, sc->d_alloc_bytes);
        cache_free(sc->device, sc->ws.fb, sizeof(float) * sc->ws.fb_capacity);
        sc->ws.fb = nullptr;
        free_ws(sc->ws);
    }
    delete sc;
    return PT_OK;
}

int pt_nif_load_ex(int32_t kind, const uint16_t* blob, int64_t n_halves, pt_nif** out) {
    if (!blob || !out) return fail(PT_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    if (kind != PT_NIF_SIREN && kind != PT_NIF_FOURIER_RELU) return fail(PT_ERR_INVALID_ARG, "unknown NIF kind");
    const int64_t want = kind == PT_NIF_SIREN ? 50307 : 50051;
    if (n_halves != want)
        return fail(PT_ERR_FORMAT, kind == PT_NIF_SIREN ? "NIF blob must hold 50307 fp16 values (SIREN 2-128x4-3)"
                                                        : "NIF blob must hold 50051 fp16 values (Fourier/ReLU NIF)");
    for (int64_t i = 0; i < n_halves; ++i)
        if ((blob[i] & 0x7C00u) == 0x7C00u) return fail(PT_ERR_DOMAIN, "non-finite NIF weight");
    int rc = check_device();
    if (rc) return rc;
    std::vector<uint8_t> img;
    if (kind == PT_NIF_SIREN) pt::nif_build_smem_image(blob, &img);
    else pt::nif_build_smem_image_fr(blob, &img);
    pt_nif* n = new pt_nif();
    n->kind = kind;
    cudaGetDevice(&n->device);
    n->smem_bytes = (int64_t)img.size();
    // one allocation and one copy: the kernel's shared-memory image (the kernels read nothing else)
    n->d_alloc_bytes = img.size();
    cudaError_t e = cache_alloc(n->device, img.size(), &n->d_smem_image);
    if (e == cudaSuccess) e = upload(n->device, n->d_smem_image, img.data(), img.size());
    if (e != cudaSuccess) {
        pt_nif_destroy(n);
        return fail(e == cudaErrorMemoryAllocation ? PT_ERR_OOM : PT_ERR_CUDA, cudaGetErrorString(e));
    }
    *out = n;
    return PT_OK;
}

int pt_nif_load(const uint16_t* blob, int64_t n_halves, pt_nif** out) {
    return pt_nif_load_ex(PT_NIF_SIREN, blob, n_halves, out);
}

int pt_nif_load_family_ex(int32_t hidden, int32_t layers, int32_t precision, const uint16_t* blob, int64_t n_halves,
                          pt_nif** out) {
    if (!blob || !out) return fail(PT_ERR_INVALID_ARG, "null argument");
    *out = nullptr;
    if (hidden < 64 || hidden > 1024 || hidden % 64 != 0 || layers < 1 || layers > 16)
        return fail(PT_ERR_INVALID_ARG, "hidden must be a multiple of 64 in [64, 1024], layers in [1, 16]");
    if (precision != PT_NIF_FP16 && precision != PT_NIF_FP8)
        return fail(PT_ERR_INVALID_ARG, "precision must be PT_NIF_FP16 or PT_NIF_FP8");
    if (n_halves != pt::mlp_blob_halves(hidden, layers))
        return fail(PT_ERR_FORMAT, "NIF family blob size does not match (hidden, layers)");
    for (int64_t i = 0; i < n_halves; ++i)
        if ((blob[i] & 0x7C00u) == 0x7C00u) return fail(PT_ERR_DOMAIN, "non-finite NIF weight");
    int rc = check_device();
    if (rc) return rc;
    pt_nif* n = new pt_nif();
    n->kind = PT_NIF_FR_FAMILY;
    cudaGetDevice(&n->device);
    std::string msg;
    rc = pt::mlp_load(n, hidden, layers, blob, precision == PT_NIF_FP8, &msg);
    if (rc) {
        pt_nif_destroy(n);
        return fail(rc, msg);
    }
    if (hidden == 128 && layers == 4) {
        // (128, 4) is the paper's network (reading R23): its fused path is the three-tile paper-NIF kernel
        // (fp16, or e4m3 with kind::f8f6f4), which reads this shared-memory image (the streamed-weight
        // family kernel serves the other sizes)
        std::vector<uint8_t> img;
        if (precision == PT_NIF_FP8) pt::nif_build_smem_image_fr8(blob, &img);
        else pt::nif_build_smem_image_fr(blob, &img);
        n->smem_bytes = (int64_t)img.size();
        n->d_alloc_bytes = img.size();
        cudaError_t e = cache_alloc(n->device, img.size(), &n->d_smem_image);
        if (e == cudaSuccess) e = upload(n->device, n->d_smem_image, img.data(), img.size());
        if (e != cudaSuccess) {
            pt_nif_destroy(n);
            return fail(e == cudaErrorMemoryAllocation ? PT_ERR_OOM : PT_ERR_CUDA, cudaGetErrorString(e));
        }
    }
    *out = n;
    return PT_OK;
}

int pt_nif_load_family(int32_t hidden, int32_t layers, const uint16_t* blob, int64_t n_halves, pt_nif** out) {
    return pt_nif_load_family_ex(hidden, layers, PT_NIF_FP16, blob, n_halves, out);
}

int pt_nif_destroy(pt_nif* n) {
    if (!n) return PT_OK;
    pt::mlp_free(n);
    cache_free(n->device, n->d_smem_image, n->d_alloc_bytes);
    delete n;
    return PT_OK;
}

int pt_render_samples(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width, int32_t height,
                      int32_t first_sample, int32_t n_samples, int32_t max_depth, uint64_t seed, int32_t wave_samples,
                      float* d_accum, void* stream) {
    if (!scene) return fail(PT_ERR_INVALID_ARG, "scene is NULL");
    pt_scene* sc = const_cast<pt_scene*>(scene);
    std::lock_guard<std::mutex> lk(sc->mu);
    return render_samples_impl(sc, nif, env_rgb, width, height, 0, height, first_sample, n_samples, max_depth, seed,
                               wave_samples, d_accum, (cudaStream_t)stream);
}

int pt_render_rows(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width, int32_t height,
                   int32_t row0, int32_t row1, int32_t first_sample, int32_t n_samples, int32_t max_depth, uint64_t seed,
                   int32_t wave_samples, float* d_accum, void* stream) {
    if (!scene) return fail(PT_ERR_INVALID_ARG, "scene is NULL");
    pt_scene* sc = const_cast<pt_scene*>(scene);
    std::lock_guard<std::mutex> lk(sc->mu);
    return render_samples_impl(sc, nif, env_rgb, width, height, row0, row1, first_sample, n_samples, max_depth, seed,
                               wave_samples, d_accum, (cudaStream_t)stream);
}

namespace {
// pt_render / pt_render_async: frame into the scene's device framebuffer, scale, copy to the host buffer
// on `st` (the scene's own stream for pt_render); synchronous when `sync`
int render_frame(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width, int32_t height,
                 int32_t spp, int32_t max_depth, uint64_t seed, float* out_rgb, void* stream, bool sync) {
    if (!scene || !out_rgb) return fail(PT_ERR_INVALID_ARG, "null argument");
    if (width < 1 || height < 1 || spp < 1 || max_depth < 1) return fail(PT_ERR_INVALID_ARG, "W, H, spp, max_depth >= 1");
    pt_scene* sc = const_cast<pt_scene*>(scene);
    std::lock_guard<std::mutex> lk(sc->mu);
    int rc = ensure_ws(sc);
    if (rc) return rc;
    const int64_t n = (int64_t)width * height * 3;
    cudaStream_t st = sync ? sc->ws.own_stream : (cudaStream_t)stream;
    if (sc->ws.fb_capacity < n) {
        // the old framebuffer may still be read by an earlier asynchronous call: cache_free returns it only
        // once the device is idle
        cache_free(sc->device, sc->ws.fb, sizeof(float) * sc->ws.fb_capacity);
        sc->ws.fb = nullptr;
        sc->ws.fb_capacity = 0;
        CU(cache_alloc(sc->device, sizeof(float) * n, reinterpret_cast<void**>(&sc->ws.fb)));
        sc->ws.fb_capacity = n;
    }
    CU(cudaMemsetAsync(sc->ws.fb, 0, sizeof(float) * n, st));
    rc = render_samples_impl(sc, nif, env_rgb, width, height, 0, height, 0, spp, max_depth, seed, 0, sc->ws.fb, st);
    if (rc) return rc;
    pt::launch_scale(sc->ws.fb, n, 1.0f / (float)spp, st);
    CU(cudaMemcpyAsync(out_rgb, sc->ws.fb, sizeof(float) * n, cudaMemcpyDeviceToHost, st));
    if (sync) CU(cudaStreamSynchronize(st));
    return PT_OK;
}
}  // namespace

int pt_render(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width, int32_t height,
              int32_t spp, int32_t max_depth, uint64_t seed, float* out_rgb) {
    return render_frame(scene, nif, env_rgb, width, height, spp, max_depth, seed, out_rgb, nullptr, true);
}

int pt_render_async(const pt_scene* scene, const pt_nif* nif, const float env_rgb[3], int32_t width, int32_t height,
                    int32_t spp, int32_t max_depth, uint64_t seed, float* out_rgb, void* stream) {
    return render_frame(scene, nif, env_rgb, width, height, spp, max_depth, seed, out_rgb, stream, false);
}

int pt_trace_primary(const pt_scene* scene, int32_t width, int32_t height, uint64_t seed, int32_t sample,
                     int32_t* d_prim, float* d_t, void* stream) {
    if (!scene || !d_prim || !d_t || width < 1 || height < 1 || sample < 0)
        return fail(PT_ERR_INVALID_ARG, "bad argument");
    const pt::Cam32 cam = pt::make_cam32(scene->cam, width, height);
    pt::launch_primary(trace_params(scene), cam, width, height, sample, seed, d_prim, d_t, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return PT_OK;
}

int pt_trace_primary_aov(const pt_scene* scene, int32_t width, int32_t height, uint64_t seed, int32_t sample,
                         int32_t* d_prim, float* d_t, float* d_pos, float* d_normal, float* d_bary2, void* stream) {
    if (!scene || !d_prim || !d_t || !d_pos || !d_normal || !d_bary2 || width < 1 || height < 1 || sample < 0)
        return fail(PT_ERR_INVALID_ARG, "bad argument");
    if ((int64_t)width * height > (1ll << 30)) return fail(PT_ERR_INVALID_ARG, "frame too large");
    const pt::Cam32 cam = pt::make_cam32(scene->cam, width, height);
    pt::launch_primary_aov(trace_params(scene), cam, width, height, sample, seed, d_prim, d_t, d_pos, d_normal, d_bary2,
                           (cudaStream_t)stream);
    CU(cudaGetLastError());
    return PT_OK;
}

int pt_trace_rays(const pt_scene* scene, const float* d_o, const float* d_d, int64_t n, int32_t* d_prim, float* d_t,
                  void* stream) {
    if (!scene || n < 0 || (n > 0 && (!d_o || !d_d || !d_prim || !d_t))) return fail(PT_ERR_INVALID_ARG, "bad argument");
    if (n == 0) return PT_OK;
    pt::launch_trace_rays(trace_params(scene), d_o, d_d, n, d_prim, d_t, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return PT_OK;
}

// Scratch query queue of the pt_nif_infer hook, per device. Every use waits for the previous one (which
// may run on another stream) through `last_use`, and growth first waits for it on the host.
struct InferScratch {
    std::mutex mu;
    float4* esc = nullptr;
    float4* esc_beta = nullptr;
    uint32_t* cnt = nullptr;
    int64_t cap = 0;
    cudaEvent_t last_use = nullptr;
};

static int nif_infer_impl(const pt_nif* nif, const float* d_uv, int64_t n, float* d_rgb, float* d_dbg, void* stream) {
    if (!nif || n < 0 || (n > 0 && (!d_uv || !d_rgb))) return fail(PT_ERR_INVALID_ARG, "bad argument");
    if (n == 0) return PT_OK;
    if (n > (1ll << 31)) return fail(PT_ERR_INVALID_ARG, "too many queries");
    cudaStream_t st = (cudaStream_t)stream;
    static InferScratch scratch[64];
    InferScratch& sc = scratch[pt::current_device()];
    std::lock_guard<std::mutex> lk(sc.mu);
    if (!sc.last_use) CU(cudaEventCreateWithFlags(&sc.last_use, cudaEventDisableTiming));
    if (n > sc.cap) {
        CU(cudaEventSynchronize(sc.last_use));     // no earlier call may still use the old queue
        cudaFree(sc.esc); cudaFree(sc.esc_beta);
        sc.esc = sc.esc_beta = nullptr;
        sc.cap = 0;
        CU(cudaMalloc(&sc.esc, sizeof(float4) * n));
        CU(cudaMalloc(&sc.esc_beta, sizeof(float4) * n));
        sc.cap = n;
    }
    if (!sc.cnt) CU(cudaMalloc(&sc.cnt, sizeof(uint32_t)));
    CU(cudaStreamWaitEvent(st, sc.last_use, 0));
    pt::launch_pack_queries(d_uv, n, sc.esc, sc.esc_beta, sc.cnt, st);
    cudaError_t e = d_dbg ? pt::launch_nif_debug(nif, sc.esc, sc.esc_beta, sc.cnt, n, d_rgb, d_dbg, st)
                          : pt::launch_nif(nif, sc.esc, sc.esc_beta, sc.cnt, n, d_rgb, 0, st);
    cudaEventRecord(sc.last_use, st);            // also on failure: the pack kernel was enqueued
    if (e != cudaSuccess) return fail(PT_ERR_CUDA, std::string("nif launch: ") + cudaGetErrorString(e));
    return PT_OK;
}

int pt_nif_infer(const pt_nif* nif, const float* d_uv, int64_t n, float* d_rgb, void* stream) {
    return nif_infer_impl(nif, d_uv, n, d_rgb, nullptr, stream);
}

// test hook (not in pt.h): raw accumulators of every layer, d_dbg[5][n][128] fp32
PT_API int pt_debug_nif_layers(const pt_nif* nif, const float* d_uv, int64_t n, float* d_rgb, float* d_dbg, void* stream) {
    if (!d_dbg) return fail(PT_ERR_INVALID_ARG, "d_dbg is NULL");
    return nif_infer_impl(nif, d_uv, n, d_rgb, d_dbg, stream);
}

int pt_get_stats(const pt_scene* scene, pt_stats* out) {
    if (!scene || !out) return fail(PT_ERR_INVALID_ARG, "null argument");
    pt_scene* sc = const_cast<pt_scene*>(scene);
    std::lock_guard<std::mutex> lk(sc->mu);
    collect_timers(sc);
    *out = sc->stats;
    if (sc->ws.d_stats) {
        unsigned long long h[4] = {0, 0, 0, 0};
        CU(cudaDeviceSynchronize());
        CU(cudaMemcpy(h, sc->ws.d_stats, sizeof(h), cudaMemcpyDeviceToHost));
        out->paths = (int64_t)h[0];
        out->segments = (int64_t)h[1];
        out->escaped = (int64_t)h[2];
    }
    out->node_visits = out->prim_tests = out->fp64_rechecks = -1;
    if (pt::trav_counts(&out->node_visits, &out->prim_tests, &out->fp64_rechecks)) CU(cudaGetLastError());
    return PT_OK;
}

int pt_set_profiling(pt_scene* scene, int32_t enabled) {
    if (!scene) return fail(PT_ERR_INVALID_ARG, "null argument");
    std::lock_guard<std::mutex> lk(scene->mu);
    scene->profiling = enabled != 0;
    return PT_OK;
}

// test hook (not in pt.h): per-segment records of single paths through the render kernels' shade_segment
// (first-divergence classifier): paths i = (pixel d_pix[i / n_s], sample s0 + i % n_s)
PT_API int pt_debug_path_records(const pt_scene* scene, int32_t use_nif, const float env_rgb[3], int32_t width,
                                 int32_t height, int32_t max_depth, uint64_t seed, const int32_t* d_pix, int32_t n_pix,
                                 int32_t s0, int32_t n_s, int32_t* d_prims, uint32_t* d_flags, float* d_esc_dir,
                                 float* d_L, void* stream) {
    if (!scene || !d_pix || !d_prims || !d_flags || !d_esc_dir || !d_L || n_pix < 0 || n_s < 1 || max_depth < 1 ||
        (!use_nif && !env_rgb) || (int64_t)width * height * n_s >= (1ll << 31))
        return fail(PT_ERR_INVALID_ARG, "bad argument");
    const pt::Cam32 cam = pt::make_cam32(scene->cam, width, height);
    const float3 env = env_rgb ? make_float3(env_rgb[0], env_rgb[1], env_rgb[2]) : make_float3(0, 0, 0);
    pt::launch_path_record(trace_params(scene), cam, width, height, s0, n_s, max_depth, seed, use_nif ? 1 : 0, env, d_pix,
                           n_pix, d_prims, d_flags, d_esc_dir, d_L, (cudaStream_t)stream);
    CU(cudaGetLastError());
    return PT_OK;
}

// host-only test hooks of the BVH builder (no GPU needed; not in pt.h)
PT_API int pt_debug_build_bvh(const pt_triangle* tris, int64_t n_tris, const pt_sphere* spheres, int64_t n_spheres,
                       int64_t* stats /* [4]: nodes, leaves, depth, pool units */, uint32_t* pool_out,
                       int64_t pool_cap_units) {
    pt::HostBvh bvh;
    std::string msg;
    int rc = pt::build_wide_bvh(tris, n_tris, spheres, n_spheres, &bvh, &msg);
    if (rc) return fail(rc, msg);
    if (stats) {
        stats[0] = bvh.n_nodes;
        stats[1] = bvh.n_leaves;
        stats[2] = bvh.max_depth;
        stats[3] = bvh.units;
    }
    if (pool_out && pool_cap_units >= bvh.units && bvh.units > 0)
        std::memcpy(pool_out, bvh.pool.get(), sizeof(uint4) * bvh.units);
    return PT_OK;
}

PT_API uint16_t pt_debug_f16_round(double x, int32_t up) { return up ? pt::f16_round_up(x) : pt::f16_round_down(x); }

}  // extern "C"
