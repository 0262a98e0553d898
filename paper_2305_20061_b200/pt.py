"""Thin Python binding of libpt_b200.so (include/pt.h). Argument marshalling only: every step of the
hot path runs in the library's CUDA kernels. PyTorch provides device memory and streams.

There is no fallback: if the shared library is missing or has no sm_100 device, calls raise."""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import scenes

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PT_B200_LIB") or os.path.join(_PKG, "libpt_b200.so")   # override: tuning experiments
_lib = None
_lock = threading.Lock()


class PtError(RuntimeError):
    pass


class PtStats(C.Structure):
    _fields_ = [("paths", C.c_int64), ("segments", C.c_int64), ("escaped", C.c_int64), ("waves", C.c_int64),
                ("launches", C.c_int64), ("t_raygen_ms", C.c_double), ("t_traverse_ms", C.c_double),
                ("t_shade_ms", C.c_double), ("t_nif_ms", C.c_double), ("t_accum_ms", C.c_double),
                ("nif_launches", C.c_int64), ("traverse_launches", C.c_int64),
                ("node_visits", C.c_int64), ("prim_tests", C.c_int64), ("fp64_rechecks", C.c_int64)]


EXPORTED = ["pt_scene_create", "pt_scene_destroy", "pt_nif_load", "pt_nif_load_ex", "pt_nif_load_family",
            "pt_nif_load_family_ex", "pt_nif_destroy", "pt_render", "pt_render_async",
            "pt_render_samples", "pt_render_rows", "pt_trace_primary", "pt_trace_primary_aov", "pt_trace_rays", "pt_nif_infer", "pt_get_stats",
            "pt_set_profiling", "pt_last_error", "pt_version"]


def lib():
    """Load libpt_b200.so (raises if it was not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise PtError(f"{LIB_PATH} not built: run __graft_entry__.build() (no CPU fallback exists)")
            L = C.CDLL(LIB_PATH)
            P, I64, I32, U64 = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64
            L.pt_scene_create.argtypes = [P, I64, P, I64, P, I32, P, C.POINTER(P)]
            L.pt_scene_destroy.argtypes = [P]
            L.pt_nif_load.argtypes = [P, I64, C.POINTER(P)]
            L.pt_nif_load_ex.argtypes = [I32, P, I64, C.POINTER(P)]
            L.pt_nif_load_family.argtypes = [I32, I32, P, I64, C.POINTER(P)]
            L.pt_nif_load_family_ex.argtypes = [I32, I32, I32, P, I64, C.POINTER(P)]
            L.pt_nif_destroy.argtypes = [P]
            L.pt_render.argtypes = [P, P, P, I32, I32, I32, I32, U64, P]
            L.pt_render_async.argtypes = [P, P, P, I32, I32, I32, I32, U64, P, P]
            L.pt_render_samples.argtypes = [P, P, P, I32, I32, I32, I32, I32, U64, I32, P, P]
            L.pt_render_rows.argtypes = [P, P, P, I32, I32, I32, I32, I32, I32, I32, U64, I32, P, P]
            L.pt_trace_primary.argtypes = [P, I32, I32, U64, I32, P, P, P]
            L.pt_trace_primary_aov.argtypes = [P, I32, I32, U64, I32, P, P, P, P, P, P]
            L.pt_trace_rays.argtypes = [P, P, P, I64, P, P, P]
            L.pt_nif_infer.argtypes = [P, P, I64, P, P]
            L.pt_debug_nif_layers.argtypes = [P, P, I64, P, P, P]
            L.pt_get_stats.argtypes = [P, C.POINTER(PtStats)]
            L.pt_set_profiling.argtypes = [P, I32]
            L.pt_last_error.restype = C.c_char_p
            L.pt_version.restype = C.c_char_p
            L.pt_debug_build_bvh.argtypes = [P, I64, P, I64, P, P, I64]
            L.pt_debug_path_records.argtypes = [P, I32, P, I32, I32, I32, U64, P, I32, I32, I32, P, P, P, P, P]
            L.pt_debug_f16_round.restype = C.c_uint16
            L.pt_debug_f16_round.argtypes = [C.c_double, I32]
            if hasattr(L, "pt_debug_nif_trace"):
                L.pt_debug_nif_trace.argtypes = [P]
            _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise PtError(f"pt error {rc}: {lib().pt_last_error().decode()}")


def _p(a):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _dp(t):
    """device pointer of a CUDA torch tensor"""
    assert t.is_cuda and t.is_contiguous()
    return C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


class Scene:
    """pt_scene_create over scenes.Scene arrays (copied by the library)."""

    def __init__(self, sc: scenes.Scene):
        self.src = sc
        t = np.ascontiguousarray(sc.tris)
        s = np.ascontiguousarray(sc.spheres)
        m = np.ascontiguousarray(sc.materials)
        c = np.ascontiguousarray(sc.camera)
        h = C.c_void_p()
        _check(lib().pt_scene_create(_p(t), t.shape[0], _p(s), s.shape[0], _p(m), m.shape[0], _p(c), C.byref(h)))
        self._lib = lib()
        self.h = h

    def close(self):
        # the library handle is held by the object: module globals may be gone at interpreter exit
        if getattr(self, "h", None):
            self._lib.pt_scene_destroy(self.h)
            self.h = None

    __del__ = close

    def set_profiling(self, on: bool):
        _check(lib().pt_set_profiling(self.h, int(on)))

    def stats(self) -> dict:
        st = PtStats()
        _check(lib().pt_get_stats(self.h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in PtStats._fields_}


NIF_SIREN = 0          # PT_NIF_SIREN: SIREN 2-128x4-3 (scenes.siren_blob)
NIF_FOURIER_RELU = 1   # PT_NIF_FOURIER_RELU: the paper's Fourier/ReLU/YUV NIF (scenes.fourier_relu_blob)
NIF_FR_FAMILY = 2      # PT_NIF_FR_FAMILY: the size-sweep family (scenes.fourier_relu_family_blob)


class Nif:
    def __init__(self, blob: np.ndarray, kind: int = NIF_SIREN, hidden: int = 0, layers: int = 0, fp8: bool = False):
        """kind NIF_FR_FAMILY needs (hidden, layers) (+ fp8: e4m3 weights/activations):
        pt_nif_load_family_ex; else pt_nif_load_ex."""
        b = np.ascontiguousarray(blob, dtype=np.uint16)
        h = C.c_void_p()
        if kind == NIF_FR_FAMILY:
            _check(lib().pt_nif_load_family_ex(int(hidden), int(layers), int(bool(fp8)), _p(b), b.size, C.byref(h)))
        else:
            _check(lib().pt_nif_load_ex(int(kind), _p(b), b.size, C.byref(h)))
        self._lib = lib()
        self.h = h
        self.kind = int(kind)

    def close(self):
        # the library handle is held by the object: module globals may be gone at interpreter exit
        if getattr(self, "h", None):
            self._lib.pt_nif_destroy(self.h)
            self.h = None

    __del__ = close


def _env(env_rgb):
    return None if env_rgb is None else np.ascontiguousarray(env_rgb, dtype=np.float32)


def render(scene: Scene, nif: Nif | None, width, height, spp, max_depth, seed=0, env_rgb=None, out=None) -> np.ndarray:
    """pt_render: full frame, mean over spp, host float32 [H][W][3]. `out` (optional): a C-contiguous
    float32 host array of H*W*3 elements to write into (e.g. a view of pinned memory)."""
    if out is None:
        out = np.empty((height, width, 3), np.float32)
    elif out.dtype != np.float32 or not out.flags["C_CONTIGUOUS"] or out.size != height * width * 3:
        raise PtError(-1, "out must be a C-contiguous float32 array of height * width * 3 elements")
    env = _env(env_rgb if env_rgb is not None else ((1.0, 1.0, 1.0) if nif is None else None))
    _check(lib().pt_render(scene.h, nif.h if nif else None, _p(env), width, height, spp, max_depth, seed, _p(out)))
    return out


def render_async(scene: Scene, nif: Nif | None, width, height, spp, max_depth, seed, out, env_rgb=None,
                 stream=None):
    """pt_render_async: enqueue a full frame (mean over spp) into the host array `out` (C-contiguous
    float32, H*W*3 elements, page-locked for an asynchronous copy) on `stream` (a torch CUDA stream;
    default: the current one). `out` holds the frame once the stream is synchronised."""
    if out.dtype != np.float32 or not out.flags["C_CONTIGUOUS"] or out.size != height * width * 3:
        raise PtError(-1, "out must be a C-contiguous float32 array of height * width * 3 elements")
    env = _env(env_rgb if env_rgb is not None else ((1.0, 1.0, 1.0) if nif is None else None))
    _check(lib().pt_render_async(scene.h, nif.h if nif else None, _p(env), width, height, spp, max_depth, seed,
                                 _p(out), _stream(stream)))
    return out


def render_samples(scene: Scene, nif: Nif | None, width, height, first_sample, n_samples, max_depth, seed, accum,
                   env_rgb=None, wave_samples=0, stream=None):
    """pt_render_samples: accum (CUDA float32 tensor [H*W*3]) += per-pixel sample sums."""
    env = _env(env_rgb if env_rgb is not None else ((1.0, 1.0, 1.0) if nif is None else None))
    _check(lib().pt_render_samples(scene.h, nif.h if nif else None, _p(env), width, height, first_sample, n_samples,
                                   max_depth, seed, wave_samples, _dp(accum), _stream(stream)))


def render_rows(scene: Scene, nif: Nif | None, width, height, row0, row1, first_sample, n_samples, max_depth, seed,
                accum, env_rgb=None, wave_samples=0, stream=None):
    """pt_render_rows: accum (full-frame CUDA float32 [H*W*3]) rows [row0, row1) += per-pixel sample sums."""
    env = _env(env_rgb if env_rgb is not None else ((1.0, 1.0, 1.0) if nif is None else None))
    _check(lib().pt_render_rows(scene.h, nif.h if nif else None, _p(env), width, height, row0, row1, first_sample,
                                n_samples, max_depth, seed, wave_samples, _dp(accum), _stream(stream)))


def trace_primary(scene: Scene, width, height, seed, sample, stream=None):
    import torch
    prim = torch.empty(width * height, dtype=torch.int32, device="cuda")
    t = torch.empty(width * height, dtype=torch.float32, device="cuda")
    _check(lib().pt_trace_primary(scene.h, width, height, seed, sample, _dp(prim), _dp(t), _stream(stream)))
    return prim, t


def trace_primary_aov(scene: Scene, width, height, seed, sample, stream=None):
    """pt_trace_primary_aov: (prim, t, hit point [n][3], normal [n][3], (b1, b2) [n][2]) CUDA tensors."""
    import torch
    n = width * height
    prim = torch.empty(n, dtype=torch.int32, device="cuda")
    t = torch.empty(n, dtype=torch.float32, device="cuda")
    pos = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    nrm = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    bary2 = torch.empty((n, 2), dtype=torch.float32, device="cuda")
    _check(lib().pt_trace_primary_aov(scene.h, width, height, seed, sample, _dp(prim), _dp(t), _dp(pos), _dp(nrm),
                                      _dp(bary2), _stream(stream)))
    return prim, t, pos, nrm, bary2


def trace_rays(scene: Scene, o, d, stream=None):
    import torch
    o = o.contiguous().float()
    d = d.contiguous().float()
    n = o.shape[0]
    prim = torch.empty(n, dtype=torch.int32, device="cuda")
    t = torch.empty(n, dtype=torch.float32, device="cuda")
    _check(lib().pt_trace_rays(scene.h, _dp(o), _dp(d), n, _dp(prim), _dp(t), _stream(stream)))
    return prim, t


def nif_infer(nif: Nif, uv, out=None, stream=None):
    """exp(y) for (u, v) queries: uv CUDA float32 [n][2] -> [n][3]."""
    import torch
    uv = uv.contiguous().float()
    n = uv.shape[0]
    if out is None:
        out = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    _check(lib().pt_nif_infer(nif.h, _dp(uv), n, _dp(out), _stream(stream)))
    return out


def nif_debug_layers(nif: Nif, uv, stream=None):
    """Raw fp32 accumulators of the 5 layers [5][n][128] (pre-activations; layer 5 in cols 0..2)."""
    import torch
    uv = uv.contiguous().float()
    n = uv.shape[0]
    out = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    dbg = torch.zeros((5, n, 128), dtype=torch.float32, device="cuda")
    _check(lib().pt_debug_nif_layers(nif.h, _dp(uv), n, _dp(out), _dp(dbg), _stream(stream)))
    return out, dbg


def debug_path_records(scene: Scene, width, height, max_depth, seed, pix, s0, n_s, use_nif=True, env_rgb=None):
    """Per-segment records of single paths through the render kernels (first-divergence classifier): dict of
    prim [n][D] (-2 past the end), flags [n][D] (1 reflect, 2 roulette kill), esc_dir [n][3], L [n][3]
    (numpy; path i = pixel pix[i // n_s], sample s0 + i % n_s)."""
    import torch
    pix_t = torch.as_tensor(np.ascontiguousarray(pix, dtype=np.int32)).cuda()
    n = len(pix) * n_s
    prims = torch.empty((n, max_depth), dtype=torch.int32, device="cuda")
    flags = torch.empty((n, max_depth), dtype=torch.int32, device="cuda")
    esc = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    L = torch.empty((n, 3), dtype=torch.float32, device="cuda")
    env = _env(env_rgb if env_rgb is not None else (1.0, 1.0, 1.0))
    _check(lib().pt_debug_path_records(scene.h, int(bool(use_nif)), _p(env), width, height, max_depth, seed,
                                       _dp(pix_t), len(pix), s0, n_s, _dp(prims), _dp(flags), _dp(esc), _dp(L),
                                       _stream(None)))
    torch.cuda.synchronize()
    return {"prim": prims.cpu().numpy(), "flags": flags.cpu().numpy(), "esc_dir": esc.cpu().numpy(),
            "L": L.cpu().numpy()}


def debug_build_bvh(sc: scenes.Scene, with_pool=False):
    """Host-only BVH build (no GPU): stats dict and optionally the raw pool (uint32 [units][4])."""
    t = np.ascontiguousarray(sc.tris)
    s = np.ascontiguousarray(sc.spheres)
    st = np.zeros(4, np.int64)
    _check(lib().pt_debug_build_bvh(_p(t), t.shape[0], _p(s), s.shape[0], _p(st), None, 0))
    out = {"nodes": int(st[0]), "leaves": int(st[1]), "depth": int(st[2]), "units": int(st[3])}
    if with_pool:
        pool = np.zeros((max(1, out["units"]), 4), np.uint32)
        _check(lib().pt_debug_build_bvh(_p(t), t.shape[0], _p(s), s.shape[0], _p(st), _p(pool), pool.shape[0]))
        return out, pool[: out["units"]]
    return out


def f16_round(x: float, up: bool) -> int:
    return int(lib().pt_debug_f16_round(float(x), int(up)))


def version() -> str:
    return lib().pt_version().decode()
