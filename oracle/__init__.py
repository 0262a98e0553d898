"""ctypes wrapper of the fp64 CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg, never by the product package. It shares no code with the CUDA path; both
read the seeded arrays of paper_2305_20061_b200/scenes.py (an input generator with none of the
method's arithmetic). Every function here is argument marshalling; the arithmetic is in oracle.c,
whose header cites the paper passages it follows.

Parity status per function:
  philox            pinned: Random123 known-answer vectors + cuRAND host routine (tests/test_oracle_rng.py)
  closest_hit       pinned: brute force (bit-exact), closed-form axis-aligned cases, watertightness
  camera_rays       pinned: centre-pixel/forward-axis identity, corner symmetry
  equirect          pinned: SPEC.md:441-443 worked values, inverse round trip
  nif_eval          pinned: zero net (exp(b5)), hand-computed one-unit nets, torch.float64 full SIREN
  fr_eval           pinned: zero net (M b4), single-frequency closed form through the concat skip,
                    torch.float64 full network (the paper's Fourier/ReLU/YUV NIF, reading R4)
  scatter           pinned: cosine moments E[cos]=2/3, E[cos^2]=1/2; mirror; Fresnel(0)=0.04; Snell; TIR
  render            pinned: furnace 1 (empty scene == c exactly), furnace 2 (convex sphere == rho*c),
                    furnace 3 (dielectric: L in {0, c}), emitter front/back, RR unbiasedness
                    (full images beyond these: parity unpinned -- Monte Carlo)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "_oracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (fp64, -ffp-contract=off: no fused ops)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
                               "-pthread", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            P, I64, I32, U64, D = C.c_void_p, C.c_int64, C.c_int32, C.c_uint64, C.c_double
            L.orc_scene_create.restype = P
            L.orc_scene_create.argtypes = [P, I64, P, I64, P, I32, P]
            L.orc_scene_destroy.argtypes = [P]
            L.orc_scene_n_nodes.restype = I64
            L.orc_scene_n_nodes.argtypes = [P]
            L.orc_philox.argtypes = [P, P, I64, P]
            L.orc_closest_hit.argtypes = [P, P, P, I64, C.c_int, P, P, P, P]
            L.orc_camera_rays.argtypes = [P, I32, I32, U64, I32, P, I64, P]
            L.orc_equirect.argtypes = [P, I64, P]
            L.orc_camera_dir.argtypes = [P, I32, I32, I32, I32, C.c_float, C.c_float, P]
            L.orc_roulette.restype = C.c_int
            L.orc_roulette.argtypes = [P, I32, D]
            L.orc_nif_eval.argtypes = [P, P, I64, P]
            L.orc_fr_eval.argtypes = [P, P, I64, P]
            L.orc_fr_eval_hl.argtypes = [I32, I32, P, P, I64, P]
            L.orc_fr_eval_hl_fp8.argtypes = [I32, I32, P, P, I64, P]
            L.orc_e4m3_round.restype = D
            L.orc_e4m3_round.argtypes = [D]
            L.orc_render_fr.restype = C.c_int
            L.orc_render_fr.argtypes = [P, I32, I32, P, I32, I32, I32, U64, P, I64, I32, I32, I32, P, P]
            L.orc_render_fr_ex.restype = C.c_int
            L.orc_render_fr_ex.argtypes = [P, I32, I32, P, I32, I32, I32, I32, U64, P, I64, I32, I32, I32, P, P]
            L.orc_fr_concat_layer.restype = C.c_int
            L.orc_fr_concat_layer.argtypes = [I32]
            L.orc_scatter.argtypes = [C.c_int, P, P, D, P, P, P, P]
            L.orc_render.restype = C.c_int
            L.orc_render.argtypes = [P, P, P, I32, I32, I32, U64, P, I64, I32, I32, I32, P, P]
            L.orc_trace_one.restype = I32
            L.orc_trace_one.argtypes = [P, P, P, I32, I32, I32, U64, I64, I32, P, P]
            L.orc_primary.argtypes = [P, I32, I32, U64, I32, P, I64, P, P, P]
            L.orc_trace_paths.argtypes = [P, P, P, I32, I32, I32, U64, P, I64, I32, I32, P, P, P, P, P, P, P, P]
            L.orc_primary_aov.argtypes = [P, I32, I32, U64, I32, P, I64, P, P, P, P, P]
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OracleScene:
    """fp64 oracle scene (own BVH-2) built from scenes.Scene arrays."""

    def __init__(self, scene):
        self.scene = scene
        self._keep = [np.ascontiguousarray(scene.tris), np.ascontiguousarray(scene.spheres),
                      np.ascontiguousarray(scene.materials), np.ascontiguousarray(scene.camera)]
        t, s, m, c = self._keep
        self.h = lib().orc_scene_create(_p(t), t.shape[0], _p(s), s.shape[0], _p(m), m.shape[0], _p(c))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_scene_destroy(self.h)
            self.h = None

    @property
    def n_nodes(self) -> int:
        return int(lib().orc_scene_n_nodes(self.h))

    def closest_hit(self, o, d, brute=False):
        o = np.ascontiguousarray(o, dtype=np.float64).reshape(-1, 3)
        d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1, 3)
        n = o.shape[0]
        prim = np.empty(n, np.int64)
        t = np.empty(n, np.float64)
        bary = np.empty((n, 3), np.float64)
        edge = np.empty(n, np.float64)
        lib().orc_closest_hit(self.h, _p(o), _p(d), n, int(brute), _p(prim), _p(t), _p(bary), _p(edge))
        return prim, t, bary, edge

    def primary(self, width, height, seed, sample, pix):
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        n = pix.shape[0]
        prim = np.empty(n, np.int64)
        t = np.empty(n, np.float64)
        edge = np.empty(n, np.float64)
        lib().orc_primary(self.h, width, height, seed, sample, _p(pix), n, _p(prim), _p(t), _p(edge))
        return prim, t, edge

    def primary_aov(self, width, height, seed, sample, pix):
        """Table-3 AOVs of the primary hits (orc_primary_aov): prim, t, hit point [n][3], geometric
        normal [n][3], (b1, b2) [n][2]."""
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        n = pix.shape[0]
        prim = np.empty(n, np.int64)
        t = np.empty(n, np.float64)
        pos = np.empty((n, 3), np.float64)
        nrm = np.empty((n, 3), np.float64)
        bary2 = np.empty((n, 2), np.float64)
        lib().orc_primary_aov(self.h, width, height, seed, sample, _p(pix), n, _p(prim), _p(t), _p(pos), _p(nrm),
                              _p(bary2))
        return prim, t, pos, nrm, bary2

    def render(self, width, height, max_depth, seed, pix=None, s0=0, s1=1, nif_blob=None, env_rgb=(1, 1, 1),
               nthreads=None):
        """Per-pixel SUM over samples [s0, s1) of the path radiance (fp64 [n][3]) + stats dict."""
        if pix is None:
            pix = np.arange(width * height, dtype=np.int64)
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        out = np.zeros((pix.shape[0], 3), np.float64)
        st = np.zeros(5, np.int64)
        env = np.ascontiguousarray(env_rgb, dtype=np.float64)
        blob = None if nif_blob is None else np.ascontiguousarray(nif_blob, dtype=np.uint16)
        nthreads = nthreads or os.cpu_count() or 1
        lib().orc_render(self.h, _p(blob), _p(env), width, height, max_depth, seed, _p(pix), pix.shape[0],
                         s0, s1, nthreads, _p(out), _p(st))
        stats = dict(zip(["segments", "escaped", "emitted", "capped", "rr_killed"], st.tolist()))
        return out, stats

    def render_fr(self, hidden, layers, blob, width, height, max_depth, seed, pix=None, s0=0, s1=1, nthreads=None,
                  fp8=False):
        """As render, with the environment of the paper's NIF family (hidden, layers); fp8: its e4m3 model
        (reading R24, as fr_eval_hl_fp8)."""
        if pix is None:
            pix = np.arange(width * height, dtype=np.int64)
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        out = np.zeros((pix.shape[0], 3), np.float64)
        st = np.zeros(5, np.int64)
        blob = np.ascontiguousarray(blob, dtype=np.uint16)
        nthreads = nthreads or os.cpu_count() or 1
        lib().orc_render_fr_ex(self.h, int(hidden), int(layers), _p(blob), int(bool(fp8)), width, height, max_depth,
                               seed, _p(pix), pix.shape[0], s0, s1, nthreads, _p(out), _p(st))
        stats = dict(zip(["segments", "escaped", "emitted", "capped", "rr_killed"], st.tolist()))
        return out, stats

    def trace_paths(self, width, height, max_depth, seed, pix, s0, s1, nif_blob=None, env_rgb=(1, 1, 1)):
        """Per-segment records of paths (pixel pix[i // ns], sample s0 + i % ns), orc_trace_paths: dict of prim
        [n][D] (-2 past the end), edge, fres_delta (xi2 - F, < 0 reflect), rr_delta (xi3 - q, >= 0 kill) [n][D],
        ray [n][D][7] (o, d, t), uv [n][2], L [n][3], len [n]."""
        pix = np.ascontiguousarray(pix, dtype=np.int64)
        n = pix.shape[0] * (s1 - s0)
        D = max_depth
        out = {"prim": np.empty((n, D), np.int64), "edge": np.empty((n, D)), "fres_delta": np.empty((n, D)),
               "rr_delta": np.empty((n, D)), "ray": np.empty((n, D, 7)), "uv": np.empty((n, 2)),
               "L": np.empty((n, 3)), "len": np.empty(n, np.int32)}
        env = np.ascontiguousarray(env_rgb, dtype=np.float64)
        blob = None if nif_blob is None else np.ascontiguousarray(nif_blob, dtype=np.uint16)
        lib().orc_trace_paths(self.h, _p(blob), _p(env), width, height, max_depth, seed, _p(pix), pix.shape[0], s0,
                              s1, _p(out["prim"]), _p(out["edge"]), _p(out["fres_delta"]), _p(out["rr_delta"]),
                              _p(out["ray"]), _p(out["uv"]), _p(out["L"]), _p(out["len"]))
        return out

    def trace_one(self, width, height, max_depth, seed, p, s, nif_blob=None, env_rgb=(1, 1, 1)):
        L = np.zeros(3, np.float64)
        prims = np.full(64, -2, np.int64)
        env = np.ascontiguousarray(env_rgb, dtype=np.float64)
        blob = None if nif_blob is None else np.ascontiguousarray(nif_blob, dtype=np.uint16)
        n = lib().orc_trace_one(self.h, _p(blob), _p(env), width, height, max_depth, seed, p, s, _p(L), _p(prims))
        return L, prims[:n]


def philox(ctr, key):
    ctr = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.empty_like(ctr)
    lib().orc_philox(_p(ctr), _p(key), ctr.shape[0], _p(out))
    return out


def camera_rays(camera, width, height, seed, sample, pix):
    pix = np.ascontiguousarray(pix, dtype=np.int64)
    cam = np.ascontiguousarray(camera)
    out = np.empty((pix.shape[0], 3), np.float32)
    lib().orc_camera_rays(_p(cam), width, height, seed, sample, _p(pix), pix.shape[0], _p(out))
    return out


def camera_dir(camera, width, height, x, y, xi0, xi1):
    """fp32 pinhole direction for pixel (x, y) with sub-pixel jitter (xi0, xi1)."""
    cam = np.ascontiguousarray(camera)
    out = np.empty(3, np.float32)
    lib().orc_camera_dir(_p(cam), width, height, x, y, float(xi0), float(xi1), _p(out))
    return out


def roulette(beta, depth, xi3):
    """Returns (survived, beta') for one Russian-roulette decision."""
    b = np.ascontiguousarray(beta, dtype=np.float64).copy()
    ok = lib().orc_roulette(_p(b), depth, float(xi3))
    return bool(ok), b


def equirect(d):
    d = np.ascontiguousarray(d, dtype=np.float64).reshape(-1, 3)
    uv = np.empty((d.shape[0], 2), np.float64)
    lib().orc_equirect(_p(d), d.shape[0], _p(uv))
    return uv


def nif_eval(blob, uv):
    """log-RGB y = MLP(u, v) in fp64 [n][3]; the environment radiance is exp(y)."""
    blob = np.ascontiguousarray(blob, dtype=np.uint16)
    uv = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
    y = np.empty((uv.shape[0], 3), np.float64)
    lib().orc_nif_eval(_p(blob), _p(uv), uv.shape[0], _p(y))
    return y


def fr_eval(blob, uv):
    """The paper's Fourier/ReLU/YUV NIF in fp64: RGB log radiance [n][3] (env = exp)."""
    blob = np.ascontiguousarray(blob, dtype=np.uint16)
    uv = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
    y = np.empty((uv.shape[0], 3), np.float64)
    lib().orc_fr_eval(_p(blob), _p(uv), uv.shape[0], _p(y))
    return y


def fr_eval_hl(hidden, layers, blob, uv):
    """The paper's NIF family of the size sweep (hidden size H, L dense-ReLU layers; reading R23) in
    fp64: RGB log radiance [n][3]."""
    blob = np.ascontiguousarray(blob, dtype=np.uint16)
    uv = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
    y = np.empty((uv.shape[0], 3), np.float64)
    lib().orc_fr_eval_hl(int(hidden), int(layers), _p(blob), _p(uv), uv.shape[0], _p(y))
    return y


def fr_eval_hl_fp8(hidden, layers, blob, uv):
    """The fp8 (e4m3) variant of the family (weights, features and hidden activations rounded to e4m3)."""
    blob = np.ascontiguousarray(blob, dtype=np.uint16)
    uv = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
    y = np.empty((uv.shape[0], 3), np.float64)
    lib().orc_fr_eval_hl_fp8(int(hidden), int(layers), _p(blob), _p(uv), uv.shape[0], _p(y))
    return y


def e4m3_round(x):
    return float(lib().orc_e4m3_round(float(x)))


def fr_concat_layer(layers):
    return int(lib().orc_fr_concat_layer(int(layers)))


def scatter(kind, d, ng, xi, ior=1.5):
    d = np.ascontiguousarray(d, dtype=np.float64)
    ng = np.ascontiguousarray(ng, dtype=np.float64)
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    wi = np.empty(3, np.float64)
    F = np.zeros(1, np.float64)
    side = np.zeros(1, np.int32)
    lib().orc_scatter(kind, _p(d), _p(ng), ior, _p(xi), _p(wi), _p(F), _p(side))
    return wi, float(F[0]), int(side[0])


def u01(x):
    """The (x >> 8) * 2^-24 conversion, exact (reading R13)."""
    return (np.asarray(x, dtype=np.uint32) >> 8).astype(np.float64) * 2.0 ** -24
