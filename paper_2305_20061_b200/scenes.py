"""Seeded synthetic inputs for the neural path tracer (BASELINE.json configs 0-4).

This module is the ONE place both the CUDA path and the fp64 oracle get their inputs from. It holds
none of the method's arithmetic (no ray tracing, no shading, no NIF evaluation, no path-sampling RNG):
only scene geometry, materials, cameras and the HDR-NIF weight blob, written as plain numpy arrays in
the byte layout of the C-ABI structs declared in ``include/pt.h``.

Citations: PAPER.md = /root/reference/PAPER.md (line numbers), SURVEY.md §8c "Scene/camera pins".
The paper's own scenes and HDRIs are not distributed; these generators are the
stand-ins that BASELINE.json names (its ``configs`` list).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------------------------------
# Byte layouts (must match include/pt.h)
# ---------------------------------------------------------------------------------------------------
TRI_DTYPE = np.dtype([("v0", "<f4", 3), ("v1", "<f4", 3), ("v2", "<f4", 3), ("material", "<u4")])   # 40 B
SPHERE_DTYPE = np.dtype([("center", "<f4", 3), ("radius", "<f4"), ("material", "<u4")])                # 20 B
MAT_DTYPE = np.dtype([("kind", "<u4"), ("albedo", "<f4", 3), ("emission", "<f4", 3), ("ior", "<f4")])   # 32 B
CAM_DTYPE = np.dtype([("eye", "<f4", 3), ("look_at", "<f4", 3), ("up", "<f4", 3), ("vfov_deg", "<f4")])  # 40 B

LAMBERT, MIRROR, DIELECTRIC, EMISSIVE = 0, 1, 2, 3

# SIREN NIF (BASELINE.json configs: "SIREN 2->128->128->128->128->3, w0=30")
NIF_HIDDEN = 128
NIF_LAYERS = [(2, 128), (128, 128), (128, 128), (128, 128), (128, 3)]
NIF_W0 = 30.0
NIF_N_HALVES = sum(o * i + o for i, o in NIF_LAYERS)  # 50,307
assert NIF_N_HALVES == 50307


@dataclass
class Scene:
    name: str
    tris: np.ndarray          # TRI_DTYPE [T]
    spheres: np.ndarray       # SPHERE_DTYPE [S]
    materials: np.ndarray     # MAT_DTYPE [M]
    camera: np.ndarray        # CAM_DTYPE scalar record
    meta: dict = field(default_factory=dict)

    @property
    def n_tris(self) -> int:
        return int(self.tris.shape[0])

    @property
    def n_spheres(self) -> int:
        return int(self.spheres.shape[0])


@dataclass
class RenderConfig:
    index: int
    name: str
    width: int
    height: int
    spp: int
    max_depth: int
    use_nif: bool
    env_rgb: tuple = (1.0, 1.0, 1.0)
    seed: int = 0
    wave_samples: int = 1     # k: samples per wavefront wave (SURVEY.md §8a "Wave")

    @property
    def n_pix(self) -> int:
        return self.width * self.height

    @property
    def paths(self) -> int:
        return self.n_pix * self.spp


# BASELINE.json "configs" (index order), SURVEY.md §8a wave sizes
CONFIGS = [
    RenderConfig(0, "box_nif_tiny", 64, 64, 4, 4, True, wave_samples=4),
    RenderConfig(1, "box_nif", 512, 512, 16, 8, True, wave_samples=16),
    RenderConfig(2, "spheres_nif", 1024, 1024, 64, 12, True, wave_samples=64),
    RenderConfig(3, "small_bvh_nif", 1920, 1080, 32, 8, True, wave_samples=32),
    RenderConfig(4, "large_bvh", 3840, 2160, 64, 8, False, env_rgb=(1.0, 1.0, 1.0), wave_samples=32),
]


def _camera(eye, look_at, up, vfov):
    c = np.zeros((), dtype=CAM_DTYPE)
    c["eye"] = eye
    c["look_at"] = look_at
    c["up"] = up
    c["vfov_deg"] = vfov
    return c


def _materials(rows):
    m = np.zeros(len(rows), dtype=MAT_DTYPE)
    for i, (kind, albedo, emission, ior) in enumerate(rows):
        m[i]["kind"] = kind
        m[i]["albedo"] = albedo
        m[i]["emission"] = emission
        m[i]["ior"] = ior
    return m


def _quad(p0, p1, p2, p3, mat):
    """Two triangles (p0,p1,p2), (p0,p2,p3); geometric normal = (p1-p0) x (p2-p0)."""
    t = np.zeros(2, dtype=TRI_DTYPE)
    t[0]["v0"], t[0]["v1"], t[0]["v2"] = p0, p1, p2
    t[1]["v0"], t[1]["v1"], t[1]["v2"] = p0, p2, p3
    t["material"] = mat
    return t


# ---------------------------------------------------------------------------------------------------
# Config 0/1: Box + NIF (BASELINE.json configs[0..1]; SURVEY.md §8c pins row "0, 1")
# ---------------------------------------------------------------------------------------------------
def box_scene(seed: int = 0) -> Scene:
    """Unit box [-0.5,0.5]^3 missing its z=+0.5 face; 5 Lambertian faces (albedo U[0.2,0.8]^3 each,
    in the order floor, ceiling, back, left, right); emissive quad at y=0.499, x,z in [-0.15,0.15],
    facing -y, E=(5,5,5). Camera eye (0,0,2), look_at 0, up +y, vfov 40 deg."""
    rng = np.random.default_rng([seed, 1])
    alb = rng.uniform(0.2, 0.8, size=(5, 3)).astype(np.float32)
    mats = _materials([(LAMBERT, alb[i], (0, 0, 0), 1.0) for i in range(5)] +
                      [(EMISSIVE, (0, 0, 0), (5.0, 5.0, 5.0), 1.0)])
    h = 0.5
    # windings chosen so the geometric normal points into the box
    floor = _quad((-h, -h, -h), (-h, -h, h), (h, -h, h), (h, -h, -h), 0)        # +y
    ceil = _quad((-h, h, -h), (h, h, -h), (h, h, h), (-h, h, h), 1)             # -y
    back = _quad((-h, -h, -h), (h, -h, -h), (h, h, -h), (-h, h, -h), 2)         # +z
    left = _quad((-h, -h, -h), (-h, h, -h), (-h, h, h), (-h, -h, h), 3)         # +x
    right = _quad((h, -h, -h), (h, -h, h), (h, h, h), (h, h, -h), 4)            # -x
    e, y = 0.15, 0.499
    light = _quad((-e, y, -e), (e, y, -e), (e, y, e), (-e, y, e), 5)           # -y (faces down)
    tris = np.concatenate([floor, ceil, back, left, right, light])
    return Scene("box", tris, np.zeros(0, dtype=SPHERE_DTYPE), mats,
                 _camera((0, 0, 2), (0, 0, 0), (0, 1, 0), 40.0))


# ---------------------------------------------------------------------------------------------------
# Config 2: Spheres + NIF
# ---------------------------------------------------------------------------------------------------
def spheres_scene(seed: int = 0, n_spheres: int = 64) -> Scene:
    """64 spheres r~U[0.05,0.3], c~U[-2,2]^3 by sequential rejection (non-overlapping); material by
    index i mod 4: 0,1 Lambertian U[0.2,0.8]^3, 2 mirror (0.9), 3 dielectric IOR 1.5. Ground quad
    y=-2.3, x,z in [-20,20], albedo 0.5. Camera eye (0,0.5,7) -> (0,-0.5,0), vfov 45."""
    rng = np.random.default_rng([seed, 2])
    cs, rs = [], []
    while len(cs) < n_spheres:
        r = float(rng.uniform(0.05, 0.3))
        c = rng.uniform(-2.0, 2.0, size=3)
        if all(np.linalg.norm(c - c2) >= r + r2 for c2, r2 in zip(cs, rs)):
            cs.append(c)
            rs.append(r)
    rows = []
    sph = np.zeros(n_spheres, dtype=SPHERE_DTYPE)
    for i in range(n_spheres):
        k = i % 4
        if k < 2:
            rows.append((LAMBERT, rng.uniform(0.2, 0.8, size=3), (0, 0, 0), 1.0))
        elif k == 2:
            rows.append((MIRROR, (0.9, 0.9, 0.9), (0, 0, 0), 1.0))
        else:
            rows.append((DIELECTRIC, (1.0, 1.0, 1.0), (0, 0, 0), 1.5))
        sph[i]["center"] = cs[i]
        sph[i]["radius"] = rs[i]
        sph[i]["material"] = i
    rows.append((LAMBERT, (0.5, 0.5, 0.5), (0, 0, 0), 1.0))
    g, y = 20.0, -2.3
    ground = _quad((-g, y, -g), (-g, y, g), (g, y, g), (g, y, -g), n_spheres)   # +y
    return Scene("spheres", ground, sph, _materials(rows),
                 _camera((0, 0.5, 7), (0, -0.5, 0), (0, 1, 0), 45.0))


# ---------------------------------------------------------------------------------------------------
# Geodesic icosphere + fBm displacement (configs 3, 4). SURVEY.md §8c ambiguity #16/#17.
# ---------------------------------------------------------------------------------------------------
def _icosahedron():
    p = (1.0 + math.sqrt(5.0)) / 2.0
    v = np.array([(-1, p, 0), (1, p, 0), (-1, -p, 0), (1, -p, 0),
                  (0, -1, p), (0, 1, p), (0, -1, -p), (0, 1, -p),
                  (p, 0, -1), (p, 0, 1), (-p, 0, -1), (-p, 0, 1)], dtype=np.float64)
    f = np.array([(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
                  (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
                  (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
                  (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)], dtype=np.int64)
    return v / np.linalg.norm(v, axis=1, keepdims=True), f


def geodesic_sphere(freq: int):
    """Frequency-n geodesic subdivision of the icosahedron: 20 n^2 triangles, 10 n^2 + 2 vertices.
    Grid points are keyed canonically (sorted icosahedron-vertex ids with integer weights) so every
    vertex shared by two faces is computed once: the mesh is watertight by construction."""
    V, F = _icosahedron()
    key_to_idx: dict = {}
    pts = []

    def vid(ids, ws):
        key = tuple(sorted((int(i), int(w)) for i, w in zip(ids, ws) if w != 0))
        j = key_to_idx.get(key)
        if j is None:
            s = np.zeros(3)
            for i, w in key:
                s = s + w * V[i]
            s = s / np.linalg.norm(s)
            j = len(pts)
            key_to_idx[key] = j
            pts.append(s)
        return j

    faces = []
    n = freq
    for a, b, c in F:
        grid = {}
        for i in range(n + 1):
            for j in range(n + 1 - i):
                k = n - i - j
                grid[(i, j)] = vid((a, b, c), (k, i, j))
        for i in range(n):
            for j in range(n - i):
                faces.append((grid[(i, j)], grid[(i + 1, j)], grid[(i, j + 1)]))
                if j + 1 <= n - i - 1:
                    faces.append((grid[(i + 1, j)], grid[(i + 1, j + 1)], grid[(i, j + 1)]))
    return np.array(pts, dtype=np.float64), np.array(faces, dtype=np.int64)


def _value_noise_table(rng, size=256):
    perm = rng.permutation(size)
    vals = rng.uniform(-1.0, 1.0, size=size)
    return np.concatenate([perm, perm]), vals


def fbm(p: np.ndarray, rng, octaves=5, lacunarity=2.0, gain=0.5, base_freq=2.0) -> np.ndarray:
    """Seeded 3-D value-noise fBm, range about [-1, 1] (SURVEY.md ambiguity #17)."""
    perm, vals = _value_noise_table(rng)
    out = np.zeros(p.shape[0])
    amp, freq, norm = 1.0, base_freq, 0.0
    for _ in range(octaves):
        q = p * freq
        q0 = np.floor(q)
        f = q - q0
        f = f * f * (3 - 2 * f)
        i0 = q0.astype(np.int64) & 255
        acc = np.zeros(p.shape[0])
        for dx in (0, 1):
            for dy in (0, 1):
                for dz in (0, 1):
                    h = perm[(perm[(perm[(i0[:, 0] + dx) & 255] + ((i0[:, 1] + dy) & 255)) & 511]
                              + ((i0[:, 2] + dz) & 255)) & 511]
                    w = ((f[:, 0] if dx else 1 - f[:, 0]) * (f[:, 1] if dy else 1 - f[:, 1]) *
                         (f[:, 2] if dz else 1 - f[:, 2]))
                    acc += w * vals[h & 255]
        out += amp * acc
        norm += amp
        amp *= gain
        freq *= lacunarity
    return out / norm


def displaced_sphere(freq: int, center, radius: float, amp: float, rng):
    P, F = geodesic_sphere(freq)
    d = fbm(P, rng)
    Q = (P * (radius * (1.0 + amp * d))[:, None] + np.asarray(center, dtype=np.float64)).astype(np.float32)
    return Q, F


def _mesh_tris(Q, F, mats_per_tri):
    t = np.zeros(F.shape[0], dtype=TRI_DTYPE)
    t["v0"] = Q[F[:, 0]]
    t["v1"] = Q[F[:, 1]]
    t["v2"] = Q[F[:, 2]]
    t["material"] = mats_per_tri
    return t


def small_bvh_scene(seed: int = 0, freq: int = 71) -> Scene:
    """Config 3: frequency-71 geodesic icosphere (100,820 tris), R=1 at origin, radial fBm
    displacement amplitude 0.1; per-triangle coin: Lambertian from a 16-entry palette U[0.2,0.8]^3
    or mirror 0.9. Camera eye (0,0,3.2), look_at 0, vfov 40, 16:9."""
    rng = np.random.default_rng([seed, 3])
    Q, F = displaced_sphere(freq, (0, 0, 0), 1.0, 0.1, rng)
    pal = rng.uniform(0.2, 0.8, size=(16, 3))
    rows = [(LAMBERT, pal[i], (0, 0, 0), 1.0) for i in range(16)] + [(MIRROR, (0.9, 0.9, 0.9), (0, 0, 0), 1.0)]
    coin = rng.random(F.shape[0]) < 0.5
    pick = rng.integers(0, 16, size=F.shape[0])
    mat = np.where(coin, 16, pick).astype(np.uint32)
    return Scene("small_bvh", _mesh_tris(Q, F, mat), np.zeros(0, dtype=SPHERE_DTYPE), _materials(rows),
                 _camera((0, 0, 3.2), (0, 0, 0), (0, 1, 0), 40.0))


def large_bvh_scene(seed: int = 0, freq: int = 63, n_objects: int = 64) -> Scene:
    """Config 4: 64 frequency-63 displaced icospheres (79,380 tris each; 5,080,320 total), R~U[0.5,1],
    centres U[0,10]^3 (overlap allowed), per-sphere fBm seed, Lambertian U[0.2,0.8]^3 per sphere.
    Camera eye (5,5,-8) -> (5,5,5), vfov 60."""
    rng = np.random.default_rng([seed, 4])
    P, F = geodesic_sphere(freq)
    parts, rows = [], []
    for i in range(n_objects):
        c = rng.uniform(0.0, 10.0, size=3)
        r = float(rng.uniform(0.5, 1.0))
        sub = np.random.default_rng([seed, 4, i])
        d = fbm(P, sub)
        Q = (P * (r * (1.0 + 0.1 * d))[:, None] + c).astype(np.float32)
        parts.append(_mesh_tris(Q, F, np.full(F.shape[0], i, dtype=np.uint32)))
        rows.append((LAMBERT, rng.uniform(0.2, 0.8, size=3), (0, 0, 0), 1.0))
    return Scene("large_bvh", np.concatenate(parts), np.zeros(0, dtype=SPHERE_DTYPE), _materials(rows),
                 _camera((5, 5, -8), (5, 5, 5), (0, 1, 0), 60.0))


def empty_scene(vfov=40.0) -> Scene:
    return Scene("empty", np.zeros(0, dtype=TRI_DTYPE), np.zeros(0, dtype=SPHERE_DTYPE),
                 _materials([(LAMBERT, (0.5, 0.5, 0.5), (0, 0, 0), 1.0)]),
                 _camera((0, 0, 2), (0, 0, 0), (0, 1, 0), vfov))


def single_sphere_scene(kind=LAMBERT, albedo=(0.5, 0.5, 0.5), ior=1.5, radius=0.5) -> Scene:
    """Furnace-test scene (SURVEY.md §8c pins 'Furnace 2/3'): one sphere at the origin."""
    s = np.zeros(1, dtype=SPHERE_DTYPE)
    s[0]["center"] = (0, 0, 0)
    s[0]["radius"] = radius
    s[0]["material"] = 0
    return Scene("sphere", np.zeros(0, dtype=TRI_DTYPE), s, _materials([(kind, albedo, (0, 0, 0), ior)]),
                 _camera((0, 0, 2), (0, 0, 0), (0, 1, 0), 40.0))


def random_soup(n_tris: int, n_spheres: int, seed: int, extent=1.0) -> Scene:
    """Random triangle/sphere soup for intersection brute-force pins."""
    rng = np.random.default_rng([seed, 9])
    t = np.zeros(n_tris, dtype=TRI_DTYPE)
    c = rng.uniform(-extent, extent, size=(n_tris, 1, 3))
    e = rng.normal(scale=0.25 * extent, size=(n_tris, 3, 3))
    v = (c + e).astype(np.float32)
    t["v0"], t["v1"], t["v2"] = v[:, 0], v[:, 1], v[:, 2]
    t["material"] = 0
    s = np.zeros(n_spheres, dtype=SPHERE_DTYPE)
    s["center"] = rng.uniform(-extent, extent, size=(n_spheres, 3))
    s["radius"] = rng.uniform(0.05, 0.3, size=n_spheres) * extent
    s["material"] = 0
    return Scene("soup", t, s, _materials([(LAMBERT, (0.5, 0.5, 0.5), (0, 0, 0), 1.0)]),
                 _camera((0, 0, 3 * extent), (0, 0, 0), (0, 1, 0), 50.0))


def scene_for_config(index: int, seed: int = 0) -> Scene:
    if index in (0, 1):
        return box_scene(seed)
    if index == 2:
        return spheres_scene(seed)
    if index == 3:
        return small_bvh_scene(seed)
    if index == 4:
        return large_bvh_scene(seed)
    raise ValueError(f"no config {index}")


# ---------------------------------------------------------------------------------------------------
# HDR-NIF weights: SIREN, seeded init, w0 folded before fp16 rounding (SURVEY.md §8c ambiguity #2)
# ---------------------------------------------------------------------------------------------------
def siren_blob(seed: int = 0, out_scale: float = 1.0) -> np.ndarray:
    """fp16 blob of 50,307 halves: for l = 1..5, W_l row-major [out][in] then b_l[out].
    Canonical SIREN init (first layer W ~ U(-1/in, 1/in); others U(+-sqrt(6/in)/w0); biases
    U(+-1/sqrt(in))). Layers 1-4 store W' = fp16(w0 W), b' = fp16(w0 b) so every sine layer is
    sin(W' x + b'); layer 5 stores W_5, b_5 unscaled (times ``out_scale``, a test knob that widens the
    output range; 1.0 is the BASELINE network). The blob *is* the network: both sides evaluate it."""
    rng = np.random.default_rng([seed, 5])
    parts = []
    for li, (fin, fout) in enumerate(NIF_LAYERS):
        if li == 0:
            bound = 1.0 / fin
        else:
            bound = math.sqrt(6.0 / fin) / NIF_W0
        W = rng.uniform(-bound, bound, size=(fout, fin))
        b = rng.uniform(-1.0 / math.sqrt(fin), 1.0 / math.sqrt(fin), size=fout)
        if li < 4:
            W, b = NIF_W0 * W, NIF_W0 * b
        else:
            W, b = out_scale * W, out_scale * b
        parts.append(W.reshape(-1))
        parts.append(b)
    flat = np.concatenate(parts).astype(np.float16)
    assert flat.size == NIF_N_HALVES
    return flat.view(np.uint16).copy()


# The paper's own HDR-NIF (Sec. 3.2; reading R4):
# Fourier features (F = 40: sin and cos of 2 pi B x for 20 frequency rows B, x = (u, v)) -> 4 dense ReLU
# layers of width H = 128, where layer 1 ("the last odd layer before the middle") outputs H - F = 88
# units and is concatenated with the 40 Fourier features -> linear 128 -> 3 (YUV, log space) -> fixed
# YUV -> RGB matrix -> exp. 50,011 trainable parameters (97.7 KiB in fp16, "97 KiB")
# plus the 20 x 2 frequency matrix.
FR_FREQS = 20
FR_FEATURES = 2 * FR_FREQS
FR_LAYERS = [(FR_FEATURES, 128), (128, 128 - FR_FEATURES), (128, 128), (128, 128), (128, 3)]
FR_N_HALVES = 2 * FR_FREQS + sum(o * i + o for i, o in FR_LAYERS)   # 50,051
assert FR_N_HALVES == 50051
# BT.601 YUV -> RGB ("The network's final layer is a static colour-conversion matrix (defaulting to YUV
# to RGB)"): rows R, G, B; columns Y, U, V
YUV_TO_RGB = np.array([[1.0, 0.0, 1.13983],
                       [1.0, -0.39465, -0.58060],
                       [1.0, 2.03211, 0.0]])


def fourier_relu_blob(seed: int = 0, sigma: float = 6.0) -> np.ndarray:
    """fp16 blob of the paper's NIF, 50,051 halves: B[20][2] (frequencies, cycles per unit of u/v),
    then for each of the 5 layers W[out][in], b[out]. Untrained seeded init: B ~ N(0, sigma^2), ReLU
    layers He-uniform, biases U(+-0.05), output layer scaled by 0.1 with b = (0.5, 0, 0) (Y offset)."""
    rng = np.random.default_rng([seed, 7])
    parts = [rng.normal(0.0, sigma, size=(FR_FREQS, 2)).reshape(-1)]
    for li, (fin, fout) in enumerate(FR_LAYERS):
        bound = math.sqrt(6.0 / fin)
        W = rng.uniform(-bound, bound, size=(fout, fin))
        b = rng.uniform(-0.05, 0.05, size=fout)
        if li == len(FR_LAYERS) - 1:
            W = 0.1 * W
            b = np.array([0.5, 0.0, 0.0])
        parts.append(W.reshape(-1))
        parts.append(b)
    flat = np.concatenate(parts).astype(np.float16)
    assert flat.size == FR_N_HALVES
    return flat.view(np.uint16).copy()


# The NIF family of the size sweep (reading R23): hidden
# size H, L dense-ReLU layers; the concat layer c is the largest odd index below L / 2 (0 if none) and
# outputs H - 40 units. (H, L) = (128, 4) is FR_LAYERS.
NIF_SWEEP = [(64, 2), (128, 4), (256, 4), (1024, 8)]


def fr_concat_layer(layers: int) -> int:
    c = 0
    for l in range(1, layers):
        if 2 * l < layers and l % 2 == 1:
            c = l
    return c


def fr_family_layers(hidden: int, layers: int):
    """[(fan_in, fan_out)] of the L dense-ReLU layers and the linear output layer."""
    c = fr_concat_layer(layers)
    dims = []
    for l in range(layers + 1):
        fin = FR_FEATURES if l == 0 else hidden
        fout = 3 if l == layers else (hidden - FR_FEATURES if l == c else hidden)
        dims.append((fin, fout))
    return dims


def fr_family_halves(hidden: int, layers: int) -> int:
    return 2 * FR_FREQS + sum(o * i + o for i, o in fr_family_layers(hidden, layers))


def fourier_relu_family_blob(hidden: int, layers: int, seed: int = 0, sigma: float = 6.0) -> np.ndarray:
    """fp16 blob of a sweep member: B[20][2] then W_l[out][in], b_l[out] for the L + 1 layers; the same
    untrained seeded init as fourier_relu_blob (He-uniform ReLU layers, output scaled by 0.1, b_out =
    (0.5, 0, 0)). (128, 4) reproduces fourier_relu_blob's layer shapes (not its values)."""
    rng = np.random.default_rng([seed, 11, hidden, layers])
    dims = fr_family_layers(hidden, layers)
    parts = [rng.normal(0.0, sigma, size=(FR_FREQS, 2)).reshape(-1)]
    for li, (fin, fout) in enumerate(dims):
        bound = math.sqrt(6.0 / fin)
        W = rng.uniform(-bound, bound, size=(fout, fin))
        b = rng.uniform(-0.05, 0.05, size=fout)
        if li == len(dims) - 1:
            W = 0.1 * W
            b = np.array([0.5, 0.0, 0.0])
        parts.append(W.reshape(-1))
        parts.append(b)
    flat = np.concatenate(parts).astype(np.float16)
    assert flat.size == fr_family_halves(hidden, layers)
    return flat.view(np.uint16).copy()


def fourier_relu_from_blob(blob: np.ndarray):
    """(B [20][2], [(W, b)] x 5) as float64 arrays (exact widening)."""
    h = np.asarray(blob, dtype=np.uint16).view(np.float16).astype(np.float64)
    B = h[:2 * FR_FREQS].reshape(FR_FREQS, 2)
    off = 2 * FR_FREQS
    out = []
    for fin, fout in FR_LAYERS:
        W = h[off:off + fin * fout].reshape(fout, fin)
        off += fin * fout
        b = h[off:off + fout]
        off += fout
        out.append((W, b))
    return B, out


def nif_layers_from_blob(blob: np.ndarray):
    """Split a blob into [(W[out][in], b[out])] as float64 arrays (exact widening)."""
    h = np.asarray(blob, dtype=np.uint16).view(np.float16).astype(np.float64)
    out, off = [], 0
    for fin, fout in NIF_LAYERS:
        W = h[off:off + fin * fout].reshape(fout, fin)
        off += fin * fout
        b = h[off:off + fout]
        off += fout
        out.append((W, b))
    return out


def query_uv(n: int, seed: int = 0) -> np.ndarray:
    """NIF microbenchmark queries: (u, v) ~ U[0,1)^2, float32 [n][2]."""
    rng = np.random.default_rng([seed, 6])
    return rng.random((n, 2), dtype=np.float32)
