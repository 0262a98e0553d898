"""Pins for the oracle's camera (reading R22), equirect map,
scattering (readings R9/R10) and Russian roulette (reading R8)."""
import math

import numpy as np
import pytest

from paper_2305_20061_b200 import scenes


def _frame(cam, W, H):
    e = cam["eye"].astype(np.float64)
    f = cam["look_at"].astype(np.float64) - e
    f /= np.linalg.norm(f)
    r = np.cross(f, cam["up"].astype(np.float64))
    r /= np.linalg.norm(r)
    u = np.cross(r, f)
    t = math.tan(math.radians(float(cam["vfov_deg"])) / 2)
    return f, r, u, t, t * W / H


def test_camera_centre_pixel_is_forward_axis(orc):
    cams = [scenes.box_scene().camera, scenes.spheres_scene().camera,
            scenes._camera((5, 5, -8), (5, 5, 5), (0, 1, 0), 60.0)]       # config-4 camera
    for cam in cams:
        W = H = 65
        d = orc.camera_dir(cam, W, H, 32, 32, 0.5, 0.5)
        f, *_ = _frame(cam, W, H)
        assert np.abs(d - f).max() < 2e-7


@pytest.mark.parametrize("W,H", [(64, 64), (192, 108)])
def test_camera_ray_hits_its_image_plane_point(orc, W, H):
    """d must point at (sx * t * a, sy * t) on the unit-distance image plane (pinhole model)."""
    cam = scenes.box_scene().camera
    f, r, u, t, ta = _frame(cam, W, H)
    rng = np.random.default_rng(0)
    for _ in range(200):
        x, y = rng.integers(0, W), rng.integers(0, H)
        xi = rng.random(2).astype(np.float32)
        d = orc.camera_dir(cam, W, H, x, y, xi[0], xi[1]).astype(np.float64)
        assert abs(np.linalg.norm(d) - 1) < 3e-7
        sx = 2 * (x + float(xi[0])) / W - 1
        sy = 1 - 2 * (y + float(xi[1])) / H
        assert abs(d @ r / (d @ f) - sx * ta) < 2e-6
        assert abs(d @ u / (d @ f) - sy * t) < 2e-6


def test_camera_mirror_symmetry(orc):
    cam = scenes.box_scene().camera
    W, H = 64, 48
    a = orc.camera_dir(cam, W, H, 3, 5, 0.25, 0.125)
    b = orc.camera_dir(cam, W, H, W - 1 - 3, H - 1 - 5, 0.75, 0.875)
    assert abs(a[0] + b[0]) < 2e-7 and abs(a[1] + b[1]) < 2e-7 and abs(a[2] - b[2]) < 2e-7


def test_camera_rays_use_slot0_philox_jitter(orc):
    """camera_rays(seed, sample) == camera_dir with xi = u01(Philox(p, s, 0, 0) lanes 0, 1)."""
    cam = scenes.box_scene().camera
    W, H, seed, s = 32, 16, 0x1234_5678_9ABC, 5
    pix = np.array([0, 17, 511])
    rays = orc.camera_rays(cam, W, H, seed, s, pix)
    for p, d in zip(pix, rays):
        o = orc.philox([[p, s, 0, 0]], [[seed & 0xFFFFFFFF, seed >> 32]])[0]
        xi = orc.u01(o)
        assert np.array_equal(d, orc.camera_dir(cam, W, H, p % W, p // W, xi[0], xi[1]))


def test_equirect_worked_values(orc):
    uv = orc.equirect([[0, 1, 0], [0, 0, -1], [0, -1, 0], [1, 0, 0], [0, 0, 1], [-1, 0, 0]])
    assert tuple(uv[0]) == (0.5, 0.0)      # SPEC.md:441 north pole, u = 0.5 by convention
    assert tuple(uv[1]) == (0.5, 0.5)      # SPEC.md:442 forward axis
    assert tuple(uv[2]) == (0.5, 1.0)
    assert tuple(uv[3]) == (0.75, 0.5)
    assert tuple(uv[4]) == (0.0, 0.5)      # seam: u = 1 wraps to 0
    assert tuple(uv[5]) == (0.25, 0.5)


def test_equirect_round_trip(orc):
    rng = np.random.default_rng(1)
    d = rng.normal(size=(10000, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    uv = orc.equirect(d * rng.uniform(0.5, 2, size=(10000, 1)))       # scale invariant
    assert (uv >= 0).all() and (uv < 1 + 1e-15).all() and (uv[:, 0] < 1).all()
    th, ph = uv[:, 1] * np.pi, 2 * np.pi * (uv[:, 0] - 0.5)
    back = np.stack([np.sin(th) * np.sin(ph), np.cos(th), -np.sin(th) * np.cos(ph)], 1)
    assert np.abs(back - d).max() < 1e-12


def _rand_unit(rng):
    v = rng.normal(size=3)
    return v / np.linalg.norm(v)


def test_lambert_cosine_moments(orc):
    """Cosine-weighted hemisphere: E[cos] = 2/3, E[cos^2] = 1/2, zero mean tangential component."""
    rng = np.random.default_rng(2)
    g = (np.arange(120) + 0.5) / 120
    for trial in range(3):
        n = _rand_unit(rng)
        if trial == 2:
            n = np.array([0.0, -0.0, -1.0])        # ONB branch for n.z = -1 (s = -1)
        d = -n
        t = np.cross(n, _rand_unit(rng))
        t /= np.linalg.norm(t)
        c, c2, tt = [], [], []
        for a in (np.arange(60) + 0.5) / 60:
            for b in g:
                wi, _, side = orc.scatter(scenes.LAMBERT, d, n, [a, b, 0, 0])
                assert side == 1 and abs(np.linalg.norm(wi) - 1) < 1e-14
                c.append(wi @ n)
                tt.append(wi @ t)
        c = np.array(c)
        assert c.min() > 0
        assert abs(c.mean() - 2 / 3) < 2e-3
        assert abs((c * c).mean() - 0.5) < 2e-3
        assert abs(np.mean(tt)) < 2e-3


def test_mirror_reflection(orc):
    d = np.array([1.0, -1.0, 0]) / math.sqrt(2)
    wi, _, side = orc.scatter(scenes.MIRROR, d, [0, 1.0, 0], [0.1, 0.2, 0.3, 0.4])
    assert side == 1 and np.abs(wi - np.array([1.0, 1.0, 0]) / math.sqrt(2)).max() < 1e-15
    # geometric normal facing away from the ray: face-forwarded first, same reflection
    wi2, _, _ = orc.scatter(scenes.MIRROR, d, [0, -1.0, 0], [0.1, 0.2, 0.3, 0.4])
    assert np.abs(wi2 - wi).max() < 1e-15


def test_dielectric_fresnel_snell_tir(orc):
    down = np.array([0, -1.0, 0])
    wi, F, side = orc.scatter(scenes.DIELECTRIC, down, [0, 1.0, 0], [0, 0, 0.039, 0])
    assert abs(F - 0.04) < 1e-15 and side == 1 and np.abs(wi - [0, 1, 0]).max() < 1e-15
    wi, F, side = orc.scatter(scenes.DIELECTRIC, down, [0, 1.0, 0], [0, 0, 0.5, 0])
    assert side == -1 and np.abs(wi - down).max() < 1e-15
    # Snell: entering at 30 deg -> sin(theta_t) = sin(30)/1.5
    th = math.radians(30)
    d = np.array([math.sin(th), -math.cos(th), 0])
    wi, F, side = orc.scatter(scenes.DIELECTRIC, d, [0, 1.0, 0], [0, 0, 0.99, 0])
    assert side == -1 and abs(abs(wi[0]) - 0.5 / 1.5) < 1e-14 and wi[1] < 0
    # exiting (ray inside, d . n_g > 0): Snell the other way, and TIR past the critical angle
    th = math.radians(20)
    d = np.array([math.sin(th), math.cos(th), 0])
    wi, F, side = orc.scatter(scenes.DIELECTRIC, d, [0, 1.0, 0], [0, 0, 0.999, 0])
    assert side == -1 and abs(wi[0] - 1.5 * math.sin(th)) < 1e-14 and wi[1] > 0
    crit = math.asin(1 / 1.5)
    for th, tir in ((crit - 1e-6, False), (crit + 1e-6, True), (math.radians(60), True)):
        d = np.array([math.sin(th), math.cos(th), 0])
        wi, F, side = orc.scatter(scenes.DIELECTRIC, d, [0, 1.0, 0], [0, 0, 0.999999, 0])
        assert (F == 1.0) == tir
        assert (side == 1) == tir


def test_roulette(orc):
    ok, b = orc.roulette([0.01, 0.02, 0.03], 2, 0.999)        # before depth 3: never
    assert ok and list(b) == [0.01, 0.02, 0.03]
    for xi in (0.0, 0.5, 1 - 2 ** -24):                        # p = 1 at throughput (1,1,1)
        ok, b = orc.roulette([1.0, 1.0, 1.0], 3, xi)
        assert ok and list(b) == [1.0, 1.0, 1.0]
    # unbiased: E[beta'] = beta at beta = 0.25, over a uniform xi grid
    xs = (np.arange(100000) + 0.5) / 100000
    acc = np.zeros(3)
    for xi in xs[::7]:
        ok, b = orc.roulette([0.25, 0.125, 0.0625], 5, xi)
        acc += b if ok else 0
    acc /= len(xs[::7])
    assert np.abs(acc - [0.25, 0.125, 0.0625]).max() < 1e-3
