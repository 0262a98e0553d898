"""Pins for the oracle's path loop (PAPER.md:78 no light sampling; 134 env on escape; 150 RR from
depth 3; readings R7 depth cap, R10 spawn offset). Closed forms: white/albedo furnaces, dielectric
furnace, one-sided emitter. Full images beyond these are Monte Carlo: parity unpinned."""
import numpy as np

from paper_2305_20061_b200 import scenes


def test_furnace_empty_scene_exact(orc):
    """empty scene, constant env c -> every pixel exactly c."""
    sc = orc.OracleScene(scenes.empty_scene())
    c = (0.3, 0.7, 1.9)
    out, st = sc.render(16, 8, 5, seed=3, s0=0, s1=4, env_rgb=c)
    assert np.array_equal(out / 4, np.broadcast_to(c, out.shape))
    assert st["escaped"] == 16 * 8 * 4 and st["segments"] == 16 * 8 * 4


def test_furnace_convex_lambert_sphere(orc):
    """One convex Lambertian sphere, constant env 1: each sample is exactly rho (hit, one outward
    bounce, escape) or 1 (miss); RR never fires before depth 3."""
    rho = (0.25, 0.5, 0.75)
    for kind, expect in ((scenes.LAMBERT, rho), (scenes.MIRROR, rho)):
        sc = orc.OracleScene(scenes.single_sphere_scene(kind=kind, albedo=rho))
        W = H = 24
        for p in range(0, W * H, 37):
            for s in range(3):
                L, prims = sc.trace_one(W, H, 4, 7, p, s)
                if prims[0] < 0:
                    assert list(L) == [1.0, 1.0, 1.0] and len(prims) == 1
                else:
                    assert list(L) == list(expect) and len(prims) == 2 and prims[1] == -1
        out, st = sc.render(W, H, 4, seed=7, s0=0, s1=8)
        k = (out[:, 0] - 8) / (rho[0] - 1)          # number of sphere hits per pixel
        assert np.allclose(k, np.round(k), atol=1e-9)
        for ch in range(3):
            assert np.allclose(out[:, ch], k * rho[ch] + (8 - k), atol=1e-12)
        assert ((k > 0) & (k < 8)).any() and (k == 8).any() and (k == 0).any()


def test_furnace_dielectric_sphere(orc):
    """Dielectric (tint 1) under constant env 1: throughput is never scaled and RR keeps q = 1, so
    every sample is exactly 1 (escaped) or 0 (capped at max_depth)."""
    sc = orc.OracleScene(scenes.single_sphere_scene(kind=scenes.DIELECTRIC))
    W = H = 32
    for md in (3, 12):
        out, st = sc.render(W, H, md, seed=1, s0=0, s1=4)
        assert np.allclose(out, np.round(out), atol=0) and (out[:, 0] == out[:, 1]).all()
        capped = 4 * W * H - out[:, 0].sum()
        assert capped == st["capped"] and st["rr_killed"] == 0
        if md == 3:
            assert capped > 0


def test_emitter_one_sided(orc):
    box = scenes.box_scene()
    sc = orc.OracleScene(box)
    W = H = 64
    found = 0
    for p in range(W * H):
        L, prims = sc.trace_one(W, H, 4, 0, p, 0)
        if prims[0] in (10, 11):                # the emissive ceiling quad, seen from below
            assert list(L) == [5.0, 5.0, 5.0] and len(prims) == 1
            found += 1
    assert found > 20
    # same quad seen from its back: terminates with no contribution
    q = box.tris[10:12].copy()
    q["v0"][:, 1] = q["v1"][:, 1] = q["v2"][:, 1] = -0.2
    q["material"] = 0
    mats = scenes._materials([(scenes.EMISSIVE, (0, 0, 0), (5, 5, 5), 1.0)])
    cam = scenes._camera((0, 1, 0.01), (0, 0, 0), (0, 0, -1), 40.0)     # above, looking down at +y back
    sc2 = orc.OracleScene(scenes.Scene("q", q, np.zeros(0, dtype=scenes.SPHERE_DTYPE), mats, cam))
    L, prims = sc2.trace_one(8, 8, 4, 0, 4 * 8 + 4, 0, env_rgb=(2, 2, 2))
    assert prims[0] in (0, 1) and list(L) == [0.0, 0.0, 0.0]


def test_depth_cap_and_thread_invariance(orc):
    sc = orc.OracleScene(scenes.box_scene())
    blob = scenes.siren_blob(0)
    W = H = 32
    a, sta = sc.render(W, H, 4, 0, s0=0, s1=2, nif_blob=blob, nthreads=1)
    b, stb = sc.render(W, H, 4, 0, s0=0, s1=2, nif_blob=blob, nthreads=5)
    assert np.array_equal(a, b) and sta == stb
    # max_depth 1: only direct env or emitter; every path is 1 segment
    c, stc = sc.render(W, H, 1, 0, s0=0, s1=2, nif_blob=blob)
    assert stc["segments"] == W * H * 2
    assert stc["escaped"] + stc["emitted"] + stc["capped"] == W * H * 2
    # sample ranges add up: [0,1) + [1,2) == [0,2)
    d0, _ = sc.render(W, H, 4, 0, s0=0, s1=1, nif_blob=blob)
    d1, _ = sc.render(W, H, 4, 0, s0=1, s1=2, nif_blob=blob)
    assert np.allclose(d0 + d1, a, rtol=1e-15, atol=0)


def test_divergence_classifier_on_synthetic_records(orc):
    """tools/divergence.classify against hand-made differences of an oracle record set (no GPU): identical
    records -> "same"; a roulette flip inside the xi band -> "roulette", outside -> "unexplained"; a
    different primitive far from every edge -> "unexplained"; a near-edge hit -> "edge"."""
    import os
    import sys
    import numpy as np
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import divergence
    from paper_2305_20061_b200 import scenes
    c = scenes.CONFIGS[0]
    sc = scenes.scene_for_config(0)
    pix = np.arange(64 * 20, 64 * 20 + 64)
    o = orc.OracleScene(sc).trace_paths(c.width, c.height, 8, 0, pix, 0, 4, nif_blob=scenes.siren_blob(0))
    # GPU-like records equal to the oracle's decisions
    flags = np.where(np.isfinite(o["fres_delta"]) & (o["fres_delta"] < 0), 1, 0) | \
        np.where(np.isfinite(o["rr_delta"]) & (o["rr_delta"] >= 0), 2, 0)
    dirs = o["ray"][np.arange(len(o["len"])), o["len"] - 1, 3:6]
    g = {"prim": o["prim"].copy(), "flags": flags, "esc_dir": dirs, "L": o["L"]}
    cls, _ = divergence.classify(sc, g, o)
    assert set(cls) == {"same"}
    # a roulette decision flipped: inside / outside the band
    i, j = next((i, j) for i in range(len(cls)) for j in range(8) if np.isfinite(o["rr_delta"][i, j]))
    g2 = {k: v.copy() for k, v in g.items()}
    g2["flags"][i, j] ^= 2
    o2 = {k: v.copy() for k, v in o.items()}
    o2["rr_delta"][i, j] = 5e-5 if o["rr_delta"][i, j] >= 0 else -5e-5
    assert divergence.classify(sc, g2, o2)[0][i] == "roulette"
    o2["rr_delta"][i, j] = 0.3 if o["rr_delta"][i, j] >= 0 else -0.3
    assert divergence.classify(sc, g2, o2)[0][i] == "unexplained"
    # a different triangle on a first-segment hit far from any edge -> unexplained; near the edge -> edge
    i = next(i for i in range(len(cls)) if o["prim"][i, 0] >= 0 and o["edge"][i, 0] > 0.05)
    g3 = {k: v.copy() for k, v in g.items()}
    g3["prim"][i, 0] = (o["prim"][i, 0] + 6) % sc.n_tris
    assert divergence.classify(sc, g3, o)[0][i] == "unexplained"
    o3 = {k: v.copy() for k, v in o.items()}
    o3["edge"][i, 0] = 1e-5
    assert divergence.classify(sc, g3, o3)[0][i] == "edge"
