"""Pins for the oracle's closest-hit (PAPER.md:97 watertight triangle test, PAPER.md:101 BVH;
DESIGN.md readings R11 tie-break (t, id), R12 t > 0 strictly / smaller positive sphere root).

The BVH is pinned to the brute-force definition (bit-exact); the fp64 tests are pinned to closed-form
values on axis-aligned cases and to watertightness on a closed mesh."""
import numpy as np
import pytest

from paper_2305_20061_b200 import scenes


def _rays(rng, n, extent):
    o = rng.uniform(-2 * extent, 2 * extent, size=(n, 3))
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    # a quarter of the rays aimed at the soup centre so most of them hit something
    aim = rng.uniform(-0.5 * extent, 0.5 * extent, size=(n // 4, 3)) - o[: n // 4]
    d[: n // 4] = aim / np.linalg.norm(aim, axis=1, keepdims=True)
    # axis-aligned directions exercise the zero-direction slab branch
    d[n // 4: n // 4 + 64] = np.eye(3)[rng.integers(0, 3, 64)] * rng.choice([-1, 1], (64, 1))
    return o, d


@pytest.mark.parametrize("seed,n_tris,n_sph", [(0, 200, 0), (1, 50, 20), (2, 1000, 40), (3, 0, 64)])
def test_bvh_equals_brute_force(orc, seed, n_tris, n_sph):
    sc = scenes.random_soup(n_tris, n_sph, seed)
    o_sc = orc.OracleScene(sc)
    rng = np.random.default_rng(seed)
    o, d = _rays(rng, 10000, 1.0)
    a = o_sc.closest_hit(o, d, brute=False)
    b = o_sc.closest_hit(o, d, brute=True)
    assert (a[0] >= 0).mean() > 0.2
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1])
    assert np.array_equal(a[2], b[2])


def _tri_scene(tris):
    t = np.zeros(len(tris), dtype=scenes.TRI_DTYPE)
    for i, (v0, v1, v2) in enumerate(tris):
        t[i]["v0"], t[i]["v1"], t[i]["v2"] = v0, v1, v2
    return scenes.Scene("t", t, np.zeros(0, dtype=scenes.SPHERE_DTYPE), scenes.empty_scene().materials,
                        scenes.empty_scene().camera)


def test_triangle_closed_form(orc):
    sc = orc.OracleScene(_tri_scene([((0, 0, 0), (1, 0, 0), (0, 1, 0))]))
    prim, t, bary, edge = sc.closest_hit([[0.25, 0.25, 2.0]], [[0, 0, -1.0]])
    assert prim[0] == 0 and t[0] == 2.0
    assert list(bary[0]) == [0.5, 0.25, 0.25]        # weights of (v0, v1, v2)
    assert edge[0] == 0.25
    # from below, facing the other side: still a hit (two-sided test), same t
    prim, t, bary, _ = sc.closest_hit([[0.25, 0.25, -3.0]], [[0, 0, 1.0]])
    assert prim[0] == 0 and t[0] == 3.0
    # centroid of a larger triangle, oblique ray: barycentrics 1/3 each
    sc2 = orc.OracleScene(_tri_scene([((0, 0, 0), (3, 0, 0), (0, 3, 0))]))
    o = np.array([[1.0, 1.0, 0.0]]) + np.array([[0.3, -0.2, 1.0]]) * 4
    prim, t, bary, _ = sc2.closest_hit(o, -np.array([[0.3, -0.2, 1.0]]))
    assert prim[0] == 0 and abs(t[0] - 4.0) < 1e-14
    assert np.allclose(bary[0], 1 / 3, atol=1e-15, rtol=0)
    # misses: outside an edge, behind the origin (t < 0), origin on the triangle (t = 0)
    assert sc.closest_hit([[0.75, 0.75, 1.0]], [[0, 0, -1.0]])[0][0] == -1
    assert sc.closest_hit([[0.25, 0.25, 1.0]], [[0, 0, 1.0]])[0][0] == -1
    assert sc.closest_hit([[0.25, 0.25, 0.0]], [[0, 0, -1.0]])[0][0] == -1


def test_tie_break_smallest_id(orc):
    v = ((0, 0, 0), (1, 0, 0), (0, 1, 0))
    sc = orc.OracleScene(_tri_scene([v, v, v]))
    for brute in (False, True):
        prim, t, _, _ = sc.closest_hit([[0.2, 0.2, 1.0]], [[0, 0, -1.0]], brute=brute)
        assert prim[0] == 0 and t[0] == 1.0


def test_sphere_closed_form(orc):
    s = np.zeros(1, dtype=scenes.SPHERE_DTYPE)
    s[0]["center"] = (0, 0, -5)
    s[0]["radius"] = 1.0
    sc = scenes.Scene("s", np.zeros(0, dtype=scenes.TRI_DTYPE), s, scenes.empty_scene().materials,
                      scenes.empty_scene().camera)
    o_sc = orc.OracleScene(sc)
    prim, t, _, edge = o_sc.closest_hit([[0, 0, 0.0], [0, 0, -5.0], [0, 0, 0.0], [0, 2, 0.0]],
                                        [[0, 0, -1.0], [1, 0, 0.0], [0, 0, 1.0], [0, 0, -1.0]])
    assert prim[0] == 0 and t[0] == 4.0 and edge[0] == 1.0     # head-on: graze measure 1
    assert prim[1] == 0 and t[1] == 1.0                         # from the centre: far root
    assert prim[2] == -1                                        # sphere behind the ray
    assert prim[3] == -1                                        # passes above
    # non-unit direction: t scales inversely
    prim, t, _, _ = o_sc.closest_hit([[0, 0, 0.0]], [[0, 0, -2.0]])
    assert t[0] == 2.0


def test_watertight_closed_mesh(orc):
    """Rays from inside a closed geodesic sphere never escape, including rays aimed exactly at
    shared vertices and edge midpoints (the cases a non-watertight test can miss)."""
    P, F = scenes.geodesic_sphere(4)
    Q = P.astype(np.float32)
    t = np.zeros(F.shape[0], dtype=scenes.TRI_DTYPE)
    t["v0"], t["v1"], t["v2"] = Q[F[:, 0]], Q[F[:, 1]], Q[F[:, 2]]
    sc = scenes.Scene("g", t, np.zeros(0, dtype=scenes.SPHERE_DTYPE), scenes.empty_scene().materials,
                      scenes.empty_scene().camera)
    o_sc = orc.OracleScene(sc)
    mids = 0.5 * (Q[F[:, 0]].astype(np.float64) + Q[F[:, 1]])
    rng = np.random.default_rng(0)
    targets = np.concatenate([Q.astype(np.float64), mids, rng.normal(size=(5000, 3))])
    for origin in ([0, 0, 0], [0.1, -0.2, 0.05]):
        o = np.broadcast_to(np.array(origin, dtype=np.float64), targets.shape)
        d = targets - o
        prim, t, _, _ = o_sc.closest_hit(o, d)
        assert (prim >= 0).all()


def test_empty_scene_misses(orc):
    o_sc = orc.OracleScene(scenes.empty_scene())
    prim, t, _, _ = o_sc.closest_hit([[0, 0, 0.0]], [[0, 0, 1.0]])
    assert prim[0] == -1 and np.isinf(t[0])


@pytest.mark.parametrize("freq,n_rays", [(17, None), (71, 1500)])
def test_bvh_equals_brute_at_shared_vertices_and_edges(orc, freq, n_rays):
    """The oracle's BVH returns exactly the brute-force (t, id) minimum (reading R11) also where hits tie:
    rays from inside a closed geodesic mesh at its shared vertices (3-6 triangles at one t), edge midpoints
    and centroids, from three origins. (A cull of boxes entered strictly beyond the best t without a
    rounding margin returned a larger id on ~1 % of these rays.)"""
    P, F = scenes.geodesic_sphere(freq)
    Q = P.astype(np.float32)
    t = np.zeros(F.shape[0], dtype=scenes.TRI_DTYPE)
    t["v0"], t["v1"], t["v2"] = Q[F[:, 0]], Q[F[:, 1]], Q[F[:, 2]]
    sc = scenes.Scene("g", t, np.zeros(0, dtype=scenes.SPHERE_DTYPE), scenes.empty_scene().materials,
                      scenes.empty_scene().camera)
    o_sc = orc.OracleScene(sc)
    e = np.unique(np.sort(np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]]), 1), axis=0)
    Q64 = Q.astype(np.float64)
    tg = np.concatenate([Q, (0.5 * (Q64[e[:, 0]] + Q64[e[:, 1]])).astype(np.float32),
                         Q64[F].mean(1).astype(np.float32)])
    if n_rays is not None:
        tg = tg[np.linspace(0, len(tg) - 1, n_rays).astype(np.int64)]
    for origin in ([0, 0, 0], [0.1, -0.2, 0.05], [0.37, 0.41, -0.29]):
        o = np.broadcast_to(np.asarray(origin, np.float32), tg.shape).astype(np.float64)
        d = (tg - o.astype(np.float32)).astype(np.float32).astype(np.float64)
        pb, tb, _, _ = o_sc.closest_hit(o, d, brute=False)
        pf, tf, _, _ = o_sc.closest_hit(o, d, brute=True)
        assert np.array_equal(pb, pf) and np.array_equal(tb, tf)
        assert (pf >= 0).all()


@pytest.mark.parametrize("cfg", [0, 2])
def test_primary_aov_invariants(orc, cfg):
    """oracle.primary_aov (the Table-3 AOVs) against identities it does not compute
    with: a triangle hit point equals the barycentric combination of the vertices, (1 - b1 - b2) v0 +
    b1 v1 + b2 v2, its normal is unit and orthogonal to both edges; a sphere hit point lies on the sphere
    and its normal is the unit radial direction; prim and t equal oracle.primary."""
    c = scenes.CONFIGS[cfg]
    sc = scenes.scene_for_config(cfg)
    o_sc = orc.OracleScene(sc)
    W, H = 64, 48
    pix = np.arange(W * H, dtype=np.int64)
    prim, t, pos, nrm, b2 = o_sc.primary_aov(W, H, 3, 1, pix)
    p2, t2, _ = o_sc.primary(W, H, 3, 1, pix)
    assert np.array_equal(prim, p2) and np.array_equal(t, t2)
    nt = sc.n_tris
    tri = (prim >= 0) & (prim < nt)
    sph = prim >= nt
    assert tri.sum() > 100 and (cfg != 2 or sph.sum() > 100)
    v0 = sc.tris["v0"][prim[tri]].astype(np.float64)
    v1 = sc.tris["v1"][prim[tri]].astype(np.float64)
    v2 = sc.tris["v2"][prim[tri]].astype(np.float64)
    b1, bb2 = b2[tri, 0], b2[tri, 1]
    comb = (1 - b1 - bb2)[:, None] * v0 + b1[:, None] * v1 + bb2[:, None] * v2
    scale = 1 + np.abs(pos[tri]).max(1)
    assert (np.abs(comb - pos[tri]).max(1) <= 1e-12 * scale).all()
    assert np.allclose(np.linalg.norm(nrm[tri], axis=1), 1, atol=1e-14)
    assert np.abs((nrm[tri] * (v1 - v0)).sum(1)).max() <= 1e-13
    assert np.abs((nrm[tri] * (v2 - v0)).sum(1)).max() <= 1e-13
    if sph.any():
        s = sc.spheres[prim[sph] - nt]
        cen = s["center"].astype(np.float64)
        r = s["radius"].astype(np.float64)
        # (the quadratic's cancellation at |oc| ~ 7 >> r leaves ~1e-12 relative in t)
        assert np.allclose(np.linalg.norm(pos[sph] - cen, axis=1), r, rtol=1e-9, atol=0)
        assert np.allclose(nrm[sph], (pos[sph] - cen) / r[:, None], rtol=0, atol=1e-14)
        assert np.allclose(np.linalg.norm(nrm[sph], axis=1), 1, atol=1e-9)
    miss = prim < 0
    assert (pos[miss] == 0).all() and (nrm[miss] == 0).all()
