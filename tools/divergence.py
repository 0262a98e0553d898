#!/usr/bin/env python
"""First-divergence classifier (SURVEY 8c precision plan #3; Sec. 4.2: paths may hit
"adjacent (but still valid within machine precision) primitives"). The GPU renders single paths through
its own shade_segment (pt_debug_path_records: per segment the hit primitive, the Fresnel and roulette
decisions, the escape direction); the fp64 oracle traces the same paths (orc_trace_paths: the segment's
ray, hit, edge measure and signed decision deltas). Every path whose segments differ is classified at its
FIRST difference:
  edge      the two hits differ and one of the rays passes within DELTA_EDGE (barycentric / graze units) of
            a primitive boundary: the oracle's own hit is near its edge, or the oracle ray nearly hits the
            GPU's primitive (adjacent primitives, silhouettes);
  tie       both hit, the oracle ray also hits the GPU's primitive, at |dt| <= DELTA_T t (overlapping
            geometry);
  fresnel   same hit, the dielectric's reflect/refract choice differs with |xi2 - F| <= DELTA_XI;
  roulette  same hit, the roulette outcome differs with |xi3 - q| <= DELTA_XI;
  seam      same segments, the escape directions map to (u, v) on opposite sides of the equirect seam;
  unexplained  anything else (a bug).
  python tools/divergence.py [CONFIG] [ROW0 ROWS COL0 COLS]   -> JSON histogram"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

DELTA_EDGE = 1e-3
DELTA_T = 1e-4
DELTA_XI = 1e-4
CLASSES = ("same", "edge", "tie", "fresnel", "roulette", "seam", "unexplained")


def _prim_measure(scene, prim, o, d):
    """fp64 (measure, t) of the ray (o, d) against primitive `prim`: triangles -> min barycentric of the
    ray/plane intersection (>= 0 inside) and its t; spheres -> graze 1 - (d_perp / r)^2 (>= 0 hits) and the
    nearest root's t (nan if it misses)."""
    nt = scene.n_tris
    if prim < nt:
        t3 = scene.tris[prim]
        v0, v1, v2 = (np.asarray(t3[k], np.float64) for k in ("v0", "v1", "v2"))
        e1, e2 = v1 - v0, v2 - v0
        pv = np.cross(d, e2)
        det = e1 @ pv
        if det == 0:
            return -np.inf, np.nan
        tv = o - v0
        b1 = (tv @ pv) / det
        qv = np.cross(tv, e1)
        b2 = (d @ qv) / det
        t = (e2 @ qv) / det
        return min(1 - b1 - b2, b1, b2), t
    sp = scene.spheres[prim - nt]
    c = np.asarray(sp["center"], np.float64)
    r = float(sp["radius"])
    dn = d / np.linalg.norm(d)
    oc = o - c
    b = oc @ dn
    dperp2 = oc @ oc - b * b
    g = 1 - dperp2 / (r * r)
    if g < 0:
        return g, np.nan
    sq = np.sqrt(max(0.0, r * r - dperp2))
    t = (-b - sq) if -b - sq > 0 else (-b + sq)
    return g, t / np.linalg.norm(d)


def _u_of(d):
    d = np.asarray(d, np.float64)
    if d[0] == 0 and d[2] == 0:
        return 0.5
    u = 0.5 + np.arctan2(d[0], -d[2]) / (2 * np.pi)
    return u - 1.0 if u >= 1.0 else u


def classify(scene, g, o):
    """Class of every path (list of str) and the details of the non-"same" ones."""
    n, D = o["prim"].shape
    classes, details = [], []
    for i in range(n):
        cls, det = "same", None
        for j in range(D):
            pg, po = int(g["prim"][i, j]), int(o["prim"][i, j])
            if pg == -2 and po == -2:
                break
            if pg != po:
                ray = o["ray"][i, j]
                oo, dd, to = ray[:3], ray[3:6], ray[6]
                e_o = o["edge"][i, j]
                if pg >= 0:
                    m, tg = _prim_measure(scene, pg, oo, dd)
                else:
                    m, tg = -np.inf, np.nan
                if po == -2 or pg == -2:
                    # one path has ended while the other traced another segment: the previous segment's
                    # termination (roulette) decided differently
                    k = j - 1
                    dl = o["rr_delta"][i, k] if k >= 0 else np.inf
                    cls = "roulette" if np.isfinite(dl) and abs(dl) <= DELTA_XI else "unexplained"
                    det = {"seg": j, "gpu": pg, "oracle": po, "rr_delta": float(dl)}
                elif (po >= 0 and e_o <= DELTA_EDGE) or (pg >= 0 and abs(m) <= DELTA_EDGE) or \
                        (po < 0 and pg >= 0 and m >= -DELTA_EDGE):
                    cls = "edge"
                elif po >= 0 and pg >= 0 and m > 0 and np.isfinite(tg) and abs(tg - to) <= DELTA_T * to:
                    cls = "tie"
                else:
                    cls = "unexplained"
                if det is None:
                    det = {"seg": j, "gpu": pg, "oracle": po, "oracle_edge": float(e_o), "gpu_prim_measure": float(m),
                           "t_oracle": float(to), "t_gpu_prim": float(tg) if np.isfinite(tg) else None}
                break
            if pg < 0:      # both escaped: the equirect u of both directions
                if o["uv"][i, 0] >= 0 and abs(_u_of(g["esc_dir"][i]) - o["uv"][i, 0]) > 0.5:
                    cls, det = "seam", {"seg": j, "u_gpu": _u_of(g["esc_dir"][i]), "u_oracle": float(o["uv"][i, 0])}
                break
            fl = int(g["flags"][i, j])
            fd, rd = o["fres_delta"][i, j], o["rr_delta"][i, j]
            if np.isfinite(fd) and bool(fl & 1) != (fd < 0):
                cls = "fresnel" if abs(fd) <= DELTA_XI else "unexplained"
                det = {"seg": j, "fres_delta": float(fd)}
                break
            if np.isfinite(rd) and bool(fl & 2) != (rd >= 0):
                cls = "roulette" if abs(rd) <= DELTA_XI else "unexplained"
                det = {"seg": j, "rr_delta": float(rd)}
                break
        classes.append(cls)
        if cls != "same":
            details.append({"path": i, "class": cls, **(det or {})})
    return classes, details


def run(cfg_index=3, row0=496, rows=16, col0=896, cols=128, seed=0):
    import oracle
    from paper_2305_20061_b200 import pt, scenes
    c = scenes.CONFIGS[cfg_index]
    sc = scenes.scene_for_config(cfg_index)
    blob = scenes.siren_blob(0) if c.use_nif else None
    pix = ((np.arange(row0, row0 + rows)[:, None] * c.width) + np.arange(col0, col0 + cols)[None, :]).reshape(-1)
    S = pt.Scene(sc)
    g = pt.debug_path_records(S, c.width, c.height, c.max_depth, seed, pix, 0, c.spp, use_nif=c.use_nif,
                              env_rgb=None if c.use_nif else c.env_rgb)
    o = oracle.OracleScene(sc).trace_paths(c.width, c.height, c.max_depth, seed, pix, 0, c.spp, nif_blob=blob,
                                           env_rgb=c.env_rgb)
    classes, details = classify(sc, g, o)
    hist = {k: int(sum(1 for x in classes if x == k)) for k in CLASSES}
    return {"config": cfg_index, "crop": [row0, rows, col0, cols], "paths": len(classes), "segments_oracle":
            int(o["len"].sum()), "histogram": hist, "examples": details[:20],
            "thresholds": {"edge": DELTA_EDGE, "t": DELTA_T, "xi": DELTA_XI}}, g, o


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    res, _, _ = run(*a) if a else run()
    print(json.dumps(res, indent=1))
