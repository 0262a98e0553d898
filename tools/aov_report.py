#!/usr/bin/env python
"""Table-3 analogue: worst-component mean squared error of primary
hit points and geometric normals, GPU (fp32 rays, certified-fp32/fp64 closest hit) vs the fp64 oracle,
per config (sample 0). Hit point = o + t d with the GPU's t; normals of the hit primitive (fp32 on the
GPU side as in the shading kernel, fp64 on the oracle side). Writes JSON to stdout."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2305_20061_b200 import pt, scenes  # noqa: E402


def normals(sc, prim, P, dtype):
    n = np.zeros((len(prim), 3), dtype)
    T = sc.n_tris
    tri = prim < T
    if tri.any():
        t = sc.tris[prim[tri]]
        v0, v1, v2 = (t[k].astype(dtype) for k in ("v0", "v1", "v2"))
        c = np.cross(v1 - v0, v2 - v0)
        n[tri] = c / np.linalg.norm(c, axis=1, keepdims=True)
    sp = ~tri
    if sp.any():
        s = sc.spheres[prim[sp] - T]
        n[sp] = (P[sp] - s["center"].astype(dtype)) / s["radius"].astype(dtype)[:, None]
    return n


rows = {}
for cfg in range(5):
    c = scenes.CONFIGS[cfg]
    sc = scenes.scene_for_config(cfg)
    W, H = c.width, c.height
    step = 1 if cfg < 3 else 16
    pix = np.arange(0, W * H, step, dtype=np.int64)
    prim_g, t_g = pt.trace_primary(pt.Scene(sc), W, H, c.seed, 0)
    prim_g = prim_g.cpu().numpy()[pix]
    t_g = t_g.cpu().numpy()[pix]
    osc = oracle.OracleScene(sc)
    prim_o, t_o, edge = osc.primary(W, H, c.seed, 0, pix)
    d32 = oracle.camera_rays(sc.camera, W, H, c.seed, 0, pix)
    eye = sc.camera["eye"].astype(np.float64)
    both = (prim_g >= 0) & (prim_o >= 0) & (prim_g == prim_o)
    Pg = (eye.astype(np.float32) + t_g[both, None] * d32[both]).astype(np.float32)
    Po = eye + t_o[both, None] * d32[both].astype(np.float64)
    ng = normals(sc, prim_g[both], Pg, np.float32).astype(np.float64)
    no = normals(sc, prim_o[both], Po, np.float64)
    rows[cfg] = {"pixels": int(len(pix)), "hit_id_agreement": float((prim_g == prim_o).mean()),
                 "hit_mse_worst": float(((Pg.astype(np.float64) - Po) ** 2).mean(0).max()),
                 "normal_mse_worst": float(((ng - no) ** 2).mean(0).max()),
                 "max_rel_t_err": float(np.max(np.abs(t_g[both] - t_o[both]) / t_o[both]))}
print(json.dumps(rows, indent=1))
