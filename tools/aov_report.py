#!/usr/bin/env python
"""Table-3 analogue: worst-component mean squared error of primary hit
points and geometric normals, the render kernels' own values (pt_trace_primary_aov: P = o + t d and the
shading's normal code, fp32) against the fp64 oracle (orc_primary_aov), per config, sample 0. Pixels:
configs 0-2 full frames, config 3 every 8th row, config 4 every 16th pixel. Writes JSON to stdout.
(tests/test_gpu_aov.py gates the same quantities.)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2305_20061_b200 import pt, scenes  # noqa: E402


def aov_pixels(cfg):
    c = scenes.CONFIGS[cfg]
    if cfg < 3:
        return np.arange(c.n_pix, dtype=np.int64)
    if cfg == 3:
        rows = np.arange(0, c.height, 8)
        return (rows[:, None] * c.width + np.arange(c.width)[None, :]).reshape(-1).astype(np.int64)
    return np.arange(0, c.n_pix, 16, dtype=np.int64)


def aov_compare(cfg, sc=None):
    """(row dict, arrays) of the GPU-vs-oracle AOV comparison of one config."""
    c = scenes.CONFIGS[cfg]
    sc = sc if sc is not None else scenes.scene_for_config(cfg)
    W, H = c.width, c.height
    pix = aov_pixels(cfg)
    S = pt.Scene(sc)
    prim_g, t_g, pos_g, nrm_g, b_g = (x.cpu().numpy() for x in pt.trace_primary_aov(S, W, H, c.seed, 0))
    S.close()
    prim_g, t_g, pos_g, nrm_g, b_g = prim_g[pix], t_g[pix], pos_g[pix], nrm_g[pix], b_g[pix]
    osc = oracle.OracleScene(sc)
    prim_o, t_o, pos_o, nrm_o, b_o = osc.primary_aov(W, H, c.seed, 0, pix)
    _, _, edge = osc.primary(W, H, c.seed, 0, pix)
    eq = prim_g == prim_o
    both = eq & (prim_o >= 0)
    tri = both & (prim_o < sc.n_tris)
    dP = pos_g[both].astype(np.float64) - pos_o[both]
    dn = nrm_g[both].astype(np.float64) - nrm_o[both]
    db = b_g[tri].astype(np.float64) - b_o[tri]
    row = {"pixels": int(len(pix)), "hits": int(both.sum()), "hit_id_agreement": float(eq.mean()),
           "mismatches": int((~eq).sum()), "mismatch_max_edge": float(edge[~eq].max()) if (~eq).any() else None,
           "hit_mse_worst": float((dP ** 2).mean(0).max()) if both.any() else 0.0,
           "normal_mse_worst": float((dn ** 2).mean(0).max()) if both.any() else 0.0,
           "hit_max_abs": float(np.abs(dP).max()) if both.any() else 0.0,
           "normal_max_abs": float(np.abs(dn).max()) if both.any() else 0.0,
           "bary_max_abs": float(np.abs(db).max()) if tri.any() else 0.0,
           "bary_median_abs": float(np.median(np.abs(db))) if tri.any() else 0.0,
           "max_rel_t_err": float(np.max(np.abs(t_g[both] - t_o[both]) / t_o[both])) if both.any() else 0.0}
    arrays = {"eye": np.asarray(sc.camera["eye"], np.float64).reshape(3), "t": t_o[both], "dP": dP, "dn": dn,
              "db": db}
    return row, arrays


if __name__ == "__main__":
    rows = {}
    for cfg in range(5):
        rows[cfg] = aov_compare(cfg)[0]
        print(cfg, rows[cfg], file=sys.stderr, flush=True)
    print(json.dumps(rows, indent=1))
