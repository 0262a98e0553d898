#!/usr/bin/env python
"""Traversal microbenchmark (SURVEY 8d "Trav-u") for a config's scene, CUDA-event timing:
  * coherent: primary rays of a res x res frame (pt_trace_primary);
  * incoherent: the same number of rays with origins uniform in the scene's bounding box and directions
    uniform on the sphere (seeded; pt_trace_rays) -- a stand-in for bounce-1 diffuse rays that is at
    least as incoherent (every ray starts somewhere else and points anywhere).
One JSON line per kind: rays/s, ms, hit fraction."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--res", type=int, default=2048)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
src = scenes.scene_for_config(a.config)
sc = pt.Scene(src)
W = H = a.res
for i in range(3):                       # keep the outputs alive, as the timed loop does (allocator warm-up)
    prim, t = pt.trace_primary(sc, W, H, 0, i)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(a.iters):
    prim, t = pt.trace_primary(sc, W, H, 0, i)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(json.dumps({"config": a.config, "kind": "primary", "rays": W * H, "ms": ms, "rays_per_s": W * H / (ms / 1e3),
                  "hit_frac": float((prim >= 0).float().mean())}))

# incoherent rays
g = torch.Generator(device="cuda").manual_seed(7)
pts = [src.tris["v0"], src.tris["v1"], src.tris["v2"]] if src.n_tris else []
if src.n_spheres:
    pts.append(src.spheres["center"])
allp = torch.from_numpy(__import__("numpy").concatenate(pts).astype("float32"))
lo, hi = allp.min(0).values.cuda(), allp.max(0).values.cuda()
n = W * H
o = lo + (hi - lo) * torch.rand((n, 3), device="cuda", generator=g)
d = torch.nn.functional.normalize(torch.randn((n, 3), device="cuda", generator=g), dim=1)
for _ in range(3):
    prim, t = pt.trace_rays(sc, o, d)
torch.cuda.synchronize()
e0.record()
for i in range(a.iters):
    prim, t = pt.trace_rays(sc, o, d)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(json.dumps({"config": a.config, "kind": "incoherent", "rays": n, "ms": ms, "rays_per_s": n / (ms / 1e3),
                  "hit_frac": float((prim >= 0).float().mean())}))
