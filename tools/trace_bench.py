#!/usr/bin/env python
"""Traversal microbenchmark (SURVEY 8d "Trav-u"): closest hits of primary rays (pt_trace_primary) and
of the bounce-1 diffuse rays of a render, for a config's scene; CUDA-event timing."""
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
sc = pt.Scene(scenes.scene_for_config(a.config))
W = H = a.res
for _ in range(2):
    pt.trace_primary(sc, W, H, 0, 0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(a.iters):
    prim, t = pt.trace_primary(sc, W, H, 0, i)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(json.dumps({"config": a.config, "rays": W * H, "ms": ms, "rays_per_s": W * H / (ms / 1e3),
                  "hit_frac": float((prim >= 0).float().mean())}))
