#!/usr/bin/env python
"""Host BVH build and pt_scene_create times per config and builder thread count (PT_BVH_THREADS), one
JSON line per (config, threads): build = pt_debug_build_bvh (host only), create = pt_scene_create (build +
upload; needs the GPU)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = r'''
import json, os, sys, time
sys.path.insert(0, {root!r})
from paper_2305_20061_b200 import pt, scenes
cfg = int(sys.argv[1])
sc = scenes.scene_for_config(cfg)
st = pt.debug_build_bvh(sc)
b = []
for _ in range(3):
    t = time.perf_counter(); pt.debug_build_bvh(sc); b.append(1e3 * (time.perf_counter() - t))
c = []
try:
    import torch
    if torch.cuda.is_available():
        for _ in range(3):
            t = time.perf_counter(); S = pt.Scene(sc); torch.cuda.synchronize(); c.append(1e3 * (time.perf_counter() - t)); S.close()
except Exception as e:
    c = [str(e)]
print(json.dumps({{"config": cfg, "threads": os.environ.get("PT_BVH_THREADS", "auto"), "cores": os.cpu_count(),
                  "build_ms": min(b), "create_ms": min(c) if c and not isinstance(c[0], str) else c, **st}}))
'''.format(root=ROOT)

for cfg in (3, 4):
    for th in (["1", "4", ""] if "--sweep" in sys.argv else [""]):
        env = dict(os.environ)
        if th:
            env["PT_BVH_THREADS"] = th
        p = subprocess.run([sys.executable, "-c", CODE, str(cfg)], env=env, capture_output=True, text=True)
        print(p.stdout.strip() or p.stderr[-500:], flush=True)
        phases = [l for l in p.stderr.splitlines() if l.startswith("bvh ")]
        if phases:   # PT_BVH_TIMING=1: the builder's phase times of the last build
            print("   " + " | ".join(x[4:].strip() for x in phases[-6:]), flush=True)
