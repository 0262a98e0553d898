#!/usr/bin/env python
"""spp sweep (the paper's Fig. roofline: ray I/O is hidden above 256 spp
on the IPU). On B200 the per-frame fixed costs are kernel launches, the shrinking tail bounces and the
accumulate pass; this measures samples/s of config 1's scene (512 x 512, depth 8, SIREN NIF) as spp grows
(waves of up to 16 samples; from 32 spp also waves of 32 samples = 8.4 M paths), one JSON line per
(spp, wave size)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

c = scenes.CONFIGS[1]
S = pt.Scene(scenes.scene_for_config(1))
N = pt.Nif(scenes.siren_blob(0))
acc = torch.zeros(c.width * c.height * 3, device="cuda")
for spp, kmax in [(s_, 16) for s_ in (1, 2, 4, 8, 16, 32, 64, 128, 256)] + [(s_, 32) for s_ in (32, 64, 128, 256)]:
    k = min(spp, kmax)
    reps = max(2, 64 // spp)
    for _ in range(2):
        pt.render_samples(S, N, c.width, c.height, 0, spp, c.max_depth, 0, acc, wave_samples=k)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        pt.render_samples(S, N, c.width, c.height, 0, spp, c.max_depth, 0, acc, wave_samples=k)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"spp": spp, "wave_samples": k, "ms_per_frame": ms,
                      "samples_per_s": c.width * c.height * spp / (ms / 1e3)}), flush=True)
