#!/usr/bin/env python
"""NIF size sweep (Fig. nrf-vs-blender: H64 L2 311.8 M, H256 L4 149.1 M,
H1024 L8 9.3 M paths/s on one GC200 with the Spheres scene).

For each member of the paper's NIF family (pt_nif_load_family: the fused streamed-weight kernel for
H <= 256, the layered tcgen05 GEMM path for H1024; fp16 and fp8 each), the fused
paper NIF (H128 L4, PT_NIF_FOURIER_RELU) and the SIREN of the hot path:
  * inference microbenchmark: N uniform (u, v) queries, CUDA events, inferences/s and dense tensor
    TFLOP/s (2 x sum of fan_in x fan_out over the layers) against the measured bf16 peak;
  * render: config 2 (Spheres, 1024^2, depth 12) at --spp samples per pixel, samples/s and NIF share.
Prints one JSON line per network."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--spp", type=int, default=8)
ap.add_argument("--render", type=int, default=1)
a = ap.parse_args()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))


def flops_of(dims):
    return 2 * sum(i * o for i, o in dims)


nets = [("siren", pt.Nif(scenes.siren_blob(0)), 3 * 2 * 128 * 128 + 2 * (2 * 128 + 128 * 3)),
        ("paper_fused_H128L4", pt.Nif(scenes.fourier_relu_blob(0), kind=pt.NIF_FOURIER_RELU),
         flops_of(scenes.FR_LAYERS))]
for fp8 in (False, True):
    for H, L in scenes.NIF_SWEEP:
        path = "fused" if H <= 256 else "layered"      # mlp_kernel.cu use_fused()
        nets.append((f"paper_family_{path}_H{H}L{L}" + ("_fp8" if fp8 else ""),
                     pt.Nif(scenes.fourier_relu_family_blob(H, L, seed=1), kind=pt.NIF_FR_FAMILY, hidden=H, layers=L,
                            fp8=fp8),
                     flops_of(scenes.fr_family_layers(H, L))))

c = scenes.CONFIGS[2]
S = pt.Scene(scenes.scene_for_config(2)) if a.render else None
for name, nif, flop in nets:
    n = a.n if "H1024" not in name else a.n // 4
    uv = torch.from_numpy(scenes.query_uv(n, 3)).cuda()
    out = torch.empty((n, 3), device="cuda")
    for _ in range(2):
        pt.nif_infer(nif, uv, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        pt.nif_infer(nif, uv, out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    rate = n / (ms / 1e3)
    tf = rate * flop / 1e12
    # the peak of the arithmetic type: fp8 dense = 2 x the measured bf16 peak (the guide's nominal ratio)
    pk = 2.0 if name.endswith("_fp8") else 1.0
    res = {"net": name, "queries": n, "ms": ms, "inferences_per_s": rate, "flop_per_inference": flop,
           "tflops": tf, "frac_burst": tf / (pk * peaks["bf16_tflops"]),
           "frac_sustained": tf / (pk * peaks["bf16_tflops_sustained"])}
    if a.render:
        acc = torch.zeros(c.width * c.height * 3, device="cuda")
        pt.render_samples(S, nif, c.width, c.height, 0, a.spp, c.max_depth, 0, acc, wave_samples=a.spp)
        S.set_profiling(True)
        torch.cuda.synchronize()
        e0.record()
        pt.render_samples(S, nif, c.width, c.height, 0, a.spp, c.max_depth, 0, acc, wave_samples=a.spp)
        e1.record()
        torch.cuda.synchronize()
        st = S.stats()
        S.set_profiling(False)
        rms = e0.elapsed_time(e1)
        res["render"] = {"config": "configs[2] spheres 1024x1024 depth 12", "spp": a.spp,
                         "samples_per_s": c.width * c.height * a.spp / (rms / 1e3), "ms": rms,
                         "nif_ms": st["t_nif_ms"], "trace_ms": st["t_traverse_ms"], "escaped": st["escaped"]}
    print(json.dumps(res), flush=True)
