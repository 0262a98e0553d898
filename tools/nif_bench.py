#!/usr/bin/env python
"""NIF microbenchmark (SURVEY 8d "NIF-u"): the fused kernel on 2^24 uniform (u,v) queries, timed with
CUDA events on the launching stream; reports inferences/s and the tensor fraction of the measured peak.
Optional --check compares 4096 outputs with the fp64 oracle."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 24)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--check", action="store_true")
ap.add_argument("--tag", default="")
ap.add_argument("--kind", type=int, default=0, help="0 SIREN, 1 the paper's Fourier/ReLU NIF")
a = ap.parse_args()
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
blob = scenes.siren_blob(0) if a.kind == 0 else scenes.fourier_relu_blob(0)
nif = pt.Nif(blob, kind=a.kind)
uv = torch.from_numpy(scenes.query_uv(a.n, 3)).cuda()
out = torch.empty((a.n, 3), device="cuda")
for _ in range(3):
    pt.nif_infer(nif, uv, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    pt.nif_infer(nif, uv, out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
rate = a.n / (ms / 1e3)
# dense flops per inference: SIREN 3 hidden 128x128 layers; paper NIF 40x128 + 128x88 + 2 x 128x128
# (both 98,304; the tiny input/output layers are not counted)
tf = rate * 98304 / 1e12
res = {"tag": a.tag, "kind": a.kind, "n": a.n, "ms": ms, "inferences_per_s": rate, "tflops_hidden": tf,
       "frac_burst": tf / peaks["bf16_tflops"], "frac_sustained": tf / peaks["bf16_tflops_sustained"],
       "note": "includes the tiny query-pack kernel of pt_nif_infer"}
if a.check:
    import oracle
    k = 4096
    q = scenes.query_uv(a.n, 3)[:k].astype(np.float64)
    y = oracle.nif_eval(blob, q) if a.kind == 0 else oracle.fr_eval(blob, q)
    got = out[:k].cpu().numpy().astype(np.float64)
    res["max_abs_dy"] = float(np.abs(np.log(got) - y).max())
    res["max_rel"] = float((np.abs(got - np.exp(y)) / np.exp(y)).max())
print(json.dumps(res))
