#!/usr/bin/env python
"""One family member's inference, for ncu: python tools/family_one.py H L [n] [fp8]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

H, L = int(sys.argv[1]), int(sys.argv[2])
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << 22
fp8 = len(sys.argv) > 4 and sys.argv[4] == "fp8"
nif = pt.Nif(scenes.fourier_relu_family_blob(H, L, seed=1), kind=pt.NIF_FR_FAMILY, hidden=H, layers=L, fp8=fp8)
uv = torch.from_numpy(scenes.query_uv(n, 3)).cuda()
out = torch.empty((n, 3), device="cuda")
for _ in range(3):
    pt.nif_infer(nif, uv, out)
torch.cuda.synchronize()
print("ok", H, L, n)
