#!/usr/bin/env python
"""Warp-exit timeline of one config-1 wave (tail-analysis build, -DPT_TAIL_TRACE): when the warps of
first_bounce_kernel and path_kernel finish, relative to the first exit of each kernel; shows how long each
kernel's tail (SMs partly idle) lasts. Also event times of the NIF kernel for the same wave."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PT_B200_LIB", os.path.join(ROOT, "build/variants/libpt_tail.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

c = scenes.CONFIGS[1]
S = pt.Scene(scenes.scene_for_config(1))
N = pt.Nif(scenes.siren_blob(0))
acc = torch.zeros(c.width * c.height * 3, device="cuda")
for _ in range(3):
    pt.render_samples(S, N, c.width, c.height, 0, c.spp, c.max_depth, 0, acc, wave_samples=c.wave_samples)
torch.cuda.synchronize()
buf = np.zeros(2 * (1 << 14), np.uint64)
pt.lib().pt_debug_tail(C.c_void_p(buf.ctypes.data))
tr = buf.reshape(2, -1).astype(np.int64)
for k, name in enumerate(["first_bounce_kernel", "path_kernel"]):
    t = np.sort(tr[k][tr[k] > 0])
    t = (t - t[0]) / 1e3
    q = np.quantile(t, [0.1, 0.5, 0.9, 0.99, 1.0])
    print(f"{name}: {len(t)} warps; exit after first exit (us): p10 {q[0]:.1f} p50 {q[1]:.1f} p90 {q[2]:.1f} "
          f"p99 {q[3]:.1f} max {q[4]:.1f}")
fb_last, pk_first = tr[0][tr[0] > 0].max(), tr[1][tr[1] > 0].min()
print(f"path_kernel first warp exit - first_bounce last exit: {(pk_first - fb_last) / 1e3:.1f} us")
