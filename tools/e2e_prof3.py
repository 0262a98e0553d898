#!/usr/bin/env python
"""Where the end-to-end step time goes on configs[3] (the bench's e2e loop, pipelined input creation):
per step, host wall time of waiting for the next inputs, pt_render (kernels + scale + D2H into pinned
memory), and the handle closes; plus the device-only render time of the same call for comparison."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

cfg = scenes.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
src = scenes.scene_for_config(cfg.index)
blob = scenes.siren_blob(0)
W, H = cfg.width, cfg.height
host = torch.empty(W * H * 3, dtype=torch.float32, pin_memory=True)
hnp = host.numpy()


def make():
    torch.cuda.set_device(0)
    return pt.Scene(src), pt.Nif(blob)


rows = []
with ThreadPoolExecutor(max_workers=1) as ex:
    fut = ex.submit(make)
    for it in range(12):
        t0 = time.perf_counter()
        S, N = fut.result()
        t1 = time.perf_counter()
        fut = ex.submit(make)
        pt.render(S, N, W, H, cfg.spp, cfg.max_depth, cfg.seed, out=hnp)
        t2 = time.perf_counter()
        S.close()
        N.close()
        t3 = time.perf_counter()
        rows.append((1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t3 - t0)))
    fut.result()
r = np.array(rows[2:])
print("median ms: wait inputs %.2f  pt_render %.2f  close %.2f  step %.2f" % tuple(np.median(r, 0)))
# device-only: the same render into a device accumulator, CUDA events
S, N = make()
acc = torch.zeros(W * H * 3, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for it in range(6):
    acc.zero_()
    torch.cuda.synchronize()
    e0.record()
    pt.render_samples(S, N, W, H, 0, cfg.spp, cfg.max_depth, cfg.seed, acc, wave_samples=cfg.wave_samples)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
print("device render (events, no L2 flush) median %.2f ms" % np.median(ms[1:]))
t0 = time.perf_counter()
for _ in range(5):
    host.copy_(acc)
torch.cuda.synchronize()
print("D2H of the %d-byte frame into pinned memory: %.3f ms" % (acc.numel() * 4, 1e3 * (time.perf_counter() - t0) / 5))
