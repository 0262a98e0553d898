#!/usr/bin/env python
"""Run the trace build of the SIREN NIF kernel (PT_NIF_TRACE) and print the per-step timeline of CTA 0:
MMA wait/issue stamps and epilogue wake/done stamps (cycles); 4 MMA stages per tile (stage 0 = the previous
tile's output layer + layer 1), 2 slots."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("PT_B200_LIB", os.path.join(ROOT, "build/variants/libpt_trace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

n = 148 * 128 * 40
nif = pt.Nif(scenes.siren_blob(0))
uv = torch.from_numpy(scenes.query_uv(n, 3)).cuda()
for _ in range(3):
    pt.nif_infer(nif, uv)
torch.cuda.synchronize()
buf = np.zeros(3 * 4096 * 2, np.uint64)
pt.lib().pt_debug_nif_trace(C.c_void_p(buf.ctypes.data))
tr = buf.reshape(3, 4096, 2).astype(np.int64)
nrec = int((tr[0, :, 1] > 0).sum())
t0 = tr[0, 0, 0]
print("rec  stage slot | mma_wait_done  mma_issued | epiA_wake epiA_done | epiB_wake epiB_done")
for r in range(min(nrec, 60)):
    layer, s = (r // 2) % 4, r % 2
    row = [tr[0, r, 0] - t0, tr[0, r, 1] - t0, tr[1, r, 0] - t0, tr[1, r, 1] - t0, tr[2, r, 0] - t0, tr[2, r, 1] - t0]
    print(f"{r:4d} {layer:5d} {s:4d} | " + " ".join(f"{v:10d}" for v in row))
# per step averages over the steady state
d = np.diff(tr[0, 10:nrec, 0])
print("mean cycles between MMA issues:", d.mean(), " per tile:", (tr[0, nrec - 1, 0] - tr[0, 10, 0]) / ((nrec - 11) / 4))
ep = tr[1, 10:nrec, 1] - tr[1, 10:nrec, 0]
print("epilogue A busy per step:", ep.mean(), " wake latency after MMA issue:", (tr[1, 10:nrec, 0] - tr[0, 10:nrec, 1]).mean())
