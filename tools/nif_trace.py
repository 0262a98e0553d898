#!/usr/bin/env python
"""Run the trace build of the SIREN NIF kernel (PT_NIF_TRACE) and print the per-step timeline of CTA 0:
MMA wait/issue stamps and epilogue wake/done stamps (cycles); 4 MMA stages per tile (stage 0 = the previous
tile's output layer + layer 1), NS slots (env PT_TRACE_SLOTS, default 3 = PT_NIF_SLOTS)."""
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
NS = int(os.environ.get("PT_TRACE_SLOTS", "3"))
nif = pt.Nif(scenes.siren_blob(0))
uv = torch.from_numpy(scenes.query_uv(n, 3)).cuda()
for _ in range(3):
    pt.nif_infer(nif, uv)
torch.cuda.synchronize()
buf = np.zeros(17 * 4096 * 4, np.uint64)
pt.lib().pt_debug_nif_trace(C.c_void_p(buf.ctypes.data))
ALL = buf.reshape(17, 4096, 4).astype(np.int64)
nrec = int((ALL[0, :, 1] > 0).sum())
# record r (= layer group r) is run by epilogue team r % 2 (warps e = 8 t .. 8 t + 7, roles 1 + e)
TEAM = np.arange(4096) % 2
first = np.stack([ALL[1 + 8 * TEAM[r], r] for r in range(4096)])      # [rec][4]
last = np.stack([ALL[8 + 8 * TEAM[r], r] for r in range(4096)])
tr = np.stack([ALL[0], first, last])
t0 = tr[0, 0, 3]
print("rec stage slot | issuer: start in_ready d_free issued | team's first warp: commit released stored handed | last warp")
for r in range(min(nrec, 48)):
    layer, s = (r // NS) % 4, r % NS
    row = [tr[0, r, k] - t0 for k in (3, 2, 0, 1)] + [tr[w, r, k] - t0 for w in (1, 2) for k in (0, 2, 1, 3)]
    print(f"{r:4d} {layer:3d} {s:3d} | " + " ".join(f"{v:7d}" for v in row[:4]) + " | " +
          " ".join(f"{v:7d}" for v in row[4:8]) + " | " + " ".join(f"{v:7d}" for v in row[8:]))
a, b = 12, nrec - 1
R = slice(a, b)
m = lambda x: float(np.mean(x))
print("steady state (records %d..%d)" % (a, b))
print("  cycles per group: %.0f  per tile: %.0f" % (m(np.diff(tr[0, R, 1])), (tr[0, b, 1] - tr[0, a, 1]) / ((b - a) / 4)))
print("  issuer: wait input %.0f, wait D %.0f, issue %.0f" % (m(tr[0, R, 2] - tr[0, R, 3]), m(tr[0, R, 0] - tr[0, R, 2]),
                                                             m(tr[0, R, 1] - tr[0, R, 0])))
for w, nm in ((1, "first"), (2, "last")):
    print("  epilogue %s warp: commit seen %.0f after issue, load %.0f, sine+store %.0f, hand-over %.0f, idle before its next %.0f"
          % (nm, m(tr[w, R, 0] - tr[0, R, 1]), m(tr[w, R, 2] - tr[w, R, 0]), m(tr[w, R, 1] - tr[w, R, 2]),
             m(tr[w, R, 3] - tr[w, R, 1]), m(tr[w, a + 2:b + 2, 0] - tr[w, R, 3])))
rr = np.arange(a, b)
H = np.stack([ALL[1 + 8 * TEAM[r]:9 + 8 * TEAM[r], r, 3] for r in rr], 1)    # [8][recs]
Rl = np.stack([ALL[1 + 8 * TEAM[r]:9 + 8 * TEAM[r], r, 2] for r in rr], 1)
C = np.stack([ALL[1 + 8 * TEAM[r]:9 + 8 * TEAM[r], r, 0] for r in rr], 1)
B = np.stack([ALL[1 + 8 * TEAM[r]:9 + 8 * TEAM[r], r, 1] for r in rr], 1) - C
hand = H.max(0)
rel = Rl.max(0)
ok = rr - NS >= a
print("  slot input ready seen by the issuer %.0f after the team's last hand-over (same slot, previous layer)"
      % m(tr[0, rr[ok], 2] - hand[(rr - NS - a)[ok]]))
ok2 = rr - 2 >= a
print("  D free seen by the issuer %.0f after the team's last release (group - 2)" % m(tr[0, rr[ok2], 0] - rel[(rr - 2 - a)[ok2]]))
print("  within a team (warp k = 4 h + lane-quarter order): commit-seen lag / hand-over lag / busy (commit seen -> stored)")
for k in range(8):
    print("   warp %d: %6.0f %6.0f %6.0f" % (k, m(C[k] - C.min(0)), m(H[k] - H.min(0)), m(B[k])))
