#!/usr/bin/env python
"""Top source lines of an ncu report by warp-instructions executed and stall samples.

  python tools/ncu_lines.py REPORT [TOP] [KERNEL_INDEX]

Reads `ncu -i REPORT --launch-skip KERNEL_INDEX --launch-count 1 --page source --print-source cuda,sass`
(every source file of that kernel; the per-line rows carry the line's aggregate metrics)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
which = int(sys.argv[3]) if len(sys.argv) > 3 else 0
raw = subprocess.run(["ncu", "-i", rep, "--launch-skip", str(which), "--launch-count", "1", "--page", "source",
                      "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
hdr, fname, recs = None, "?", []
for r in csv.reader(io.StringIO(raw)):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        d = dict(zip(hdr, r))
        try:
            recs.append((f"{fname}:{r[0]}", r[1][:80], int(d["Instructions Executed"] or 0),
                         int(d["Warp Stall Sampling (All Samples)"] or 0),
                         int(d["Thread Instructions Executed"] or 0)))
        except (ValueError, KeyError):
            pass
ti = sum(x[2] for x in recs) or 1
ts = sum(x[3] for x in recs) or 1
print(f"total warp-inst {ti}  thread-inst/warp-inst {sum(x[4] for x in recs) / ti:.1f}  stall samples {ts}")
for ln, src, ins, st, thr in sorted(recs, key=lambda x: -x[2])[:top]:
    print(f"{ln:22s} inst {ins / ti:6.1%} stall {st / ts:6.1%} thr/inst {thr / max(1, ins):5.1f} | {src}")
