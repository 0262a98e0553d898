#!/usr/bin/env python
"""Summarise ncu output for profiles/: a launch list (gpu__time_duration per kernel, share of the
step) and key counters of `--set full` captures (tensor/XU/FP64 pipes, issue, occupancy, DRAM)."""
from __future__ import annotations

import collections
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "sm__cycles_elapsed.avg",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
]


def launch_list(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, mi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) <= mi:
            continue
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[mi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    out = io.StringIO()
    out.write(f"{'kernel':58s} {'launches':>8s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}\n")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"{k[:58]:58s} {n:8d} {t / 1e3:10.1f} {t / 1e3 / n:9.2f} {t / tot:6.3f}\n")
    out.write(f"{'TOTAL':58s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.1f}\n")
    return out.getvalue()


def rep_summary(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    out = io.StringIO()
    for row in rows[2:]:
        d = dict(zip(h, row))
        out.write(f"== {d.get('Kernel Name', '?')[:90]}  (id {d.get('ID', '?')})\n")
        for k in KEYS:
            if k in d and d[k] != "":
                out.write(f"  {k:90s} {d[k]}\n")
    return out.getvalue()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"### {p}")
        print(launch_list(p) if p.endswith(".csv") else rep_summary(p))
