#!/usr/bin/env python
"""DRAM traffic per launch of the hot-path kernels from an ncu metrics capture of one bench step:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \\
      --clock-control none \\
      -k regex:"first_bounce|path_kernel|siren|accumulate" --csv --log-file X.csv python bench.py --steps 1 --warmup 0 ...
  python tools/ncu_traffic.py X.csv > profiles/round1/ncu_traffic_c1.json

The bench's warm-up and timed step both appear; per-kernel averages are over every captured launch."""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, ni, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
per = collections.defaultdict(lambda: collections.defaultdict(list))
idi = h.index("ID")
launch = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("pt::", "").split("<")[0].strip()
    u = r[ui]
    f = scale.get(u)
    if f is None:     # counts with an SI prefix ("Ksector", "Minst", ...)
        f = {"K": 1e3, "M": 1e6, "G": 1e9}.get(u[:1], 1) if len(u) > 1 and u[1:2].islower() else 1
    v = float(r[vi].replace(",", "")) * f
    launch.setdefault((name, r[idi]), {})[r[ni]] = v
for (name, _), m in launch.items():
    per[name]["bytes"].append(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0))
    per[name]["ns"].append(m.get("gpu__time_duration.sum", 0))
    per[name]["inst"].append(m.get("smsp__inst_executed.sum", 0))
    per[name]["tinst"].append(m.get("smsp__thread_inst_executed.sum", 0))
    per[name]["lld"].append(m.get("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", 0))
    per[name]["lst"].append(m.get("l1tex__t_sectors_pipe_lsu_mem_local_op_st.sum", 0))
out = {}
for name, d in per.items():
    n = len(d["bytes"])
    out[name] = {"launches": n, "dram_bytes_per_launch": sum(d["bytes"]) / n,
                 "dram_bytes_total": sum(d["bytes"]), "ns_per_launch": sum(d["ns"]) / n,
                 "warp_inst_per_launch": sum(d["inst"]) / n,
                 "thread_inst_per_launch": sum(d["tinst"]) / n,
                 "simt_efficiency": (sum(d["tinst"]) / (32.0 * sum(d["inst"]))) if sum(d["inst"]) else None,
                 "local_ld_sectors_per_launch": sum(d["lld"]) / n, "local_st_sectors_per_launch": sum(d["lst"]) / n}
if len(sys.argv) > 2:     # kernel-sources hash of the capture (bench.py flags stale captures)
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
    import bench
    out["sources_sha16"] = bench.sources_sha16(bench.TRACE_SOURCES if sys.argv[2] == "trace" else bench.NIF_SOURCES)
    out["trace_sources_sha16"] = bench.sources_sha16(bench.TRACE_SOURCES)
    out["nif_sources_sha16"] = bench.sources_sha16(bench.NIF_SOURCES)
print(json.dumps(out, indent=1))
