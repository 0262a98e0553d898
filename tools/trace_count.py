#!/usr/bin/env python
"""Counting build (PT_COUNT): node visits and primitive tests per traced segment for the render
workloads of configs 1-4 and the primary rays of configs 1-3, i.e. the algorithmic traversal bytes of SURVEY 8d:
bytes/segment = visits * 64 B + prim tests * 48 B + 40 B state in + ~40 B state out."""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
lib = os.path.join(ROOT, "build/variants/libpt_count.so")
if not os.path.exists(lib):
    from paper_2305_20061_b200 import _build
    _build.build(out=lib, defines=["PT_COUNT"])
os.environ["PT_B200_LIB"] = lib
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2305_20061_b200 import pt, scenes  # noqa: E402

L = pt.lib()
L.pt_debug_trav_counts.argtypes = [C.c_void_p, C.c_int]


def counts(reset=True):
    h = np.zeros(8, np.uint64)
    torch.cuda.synchronize()
    L.pt_debug_trav_counts(C.c_void_p(h.ctypes.data), int(reset))
    return {"node_visits": int(h[0]), "prim_tests": int(h[2]), "fp64_tests": int(h[3]), "rays": int(h[4])}


out = {}
for cfg in (1, 2, 3):
    c = scenes.CONFIGS[cfg]
    S = pt.Scene(scenes.scene_for_config(cfg))
    counts()
    pt.trace_primary(S, c.width, c.height, 0, 0)
    k = counts()
    k["per_ray"] = {"visits": k["node_visits"] / k["rays"], "prims": k["prim_tests"] / k["rays"],
                    "fp64": k["fp64_tests"] / k["rays"]}
    out[f"primary_c{cfg}"] = k
# render workloads (all bounces): config 1 in full, configs 2-4 at min(spp, 4) samples per pixel (the
# per-segment averages do not depend on the sample count)
for cfg in (1, 2, 3, 4):
    c = scenes.CONFIGS[cfg]
    S = pt.Scene(scenes.scene_for_config(cfg))
    N = pt.Nif(scenes.siren_blob(0)) if c.use_nif else None
    spp = c.spp if cfg == 1 else min(c.spp, 4)
    acc = torch.zeros(c.width * c.height * 3, device="cuda")
    counts()
    pt.render_samples(S, N, c.width, c.height, 0, spp, c.max_depth, 0, acc, env_rgb=None if c.use_nif else c.env_rgb,
                      wave_samples=min(c.wave_samples, spp))
    st = S.stats()
    k = counts()
    # the public statistics of the counting build carry the same counters (pt_get_stats)
    assert (st["node_visits"], st["prim_tests"], st["fp64_rechecks"]) == (k["node_visits"], k["prim_tests"],
                                                                          k["fp64_tests"]), (st, k)
    k["spp"] = spp
    k["per_segment"] = {"visits": k["node_visits"] / k["rays"], "prims": k["prim_tests"] / k["rays"],
                        "fp64": k["fp64_tests"] / k["rays"]}
    k["alg_bytes_per_segment"] = 64 * k["per_segment"]["visits"] + 48 * k["per_segment"]["prims"] + 80
    out[f"render_c{cfg}"] = k
    del S, N
import bench  # noqa: E402  (sources hash: bench.py flags a capture taken with other kernel sources)
out["sources_sha16"] = bench.sources_sha16(bench.TRACE_SOURCES)
print(json.dumps(out, indent=1))
