#!/usr/bin/env python
"""Benchmark of the B200 neural path tracer hot path (BASELINE.json metric: samples/sec and NIF
inferences/sec; % tensor roofline for the NIF kernel).

One step = one full frame of BASELINE.json configs[1] ("Box+NIF": 512x512, 16 spp per GPU, max_depth 8,
RR from depth 3, SIREN HDR-NIF) through the whole wavefront hot path -- raygen, traverse, shade
(scatter + RR + compaction), fused tcgen05 NIF, accumulate -- plus, for N > 1, the NCCL framebuffer
reduce to rank 0. Inputs (scene BVH, NIF weights) are resident in HBM when the timed region starts.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl ours|reference]

Launch for N > 1: python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N.
--impl reference times the fp64 CPU oracle (the reference arm of this tier) on rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2305_20061_b200 import scenes  # noqa: E402

HIDDEN_FLOP_PER_INF = 3 * 2 * 128 * 128          # tensor-counted FLOPs per NIF inference
TOTAL_FLOP_PER_INF = 2 * (2 * 128 + 3 * 128 * 128 + 128 * 3)
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
L2_READ_GBS = 16409.6                       # tools/l2_bench.cu on this pool's B200 (profiles/round1/l2_bench.json)
PROFILES = os.path.join(ROOT, "profiles", "round1")


def trace_bytes_per_segment(cfg_index: int):
    """Algorithmic traversal bytes per traced segment of a config's render (counting build of the same
    kernel, tools/trace_count.py: 64 B x node visits + 48 B x primitive tests + 80 B path state)."""
    try:
        with open(os.path.join(PROFILES, "trace_count.json")) as f:
            return float(json.load(f)[f"render_c{cfg_index}"]["alg_bytes_per_segment"])
    except Exception:
        return None


def ncu_inst(kernels, cfg_index: int):
    """Warp instructions issued per wave by the named kernels (same ncu capture as ncu_traffic), or None."""
    try:
        with open(os.path.join(PROFILES, f"ncu_traffic_c{cfg_index}.json")) as f:
            d = json.load(f)
        v = float(sum(d[k]["warp_inst_per_launch"] for k in kernels))
        return v if v > 0 else None
    except Exception:
        return None


def ncu_traffic(kernels, cfg_index: int):
    """DRAM bytes (read + write) per wave of the named kernels (each launched once per wave) from the
    committed ncu capture of one bench step (tools/ncu_traffic.py), or None."""
    try:
        with open(os.path.join(PROFILES, f"ncu_traffic_c{cfg_index}.json")) as f:
            d = json.load(f)
        return float(sum(d[k]["dram_bytes_per_launch"] for k in kernels))
    except Exception:
        return None


ClockSampler_last = {}


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "bf16_tflops": float(p["bf16_tflops"]),
                "bf16_tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.lines: list[str] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def oracle_sample(cfg, rows_every: int):
    rows = np.arange(0, cfg.height, rows_every)
    pix = (rows[:, None] * cfg.width + np.arange(cfg.width)[None, :]).reshape(-1).astype(np.int64)
    return pix, f"rows 0::{rows_every} ({len(rows)} of {cfg.height}) x {cfg.width} px x {cfg.spp} spp"


def run_oracle(cfg, steps: int, warmup: int, rows_every: int):
    """Time the fp64 CPU oracle (as it stands) on a bounded sample of the workload."""
    import oracle
    sc = oracle.OracleScene(scenes.scene_for_config(cfg.index))
    blob = scenes.siren_blob(0) if cfg.use_nif else None
    pix, desc = oracle_sample(cfg, rows_every)
    cores = os.cpu_count() or 1
    for _ in range(warmup):
        sc.render(cfg.width, cfg.height, cfg.max_depth, cfg.seed, pix=pix, s0=0, s1=cfg.spp, nif_blob=blob,
                  env_rgb=cfg.env_rgb, nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(steps):
        sc.render(cfg.width, cfg.height, cfg.max_depth, cfg.seed, pix=pix, s0=0, s1=cfg.spp, nif_blob=blob,
                  env_rgb=cfg.env_rgb, nthreads=cores)
    dt = time.perf_counter() - t0
    samples = len(pix) * cfg.spp * steps
    return {"value": samples / dt, "unit": "samples/s", "cores": cores, "kind": "oracle",
            "sample": desc, "seconds": dt, "cpu": _cpu_model()}


def _cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_config(cfg, world):
    return {"workload": f"configs[{cfg.index}] {cfg.name}: {cfg.width}x{cfg.height}, {cfg.spp} spp per GPU, "
                        f"max_depth {cfg.max_depth}, RR>=3, {'SIREN HDR-NIF' if cfg.use_nif else 'constant env'}",
            "width": cfg.width, "height": cfg.height, "spp_per_gpu": cfg.spp, "max_depth": cfg.max_depth,
            "wave_samples": cfg.wave_samples, "frame_spp_total": cfg.spp * world, "seed": cfg.seed,
            "parallelism": f"sample-partitioned x{world} + NCCL framebuffer reduce" if world > 1 else "1 GPU",
            "l2": "L2 flushed (512 MiB memset) between timed steps, untimed; wave state 0.55 GB > L2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--oracle-rows-every", type=int, default=8)
    ap.add_argument("--wave-samples", type=int, default=0, help="samples per wave (default: the config's)")
    args = ap.parse_args()
    cfg = scenes.CONFIGS[args.config]
    if args.wave_samples > 0:
        import dataclasses
        cfg = dataclasses.replace(cfg, wave_samples=args.wave_samples)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_oracle(cfg, args.steps, args.warmup, rows_every=64)
        line = {"metric": "samples/sec", "value": r["value"], "unit": "samples/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * r["seconds"] / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "impl": "reference", "config": workload_config(cfg, 1),
                "cpu_baseline": {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": r["value"], "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        line["config"]["reference_sample"] = r["sample"]
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist

    from paper_2305_20061_b200 import _build, pt
    from paper_2305_20061_b200.dist import render_partitioned

    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    if rank == 0:
        _build.build()
    if world > 1:
        dist.barrier()
    pt.lib()

    W, H, spp, depth = cfg.width, cfg.height, cfg.spp, cfg.max_depth
    env = None if cfg.use_nif else cfg.env_rgb
    src = scenes.scene_for_config(cfg.index)
    blob = scenes.siren_blob(0) if cfg.use_nif else None
    S = pt.Scene(src)
    N = pt.Nif(blob) if cfg.use_nif else None
    accum = torch.zeros(W * H * 3, dtype=torch.float32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    n_total = spp * world                       # weak scaling: spp samples per GPU, disjoint index blocks
    stream = torch.cuda.current_stream()

    def block(f, c, acc):
        pt.render_samples(S, N, W, H, f, c, depth, cfg.seed, acc, env_rgb=env, wave_samples=cfg.wave_samples,
                          stream=stream)

    def step():
        accum.zero_()
        render_partitioned(block, n_total, accum, rank, world)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, per-step CUDA events on the launching stream, L2 flush untimed ----
    S.set_profiling(True)
    kt = {"raygen": 0.0, "traverse": 0.0, "shade": 0.0, "nif": 0.0, "accum": 0.0}
    escaped = segments = paths = launches = nif_launches = trav_launches = 0
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
            st = S.stats()
            for key in kt:
                kt[key] += st[f"t_{key}_ms"]
            escaped += st["escaped"]
            segments += st["segments"]
            paths += st["paths"]
            launches += st["launches"]
            nif_launches += st["nif_launches"]
            trav_launches += st["traverse_launches"]
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall = time.perf_counter() - t_wall0
    step_ms = sorted(a.elapsed_time(b) for a, b in evs)
    ms = sum(step_ms)
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    S.set_profiling(False)

    samples_per_step = W * H * spp * world
    value = samples_per_step * args.steps / (ms_max / 1e3)

    # ---- end-to-end through the public API: host arrays in, host framebuffer out ----
    e2e_steps = max(3, min(2 * args.steps, 100))      # host-side timing: more steps than the device loop
    e2e_warmup = max(1, min(args.warmup, 5))
    host_fb = torch.empty(W * H * 3, dtype=torch.float32, pin_memory=True)
    host_np = host_fb.numpy()
    auto_k = max(1, min(spp, (8 << 20) // (W * H)))       # pt_render's wave size (pt_api.cu)
    host_render = world == 1 and auto_k == cfg.wave_samples
    h2d = src.tris.nbytes + src.spheres.nbytes + src.materials.nbytes + src.camera.nbytes + (blob.nbytes if blob is not None else 0)
    te0 = None
    for it in range(e2e_warmup + e2e_steps):
        if it == e2e_warmup:            # untimed warm-up iterations first (allocator, first-launch setup)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            te0 = time.perf_counter()
        S2 = pt.Scene(src)
        N2 = pt.Nif(blob) if cfg.use_nif else None
        if host_render:
            # one GPU: pt_render, the C-ABI's host-buffer call (device accumulator, scale, read-back into
            # the caller's pinned buffer); its automatic wave size equals the config's here
            pt.render(S2, N2, W, H, spp, depth, cfg.seed, env_rgb=env, out=host_np)
        else:
            acc2 = torch.zeros(W * H * 3, dtype=torch.float32, device="cuda")

            def block2(f, c, acc, S2=S2, N2=N2):
                pt.render_samples(S2, N2, W, H, f, c, depth, cfg.seed, acc, env_rgb=env,
                                  wave_samples=cfg.wave_samples)

            render_partitioned(block2, n_total, acc2, rank, world)
            if rank == 0:
                host_fb.copy_(acc2.mul_(1.0 / n_total), non_blocking=False)
        torch.cuda.synchronize()
        S2.close()
        if N2:
            N2.close()
    te = torch.tensor([time.perf_counter() - te0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = samples_per_step * e2e_steps / float(te.item())

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    global ClockSampler_last
    ClockSampler_last = clk.summary()
    K = args.steps
    nif_ms = kt["nif"]
    infers = escaped
    kernels = {
        "trace_paths": {"ms_per_step": kt["traverse"] / K, "launches_per_step": trav_launches / K,
                        "bytes_alg": 80 * segments},
        "nif": {"ms_per_step": nif_ms / K, "launches_per_step": nif_launches / K,
                "flops_alg": HIDDEN_FLOP_PER_INF * infers},
        "accumulate": {"ms_per_step": kt["accum"] / K},
    }
    dominant = max(kernels, key=lambda n: kernels[n]["ms_per_step"])
    nif_tflops = (HIDDEN_FLOP_PER_INF * infers) / (nif_ms / 1e3) / 1e12 if nif_ms > 0 else 0.0
    nif_roof = {"bound": "tensor", "achieved": nif_tflops, "peak": peaks["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": nif_tflops / peaks["bf16_tflops_sustained"],
                "frac_burst": nif_tflops / peaks["bf16_tflops"],
                "traffic": ncu_traffic(["siren_kernel"], cfg.index),
                "kernel": "siren_kernel", "flop_per_inference": HIDDEN_FLOP_PER_INF,
                "inferences_per_launch": infers / max(1, nif_launches),
                "peak_source": peaks["source"] + " bf16 sustained (fp16 same rate)"}
    if dominant == "trace_paths":
        # traversal + shading (first_bounce_kernel + path_kernel, timed together per wave): algorithmic
        # L2 bytes per segment (counting build, tools/trace_count.py, profiles/round1/trace_count.json):
        # node visits x 64 B + primitive tests x 48 B + 80 B of path state, against the measured L2 read
        # bandwidth (tools/l2_bench.cu, profiles/round1/l2_bench.json); traffic = DRAM bytes of both
        # kernels per wave
        ms_k = kt["traverse"]
        bps = trace_bytes_per_segment(cfg.index)
        byts = (bps or 0.0) * segments
        gbs = byts / (ms_k / 1e3) / 1e9 if ms_k > 0 else 0.0
        roof = {"bound": "l2", "achieved": gbs, "peak": L2_READ_GBS, "unit": "GB/s", "frac": gbs / L2_READ_GBS,
                "traffic": ncu_traffic(["first_bounce_kernel", "path_kernel"], cfg.index),
                "kernel": "first_bounce_kernel + path_kernel",
                "bytes_per_segment": bps,
                "segments_per_wave": segments / max(1, trav_launches / 2),
                "peak_source": "measured L2 read bandwidth, tools/l2_bench.cu (MEASURED_PEAKS.json has none)",
                "hbm_frac": (80.0 * segments / (ms_k / 1e3) / 1e9) / peaks["hbm_gbs"] if ms_k > 0 else 0.0}
        # the bound in practice: instruction issue. Warp instructions per wave (ncu capture of the same
        # kernels) / the live kernel time, against 4 issue slots per SM per clock at the sampled clock
        inst = ncu_inst(["first_bounce_kernel", "path_kernel"], cfg.index)
        waves = max(1, trav_launches / 2)
        if inst and ms_k > 0:
            f_clk = (ClockSampler_last.get("sm_mhz") or 1965.0) * 1e6
            peak_issue = 4 * torch.cuda.get_device_properties(local).multi_processor_count * f_clk
            ach = inst * waves / (ms_k / 1e3)
            # instruction issue is what bounds these kernels (ncu: ~75 % issue-active, 43 % warps active
            # at the 72-register cap, L2 at ~30 %): report it as the roofline, the L2 view beside it
            l2 = roof
            roof = {"bound": "alu", "achieved": ach, "peak": peak_issue, "unit": "warp-inst/s",
                    "frac": ach / peak_issue, "traffic": l2["traffic"], "kernel": l2["kernel"],
                    "warp_inst_per_wave": inst,
                    "work": "warp instructions per wave (ncu smsp__inst_executed.sum of the same kernels on "
                            "the same workload, profiles/round1/ncu_traffic_c%d.json) / live kernel time" % cfg.index,
                    "peak_source": "4 warp-instructions issued per clock per SM (B200_PROFILING.md) x SMs x "
                                   "SM clock sampled during the timed region",
                    "l2": {k: v for k, v in l2.items() if k not in ("traffic", "kernel")}}
    else:
        roof = nif_roof
    clocks = ClockSampler_last
    line = {
        "metric": "samples/sec", "value": value, "unit": "samples/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32 trace / f64 prim tests / f16-in f32-acc NIF",
        "data": "synthetic (seeded scene generator + seeded untrained SIREN weights)",
        "config": workload_config(cfg, world),
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(host_fb.numel() * 4),
                "what": ("pt_scene_create + pt_nif_load from host arrays, pt_render into a pinned host buffer"
                         if host_render else
                         "pt_scene_create + pt_nif_load from host arrays, render, reduce, framebuffer to pinned host")},
        "gpu_launches": int(launches),
        "roofline": roof,
        "nif": {"inferences_per_s": infers / (nif_ms / 1e3) if nif_ms > 0 else None,
                "inferences_per_step": infers / K, "roofline": nif_roof},
        "kernels_ms_per_step": {k: v["ms_per_step"] for k, v in kernels.items()},
        "paths_per_step": paths / K, "segments_per_step": segments / K,
        "wall_s_timed_region": t_wall,
        "step_ms": {"median": step_ms[len(step_ms) // 2], "best": step_ms[0], "worst": step_ms[-1],
                    "note": "this rank's per-step device times (SURVEY 8d: median and best)"},
        "clocks": clocks,
    }
    if world == 1 and not args.no_cpu_baseline:
        r = run_oracle(cfg, 1, 0, rows_every=args.oracle_rows_every)
        line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["cpu_baseline"]["cpu"] = r["cpu"]
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
