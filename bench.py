#!/usr/bin/env python
"""Benchmark of the B200 neural path tracer hot path (BASELINE.json metric: samples/sec and NIF
inferences/sec; % tensor roofline for the NIF kernel).

One step = one full frame of BASELINE.json configs[3] ("Small BVH + HDR-NIF": a 100,820-triangle
displaced icosphere, 1920x1080, 32 spp per GPU, max_depth 8, RR from depth 3, SIREN HDR-NIF; the largest
single-GPU NIF workload and the paper's clock-scaling scene) through the whole
wavefront hot path -- raygen, traverse, shade (scatter + RR + compaction), fused tcgen05 NIF,
accumulate -- plus, for N > 1, the NCCL framebuffer reduce to rank 0. Inputs (scene BVH, NIF weights)
are resident in HBM when the timed region starts. The timed loop runs with the library's per-kernel
profiling OFF and no host synchronisation between steps; the per-kernel split comes from a second,
separately timed pass with profiling on. Configs 2 and 1 are measured after it under "also".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]
      [--split weak|strong]

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
PROFILE_DIRS = [os.path.join(ROOT, "profiles", "round2"), os.path.join(ROOT, "profiles", "round1")]
TRACE_SOURCES = ["paper_2305_20061_b200/csrc/trace_kernels.cu", "paper_2305_20061_b200/csrc/bvh_build.cpp",
                 "paper_2305_20061_b200/csrc/pt_internal.h"]
TRACE_KERNELS = ["first_bounce_kernel", "path_kernel"]
NIF_SOURCES = ["paper_2305_20061_b200/csrc/siren_kernel.cu", "paper_2305_20061_b200/csrc/tc_ptx.cuh"]


def sources_sha16(files) -> str:
    """Hash of the kernel sources a committed capture was taken with (tools/trace_count.py and
    tools/ncu_traffic.py store it), so a stale capture is flagged instead of silently reused."""
    import hashlib
    h = hashlib.sha256()
    for f in files:
        with open(os.path.join(ROOT, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def _profile_json(name):
    for d in PROFILE_DIRS:
        p = os.path.join(d, name)
        if os.path.exists(p):
            with open(p) as f:
                return json.load(f), os.path.relpath(p, ROOT)
    return None, None


def trace_counts(cfg_index: int):
    """Algorithmic traversal bytes per traced segment of a config's render (counting build of the same
    kernel, tools/trace_count.py: 64 B x node visits + 48 B x primitive tests + 80 B path state), with
    the file it came from and whether it was taken with the current kernel sources."""
    d, path = _profile_json("trace_count.json")
    try:
        r = d[f"render_c{cfg_index}"]
        return {"bytes_per_segment": float(r["alg_bytes_per_segment"]), "per_segment": r.get("per_segment"),
                "file": path, "current": d.get("sources_sha16") == sources_sha16(TRACE_SOURCES)}
    except Exception:
        return None


def ncu_capture(kernels, cfg_index: int, field: str, sources):
    """Per-wave sum over the named kernels of `field` (dram_bytes_per_launch, warp_inst_per_launch) from
    the committed ncu metrics capture of one bench step (tools/ncu_traffic.py), or (None, ...)."""
    d, path = _profile_json(f"ncu_traffic_c{cfg_index}.json")
    try:
        v = float(sum(d[k][field] for k in kernels))
        key = "trace_sources_sha16" if sources is TRACE_SOURCES else "nif_sources_sha16"
        return (v if v > 0 else None), path, d.get(key) == sources_sha16(sources)
    except Exception:
        return None, path, False



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


# bounded oracle samples (rows every k): cpu_baseline ~3-5 s, one reference-arm step ~1-2 s on 16 cores
ORACLE_ROWS = {0: (1, 1), 1: (8, 64), 2: (32, 256), 3: (12, 270), 4: (540, 1080)}   # cpu_baseline / reference-arm row strides (config 3: ~11 s of oracle work for the baseline)


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


def frame_samples(cfg, world, split):
    """Samples of one frame: weak scaling = cfg.spp per GPU (disjoint sample blocks), strong = cfg.spp in
    total split over the GPUs ("64 spp, split by sample index across 8 B200")."""
    return cfg.spp * world if split == "weak" else cfg.spp


def workload_config(cfg, world, split="weak"):
    n = frame_samples(cfg, world, split)
    return {"workload": f"configs[{cfg.index}] {cfg.name}: {cfg.width}x{cfg.height}, "
                        + (f"{cfg.spp} spp per GPU" if split == "weak" else f"{cfg.spp} spp split over {world} GPU(s)")
                        + f", max_depth {cfg.max_depth}, RR>=3, {'SIREN HDR-NIF' if cfg.use_nif else 'constant env'}",
            "width": cfg.width, "height": cfg.height, "spp_per_gpu": cfg.spp if split == "weak" else n / world,
            "max_depth": cfg.max_depth, "wave_samples": cfg.wave_samples, "frame_spp_total": n, "seed": cfg.seed,
            "parallelism": (f"sample-partitioned x{world} ({split} scaling) + NCCL framebuffer reduce"
                            if world > 1 else "1 GPU"),
            "l2": "L2 flushed (512 MiB memset) between timed steps, untimed; wave state > L2"}


class Renderer:
    """One config's scene + NIF handles and the per-rank frame step (device accumulator)."""

    def __init__(self, cfg, rank, world, split, stream):
        import torch

        from paper_2305_20061_b200 import pt
        self.cfg, self.rank, self.world, self.split, self.stream = cfg, rank, world, split, stream
        self.env = None if cfg.use_nif else cfg.env_rgb
        self.src = scenes.scene_for_config(cfg.index)
        self.blob = scenes.siren_blob(0) if cfg.use_nif else None
        t0 = time.perf_counter()
        self.S = pt.Scene(self.src)
        self.scene_create_ms = 1e3 * (time.perf_counter() - t0)
        self.N = pt.Nif(self.blob) if cfg.use_nif else None
        self.accum = torch.zeros(cfg.width * cfg.height * 3, dtype=torch.float32, device="cuda")
        self.n_total = frame_samples(cfg, world, split)

    def step(self):
        from paper_2305_20061_b200 import pt
        from paper_2305_20061_b200.dist import render_partitioned_rows
        c = self.cfg

        def rows(f, n, r0, r1, acc):
            if r0 == 0 and r1 == c.height:
                pt.render_samples(self.S, self.N, c.width, c.height, f, n, c.max_depth, c.seed, acc, env_rgb=self.env,
                                  wave_samples=c.wave_samples, stream=self.stream)
            else:    # (sample, row block) split when the GPU count does not divide the samples (reading R19)
                pt.render_rows(self.S, self.N, c.width, c.height, r0, r1, f, n, c.max_depth, c.seed, acc,
                               env_rgb=self.env, wave_samples=c.wave_samples, stream=self.stream)

        self.accum.zero_()
        render_partitioned_rows(rows, self.n_total, c.height, self.accum, self.rank, self.world)


def timed_steps(R, steps, flush, stream, world):
    """K steps, one CUDA event pair per step on the launching stream, L2 flush between steps (untimed),
    no host synchronisation inside the loop; returns (per-step ms, wall s, clocks)."""
    import torch
    import torch.distributed as dist
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for k in range(steps):
            flush.zero_()
            evs[k][0].record(stream)
            R.step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return [a.elapsed_time(b) for a, b in evs], time.perf_counter() - t_wall0, clk.summary()


def max_over_ranks(x, world):
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def profile_pass(R, steps):
    """Per-kernel split (library CUDA events around every kernel class) and the per-step counters of the
    last step; a separate pass, so the timed loop above runs without the profiling events."""
    import torch
    kt = {"raygen": 0.0, "traverse": 0.0, "shade": 0.0, "nif": 0.0, "accum": 0.0}
    tot = {"escaped": 0, "segments": 0, "paths": 0, "launches": 0, "nif_launches": 0, "traverse_launches": 0,
           "waves": 0}
    R.S.set_profiling(True)
    for _ in range(steps):
        R.step()
        st = R.S.stats()      # synchronises: profiling pass only
        for key in kt:
            kt[key] += st[f"t_{key}_ms"]
        for key in tot:
            tot[key] += st[key]
    R.S.set_profiling(False)
    torch.cuda.synchronize()
    per = {k: v / steps for k, v in kt.items()}
    per.update({k: v / steps for k, v in tot.items()})
    return per


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--split", choices=["weak", "strong"], default="weak",
                    help="weak: spp per GPU fixed; strong: the config's spp divided over the GPUs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-also", action="store_true", help="skip the extra config lines")
    ap.add_argument("--oracle-rows-every", type=int, default=0)
    ap.add_argument("--wave-samples", type=int, default=0, help="samples per wave (default: the config's)")
    args = ap.parse_args()
    cfg = scenes.CONFIGS[args.config]
    if args.wave_samples > 0:
        import dataclasses
        cfg = dataclasses.replace(cfg, wave_samples=args.wave_samples)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # logic test of the multi-rank path on a single-GPU box (never a measurement): every rank on cuda:0,
    # gloo instead of NCCL (the ranks' kernels are independent; only the framebuffer reduce is shared)
    shared_gpu_test = os.environ.get("PT_BENCH_SHARED_GPU_TEST") == "1"
    if shared_gpu_test:
        local = 0
    rows_cpu, rows_ref = ORACLE_ROWS[cfg.index]
    if args.oracle_rows_every > 0:
        rows_cpu = args.oracle_rows_every

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_oracle(cfg, args.steps, args.warmup, rows_every=rows_ref)
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
    from paper_2305_20061_b200.dist import render_partitioned_rows

    if world > 1:
        if shared_gpu_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    if rank == 0:
        _build.build()
    if world > 1:
        dist.barrier()
    pt.lib()

    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    R = Renderer(cfg, rank, world, args.split, stream)
    W, H, spp, depth = cfg.width, cfg.height, cfg.spp, cfg.max_depth
    for _ in range(args.warmup):
        R.step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, profiling off, no per-step host sync ----
    step_ms, t_wall, clocks = timed_steps(R, args.steps, flush, stream, world)
    ms_max = max_over_ranks(sum(step_ms), world)
    samples_per_step = W * H * R.n_total
    value = samples_per_step * args.steps / (ms_max / 1e3)
    step_sorted = sorted(step_ms)

    # ---- second pass: per-kernel split and counters (profiling on; not the headline) ----
    prof = profile_pass(R, min(args.steps, 5))

    # ---- end-to-end through the public API: host arrays in, host framebuffer out ----
    # twice the device steps (up to 40): the pipeline fill (the first step's inputs, created before any render
    # can overlap them) is inside the timed region and is amortised over the run
    e2e_steps = max(3, min(2 * args.steps, 40))
    host_fb = torch.empty(W * H * 3, dtype=torch.float32, pin_memory=True)
    host_np = host_fb.numpy()
    auto_k = max(1, min(spp, (1 << 28) // (W * H)))      # pt_render's wave size (pt_api.cu)
    host_render = world == 1 and auto_k == cfg.wave_samples
    src, blob, env = R.src, R.blob, R.env
    h2d = src.tris.nbytes + src.spheres.nbytes + src.materials.nbytes + src.camera.nbytes + (blob.nbytes if blob is not None else 0)
    create_ms = []

    def make_inputs():
        # the step's inputs through the public API: pt_scene_create (host BVH build + upload) and pt_nif_load
        torch.cuda.set_device(local)          # (the CUDA device is per host thread)
        tc = time.perf_counter()
        S2 = pt.Scene(src)
        create_ms.append(1e3 * (time.perf_counter() - tc))
        return S2, (pt.Nif(blob) if cfg.use_nif else None)

    def render_step(S2, N2):
        if host_render:
            # one GPU: pt_render, the C-ABI's host-buffer call (device accumulator, scale, read-back into
            # the caller's pinned buffer); its automatic wave size equals the config's here
            pt.render(S2, N2, W, H, spp, depth, cfg.seed, env_rgb=env, out=host_np)
        else:
            acc2 = torch.zeros(W * H * 3, dtype=torch.float32, device="cuda")

            def rows2(f, c, r0, r1, acc, S2=S2, N2=N2):
                pt.render_rows(S2, N2, W, H, r0, r1, f, c, depth, cfg.seed, acc, env_rgb=env,
                               wave_samples=cfg.wave_samples)

            render_partitioned_rows(rows2, R.n_total, H, acc2, rank, world)
            if rank == 0:
                host_fb.copy_(acc2.mul_(1.0 / R.n_total), non_blocking=False)
        torch.cuda.synchronize()
        S2.close()
        if N2:
            N2.close()

    # one GPU: frames alternate between two streams and two pinned buffers (pt_render_async), so frame
    # i's read-back overlaps frame i+1's kernels; a buffer is reused only after its stream is synchronised
    a_streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    a_bufs = [host_fb, torch.empty(W * H * 3, dtype=torch.float32, pin_memory=True)]
    inflight = [None, None]

    def retire(j):
        if inflight[j] is not None:
            a_streams[j].synchronize()        # frame read back into a_bufs[j]
            for h in inflight[j]:
                if h:
                    h.close()
            inflight[j] = None

    def render_step_async(it, S2, N2):
        j = it % 2
        retire(j)
        pt.render_async(S2, N2, W, H, spp, depth, cfg.seed, a_bufs[j].numpy(), env_rgb=env, stream=a_streams[j])
        inflight[j] = (S2, N2)

    # warm-up (untimed), then the timed, pipelined loop: step i + 1's scene and NIF are created on a second
    # host thread (ctypes releases the GIL) while step i renders -- every step still builds and uploads
    # its own inputs and reads its frame back inside the timed region
    render_step(*make_inputs())
    from concurrent.futures import ThreadPoolExecutor
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    create_ms.clear()
    te0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=1) as ex:
        fut = ex.submit(make_inputs)
        for it in range(e2e_steps):
            S2, N2 = fut.result()
            if it + 1 < e2e_steps:
                fut = ex.submit(make_inputs)
            if host_render:
                render_step_async(it, S2, N2)
            else:
                render_step(S2, N2)
        retire(0)
        retire(1)
    e2e_s = max_over_ranks(time.perf_counter() - te0, world)
    e2e_value = samples_per_step * e2e_steps / e2e_s
    # the same steps without the pipelining (each step's inputs created, then rendered), for reference
    serial_create = list(create_ms)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ts0 = time.perf_counter()
    for _ in range(e2e_steps):
        render_step(*make_inputs())
    e2e_serial = samples_per_step * e2e_steps / max_over_ranks(time.perf_counter() - ts0, world)
    create_ms[:] = serial_create

    # ---- extra configs (not the headline): value only, same timing rules ----
    also = {}
    if not args.no_also:
        for ci in (2, 1):
            if ci == cfg.index:
                continue
            c2 = scenes.CONFIGS[ci]
            R2 = Renderer(c2, rank, world, args.split, stream)
            for _ in range(3):
                R2.step()
            torch.cuda.synchronize()
            k2 = max(3, min(args.steps, 20))
            ms2, _, clk2 = timed_steps(R2, k2, flush, stream, world)
            ms2 = max_over_ranks(sum(ms2), world)
            also[f"configs[{ci}]"] = {"value": c2.width * c2.height * R2.n_total * k2 / (ms2 / 1e3),
                                      "unit": "samples/s", "ms_per_step": ms2 / k2, "steps": k2,
                                      "workload": workload_config(c2, world, args.split)["workload"],
                                      "sm_mhz": clk2.get("sm_mhz")}
            R2.S.close()
            if R2.N:
                R2.N.close()
            del R2

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peaks = load_peaks()
    K = args.steps
    infers = prof["escaped"]
    nif_ms = prof["nif"]
    waves = max(1.0, prof["waves"])
    nif_tflops = (HIDDEN_FLOP_PER_INF * infers) / (nif_ms / 1e3) / 1e12 if nif_ms > 0 else 0.0
    nif_traffic, nif_traffic_file, nif_traffic_cur = ncu_capture(["siren_kernel"], cfg.index, "dram_bytes_per_launch",
                                                                 NIF_SOURCES)
    nif_roof = {"bound": "tensor", "achieved": nif_tflops, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
                "frac": nif_tflops / peaks["bf16_tflops"],
                "frac_sustained": nif_tflops / peaks["bf16_tflops_sustained"],
                "traffic": nif_traffic, "traffic_file": nif_traffic_file, "traffic_current": nif_traffic_cur,
                "kernel": "siren_kernel", "flop_per_inference": HIDDEN_FLOP_PER_INF,
                "inferences_per_launch": infers / max(1, prof["nif_launches"]),
                "launch_ms": nif_ms / max(1, prof["nif_launches"]),
                "peak_source": peaks["source"] + " bf16 dense burst (a ~%.1f ms kernel timed alone; fp16 runs at "
                               "the same rate)" % (nif_ms / max(1, prof["nif_launches"]))}
    kernels_ms = {"trace_paths": prof["traverse"], "nif": prof["nif"], "accumulate": prof["accum"]}
    dominant = max(kernels_ms, key=kernels_ms.get)
    tc = trace_counts(cfg.index)
    ms_k = prof["traverse"]
    segs = prof["segments"]
    bps = tc["bytes_per_segment"] if tc else None
    gbs = (bps or 0.0) * segs / (ms_k / 1e3) / 1e9 if ms_k > 0 else 0.0
    tr_traffic, tr_file, tr_cur = ncu_capture(TRACE_KERNELS, cfg.index, "dram_bytes_per_launch", TRACE_SOURCES)
    inst, inst_file, inst_cur = ncu_capture(TRACE_KERNELS, cfg.index, "warp_inst_per_launch", TRACE_SOURCES)
    f_clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
    peak_issue = 4 * torch.cuda.get_device_properties(local).multi_processor_count * f_clk
    issue = None
    if inst and ms_k > 0:
        ach = inst * waves / (ms_k / 1e3)
        issue = {"bound": "alu", "achieved": ach, "peak": peak_issue, "unit": "warp-inst/s", "frac": ach / peak_issue,
                 "warp_inst_per_wave": inst, "file": inst_file, "current": inst_cur,
                 "work": "warp instructions per wave (ncu smsp__inst_executed.sum of the same kernels on the same "
                         "workload) / live kernel time",
                 "peak_source": "4 warp-instructions issued per clock per SM (B200_PROFILING.md) x SMs x SM clock "
                                "sampled during the timed region"}
    trace_roof = {"bound": "l2", "achieved": gbs, "peak": L2_READ_GBS, "unit": "GB/s", "frac": gbs / L2_READ_GBS,
                  "traffic": tr_traffic / 1.0 if tr_traffic else None, "traffic_file": tr_file,
                  "traffic_current": tr_cur, "kernel": " + ".join(TRACE_KERNELS),
                  "bytes_per_segment": bps, "per_segment": tc["per_segment"] if tc else None,
                  "counts_file": tc["file"] if tc else None, "counts_current": tc["current"] if tc else None,
                  "segments_per_wave": segs / waves, "launch_ms": ms_k / waves,
                  "peak_source": "measured L2 read bandwidth, tools/l2_bench.cu (MEASURED_PEAKS.json has none)",
                  "issue": issue}
    roof = trace_roof if dominant == "trace_paths" else nif_roof
    line = {
        "metric": "samples/sec", "value": value, "unit": "samples/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": ms_max / K, "higher_is_better": True,
        "scaling": "weak" if args.split == "weak" else "strong",
        "vs_baseline": None, "dtype": "f32 trace / f64 prim tests / f16-in f32-acc NIF",
        "data": "synthetic (seeded scene generator + seeded untrained SIREN weights)",
        "config": workload_config(cfg, world, args.split),
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(host_fb.numel() * 4),
                "what": ("every step: pt_scene_create (incl. the host BVH build) + pt_nif_load from host arrays, "
                         "pt_render_async into one of two pinned host buffers on one of two streams (a buffer is "
                         "reused after its stream is synchronised; serial_value: pt_render, synchronous)"
                         if host_render else
                         "every step: pt_scene_create + pt_nif_load from host arrays, render, reduce, framebuffer "
                         "to pinned host") + "; pipelined: step i+1's inputs are created on a second host thread "
                                             "while step i renders",
                "scene_create_ms_median": statistics.median(create_ms),
                "serial_value": e2e_serial},
        "gpu_launches": int(round(prof["launches"] * K)),
        "roofline": roof,
        "nif": {"inferences_per_s": infers / (nif_ms / 1e3) if nif_ms > 0 else None,
                "inferences_per_step": infers, "roofline": nif_roof},
        "kernels_ms_per_step": kernels_ms,
        "kernels_note": "second pass (%d steps) with the library's per-kernel CUDA events on" % min(K, 5),
        "paths_per_step": prof["paths"], "segments_per_step": segs,
        "wall_s_timed_region": t_wall,
        "step_ms": {"median": step_sorted[len(step_sorted) // 2], "best": step_sorted[0], "worst": step_sorted[-1],
                    "note": "this rank's per-step device times (SURVEY 8d: median and best)"},
        "clocks": clocks,
        "host": {"scene_create_ms": R.scene_create_ms},
        "also": also,
    }
    if world == 1 and not args.no_cpu_baseline:
        r = run_oracle(cfg, 1, 0, rows_every=rows_cpu)
        line["cpu_baseline"] = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["cpu_baseline"]["cpu"] = r["cpu"]
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
