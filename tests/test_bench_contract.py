"""bench.py's reference arm (the fp64 oracle timed on the host, this tier's base-contract reference): the
one JSON line and its keys, and the N > 1 behaviour (rank 0 alone prints; other ranks exit 0)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return [l for l in p.stdout.splitlines() if l.strip()]


def test_reference_arm_json_line():
    lines = _run({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"})
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"] == "samples/sec" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("configs[3]")   # the headline workload


def test_reference_arm_other_ranks_exit_quietly():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}) == []


@__import__("pytest").mark.gpu
def test_own_arm_json_line_on_gpu():
    """The device arm at N = 1 (short run): every key of the contract, and the rooflines' arithmetic."""
    import torch
    if not torch.cuda.is_available():
        __import__("pytest").skip("no CUDA device")
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline", "--no-also"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-2000:]
    d = json.loads([l for l in p.stdout.splitlines() if l.strip()][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks", "nif"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] == 1920 * 1080 * 3 * 4
    assert d["config"]["workload"].startswith("configs[3]")
    r = d["roofline"]
    assert r["bound"] in ("alu", "l2", "hbm", "tensor") and r["peak"] > 0 and r["achieved"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    nr = d["nif"]["roofline"]
    assert nr["bound"] == "tensor" and 0 < nr["frac"] < 1
    # the NIF kernel runs for well under a second per launch: the burst peak applies
    assert nr["peak"] == json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else True
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@__import__("pytest").mark.gpu
@__import__("pytest").mark.parametrize("split", ["weak", "strong"])
def test_own_arm_two_ranks_logic_on_one_gpu(split):
    """bench.py's multi-rank path (partition, reduce, max-over-ranks timing, rank-0 line) under torchrun
    with 2 ranks sharing cuda:0 over gloo (PT_BENCH_SHARED_GPU_TEST: a logic test, not a measurement);
    configs[0] has 4 spp, so the strong split runs 2 samples per rank."""
    import torch
    if not torch.cuda.is_available():
        __import__("pytest").skip("no CUDA device")
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, PT_BENCH_SHARED_GPU_TEST="1")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--config", "0", "--steps", "2", "--warmup", "3", "--no-also", "--split", split],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == split and d["value"] > 0
    assert d["config"]["frame_spp_total"] == (8 if split == "weak" else 4)
