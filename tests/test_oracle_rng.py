"""Pins for the oracle's counter-based RNG (Philox-4x32-10, reading R13 in DESIGN.md).

Pinned against (a) the published Random123 known-answer vectors (tests/golden) and (b) an
independent library implementation: cuRAND's curand_Philox4x32_10, compiled for the host CPU."""
import os
import shutil
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat():
    rows = []
    for line in open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[:4], v[4:6], v[6:10]))
    return rows


def test_philox_known_answers(orc):
    for ctr, key, want in _kat():
        got = orc.philox([ctr], [key])[0]
        assert [int(x) for x in got] == want


CURAND_HOST = r"""
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
int main() {
  unsigned c[4], k[2];
  while (scanf("%u %u %u %u %u %u", &c[0], &c[1], &c[2], &c[3], &k[0], &k[1]) == 6) {
    uint4 r = curand_Philox4x32_10(make_uint4(c[0], c[1], c[2], c[3]), make_uint2(k[0], k[1]));
    printf("%u %u %u %u\n", r.x, r.y, r.z, r.w);
  }
}
"""


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc (cuRAND headers) not available")
def test_philox_matches_curand_host_routine(orc, tmp_path):
    src = tmp_path / "ph.cu"
    src.write_text(CURAND_HOST)
    exe = tmp_path / "ph"
    subprocess.check_call(["nvcc", "-Wno-deprecated-gpu-targets", "-o", str(exe), str(src)])
    rng = np.random.default_rng(123)
    n = 1 << 14
    ctr = rng.integers(0, 2**32, size=(n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(n, 2), dtype=np.uint64).astype(np.uint32)
    # structured counters too: (pixel, sample, slot, stream) as the renderer uses them
    ctr[:256] = np.stack([np.arange(256), np.arange(256) % 7, np.arange(256) % 13, np.zeros(256)], 1)
    inp = "\n".join(" ".join(str(int(x)) for x in list(c) + list(k)) for c, k in zip(ctr, key))
    out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout
    want = np.array([[int(x) for x in l.split()] for l in out.strip().splitlines()], dtype=np.uint32)
    got = orc.philox(ctr, key)
    assert np.array_equal(got, want)


def test_u01_exact_range():
    import oracle
    u = oracle.u01(np.array([0, 255, 256, 0xFFFFFFFF], dtype=np.uint32))
    assert u[0] == 0.0 and u[1] == 0.0 and u[2] == 2.0 ** -24
    assert u[3] == 1.0 - 2.0 ** -24
    assert np.all(u.astype(np.float32).astype(np.float64) == u)   # exact in fp32 as well


def test_philox_uniform_moments(orc):
    n = 1 << 18
    ctr = np.zeros((n, 4), np.uint32)
    ctr[:, 0] = np.arange(n)
    out = orc.philox(ctr, np.zeros((n, 2), np.uint32))
    u = orc.u01(out.reshape(-1))
    assert abs(u.mean() - 0.5) < 4 * np.sqrt(1 / 12 / u.size)
    assert abs((u ** 2).mean() - 1 / 3) < 4 * np.sqrt(4 / 45 / u.size)
