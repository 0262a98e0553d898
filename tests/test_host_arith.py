"""Host-side pins of two arithmetic shortcuts the CUDA path relies on (emulated bit-for-bit in numpy
float32), and of the Python binding's argument checks that run before any device work.

* udiv_exact (trace_kernels.cu): q = trunc(fl32(n) * fl32(1/d)) is within one of n // d for n < 2^31 and
  quotients < 2^20, so one correction each way gives the exact quotient and remainder (slot -> (pixel,
  sample), pixel -> (x, y)); checked exhaustively near every multiple and on random draws for the
  divisors the configs use plus awkward ones."""
import numpy as np
import pytest


def _udiv_exact(n, d):
    inv = np.float32(1.0) / np.float32(d)
    q = np.trunc(n.astype(np.float32) * inv).astype(np.int64)
    r = n - q * d
    q = np.where(r < 0, q - 1, np.where(r >= d, q + 1, q))
    return q, n - q * d


@pytest.mark.parametrize("d", [1, 3, 7, 64, 100, 512, 1024, 1920, 3840, 4096, 262144, 1048576, 2073600, 8294400,
                               999983, 12345])
def test_udiv_exact(d):
    rng = np.random.default_rng(d)
    maxn = min(2 ** 31 - 1, 64 * d + d)
    n = np.concatenate([rng.integers(0, maxn, 100000), np.arange(0, min(maxn, 20000)),
                        ((np.arange(1, 65) * d)[:, None] + np.arange(-2, 3)[None, :]).ravel()])
    n = n[(n >= 0) & (n < 2 ** 31)].astype(np.int64)
    q, r = _udiv_exact(n, d)
    assert np.array_equal(q, n // d) and np.array_equal(r, n % d)


def test_render_rejects_bad_output_buffer():
    from paper_2305_20061_b200 import pt
    with pytest.raises(pt.PtError):
        pt.render(None, None, 4, 2, 1, 1, out=np.zeros(4 * 2 * 3, np.float64))     # wrong dtype
    with pytest.raises(pt.PtError):
        pt.render(None, None, 4, 2, 1, 1, out=np.zeros(4 * 2 * 3 + 1, np.float32))  # wrong size
    with pytest.raises(pt.PtError):
        pt.render(None, None, 4, 2, 1, 1, out=np.zeros((6, 8), np.float32)[:, ::2])  # not contiguous
