"""Multi-process (gloo, world size 2, CPU) tests of the sample-partitioned rendering host logic
(dist.py): partition coverage/balance, and reduce(rank blocks) == single-rank render. The renderer
used here is the fp64 oracle (the CUDA renderer needs a GPU; the partition/reduce code is the same)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2305_20061_b200.dist import render_partitioned, render_partitioned_rows, sample_block, work_blocks


def test_sample_block_partition():
    for n in (1, 4, 7, 16, 64):
        for g in (1, 2, 3, 8):
            blocks = [sample_block(n, r, g, first=5) for r in range(g)]
            covered = [s for f, c in blocks for s in range(f, f + c)]
            assert covered == list(range(5, 5 + n))
            counts = [c for _, c in blocks]
            assert max(counts) - min(counts) <= 1
    with pytest.raises(ValueError):
        sample_block(4, 2, 2)


@pytest.mark.parametrize("n,g,h", [(4, 8, 64), (4, 3, 30), (5, 2, 7), (16, 8, 5), (1, 8, 3), (64, 3, 2160),
                                   (32, 5, 1080), (7, 7, 1), (2, 16, 17)])
def test_work_blocks_cover_exactly_once_and_balance(n, g, h):
    """work_blocks (reading R19): every (sample, row) of the frame is rendered by exactly one
    rank, and the ranks' row counts differ by at most one row block's rounding."""
    seen = np.zeros((n, h), np.int64)
    work = []
    for r in range(g):
        rows = 0
        for f, c, r0, r1 in work_blocks(n, h, r, g, first=3):
            assert 0 <= r0 < r1 <= h and c >= 1
            seen[f - 3:f - 3 + c, r0:r1] += 1
            rows += c * (r1 - r0)
        work.append(rows)
    assert (seen == 1).all()
    if n % g == 0:
        assert max(work) == min(work)                     # n / g full-frame samples each
    else:
        per = n // np.gcd(n, g)                           # (sample, row block) units per rank
        assert max(work) - min(work) <= per               # units differ by at most one row each


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2305_20061_b200 import scenes
    sc = oracle.OracleScene(scenes.box_scene())
    blob = scenes.siren_blob(0)
    W = H = 12
    acc = torch.zeros(W * H * 3, dtype=torch.float64)

    def block(f, c, a):
        out, _ = sc.render(W, H, 4, 0, s0=f, s1=f + c, nif_blob=blob, nthreads=1)
        a += torch.from_numpy(out.reshape(-1))

    render_partitioned(block, 5, acc, rank, world)
    if rank == 0:
        out_q.put(acc.numpy().copy())
    dist.destroy_process_group()


def test_gloo_reduce_equals_single_rank():
    import oracle
    from paper_2305_20061_b200 import scenes
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = oracle.OracleScene(scenes.box_scene())
    ref, _ = sc.render(12, 12, 4, 0, s0=0, s1=5, nif_blob=scenes.siren_blob(0), nthreads=1)
    assert np.allclose(got, ref.reshape(-1), rtol=1e-12, atol=0)


def _worker_rows(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2305_20061_b200 import scenes
    sc = oracle.OracleScene(scenes.box_scene())
    blob = scenes.siren_blob(0)
    W, H = 10, 9
    acc = torch.zeros(W * H * 3, dtype=torch.float64)

    def rows(f, c, r0, r1, a):
        pix = np.arange(r0 * W, r1 * W, dtype=np.int64)
        out, _ = sc.render(W, H, 4, 0, pix=pix, s0=f, s1=f + c, nif_blob=blob, nthreads=1)
        a.view(H * W, 3)[r0 * W:r1 * W] += torch.from_numpy(out)

    render_partitioned_rows(rows, 3, H, acc, rank, world)      # 3 samples on 2 ranks: (sample, row-block) split
    if rank == 0:
        out_q.put(acc.numpy().copy())
    dist.destroy_process_group()


def test_gloo_row_block_split_equals_single_rank():
    """G does not divide spp: the (sample, row block) split reduced over 2 gloo ranks equals the
    single-rank render (the oracle as renderer: the partition and reduce code is the CUDA path's)."""
    import oracle
    from paper_2305_20061_b200 import scenes
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_rows, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = oracle.OracleScene(scenes.box_scene())
    ref, _ = sc.render(10, 9, 4, 0, s0=0, s1=3, nif_blob=scenes.siren_blob(0), nthreads=1)
    assert np.allclose(got, ref.reshape(-1), rtol=1e-12, atol=0)
