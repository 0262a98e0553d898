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

from paper_2305_20061_b200.dist import render_partitioned, sample_block


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
