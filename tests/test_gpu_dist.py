"""Multi-process rendering through the CUDA library: two ranks (gloo process group,
both on cuda:0 -- their kernels are independent, only the framebuffer reduce is shared) render their
(sample, row) blocks with pt_render_rows / pt_render_samples and SUM-reduce; the reduced frame equals the
single-rank frame up to fp32 summation order. Covers the sample-block split (2 | spp) and the (sample,
row block) split (2 does not divide spp: DESIGN.md reading R19)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, spp, out_q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2305_20061_b200 import pt, scenes
    from paper_2305_20061_b200.dist import render_partitioned_rows
    c = scenes.CONFIGS[0]
    S = pt.Scene(scenes.scene_for_config(0))
    N = pt.Nif(scenes.siren_blob(0))
    acc = torch.zeros(c.width * c.height * 3, dtype=torch.float32, device="cuda")

    def rows(f, n, r0, r1, a):
        pt.render_rows(S, N, c.width, c.height, r0, r1, f, n, c.max_depth, 3, a)

    blocks = render_partitioned_rows(rows, spp, c.height, acc, rank, world)
    torch.cuda.synchronize()
    out_q.put((rank, blocks, acc.cpu().numpy().copy() if rank == 0 else None))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("spp", [4, 3])
def test_two_rank_cuda_render_reduce_equals_single_rank(spp):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2305_20061_b200 import _build, pt, scenes
    _build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, spp, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = next(a for r, _, a in res if r == 0)
    blocks = {r: b for r, b, _ in res}
    if spp % world:
        assert any(r0 > 0 or r1 < 64 for b in blocks.values() for _, _, r0, r1 in b)   # row-block split used
    c = scenes.CONFIGS[0]
    ref = torch.zeros(c.width * c.height * 3, dtype=torch.float32, device="cuda")
    pt.render_samples(pt.Scene(scenes.scene_for_config(0)), pt.Nif(scenes.siren_blob(0)), c.width, c.height, 0, spp,
                      c.max_depth, 3, ref)
    ref = ref.cpu().numpy()
    assert np.allclose(got, ref, rtol=2e-6, atol=1e-6)
