"""Sample-partitioned multi-GPU rendering (BASELINE.json north_star: "Work is partitioned by sample
index across the GPUs of one 8xB200 box, with an NCCL reduce of the fp32 framebuffer over NVLink").

The paper replicates the scene and network on every chip and runs them data parallel "with no
communication between them"; the only exchange here is the single framebuffer
reduction at the end of a frame. One process per GPU; torch.distributed supplies the process group
(NCCL on GPUs, gloo in the CPU tests).

Partition rule (reading R19): rank r of G owns the contiguous sample block
[first + r*n//G + min(r, n%G), ...) so any G (including G not dividing spp) balances to within one
sample, and the union over ranks is exactly the requested range."""
from __future__ import annotations

from typing import Callable


def sample_block(n_samples: int, rank: int, world: int, first: int = 0) -> tuple[int, int]:
    """(first_sample, count) owned by `rank`."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_samples, world)
    start = first + rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def render_partitioned(render_block: Callable[[int, int, object], None], n_samples: int, accum, rank: int,
                       world: int, first: int = 0, group=None, reduce: bool = True):
    """accum += this rank's per-pixel sample sums (render_block(first, count, accum)), then
    SUM-reduce accum to rank 0. Returns the (first, count) block rendered locally."""
    import torch.distributed as dist

    f, c = sample_block(n_samples, rank, world, first)
    if c > 0:
        render_block(f, c, accum)
    if reduce and world > 1:
        dist.reduce(accum, dst=0, op=dist.ReduceOp.SUM, group=group)
    return f, c
