"""Sample-partitioned multi-GPU rendering (BASELINE.json north_star: "Work is partitioned by sample
index across the GPUs of one 8xB200 box, with an NCCL reduce of the fp32 framebuffer over NVLink").

The paper replicates the scene and network on every chip and runs them data parallel "with no
communication between them"; the only exchange here is the single framebuffer
reduction at the end of a frame. One process per GPU; torch.distributed supplies the process group
(NCCL on GPUs, gloo in the CPU tests).

Partition rule (reading R19). The work of a frame is the set of (sample, row) pairs.
  * G divides the sample count: rank r renders the contiguous sample block r (all rows).
  * otherwise (G > spp, e.g. config 0's 4 spp on 8 GPUs, or spp = 4 on 3 GPUs): every sample's rows are
    cut into B = G / gcd(spp, G) row blocks; the spp * B (sample, row block) units, in sample-major order,
    are dealt out as G equal contiguous ranges (spp / gcd units each), merged per sample into row ranges.
Every rank then does the same amount of work to within one row block's rounding, and the union over ranks
is exactly the requested (sample, row) range. The Philox counters carry the full-frame pixel index and
the sample, so the reduced frame equals the single-rank frame up to fp32 summation order."""
from __future__ import annotations

import math
from typing import Callable


def sample_block(n_samples: int, rank: int, world: int, first: int = 0) -> tuple[int, int]:
    """(first_sample, count) of the contiguous sample block owned by `rank` (balanced to +-1 sample)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(n_samples, world)
    start = first + rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def work_blocks(n_samples: int, height: int, rank: int, world: int, first: int = 0) -> list[tuple[int, int, int, int]]:
    """The (first_sample, n_samples, row0, row1) blocks owned by `rank` (module docstring rule)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if n_samples < 1 or height < 1:
        return []
    if n_samples % world == 0:
        f, c = sample_block(n_samples, rank, world, first)
        return [(f, c, 0, height)] if c > 0 else []
    g = math.gcd(n_samples, world)
    B = world // g                       # row blocks per sample
    per = n_samples // g                 # units per rank
    out: list[tuple[int, int, int, int]] = []
    for u in range(rank * per, (rank + 1) * per):
        s, b = divmod(u, B)
        r0, r1 = b * height // B, (b + 1) * height // B
        if r1 <= r0:
            continue
        if out and out[-1][0] == first + s and out[-1][3] == r0:
            out[-1] = (out[-1][0], 1, out[-1][2], r1)        # extend the row range of this sample
        else:
            out.append((first + s, 1, r0, r1))
    # merge consecutive samples that cover the same full row range into one multi-sample block
    merged: list[tuple[int, int, int, int]] = []
    for blk in out:
        if merged and merged[-1][2:] == blk[2:] and merged[-1][0] + merged[-1][1] == blk[0]:
            merged[-1] = (merged[-1][0], merged[-1][1] + blk[1], blk[2], blk[3])
        else:
            merged.append(blk)
    return merged


def reduce_sum(accum, dst: int = 0, group=None):
    """SUM-reduce `accum` to rank `dst`: NCCL on CUDA tensors; under gloo a CUDA tensor goes through a
    host copy (gloo reduces host memory)."""
    import torch.distributed as dist
    if accum.is_cuda and dist.get_backend(group) == "gloo":
        host = accum.cpu()
        dist.reduce(host, dst=dst, op=dist.ReduceOp.SUM, group=group)
        if dist.get_rank(group) == dst:
            accum.copy_(host)
        return
    dist.reduce(accum, dst=dst, op=dist.ReduceOp.SUM, group=group)


def render_partitioned(render_block: Callable[[int, int, object], None], n_samples: int, accum, rank: int,
                       world: int, first: int = 0, group=None, reduce: bool = True):
    """accum += this rank's per-pixel sample sums (render_block(first, count, accum)) over its contiguous
    sample block, then SUM-reduce accum to rank 0. Returns the (first, count) block rendered locally."""
    f, c = sample_block(n_samples, rank, world, first)
    if c > 0:
        render_block(f, c, accum)
    if reduce and world > 1:
        reduce_sum(accum, 0, group)
    return f, c


def render_partitioned_rows(render_rows: Callable[[int, int, int, int, object], None], n_samples: int, height: int,
                            accum, rank: int, world: int, first: int = 0, group=None, reduce: bool = True):
    """accum += this rank's (sample, row) blocks (render_rows(first, count, row0, row1, accum), work_blocks
    rule), then SUM-reduce accum to rank 0. Returns the blocks rendered locally."""
    blocks = work_blocks(n_samples, height, rank, world, first)
    for f, c, r0, r1 in blocks:
        render_rows(f, c, r0, r1, accum)
    if reduce and world > 1:
        reduce_sum(accum, 0, group)
    return blocks
