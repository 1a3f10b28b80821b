"""Batch sharding across GPUs.

Rows are independent (transforms.hpp:126-143 acts on one row; SPEC.md:233 makes
disjoint buffers safe), so the multi-GPU path is one process per GPU, each
transforming a contiguous row range of the global [batch][n] buffer with no
collective on the data path.  torch.distributed (NCCL over NVLink on the GPU
box, gloo in CPU tests) is used only to gather results when a caller needs them
on one rank, and for barriers / max-over-ranks timing.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_range(batch: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous partition, ceil(batch/world) rows per rank (the last ranks may
    get fewer, possibly zero).  Returns (first_row, rows)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"shard_range: bad rank {rank} of {world}")
    if batch < 0:
        raise ValueError("shard_range: negative batch")
    per = -(-batch // world) if batch else 0
    first = min(batch, rank * per)
    return first, max(0, min(per, batch - first))


def forward_shard(x_local, mode, transform: Optional[Callable] = None, **kw):
    """Transform this rank's rows in place.  `transform` defaults to the GPU
    batched call (chw_forward_batched_); tests may inject a stand-in."""
    if transform is None:
        from . import chw_forward_batched_

        transform = chw_forward_batched_
    return transform(x_local, mode, **kw)


def gather_rows(local, batch: int, group=None, dst: int = 0):
    """Gather every rank's row shard onto rank `dst` (returns the [batch][n]
    tensor there, None elsewhere).  Shards are padded to equal size for the
    collective and trimmed afterwards."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = local.shape[-1]
    per = -(-batch // world) if batch else 0
    pad = local.new_zeros((per, n))
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    if dist.get_backend(group) == "nccl":
        # NCCL has no gather: all_gather into every rank, keep dst's copy.
        outs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(outs, pad, group=group)
        bufs = outs if rank == dst else None
    else:
        dist.gather(pad, gather_list=bufs, dst=dst, group=group)
    if rank != dst:
        return None
    full = torch.cat(bufs, dim=0)
    return full[:batch]


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Slowest rank's value (timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
