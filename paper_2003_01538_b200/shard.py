"""Batch sharding across GPUs and the logits gather to the serving rank.

Every sample is independent (the reference's batch == concatenated singles,
tests/test_ensemble.py:250-264), so rank r evaluates the contiguous slice
shard_bounds(B, r, G) on its own full replica of the ensemble and the serving
rank reassembles outputs in shard order -- exact by order stability.
The only exchange is that gather: one NCCL collective over NVLink (gloo on CPU
for the host-side tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(batch: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of rank's contiguous slice: ceil(B / G) samples per rank, last ones short."""
    per = -(-batch // world)
    lo = min(batch, rank * per)
    return lo, min(batch, lo + per)


def gather_rows(local: torch.Tensor, batch: int, dst: int = 0) -> torch.Tensor | None:
    """Gather every rank's rows (shard order) onto ``dst``; returns the (B, ...) tensor there.

    Ranks pad their slice to ceil(B / G) rows so a single fixed-size collective
    suffices; padding rows are dropped on the destination.
    """
    world = dist.get_world_size()
    rank = dist.get_rank()
    per = -(-batch // world)
    lo, hi = shard_bounds(batch, rank, world)
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} rows, expected {hi - lo}")
    buf = local.new_zeros((per,) + tuple(local.shape[1:]))
    buf[: hi - lo] = local
    if rank == dst:
        parts = [torch.empty_like(buf) for _ in range(world)]
        dist.gather(buf, parts, dst=dst)
        rows = [p[: shard_bounds(batch, r, world)[1] - shard_bounds(batch, r, world)[0]]
                for r, p in enumerate(parts)]
        return torch.cat(rows, dim=0)
    dist.gather(buf, None, dst=dst)
    return None
