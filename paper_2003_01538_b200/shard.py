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


class ShardedEngine:
    """One process serving an ensemble from several GPUs: a full
    replica (an Engine) per device, the request batch split contiguously with
    shard_bounds, every shard's forward issued from its own host thread on its own
    device and stream (the native call releases the GIL), outputs reassembled in shard
    order.  Each device copies its own labels / top-k / logits to host memory, so no
    device funnels the others' results through its PCIe link.  Exact: a sample's result
    does not depend on its batch (runtime.cu plan_conv), so the sharded output equals
    the single-GPU output bitwise.

    Same ``forward`` contract as Engine, so ensemble.forward / predict / predict_u8 run
    unchanged on top of it."""

    def __init__(self, engines):
        import concurrent.futures as cf

        if not engines:
            raise ValueError("ShardedEngine needs at least one engine")
        self.engines = list(engines)
        self.members = self.engines[0].members
        self.max_batch = sum(e.max_batch for e in self.engines)
        self._pool = cf.ThreadPoolExecutor(len(self.engines), thread_name_prefix="eb-shard")

    @property
    def devices(self) -> list[int]:
        return [e.device for e in self.engines]

    def shards(self, batch: int) -> list[tuple[int, int]]:
        g = len(self.engines)
        return [shard_bounds(batch, r, g) for r in range(g)]

    def forward(self, x, input_kind: int, *, topk: int = 0, policy: int = 0, policy_k: int = 0,
                want_logits: bool = False):
        import numpy as np

        spans = [(r, lo, hi) for r, (lo, hi) in enumerate(self.shards(int(x.shape[0]))) if hi > lo]
        futs = [self._pool.submit(self.engines[r].forward, x[lo:hi], input_kind, topk=topk,
                                  policy=policy, policy_k=policy_k, want_logits=want_logits)
                for r, lo, hi in spans]
        parts = [f.result() for f in futs]
        out = {"labels": np.concatenate([p["labels"] for p in parts], axis=1)}
        for key in ("logits", "topk_idx", "topk_prob"):
            if key in parts[0]:
                out[key] = np.concatenate([p[key] for p in parts], axis=1)
        if "combined" in parts[0]:
            out["combined"] = np.concatenate([p["combined"] for p in parts])
        return out

    def warmup(self, input_kind: int, max_b: int = 0) -> None:
        for f in [self._pool.submit(e.warmup, input_kind, max_b) for e in self.engines]:
            f.result()

    def close(self):
        self._pool.shutdown(wait=True)
        for e in self.engines:
            e.close()
