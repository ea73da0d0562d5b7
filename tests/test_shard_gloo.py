"""CPU, world_size 2 (gloo): batch sharding and the logits gather to the serving rank
reassemble exactly the single-process result (the reference's batch == concatenated
singles property makes sharding exact)."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2003_01538_b200.shard import gather_rows, shard_bounds


def test_shard_bounds_cover_batch():
    for batch in (1, 2, 7, 256, 4096, 4097):
        for world in (1, 2, 4, 8):
            spans = [shard_bounds(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert all(hi >= lo for lo, hi in spans)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, batch, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = torch.arange(batch * 3 * 5, dtype=torch.float32).reshape(batch, 3, 5)  # "logits"
    lo, hi = shard_bounds(batch, rank, world)
    got = gather_rows(full[lo:hi].clone(), batch, dst=0)
    if rank == 0:
        out.put(bool(torch.equal(got, full)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("batch", [7, 64])
def test_gather_rows_two_ranks(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=10) is True
