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


class _FakeEngine:
    """Stands in for an Engine: labels = the first pixel of each sample, per member."""

    def __init__(self, device, max_batch):
        import numpy as np

        self.device, self.max_batch, self.members = device, max_batch, [(0, 0, 0, 4), (0, 0, 8, 4)]
        self.seen = []
        self.np = np

    def forward(self, x, kind, *, topk=0, policy=0, policy_k=0, want_logits=False):
        np = self.np
        self.seen.append(int(x.shape[0]))
        lab = np.stack([x.reshape(len(x), -1)[:, 0], x.reshape(len(x), -1)[:, 0] + 1]).astype(np.int32)
        out = {"labels": lab}
        if want_logits:
            out["logits"] = np.repeat(lab[..., None], 4, axis=-1).astype(np.float32)
        if topk:
            out["topk_idx"] = np.repeat(lab[..., None], topk, axis=-1)
            out["topk_prob"] = np.ones(lab.shape + (topk,), np.float32)
        if policy:
            out["combined"] = lab[0] % 2
        return out

    def close(self):
        pass


@pytest.mark.parametrize("batch", [1, 3, 8, 13])
def test_sharded_engine_reassembles_in_shard_order(batch):
    import numpy as np

    from paper_2003_01538_b200.shard import ShardedEngine

    engines = [_FakeEngine(d, 4) for d in range(4)]
    se = ShardedEngine(engines)
    x = np.arange(batch * 6, dtype=np.float32).reshape(batch, 6)
    out = se.forward(x, 0, topk=2, policy=1, want_logits=True)
    spans = [shard_bounds(batch, r, 4) for r in range(4)]
    assert [e.seen for e in engines] == [[hi - lo] if hi > lo else [] for lo, hi in spans]
    want = _FakeEngine(0, batch).forward(x, 0, topk=2, policy=1, want_logits=True)
    for k in ("labels", "logits", "topk_idx", "topk_prob", "combined"):
        assert np.array_equal(out[k], want[k]), k
    se.close()


def test_bench_spawns_ranks_for_multi_gpu(monkeypatch):
    """`bench.py --gpus N` outside torchrun launches N ranks through torch.distributed.run
    (one per GPU, rendezvous on 127.0.0.1) with NCCL's init log on, and returns its exit
    code; under torchrun a --gpus / WORLD_SIZE mismatch is an error, not a silent N = 1."""
    import subprocess
    import sys

    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parent.parent))
    import bench

    seen = {}

    def fake_run(cmd, env=None, **kw):
        seen["cmd"], seen["env"] = cmd, env
        return subprocess.CompletedProcess(cmd, 0)

    monkeypatch.setattr(bench.subprocess, "run", fake_run)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "3"])
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "3"]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"
    # torchrun already set WORLD_SIZE = 2 but --gpus 4: refuse
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setattr(bench, "__name__", "bench")
    import torch

    monkeypatch.setattr(torch.cuda, "set_device", lambda *_: None)
    with pytest.raises(SystemExit) as ex:
        bench.main()
    assert "WORLD_SIZE=2" in str(ex.value.code)
