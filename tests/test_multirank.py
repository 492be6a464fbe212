"""Multi-rank host logic on CPU (gloo, world_size 2): sentence sharding
covers every sentence exactly once, per-rank results gather back into input
order identical to a single-rank run, and the max-over-ranks timing reduction
used by bench.py.  The data path has no collective; gloo stands in for the
NCCL barrier / scalar reductions."""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1610_01108_b200.sharding import shard_sentences
from paper_1610_01108_b200.workload import WORKLOADS


def fake_decode(sent):
    # deterministic stand-in for a device decode: depends only on the sentence
    return [sum(sent) % 30000, len(sent) * 2 + 10]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sents = WORKLOADS["cfg2"].corpus()[:600]
    mine = shard_sentences([len(s) for s in sents], world, 64, 5)[rank]
    local = {i: fake_decode(sents[i]) for i in mine}
    gathered = [None] * world
    dist.all_gather_object(gathered, local)
    t = torch.tensor([float(rank + 1) * 10.0])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n = torch.tensor([float(len(mine))])
    dist.all_reduce(n, op=dist.ReduceOp.SUM)
    if rank == 0:
        merged = {}
        for g in gathered:
            assert not (set(g) & set(merged)), "sentence decoded twice"
            merged.update(g)
        q.put((sorted(merged.items()), float(t.item()), float(n.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_gathers_identical_output():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, tmax, n = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sents = WORKLOADS["cfg2"].corpus()[:600]
    assert [k for k, _ in merged] == list(range(600))
    assert [v for _, v in merged] == [fake_decode(s) for s in sents]
    assert tmax == 20.0 and n == 600.0
