"""The multi-GPU exchange logic on CPU: world_size-2 gloo process group, the
per-round best (cost, id) argmin and the frontier sharding."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_12769_b200.parallel import global_best, shard_range


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = shard_range(10, rank, world)
        # costs with a cross-rank tie: ids 3 (rank 0) and 7 (rank 1) both cost 1.0
        all_cost = torch.tensor([5.0, 4.0, 2.0, 1.0, 9.0, 3.0, 8.0, 1.0, 6.0, 1.5], dtype=torch.float64)
        ids = torch.arange(lo, hi, dtype=torch.float64)
        c, i = global_best(all_cost[lo:hi], ids)
        # empty shard contributes nothing
        c2, i2 = global_best(torch.zeros(0, dtype=torch.float64) if rank == 1 else all_cost[:2], torch.arange(
            0 if rank == 1 else 2, dtype=torch.float64))
        q.put((rank, (lo, hi), (c, i), (c2, i2)))
    finally:
        dist.destroy_process_group()


def test_global_best_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][1] == (0, 5) and out[1][1] == (5, 10)
    for r in out:
        assert r[2] == (1.0, 3.0)  # strict-< tie-break: lowest global id wins
        assert r[3] == (4.0, 1.0)


def test_shard_range_covers():
    for total in (0, 1, 7, 4096):
        for world in (1, 2, 3, 8):
            spans = [shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
