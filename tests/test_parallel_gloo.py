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


class _FakeLockstep:
    """Stand-in for LockstepSearch (host logic only): seed r of the shard
    stays active for lengths[r] rounds; its best cost falls each round."""

    def __init__(self, g0, cfg, cp, seeds, precision=None, n_threads=0):
        import numpy as np

        self.R = len(seeds)
        self.left = [3 + 5 * (int(s) % 4) for s in seeds]
        self.best = np.array([100.0 + int(s) for s in seeds])
        self.rounds = 0

    def round(self):
        self.rounds += 1
        for r in range(self.R):
            if self.left[r] > 0:
                self.left[r] -= 1
                self.best[r] -= 1.0
        return sum(1 for x in self.left if x > 0)

    def run_cb(self, max_rounds, on_round):
        """LockstepSearch.run_cb: the hook after every round (native run)."""
        active = self.R
        while active > 0 and (max_rounds is None or self.rounds < max_rounds):
            active = self.round()
            if on_round(self.rounds - 1, active, self.best):
                raise RuntimeError("stopped")

    def best_costs(self):
        return self.best.copy()


class _FakeLockstepRounds(_FakeLockstep):
    """Without run_cb: ShardedSearch drives round() itself."""

    run_cb = property()  # hasattr() is False


def _sharded_worker(rank, world, port, q, seeds, exchange_every, max_rounds, use_round, lag=4, by_round=False):
    import paper_2209_12769_b200.search as S
    from paper_2209_12769_b200.parallel import ShardedSearch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S.LockstepSearch = _FakeLockstepRounds if by_round else _FakeLockstep
        sh = ShardedSearch(None, None, None, seeds, rank, world)
        sh.lag = lag
        if rank == 1 and sh.s is not None:  # ranks at different speeds: the lagged exchange absorbs it
            import time

            f = sh.s.round
            sh.s.round = lambda: (time.sleep(0.002), f())[1]
        if use_round:
            n = 0
            while sh.round("cpu") > 0:
                n += 1
            res = sh.best_history[-1]
        else:
            res = sh.run("cpu", max_rounds=max_rounds, exchange_every=exchange_every)
        q.put((rank, res, len(sh.best_history), sh.s.rounds if sh.s is not None else 0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seeds,exchange_every,max_rounds,use_round,lag,by_round", [
    (list(range(5)), 1, None, False, 4, False),     # per-round exchange (the default), 4 in flight
    (list(range(5)), 1, None, False, 1, False),     # one in flight
    (list(range(5)), 1, None, False, 64, False),    # more in flight than rounds
    (list(range(5)), 3, None, False, 4, False),     # uneven shards: 3 + 2 seeds of different lengths
    (list(range(5)), 3, 10, False, 2, False),       # max_rounds stops the runs early
    (list(range(5)), 1, None, False, 3, True),      # without the native hook: round() per round
    ([0], 2, None, False, 4, False),                # rank 1 has no seeds at all
    (list(range(4)), None, None, True, 4, False),   # driven through round()
])
def test_sharded_search_exchange_gloo_world2(seeds, exchange_every, max_rounds, use_round, lag, by_round):
    """ShardedSearch's exchange schedule on 2 ranks: both ranks leave after the
    same number of exchanges (no rank waits in a collective the other never
    joins) and agree on the global best (cost, seed)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_sharded_worker,
                         args=(r, 2, port, q, seeds, exchange_every, max_rounds, use_round, lag, by_round))
             for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][1] == out[1][1]
    assert out[0][2] == out[1][2]  # same number of exchanges on both ranks
    # the single-process answer: every seed run to its length (or max_rounds)
    ref = _FakeLockstep(None, None, None, seeds)
    n = 0
    while any(x > 0 for x in ref.left) and (max_rounds is None or n < max_rounds):
        ref.round()
        n += 1
    j = min(range(len(seeds)), key=lambda r: (ref.best[r], r))
    assert out[0][1] == (float(ref.best[j]), float(j))
