"""Multi-GPU sharding of the candidate frontier: one process per GPU, the
batch (or the seed set) split into contiguous ranges, and one exchange per
round -- the per-round best (cost, candidate id) pair -- over
torch.distributed (NCCL on B200s; gloo in the CPU tests).

The exchange follows the reference's tie-break: a strictly lower cost wins,
so among equal costs the lowest global candidate id is kept
(search.py:124, :214).
"""

from __future__ import annotations

from typing import Optional, Sequence

import numpy as np


def _dist():
    import torch.distributed as dist

    return dist


def shard_range(total: int, rank: int, world: int):
    """Contiguous [lo, hi) share of ``total`` items for ``rank``."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def global_best(cost, ids, group=None, active=None):
    """Argmin over every rank's (cost, id) pairs; returns (cost, id) as Python
    numbers, identical on all ranks.  ``cost``/``ids`` are 1-D tensors on the
    rank's device (float64 / any numeric id).  With ``active`` (this rank's
    count of live seeds) the same single all-gather also carries the counts,
    and (cost, id, total active) is returned."""
    import torch

    dist = _dist()
    if cost.numel() == 0:
        pair = torch.tensor([float("inf"), float("inf")], dtype=torch.float64, device=cost.device)
    else:
        j = torch.argmin(cost)  # first minimum -> lowest local id among ties
        pair = torch.stack([cost[j].to(torch.float64), ids[j].to(torch.float64)])
    if active is not None:
        pair = torch.cat([pair, torch.tensor([float(active)], dtype=torch.float64, device=cost.device)])
    if not (dist.is_available() and dist.is_initialized()):
        out = (float(pair[0]), float(pair[1]))
        return out + (int(active),) if active is not None else out
    world = dist.get_world_size(group)
    gathered = torch.empty(world * pair.numel(), dtype=torch.float64, device=pair.device)
    dist.all_gather_into_tensor(gathered, pair, group=group)
    allp = gathered.view(world, -1).cpu().numpy()
    order = np.lexsort((allp[:, 1], allp[:, 0]))
    c, i = allp[order[0], 0], allp[order[0], 1]
    if active is not None:
        return float(c), float(i), int(round(allp[:, 2].sum()))
    return float(c), float(i)


class ShardedSearch:
    """R lock-stepped Alg. 1 seeds sharded across ranks.  Each rank advances its
    seeds; the global (best cost, seed) pair is exchanged over the process
    group every round (run() default, or round()), every M rounds
    (run(exchange_every=M)), or once at the end (run(exchange_every=None)).

    Lock-stepped seeds are independent searches, so the wall time of a run is
    bounded by its longest seed at any GPU count: sharding adds seeds per
    second, not speed to one seed."""

    def __init__(self, g0, cfg, cp, seeds: Sequence[int], rank: int, world: int, precision=None, n_threads=0):
        from .search import LockstepSearch

        lo, hi = shard_range(len(seeds), rank, world)
        self.local_seeds = list(seeds[lo:hi])
        self.seed_offset = lo
        self.s = LockstepSearch(g0, cfg, cp, self.local_seeds, precision, n_threads) if self.local_seeds else None
        self.best_history = []

    def round(self, device) -> int:
        """One lock-stepped round on this rank's seeds, then the per-round
        exchange: one all-gather of (best cost, seed id, active seeds) per
        rank.  Returns the active-seed count over all ranks."""
        active = self.s.round() if self.s is not None else 0
        c, i, total = self._exchange(device, active)
        self.best_history.append((c, i))
        return total

    def _exchange(self, device, active):
        """(global best cost, global seed id, total active seeds): the local
        argmin on the host, then one all-gather of 3 doubles per rank into
        buffers allocated once (a per-round call: no per-round allocations)."""
        import torch

        dist = _dist()
        best = self.s.best if self.s is not None else np.zeros(0)
        if len(best):
            j = int(np.argmin(best))  # first minimum -> lowest local id among ties
            mine = (float(best[j]), float(self.seed_offset + j))
        else:
            mine = (float("inf"), float("inf"))
        if not (dist.is_available() and dist.is_initialized()):
            return mine[0], mine[1], int(active)
        world = dist.get_world_size()
        if getattr(self, "_xbuf", None) is None or self._xbuf[0].device != torch.device(device):
            self._xbuf = (torch.empty(3, dtype=torch.float64, device=device),
                          torch.empty(3 * world, dtype=torch.float64, device=device))
        send, recv = self._xbuf
        send.copy_(torch.tensor([mine[0], mine[1], float(active)], dtype=torch.float64))
        dist.all_gather_into_tensor(recv, send)
        allp = recv.view(world, 3).cpu().numpy()
        order = np.lexsort((allp[:, 1], allp[:, 0]))  # strict <: the lowest global id among equal costs
        return float(allp[order[0], 0]), float(allp[order[0], 1]), int(round(allp[:, 2].sum()))

    def run(self, device, max_rounds: Optional[int] = None, exchange_every: Optional[int] = 1):
        """Advance every local seed to completion, exchanging the global best
        (cost, seed) pair every ``exchange_every`` rounds (default 1: every
        round, as the north star states).  ``exchange_every=None`` runs each
        shard natively to the end (fo_search_run, with its speculation and
        host/device pipelining) and exchanges once.

        The stop decision is collective: every rank counts rounds in whole
        blocks and the blocks' active-seed counts are all-reduced, so all ranks
        leave after the same number of exchanges (a rank whose seeds finished
        keeps joining the exchanges with an empty shard)."""
        import torch

        dist = _dist()
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
        if not multi:
            exchange_every = None  # nobody to exchange with: the native run, pipelined and speculating
        if exchange_every is None:
            if self.s is not None:
                self.s.run(max_rounds, results=False)  # results on demand (s.result / s.best_costs)
                best = self.s.best_costs()
            else:
                best = np.zeros(0)
            if not multi:
                if self.s is None:
                    return (float("inf"), -1.0)
                r = min(range(len(best)), key=lambda i: (best[i], i))
                self.best_history.append((float(best[r]), float(self.seed_offset + r)))
                return self.best_history[-1]
            cost = torch.as_tensor(best, dtype=torch.float64, device=device)
            ids = torch.arange(self.seed_offset, self.seed_offset + len(best), dtype=torch.float64, device=device)
            self.best_history.append(global_best(cost, ids))
            return self.best_history[-1]
        if exchange_every < 1:
            raise ValueError("exchange_every must be >= 1")
        rounds = 0
        local_active = self.s.R if self.s is not None else 0
        while True:
            block = exchange_every if max_rounds is None else min(exchange_every, max_rounds - rounds)
            for _ in range(block):
                if local_active == 0:
                    break
                local_active = self.s.round()
            rounds += block  # identical on every rank
            c, i, total = self._exchange(device, local_active)
            self.best_history.append((c, i))
            if total == 0 or (max_rounds is not None and rounds >= max_rounds):
                break
        return self.best_history[-1] if self.best_history else (float("inf"), -1.0)
