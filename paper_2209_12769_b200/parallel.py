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


def global_best(cost, ids, group=None):
    """Argmin over every rank's (cost, id) pairs; returns (cost, id) as Python
    numbers, identical on all ranks.  ``cost``/``ids`` are 1-D tensors on the
    rank's device (float64 / any numeric id)."""
    import torch

    dist = _dist()
    if cost.numel() == 0:
        pair = torch.tensor([float("inf"), float("inf")], dtype=torch.float64, device=cost.device)
    else:
        j = torch.argmin(cost)  # first minimum -> lowest local id among ties
        pair = torch.stack([cost[j].to(torch.float64), ids[j].to(torch.float64)])
    if not (dist.is_available() and dist.is_initialized()):
        return float(pair[0]), float(pair[1])
    world = dist.get_world_size(group)
    out = [torch.empty_like(pair) for _ in range(world)]
    dist.all_gather(out, pair, group=group)
    allp = torch.stack(out).cpu().numpy()
    order = np.lexsort((allp[:, 1], allp[:, 0]))
    c, i = allp[order[0]]
    return float(c), float(i)


class ShardedSearch:
    """R lock-stepped Alg. 1 seeds sharded across ranks.  Each rank advances its
    seeds; the global (best cost, seed) pair is exchanged over the process
    group at the end of the run, or every M rounds (run(exchange_every=M)), or
    every round when driven through round()."""

    def __init__(self, g0, cfg, cp, seeds: Sequence[int], rank: int, world: int, precision=None, n_threads=0):
        from .search import LockstepSearch

        lo, hi = shard_range(len(seeds), rank, world)
        self.local_seeds = list(seeds[lo:hi])
        self.seed_offset = lo
        self.s = LockstepSearch(g0, cfg, cp, self.local_seeds, precision, n_threads) if self.local_seeds else None
        self.best_history = []

    def round(self, device) -> int:
        import torch

        dist = _dist()
        active = self.s.round() if self.s is not None else 0
        best = self.s.best if self.s is not None else np.zeros(0)
        cost = torch.as_tensor(best, dtype=torch.float64, device=device)
        ids = torch.arange(self.seed_offset, self.seed_offset + len(best), dtype=torch.float64, device=device)
        self.best_history.append(global_best(cost, ids))
        a = torch.tensor([active], dtype=torch.int64, device=device)
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(a)
        return int(a.item())

    def run(self, device, max_rounds: Optional[int] = None, exchange_every: Optional[int] = None):
        """Advance every local seed to completion.  Seeds are independent, so by
        default each rank runs its shard natively (fo_search_run) and the global
        best is exchanged once at the end; exchange_every=M steps the shard M
        rounds at a time with an exchange after each block (progress reports)."""
        import torch

        dist = _dist()
        multi = dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
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
        rounds = 0
        while True:
            active = 0
            for _ in range(exchange_every):
                active = self.s.round() if self.s is not None else 0
                rounds += 1
                if active == 0 or (max_rounds is not None and rounds >= max_rounds):
                    break
            best = self.s.best if self.s is not None else np.zeros(0)
            cost = torch.as_tensor(best, dtype=torch.float64, device=device)
            ids = torch.arange(self.seed_offset, self.seed_offset + len(best), dtype=torch.float64, device=device)
            self.best_history.append(global_best(cost, ids))
            a = torch.tensor([active], dtype=torch.int64, device=device)
            if multi:
                dist.all_reduce(a)
            if int(a.item()) == 0 or (max_rounds is not None and rounds >= max_rounds):
                break
        return self.best_history[-1] if self.best_history else (float("inf"), -1.0)
