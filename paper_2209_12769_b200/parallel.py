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
        self.lag = 8  # exchanges in flight before a rank waits for the oldest (run())

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

        The exchanges are non-blocking and waited ``self.lag`` exchanges late
        (_LaggedExchange); the stop decision is collective, so all ranks post
        the same number of exchanges and leave together (a rank whose seeds
        finished keeps joining them with 0 active seeds)."""
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
        s = self.s
        native = s is not None and hasattr(s, "run_cb") and getattr(getattr(s, "cfg", None), "time_budget_s", None) is None
        import os

        if ((native or s is None) and dist.get_backend() == "nccl" and torch.device(device).type == "cuda"
                and os.environ.get("FO_XCHG_PY") != "1"):
            return self._run_nccl(device, max_rounds, exchange_every)
        ex = _LaggedExchange(self, device, self.lag)
        if native:
            # the native run (speculation, host/device pipelining) hands each
            # round's bests to the exchange thread from its per-round hook
            def on_round(rnd, active, best):
                if (rnd + 1) % exchange_every == 0:
                    ex.submit(best, active)
                return False

            ex.start()
            try:
                s.run_cb(max_rounds, on_round)
            finally:
                ex.join()
            final = s.best_costs()
        elif s is not None:
            rounds, active = 0, s.R
            while active > 0 and (max_rounds is None or rounds < max_rounds):
                active = s.round()
                rounds += 1
                if rounds % exchange_every == 0:
                    ex.post(s.best, active)
            final = s.best
        else:
            final = np.zeros(0)
        ex.finish(final)
        return self.best_history[-1] if self.best_history else (float("inf"), -1.0)


    def _run_nccl(self, device, max_rounds, exchange_every):
        """The exchange natively (fo_xchg, csrc/xchg.cpp): posted from the
        search's round hook over a communicator of its own, waited lag
        exchanges late, closed by fo_xchg_finish on every rank."""
        import ctypes as C

        import torch

        from . import _native as N
        from .errors import _raise

        dist = _dist()
        rank, world = dist.get_rank(), dist.get_world_size()
        idb = (C.c_uint8 * 128)()
        if rank == 0:
            _raise(N.lib().fo_xchg_unique_id(idb), "fo_xchg_unique_id", N.last_error())
        box = [bytes(idb)]
        dist.broadcast_object_list(box, src=0)
        idb = (C.c_uint8 * 128).from_buffer_copy(box[0])
        dev = torch.device(device)
        x = C.c_void_p()
        _raise(N.lib().fo_xchg_create(idb, rank, world, dev.index if dev.index is not None else torch.cuda.current_device(),
                                      int(self.lag), C.byref(x)), "fo_xchg_create", N.last_error())
        try:
            if self.s is not None:
                _raise(N.lib().fo_xchg_attach(self.s.h, x, int(self.seed_offset), int(exchange_every)),
                       "fo_xchg_attach", N.last_error())
                try:
                    self.s.run(max_rounds, results=False)
                finally:
                    N.lib().fo_xchg_attach(self.s.h, None, 0, 1)
            _raise(N.lib().fo_xchg_finish(x), "fo_xchg_finish", N.last_error())
            n = C.c_int64()
            N.lib().fo_xchg_history(x, None, 0, C.byref(n))
            h = np.zeros(2 * max(1, n.value))
            N.lib().fo_xchg_history(x, N.ptr(h), n.value, C.byref(n))
            self.best_history.extend((float(h[2 * i]), float(h[2 * i + 1])) for i in range(n.value))
        finally:
            N.lib().fo_xchg_destroy(x)
        return self.best_history[-1] if self.best_history else (float("inf"), -1.0)


class _LaggedExchange:
    """The per-round exchange without a per-round barrier: each post is a
    non-blocking all-gather of (best cost, seed id, active seeds), and a rank
    waits for an exchange only once ``lag`` newer ones are in flight, so a
    rank's round never waits for a slower rank's same round.  Every rank waits
    the exchanges in order and records the global best of each.

    Stop protocol: a rank whose seeds are done (or whose run hit max_rounds)
    keeps posting exchanges with 0 active seeds, one per exchange it waits,
    until it waits one whose global active count is 0.  Every rank then holds
    the same number of exchanges in flight (lag), so all ranks post the same
    number of exchanges and leave together."""

    def __init__(self, sh, device, lag):
        import collections

        import torch

        self.sh = sh
        self.dist = _dist()
        self.world = self.dist.get_world_size()
        self.lag = max(1, int(lag))
        n = self.lag + 1
        dev = torch.device(device)
        self.send = [torch.empty(3, dtype=torch.float64, device=dev) for _ in range(n)]
        self.recv = [torch.empty(3 * self.world, dtype=torch.float64, device=dev) for _ in range(n)]
        # host staging of the sends: pinned, so the copies are asynchronous
        self.hsend = torch.empty((n, 3), dtype=torch.float64, pin_memory=dev.type == "cuda")
        self.hsend_np = self.hsend.numpy()
        self.pending = collections.deque()
        self.posted = 0

    def start(self):
        """Post the exchanges from a thread of their own (submit()), so the
        search's native loop only copies its bests per round."""
        import queue
        import threading

        self.q = queue.SimpleQueue()
        self.err = None

        def loop():
            import torch

            try:
                if self.send[0].device.type == "cuda":
                    torch.cuda.set_device(self.send[0].device)
                while True:
                    item = self.q.get()
                    if item is None:
                        return
                    self.post(*item)
            except BaseException as e:  # re-raised by join()
                self.err = e

        self.th = threading.Thread(target=loop, name="fo-exchange", daemon=True)
        self.th.start()

    def submit(self, best, active):
        self.q.put((np.array(best, dtype=np.float64), int(active)))

    def join(self):
        self.q.put(None)
        self.th.join()
        if self.err is not None:
            raise self.err

    def post(self, best, active):
        if len(best):
            j = int(np.argmin(best))  # first minimum -> lowest local id among ties
            mine = (float(best[j]), float(self.sh.seed_offset + j))
        else:
            mine = (float("inf"), float("inf"))
        k = self.posted % (self.lag + 1)
        self.hsend_np[k] = (mine[0], mine[1], float(active))  # slot k's previous copy is done: its exchange was waited
        self.send[k].copy_(self.hsend[k], non_blocking=True)
        work = self.dist.all_gather_into_tensor(self.recv[k], self.send[k], async_op=True)
        self.pending.append((work, k))
        self.posted += 1
        while len(self.pending) > self.lag:
            self._wait()

    def _wait(self):
        work, k = self.pending.popleft()
        work.wait()
        allp = self.recv[k].view(self.world, 3).cpu().numpy()
        order = np.lexsort((allp[:, 1], allp[:, 0]))  # strict <: the lowest global id among equal costs
        self.sh.best_history.append((float(allp[order[0], 0]), float(allp[order[0], 1])))
        return int(round(allp[:, 2].sum()))

    def finish(self, best):
        while len(self.pending) < self.lag:
            self.post(best, 0)
        while True:
            if self._wait() == 0:
                break
            self.post(best, 0)
        while self.pending:
            self._wait()
