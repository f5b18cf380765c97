"""Alg. 1 backtracking search and the exhaustive oracle with the reference's
signatures (search.py:37-225), driven by the native engine and the device
scorer.

``backtracking_search`` reproduces the reference's trajectory for one seed.
``lockstep_search`` runs R independent seeds in lock step: every round each
active seed performs one step of Alg. 1 and all their candidates are scored
in one device batch, so each seed's trajectory equals the single-seed one.
"""

from __future__ import annotations

import ctypes as C
import heapq
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N
from .errors import InvalidConfig, LimitExceeded, _raise
from .graph import HloGraph, canonical_hash, state_arrays, state_from_arrays
from .rewrite import ALL_METHODS, OptimizationMethod, engine_graph, expand_all, method_index, methods_mask

METHOD_NAMES = ("nondup", "dup", "ar")


@dataclass(frozen=True)
class SearchConfig:
    alpha: float = 1.05
    beta: int = 10
    max_unchanged: int = 1000
    seed: int = 0
    methods: tuple = ALL_METHODS
    time_budget_s: Optional[float] = None

    def __post_init__(self) -> None:
        if self.alpha < 1:
            raise InvalidConfig("alpha must be >= 1")
        if self.beta < 1:
            raise InvalidConfig("beta must be >= 1")
        if not self.methods:
            raise InvalidConfig("method mask must be non-empty")
        if self.max_unchanged < 1:
            raise InvalidConfig("max_unchanged must be >= 1")


@dataclass(frozen=True)
class TraceRecord:
    step: int
    action: str
    cost_us: float
    best_cost_us: float
    queue_len: int
    enqueued: bool = False


@dataclass
class SearchResult:
    best_graph: HloGraph
    best_cost_us: float
    steps: int
    candidates_evaluated: int
    candidates_enqueued: int
    trace: list = field(default_factory=list)


def _require_device(cp):
    from .estimator import DeviceCostProviders

    if not isinstance(cp, DeviceCostProviders):
        raise TypeError("the native search needs device cost providers (make_cost_providers / oracle_providers)")


class LockstepSearch:
    """R lock-stepped Alg. 1 instances on one device (fo_search_*)."""

    def __init__(self, g0: HloGraph, cfg: SearchConfig, cp, seeds: Sequence[int], precision=None, n_threads=0):
        _require_device(cp)
        self.g0, self.cfg, self.cp = g0, cfg, cp
        self.dg = cp.device_graph(g0)
        self.R = len(seeds)
        c = N.SearchCfg()
        c.alpha, c.beta, c.max_unchanged = cfg.alpha, cfg.beta, cfg.max_unchanged
        c.methods_mask = methods_mask(cfg.methods)
        c.precision = N.FO_PREC_FP64 if precision is None else precision
        c.n_threads = n_threads
        ng, rg, bk, _, _, _ = state_arrays(g0)
        self._seeds = np.ascontiguousarray(seeds, np.uint64)
        h = C.c_void_p()
        st = N.lib().fo_search_create(self.dg.h, C.byref(c), N.ptr(self._seeds), self.R, N.ptr(ng), N.ptr(rg),
                                      N.ptr(bk), C.byref(h))
        _raise(st, "fo_search_create", N.last_error())
        self.h = h
        self.best = np.full(self.R, np.inf)
        self.active = self.R
        self.rounds = 0

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                N.lib().fo_search_destroy(h)
            except Exception:
                pass

    def round(self) -> int:
        a = C.c_int32()
        st = N.lib().fo_search_round(self.h, C.byref(a), N.ptr(self.best))
        _raise(st, "fo_search_round", N.last_error())
        self.active = a.value
        self.rounds += 1
        return self.active

    def run(self, max_rounds: Optional[int] = None, started: Optional[float] = None, results: bool = True):
        """Run to completion; results=False skips building the per-seed
        SearchResult objects (graphs and traces) -- see best_costs()."""
        if self.cfg.time_budget_s is None:  # whole search in native code (fo_search_run)
            a = C.c_int32()
            st = N.lib().fo_search_run(self.h, int(max_rounds or 0), C.byref(a))
            _raise(st, "fo_search_run", N.last_error())
            self.active = a.value
            n = C.c_int64()
            N.lib().fo_search_rounds(self.h, C.byref(n))
            self.rounds = int(n.value)
            return [self.result(r) for r in range(self.R)] if results else None
        t0 = time.monotonic() if started is None else started
        st = N.lib().fo_search_start(self.h, N.ptr(self.best))  # eval_cost(g0) precedes the budget check
        _raise(st, "fo_search_start", N.last_error())
        while self.active > 0:
            if max_rounds is not None and self.rounds >= max_rounds:
                break
            if self.cfg.time_budget_s is not None and time.monotonic() - t0 > self.cfg.time_budget_s:
                break
            self.round()
        return [self.result(r) for r in range(self.R)]

    def run_cb(self, max_rounds: Optional[int], on_round):
        """fo_search_run with on_round(round, active, best) called after every
        round (best: the seeds' best costs so far, a view valid during the
        call).  A truthy return, or an exception, stops the run."""
        err = []

        def _fn(ctx, rnd, active, best, R):
            try:
                return 1 if on_round(int(rnd), int(active), np.ctypeslib.as_array(best, (int(R),))) else 0
            except BaseException as e:  # re-raised below, after the native run unwinds
                err.append(e)
                return 1

        cb = N.ROUND_FN(_fn)
        a = C.c_int32()
        st = N.lib().fo_search_run_cb(self.h, int(max_rounds or 0), C.cast(cb, C.c_void_p), None, C.byref(a))
        if err:
            raise err[0]
        _raise(st, "fo_search_run_cb", N.last_error())
        self.active = a.value
        n = C.c_int64()
        N.lib().fo_search_rounds(self.h, C.byref(n))
        self.rounds = int(n.value)

    def best_costs(self) -> np.ndarray:
        """Best cost found by every seed (no graph or trace reconstruction)."""
        out = np.zeros(self.R)
        for r in range(self.R):
            c = C.c_double()
            st = N.lib().fo_search_result(self.h, r, C.byref(c), None, None, None, None, None, 0)
            _raise(st, "search", N.last_error())
            out[r] = c.value
        return out

    def counters(self, r: int):
        """(steps, candidates_evaluated, candidates_enqueued, trace length) of seed r."""
        cnt = np.zeros(4, np.int64)
        st = N.lib().fo_search_result(self.h, r, None, N.ptr(cnt), None, None, None, None, 0)
        _raise(st, "search", N.last_error())
        return tuple(int(x) for x in cnt)

    def timing(self):
        d, e, s = C.c_double(), C.c_double(), C.c_int64()
        N.lib().fo_search_timing(self.h, C.byref(d), C.byref(e), C.byref(s))
        return {"device_ms": d.value, "expand_ms": e.value, "scored": s.value}

    def result(self, r: int, with_trace: bool = True) -> SearchResult:
        V, A = self.dg.V, self.dg.A
        best = C.c_double()
        cnt = np.zeros(4, np.int64)
        ng, rg, bk = np.zeros(V, np.int32), np.zeros(V, np.int32), np.zeros(A, np.int32)
        st = N.lib().fo_search_result(self.h, r, C.byref(best), N.ptr(cnt), N.ptr(ng), N.ptr(rg), N.ptr(bk), None, 0)
        trace = []
        if with_trace and cnt[3] > 0:
            buf = (N.TraceRec * int(cnt[3]))()
            N.lib().fo_search_result(self.h, r, None, None, None, None, None, buf, int(cnt[3]))
            trace = [TraceRecord(t.step, METHOD_NAMES[t.method], t.cost_us, t.best_cost_us, t.queue_len,
                                 bool(t.enqueued)) for t in buf]
        _raise(st, "search", N.last_error())
        return SearchResult(state_from_arrays(self.g0, ng, rg, bk), best.value, int(cnt[0]), int(cnt[1]), int(cnt[2]),
                            trace)


def _is_device(cp) -> bool:
    from .estimator import DeviceCostProviders

    return isinstance(cp, DeviceCostProviders)


def _host_driven_search(g0: HloGraph, cfg: SearchConfig, cp) -> SearchResult:
    """Alg. 1 (search.py:84-155) for arbitrary Python CostProviders: the same
    bookkeeping, one candidate at a time -- the rewrites run in the native
    engine on the caller's random.Random, each cost() evaluates the
    callbacks in Python and simulates on the device (simulator.simulate)."""
    import random

    from .rewrite import random_apply
    from .simulator import cost

    rng = random.Random(cfg.seed)
    t0 = time.monotonic()
    cache = {}
    evaluated = 0

    def eval_cost(g, h):
        nonlocal evaluated
        if h not in cache:
            cache[h] = cost(g, cp)
            evaluated += 1
        return cache[h]

    h0 = canonical_hash(g0)
    best, best_cost = g0, eval_cost(g0, h0)
    seen = {h0}
    queue = [(best_cost, 0, h0, g0)]
    seq, enqueued, unchanged, steps = 1, 0, 0, 0
    trace = []
    chosen = {method_index(m) for m in cfg.methods}
    methods = [m for m in ALL_METHODS if method_index(m) in chosen]
    while queue and unchanged < cfg.max_unchanged:
        if cfg.time_budget_s is not None and time.monotonic() - t0 > cfg.time_budget_s:
            break
        _, _, cur_h, cur = heapq.heappop(queue)
        steps += 1
        requeued = False
        for m in methods:
            n = rng.randint(0, cfg.beta)
            out = random_apply(cur, m, n, rng)
            h = canonical_hash(out.graph) if out.applied else cur_h
            c = eval_cost(out.graph, h)
            if c < best_cost:
                best, best_cost, unchanged = out.graph, c, 0
            else:
                unchanged += 1
            entered = False
            if c <= cfg.alpha * best_cost:
                if h not in seen:  # a new state
                    seen.add(h)
                    heapq.heappush(queue, (c, seq, h, out.graph))
                    seq, enqueued, entered = seq + 1, enqueued + 1, True
                elif h == cur_h and not requeued:  # the state came back: one copy stays in rotation
                    heapq.heappush(queue, (c, seq, h, out.graph))
                    seq, requeued, entered = seq + 1, True, True
            trace.append(TraceRecord(steps, m.value, c, best_cost, len(queue), entered))
    return SearchResult(best, best_cost, steps, evaluated, enqueued, trace)


def backtracking_search(g0: HloGraph, cfg: SearchConfig, cp, precision=None) -> SearchResult:
    """Best fusion state found from g0; never worse than g0 (search.py:84-155).
    Device providers run the native lock-stepped driver; arbitrary Python
    CostProviders run the same algorithm one candidate at a time."""
    if not _is_device(cp):
        return _host_driven_search(g0, cfg, cp)
    return LockstepSearch(g0, cfg, cp, [cfg.seed], precision).run()[0]


def lockstep_search(g0: HloGraph, cfg: SearchConfig, cp, seeds: Sequence[int], precision=None, n_threads=0):
    """Independent searches for every seed, advanced in lock step."""
    return LockstepSearch(g0, cfg, cp, seeds, precision, n_threads).run()


def exhaustive_search(g0: HloGraph, cp, max_ops: int = 8, max_tensors: int = 4) -> SearchResult:
    """BFS closure of the three rewrites with state dedupe (search.py:158-225);
    each BFS level is scored as one device batch."""
    if len(g0.ops) > max_ops:
        raise LimitExceeded(f"{len(g0.ops)} ops exceeds limit {max_ops}")
    if len(g0.allreduces) > max_tensors:
        raise LimitExceeded(f"{len(g0.allreduces)} tensors exceeds limit {max_tensors}")
    if not _is_device(cp):
        return _host_exhaustive(g0, cp)
    dg = cp.device_graph(g0)
    ng, rg, bk, vb, _, _ = state_arrays(g0)
    h0 = int(dg.state_hash(ng, rg, bk)[0])
    seen = {h0}
    c0 = dg.score_host(ng[None], rg[None], bk[None], vb, N.FO_PREC_FP64)
    _raise(int(c0[1][0]), "cost")
    best = (ng, rg, bk)
    best_cost = float(c0[0][0])
    evaluated, steps = 1, 0
    frontier = [(ng, rg, bk)]
    gb = 2 * dg.V + 2
    while frontier:
        level = []
        for s in frontier:
            steps += 1
            cn, cr, cb = expand_all(g0, *s)
            if len(cn) == 0:
                continue
            hs = dg.state_hash(cn, cr, cb)
            for i in range(len(cn)):
                h = int(hs[i])
                if h in seen:
                    continue
                seen.add(h)
                level.append((cn[i], cr[i], cb[i]))
        if not level:
            break
        cost, st = dg.score_host(np.stack([x[0] for x in level]), np.stack([x[1] for x in level]),
                                 np.stack([x[2] for x in level]), gb, N.FO_PREC_FP64)
        for i, x in enumerate(level):
            _raise(int(st[i]), "cost")
            evaluated += 1
            if cost[i] < best_cost:  # strict: first in enumeration order wins (search.py:214-215)
                best, best_cost = x, float(cost[i])
        frontier = level
    return SearchResult(state_from_arrays(g0, *best), best_cost, steps, evaluated, len(seen) - 1)


# --- heuristic baselines (search.py:228-302) ---------------------------------


def topo_order(g: HloGraph) -> list:
    """Deterministic topological order of group ids over the contracted graph,
    ties to the group with the smallest member op id (graph.py:536-556), from
    the native engine.  CycleError when the contraction is cyclic."""
    dg = engine_graph(g)
    ng, rg, bk, _, gids, _ = state_arrays(g)
    out = np.empty(max(len(gids), 1), np.int32)
    n = C.c_int32(0)
    st = N.lib().fo_topo_order(dg.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), N.ptr(out), C.byref(n))
    _raise(st, "topo_order", N.last_error())
    return [gids[int(x)] for x in out[:n.value]]


def greedy_postorder_fusion(g: HloGraph) -> HloGraph:
    """Walk ops in post order (reverse topological) and non-duplicate-fuse each
    op's current group with its first fusible predecessor when the rewrite is
    valid (search.py:228-244), in the native engine."""
    dg = engine_graph(g)
    ng, rg, bk, _, _, _ = state_arrays(g)
    on, orr, ob = np.empty_like(ng), np.empty_like(rg), np.empty_like(bk)
    st = N.lib().fo_greedy_postorder(dg.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), N.ptr(on), N.ptr(orr), N.ptr(ob))
    _raise(st, "greedy_postorder_fusion", N.last_error())
    return state_from_arrays(g, on, orr, ob)


def threshold_allreduce_fusion(g: HloGraph, threshold_bytes: int, cp=None) -> HloGraph:
    """Scan buckets in tensor production order and merge consecutive neighbours
    while the merged size stays within the threshold (search.py:247-302).
    With cost providers the order is the simulated start order (the device
    simulator), otherwise the contracted topological production order."""
    if threshold_bytes <= 0:
        raise InvalidConfig("threshold must be > 0")
    if not g.buckets:
        return g
    dg = engine_graph(g)
    ng, rg, bk, _, _, bids = state_arrays(g)
    order = None
    if cp is not None:
        from .simulator import simulate

        tl = simulate(g, cp)
        start_of = {bid: (start, bid) for bid, start, _ in tl.comm_events}
        rank = {b: i for i, b in enumerate(bids)}
        order = np.array([rank[b] for b in sorted(bids, key=lambda b: start_of[b])], np.int32)
    on, orr, ob = np.empty_like(ng), np.empty_like(rg), np.empty_like(bk)
    st = N.lib().fo_threshold_ar(dg.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), int(threshold_bytes),
                                 None if order is None else N.ptr(order), 0 if order is None else len(order),
                                 N.ptr(on), N.ptr(orr), N.ptr(ob))
    _raise(st, "threshold_allreduce_fusion", N.last_error())
    return state_from_arrays(g, on, orr, ob)


def _host_exhaustive(g0: HloGraph, cp) -> SearchResult:
    """exhaustive_search (search.py:158-225) for arbitrary Python CostProviders:
    BFS over the native engine's single rewrites, cost() per new state."""
    from .rewrite import engine_graph
    from .simulator import cost

    dg = engine_graph(g0)
    ng, rg, bk, _, _, _ = state_arrays(g0)
    seen = {int(dg.state_hash(ng, rg, bk)[0])}
    best, best_cost = g0, cost(g0, cp)
    evaluated, steps = 1, 0
    frontier = [(ng, rg, bk)]
    while frontier:
        level = []
        for st in frontier:
            steps += 1
            cn, cr, cb = expand_all(g0, *st)
            if len(cn) == 0:
                continue
            hs = dg.state_hash(cn, cr, cb)
            for i in range(len(cn)):
                h = int(hs[i])
                if h in seen:
                    continue
                seen.add(h)
                level.append((cn[i], cr[i], cb[i]))
        for x in level:
            gx = state_from_arrays(g0, *x)
            c = cost(gx, cp)
            evaluated += 1
            if c < best_cost:  # strict: the first in enumeration order wins (search.py:214-215)
                best, best_cost = gx, c
        frontier = level
    return SearchResult(best, best_cost, steps, evaluated, len(seen) - 1)
