"""The search's batch-expand moves, executed by the native engine
(csrc/engine.cpp) with the reference's enumeration order, id assignment and
validity rule (rewrite.py:28-263 of the reference)."""

from __future__ import annotations

import ctypes as C
import random
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import _native as N
from .errors import _raise
from .graph import HloGraph, state_arrays, state_from_arrays


class OptimizationMethod(Enum):
    NON_DUPLICATE_FUSION = "nondup"
    DUPLICATE_FUSION = "dup"
    ALLREDUCE_FUSION = "ar"


METHOD_INDEX = {OptimizationMethod.NON_DUPLICATE_FUSION: 0, OptimizationMethod.DUPLICATE_FUSION: 1,
                OptimizationMethod.ALLREDUCE_FUSION: 2}
ALL_METHODS = tuple(METHOD_INDEX)


@dataclass(frozen=True)
class RewriteOutcome:
    graph: HloGraph
    applied: bool
    description: str


_engines = {}


def engine_graph(g: HloGraph):
    """A device handle used only for its host-side engine (no cost model needed)."""
    from .simulator import _plain_providers

    return _plain_providers().device_graph(g)


def random_apply(g: HloGraph, method: OptimizationMethod, n: int, rng: random.Random) -> RewriteOutcome:
    """Apply ``method`` up to n times on uniformly drawn legal choices
    (rewrite.py:222-263).  Consumes ``rng`` exactly like the reference."""
    if n < 0:
        raise ValueError("n must be >= 0")
    dg = engine_graph(g)
    ng, rg, bk, _, _, _ = state_arrays(g)
    version, internal, gauss = rng.getstate()
    mt = np.array(internal, dtype=np.uint32)
    applied = C.c_int32()
    st = N.lib().fo_random_apply(dg.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), METHOD_INDEX[method], n, N.ptr(mt),
                                 C.byref(applied))
    _raise(st, "fo_random_apply", N.last_error())
    rng.setstate((version, tuple(int(x) for x in mt), gauss))
    if not applied.value:
        return RewriteOutcome(g, False, f"{method.value}: no change")
    return RewriteOutcome(state_from_arrays(g, ng, rg, bk), True, f"{method.value}: applied")


def expand_all(g: HloGraph, ng, rg, bk):
    """Every accepted single rewrite (exhaustive_search order, search.py:185-206)."""
    dg = engine_graph(g)
    cap = 2 * dg.V * dg.V + dg.A * dg.A + 16
    cap = min(cap, 1 << 16)
    ng_o = np.zeros((cap, dg.V), np.int32)
    rg_o = np.zeros((cap, dg.V), np.int32)
    bk_o = np.zeros((cap, dg.A), np.int32)
    n = C.c_int32()
    st = N.lib().fo_expand_all(dg.h, N.ptr(np.ascontiguousarray(ng, np.int32)), N.ptr(np.ascontiguousarray(rg, np.int32)),
                               N.ptr(np.ascontiguousarray(bk, np.int32)), cap, N.ptr(ng_o), N.ptr(rg_o), N.ptr(bk_o),
                               C.byref(n))
    _raise(st, "fo_expand_all", N.last_error())
    k = n.value
    return ng_o[:k], rg_o[:k], bk_o[:k]


def make_candidates(g: HloGraph, seeds, beta: int = 10, methods=ALL_METHODS, base=None, n_threads: int = 0):
    """Random batch: candidate k = Random(seeds[k]) then accumulating
    random_apply for each method with n = randint(0, beta).
    Returns (ngid[K,V], rgid[K,V], bkt[K,A], gid_bound) with engine ids."""
    mask = sum(1 << METHOD_INDEX[m] for m in methods)
    return engine_graph(g).make_candidates(seeds, beta, mask, base, n_threads)
