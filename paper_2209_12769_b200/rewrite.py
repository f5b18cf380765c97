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
from .errors import NotNeighbors, _raise
from .graph import HloGraph, state_arrays, state_from_arrays


class OptimizationMethod(Enum):
    NON_DUPLICATE_FUSION = "nondup"
    DUPLICATE_FUSION = "dup"
    ALLREDUCE_FUSION = "ar"


METHOD_INDEX = {OptimizationMethod.NON_DUPLICATE_FUSION: 0, OptimizationMethod.DUPLICATE_FUSION: 1,
                OptimizationMethod.ALLREDUCE_FUSION: 2}
ALL_METHODS = tuple(METHOD_INDEX)
_VALUE_INDEX = {m.value: i for m, i in METHOD_INDEX.items()}


def method_index(method) -> int:
    """Engine slot of a method.  Keyed by the enum's value, so the reference's
    own ``fuseopt.OptimizationMethod`` members (same values, rewrite.py:28-33
    of the reference) and plain value strings work as well as this package's."""
    value = getattr(method, "value", method)
    try:
        return _VALUE_INDEX[value]
    except (KeyError, TypeError):
        raise KeyError(method) from None


def methods_mask(methods) -> int:
    """Bit mask of a method collection (SearchConfig.methods)."""
    return sum(1 << method_index(m) for m in set(methods))


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


def _pairs(g: HloGraph, kind: int):
    dg = engine_graph(g)
    ng, rg, bk, _, gids, bids = state_arrays(g)
    cap = 4 * (len(g.edges) + len(g.allreduces) ** 2 + 16)
    out = np.zeros(2 * cap, np.int32)
    n = C.c_int32()
    st = N.lib().fo_rewrite_pairs(dg.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), kind, N.ptr(out), cap, C.byref(n))
    _raise(st, "fo_rewrite_pairs", N.last_error())
    ids = bids if kind == 2 else gids  # ranks back to the graph's ids
    return [(ids[out[2 * i]], ids[out[2 * i + 1]]) for i in range(n.value)]


def fusible_pairs(g: HloGraph):
    """(consumer group, predecessor group) pairs eligible for op fusion, in the
    reference's order (rewrite.py:49-61)."""
    return _pairs(g, 0)


def bucket_pairs(g: HloGraph):
    """(bucket, neighbour) pairs eligible for AllReduce fusion (rewrite.py:212-219)."""
    return _pairs(g, 2)


def neighbors_allreduce(g: HloGraph, bucket_id: int) -> set:
    """Buckets whose producing groups touch this bucket's (rewrite.py:156-178)."""
    g.bucket(bucket_id)  # KeyError for an unknown bucket, as the reference
    return {o for b, o in _pairs(g, 2) if b == bucket_id}


def _apply(g: HloGraph, method: int, a: int, b: int, what: str) -> RewriteOutcome:
    dg = engine_graph(g)
    ng, rg, bk, _, gids, bids = state_arrays(g)
    ids = bids if method == 2 else gids
    rank = {x: i for i, x in enumerate(ids)}
    applied = C.c_int32()
    st = N.lib().fo_rewrite_apply(dg.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), method, rank[a], rank[b], C.byref(applied))
    _raise(st, "fo_rewrite_apply", N.last_error())
    if not applied.value:
        return RewriteOutcome(g, False, "rejected: group contraction (with bucket dependencies) is cyclic")
    return RewriteOutcome(state_from_arrays(g, ng, rg, bk), True, f"{what}: {b} into {a}")


def _op_fusion_checks(g: HloGraph, op_gid: int, pred_gid: int, dup: bool):
    """The reference's rejection reasons in its order (rewrite.py:70-79,
    :108-122); None when only the acyclicity test remains."""
    og, pg = g.group(op_gid), g.group(pred_gid)  # KeyError for unknown groups
    if op_gid == pred_gid:
        return "cannot fuse a group with itself"
    if (op_gid, pred_gid) not in set(_pairs(g, 3)):
        return f"group {pred_gid} is not a direct predecessor of {op_gid}"
    if not all(g.op(m).kind == "compute" for m in og.member_ops | pg.member_ops):
        return "parameter or control op in fusion"
    if og.member_ops & pg.member_ops:
        return "groups share a member"
    if dup and any(m in x.duplicated_ops for x in g.groups for m in pg.member_ops):
        return "a predecessor member already has a replica"
    return None


def fuse_nondup(g: HloGraph, op_gid: int, pred_gid: int) -> RewriteOutcome:
    """Merge the predecessor group into the consumer group (rewrite.py:64-96)."""
    why = _op_fusion_checks(g, op_gid, pred_gid, False)
    if why:
        return RewriteOutcome(g, False, f"rejected: {why}")
    return _apply(g, 0, op_gid, pred_gid, "nondup")


def fuse_dup(g: HloGraph, op_gid: int, pred_gid: int) -> RewriteOutcome:
    """Merge the predecessor into the consumer and leave a replica for its other
    consumers; degrades to non-duplicate fusion without any (rewrite.py:99-153)."""
    why = _op_fusion_checks(g, op_gid, pred_gid, True)
    if why:
        return RewriteOutcome(g, False, f"rejected: {why}")
    return _apply(g, 1, op_gid, pred_gid, "dup")


def fuse_allreduce(g: HloGraph, bucket_id: int, neighbor_id: int) -> RewriteOutcome:
    """Merge two neighbouring buckets (rewrite.py:181-209); NotNeighbors otherwise."""
    if neighbor_id not in neighbors_allreduce(g, bucket_id):
        raise NotNeighbors(f"bucket {neighbor_id} is not a neighbor of {bucket_id}")
    return _apply(g, 2, bucket_id, neighbor_id, "ar")


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
    st = N.lib().fo_random_apply(dg.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), method_index(method), n, N.ptr(mt),
                                 C.byref(applied))
    _raise(st, "fo_random_apply", N.last_error())
    rng.setstate((version, tuple(int(x) for x in mt), gauss))
    if not applied.value:
        return RewriteOutcome(g, False, f"{getattr(method, 'value', method)}: no change")
    return RewriteOutcome(state_from_arrays(g, ng, rg, bk), True, f"{getattr(method, 'value', method)}: applied")


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
    mask = methods_mask(methods)
    return engine_graph(g).make_candidates(seeds, beta, mask, base, n_threads)
