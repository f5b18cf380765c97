"""Feature-level estimator API: SubgraphFeatures, featurize and predict_fused
(estimator.py:99-191, :462-470).

featurize is host-side bookkeeping over one group (the reference's own feature
extraction, restated); predict_fused evaluates the loaded estimator on the
B200 through fo_predict_features -- the same closed forms and the same
message-passing forward the scoring kernels run per fused group, so
predict_fused(model, featurize(g, group, profile)) equals the duration the
device simulator uses for that group.
"""

from __future__ import annotations

import ctypes as C
import hashlib
from collections import OrderedDict
from dataclasses import dataclass
from typing import NamedTuple

import numpy as np

from . import _native as N
from .errors import _raise
from .estimator import EstimatorModel, EstimatorVariant, Profile, _vocab_slots, lookup
from .graph import HloGraph, OpNode, build_graph


@dataclass(frozen=True)
class SubgraphFeatures:
    """Per-member node features plus whole-group aggregates of one fused op
    (estimator.py:99-128): nodes in ascending member op id, ``edges`` as
    member-local (src, dst, bytes) triples in the graph's edge order."""

    op_codes: tuple
    compute_us: tuple
    in_bytes: tuple
    out_bytes: tuple
    edges: tuple
    member_count: int
    total_compute_us: float
    internal_bytes: int
    external_in_bytes: int
    external_out_bytes: int
    longest_path_len: int

    def aggregate_vector(self) -> np.ndarray:
        return np.array([self.member_count, self.total_compute_us, self.internal_bytes, self.external_in_bytes,
                         self.external_out_bytes, self.longest_path_len], dtype=np.float64)


class GroupIO(NamedTuple):
    internal_bytes: int
    external_in_bytes: int
    external_out_bytes: int


def group_io(g: HloGraph, gid: int) -> GroupIO:
    """Internal / external-in / external-out bytes of one group
    (graph.py:181-213): an output is external when an AllReduce, a copy of a
    consumer outside the group, or nothing reads it, and it is charged once,
    to its export group (the replica group when duplicated, graph.py:158)."""
    groups_of = {o.id: [] for o in g.ops}
    normal, replica = {}, {}
    members = {}
    for gr in g.groups:
        members[gr.id] = gr.member_ops
        for m in gr.member_ops:
            groups_of[m].append(gr.id)
            (replica if m in gr.duplicated_ops else normal)[m] = gr.id
    if gid not in members:
        raise KeyError(f"no group {gid}")
    mine = members[gid]
    internal = ext_in = ext_out = 0
    visible = set()
    has_out = set()
    for e in g.edges:
        has_out.add(e.src)
        for h in groups_of[e.dst]:
            if e.src in members[h]:
                if h == gid:
                    internal += e.bytes
            else:
                if h == gid:
                    ext_in += e.bytes
                visible.add(e.src)
    producers = {a.producer_op for a in g.allreduces}
    for o in g.ops:
        if o.id in mine and replica.get(o.id, normal.get(o.id)) == gid and (
                o.id in visible or o.id not in has_out or o.id in producers):
            ext_out += o.out_bytes
    return GroupIO(internal, ext_in, ext_out)


def _longest_path_nodes(n: int, edges) -> int:
    """Nodes on the longest internal path (estimator.py:131-154)."""
    if n == 0:
        return 0
    succs = [[] for _ in range(n)]
    indeg = [0] * n
    for i, j, _ in edges:
        succs[i].append(j)
        indeg[j] += 1
    frontier = [i for i in range(n) if indeg[i] == 0]
    order = list(frontier)
    while frontier:
        nxt = []
        for u in frontier:
            for v in succs[u]:
                indeg[v] -= 1
                if indeg[v] == 0:
                    nxt.append(v)
        order.extend(nxt)
        frontier = nxt
    depth = [1] * n
    for u in order:
        for v in succs[u]:
            depth[v] = max(depth[v], depth[u] + 1)
    return max(depth)


def featurize(g: HloGraph, group, profile: Profile) -> SubgraphFeatures:
    """Feature extraction for one group (estimator.py:157-191); replica
    members contribute like ordinary members."""
    members = sorted(group.member_ops)
    local = {m: i for i, m in enumerate(members)}
    in_b = {m: 0 for m in members}
    for e in g.edges:
        if e.dst in in_b:
            in_b[e.dst] += e.bytes
    ops = [g.op(m) for m in members]
    compute = [lookup(profile, o) for o in ops]
    edges = tuple((local[e.src], local[e.dst], e.bytes) for e in g.edges
                  if e.src in group.member_ops and e.dst in group.member_ops)
    io = group_io(g, group.id)
    return SubgraphFeatures(op_codes=tuple(o.op_code for o in ops), compute_us=tuple(compute),
                            in_bytes=tuple(in_b[m] for m in members), out_bytes=tuple(o.out_bytes for o in ops),
                            edges=edges, member_count=len(members), total_compute_us=float(sum(compute)),
                            internal_bytes=io.internal_bytes, external_in_bytes=io.external_in_bytes,
                            external_out_bytes=io.external_out_bytes,
                            longest_path_len=_longest_path_nodes(len(members), edges))


# -- device evaluation ---------------------------------------------------------

_HANDLES: "OrderedDict[bytes, tuple]" = OrderedDict()
_MAX_HANDLES = 8


def _fingerprint(model: EstimatorModel) -> bytes:
    h = hashlib.blake2b(digest_size=16)
    h.update(f"{model.variant.value}|{model.layers}|{model.hidden}|{model.out_scale!r}|{model.vocab!r}".encode())
    for k in sorted(model.params):
        a = np.ascontiguousarray(model.params[k], np.float64)
        h.update(k.encode() + repr(a.shape).encode() + a.tobytes())
    for norm in (model.node_norm, model.agg_norm):
        if norm is None:
            h.update(b"-")
        else:
            for a in norm:
                h.update(np.ascontiguousarray(a, np.float64).tobytes())
    return h.digest()


def _handle(model: EstimatorModel, precision: int):
    """A device handle carrying ``model`` (a one-op graph; the estimator state
    is what matters), cached by model content."""
    from .comm import CommModelParams
    from .estimator import DeviceCostProviders

    key = _fingerprint(model) + bytes([precision])
    ent = _HANDLES.get(key)
    if ent is not None:
        _HANDLES.move_to_end(key)
        return ent[1]
    op0 = OpNode(0, model.vocab[0] if model.vocab else "op", input_shape_key="k", out_bytes=0, compute_us=1.0)
    g = build_graph([op0])
    cp = DeviceCostProviders("profile", profile=Profile({(op0.op_code, "k"): 1.0}),
                             comm_params=CommModelParams(0.0, 0.0), model=model, precision=precision)
    dg = cp.device_graph(g)
    _HANDLES[key] = (cp, dg, g)
    while len(_HANDLES) > _MAX_HANDLES:
        _HANDLES.popitem(last=False)
    return dg


def predict_fused(model: EstimatorModel, f: SubgraphFeatures, precision: int = N.FO_PREC_FP64) -> float:
    """Strictly positive execution-time prediction for a fused group
    (estimator.py:462-470), computed on the B200 (fo_predict_features)."""
    dg = _handle(model, precision)
    n = int(f.member_count)
    slots = (_vocab_slots(model, f.op_codes) if model.variant is EstimatorVariant.MESSAGE_PASSING
             else np.zeros(n, np.int32))
    c = np.ascontiguousarray(f.compute_us, np.float64)
    ib = np.ascontiguousarray(f.in_bytes, np.int64)
    ob = np.ascontiguousarray(f.out_bytes, np.int64)
    ed = np.ascontiguousarray([(int(i), int(j)) for i, j, _ in f.edges], np.int32).reshape(-1, 2)
    agg = np.ascontiguousarray(f.aggregate_vector(), np.float64)
    out = C.c_double(0.0)
    p = lambda a: a.ctypes.data if a.size else None  # noqa: E731
    st = N.lib().fo_predict_features(dg.h, n, p(slots), p(c), p(ib), p(ob), len(ed), p(ed), agg.ctypes.data,
                                     precision, C.byref(out))
    _raise(st, "fo_predict_features", N.last_error())
    return float(out.value)
