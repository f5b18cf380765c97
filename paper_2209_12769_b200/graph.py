"""Graph value types with the reference's field names (graph.py:35-299) and its
JSON document format (graph.py:611-743), so graphs, strategies and fixtures
move between the two packages unchanged.

Only what the scoring path needs lives here: the structural validation,
statistics and contraction queries of the reference stay in the reference.
The contraction itself runs on the device (csrc/score.cu).
"""

from __future__ import annotations

import gzip
import hashlib
import json
from dataclasses import dataclass
from typing import Iterable, NamedTuple, Optional, Sequence

from .errors import GraphFormatError

KIND_COMPUTE = "compute"
KIND_PARAMETER = "parameter"
KIND_CONTROL = "control"
OP_KINDS = (KIND_COMPUTE, KIND_PARAMETER, KIND_CONTROL)
KIND_CODE = {KIND_COMPUTE: 0, KIND_PARAMETER: 1, KIND_CONTROL: 2}


@dataclass(frozen=True)
class OpNode:
    id: int
    op_code: str
    kind: str = KIND_COMPUTE
    input_shape_key: str = ""
    out_bytes: int = 0
    compute_us: Optional[float] = None


@dataclass(frozen=True)
class DataEdge:
    src: int
    dst: int
    bytes: int = 0


@dataclass(frozen=True)
class AllReduceInstr:
    id: int
    producer_op: int
    tensor_bytes: int
    bucket: int


@dataclass(frozen=True)
class FusionGroup:
    id: int
    member_ops: frozenset
    duplicated_ops: frozenset = frozenset()

    def __post_init__(self) -> None:
        object.__setattr__(self, "member_ops", frozenset(self.member_ops))
        object.__setattr__(self, "duplicated_ops", frozenset(self.duplicated_ops))


@dataclass(frozen=True)
class TensorBucket:
    id: int
    members: tuple
    total_bytes: int


@dataclass(frozen=True)
class GraphMeta:
    name: str = "unnamed"
    devices: int = 2
    seed: int = 0


@dataclass(frozen=True)
class HloGraph:
    meta: GraphMeta
    ops: tuple
    edges: tuple
    allreduces: tuple
    groups: tuple
    buckets: tuple

    def op(self, op_id: int) -> OpNode:
        return _lookup(self, "_op_by_id", self.ops)[op_id]

    def group(self, gid: int) -> FusionGroup:
        return _lookup(self, "_group_by_id", self.groups)[gid]

    def bucket(self, bid: int) -> TensorBucket:
        return _lookup(self, "_bucket_by_id", self.buckets)[bid]


def _lookup(g, attr, items):
    table = g.__dict__.get(attr)
    if table is None:
        table = {x.id: x for x in items}
        object.__setattr__(g, attr, table)
    return table


def build_graph(ops: Iterable[OpNode], edges: Iterable[DataEdge] = (), allreduces=(), groups=None, buckets=None,
                meta: GraphMeta = GraphMeta()) -> HloGraph:
    """Unfused default state unless groups/buckets are given: group id = op
    id, bucket id = AllReduce id (graph.py:302-340)."""
    ops = tuple(sorted(ops, key=lambda o: o.id))
    edges = tuple(sorted(edges, key=lambda e: (e.src, e.dst)))
    triples = sorted(tuple(t) for t in allreduces)
    if groups is None:
        groups = [FusionGroup(o.id, frozenset((o.id,))) for o in ops]
    if buckets is None:
        specs = [(t[0], (t[0],)) for t in triples]
    else:
        specs = sorted((int(b), tuple(m)) for b, m in buckets)
    owner = {}
    for bid, members in specs:
        for m in members:
            owner[m] = bid
    size = {t[0]: t[2] for t in triples}
    ars = tuple(AllReduceInstr(i, p, n, owner.get(i, i)) for i, p, n in triples)
    bks = tuple(TensorBucket(bid, tuple(m), sum(size[x] for x in m if x in size)) for bid, m in specs)
    return HloGraph(meta, ops, edges, ars, tuple(sorted(groups, key=lambda x: x.id)), bks)


def with_fusion_state(g: HloGraph, groups, buckets=None, allreduces=None) -> HloGraph:
    """Same static graph, new fusion state (graph.py:746-760)."""
    return HloGraph(g.meta, g.ops, g.edges, g.allreduces if allreduces is None else tuple(allreduces),
                    tuple(sorted(groups, key=lambda x: x.id)),
                    g.buckets if buckets is None else tuple(sorted(buckets, key=lambda b: b.id)))


def canonical_hash(g: HloGraph) -> int:
    """64-bit digest with the reference's equality semantics (graph.py:559-580):
    graph content plus the fusion state with ids canonicalised away."""
    h = hashlib.blake2b(digest_size=8)
    h.update(repr((g.meta.name, g.meta.devices, g.meta.seed)).encode())
    for o in sorted(g.ops, key=lambda o: o.id):
        h.update(repr((o.id, o.op_code, o.kind, o.input_shape_key, o.out_bytes, o.compute_us)).encode())
    h.update(repr(sorted((e.src, e.dst, e.bytes) for e in g.edges)).encode())
    h.update(repr(sorted((a.id, a.producer_op, a.tensor_bytes) for a in g.allreduces)).encode())
    h.update(repr(sorted((tuple(sorted(x.member_ops)), tuple(sorted(x.duplicated_ops))) for x in g.groups)).encode())
    h.update(repr(sorted(tuple(sorted(b.members)) for b in g.buckets)).encode())
    return int.from_bytes(h.digest(), "little")


# ---------------------------------------------------------------------------
# JSON documents (the reference's format, graph.py:611-743)

_KEYS = {
    "top": {"meta", "ops", "edges", "allreduce", "groups", "buckets"},
    "meta": {"name", "devices", "seed"},
    "op": {"id", "op_code", "kind", "input_shape_key", "out_bytes", "compute_us"},
    "edge": {"src", "dst", "bytes"},
    "allreduce": {"id", "producer_op", "tensor_bytes"},
    "group": {"id", "members", "duplicated"},
    "bucket": {"id", "members"},
}


def _keys(obj, kind):
    extra = set(obj) - _KEYS[kind]
    if extra:
        raise GraphFormatError(f"{kind}: unknown keys {sorted(extra)}")


def graph_from_doc(doc: dict) -> HloGraph:
    if not isinstance(doc, dict):
        raise GraphFormatError("graph document must be an object")
    _keys(doc, "top")
    m = doc.get("meta", {})
    _keys(m, "meta")
    meta = GraphMeta(str(m.get("name", "unnamed")), int(m.get("devices", 2)), int(m.get("seed", 0)))
    try:
        ops = []
        for o in doc.get("ops", []):
            _keys(o, "op")
            cu = o.get("compute_us")
            ops.append(OpNode(int(o["id"]), str(o["op_code"]), str(o.get("kind", KIND_COMPUTE)),
                              str(o.get("input_shape_key", "")), int(o.get("out_bytes", 0)),
                              None if cu is None else float(cu)))
        edges = []
        for e in doc.get("edges", []):
            _keys(e, "edge")
            edges.append(DataEdge(int(e["src"]), int(e["dst"]), int(e.get("bytes", 0))))
        ars = []
        for a in doc.get("allreduce", []):
            _keys(a, "allreduce")
            ars.append((int(a["id"]), int(a["producer_op"]), int(a["tensor_bytes"])))
        groups = None
        if "groups" in doc:
            groups = []
            for x in doc["groups"]:
                _keys(x, "group")
                groups.append(FusionGroup(int(x["id"]), frozenset(int(v) for v in x["members"]),
                                          frozenset(int(v) for v in x.get("duplicated", []))))
        buckets = None
        if "buckets" in doc:
            buckets = []
            for b in doc["buckets"]:
                _keys(b, "bucket")
                buckets.append((int(b["id"]), [int(v) for v in b["members"]]))
    except (KeyError, TypeError, ValueError) as exc:
        raise GraphFormatError(f"bad graph record: {exc}") from exc
    return build_graph(ops, edges, ars, groups=groups, buckets=buckets, meta=meta)


def graph_to_doc(g: HloGraph, explicit_state: bool = False) -> dict:
    doc = {
        "meta": {"name": g.meta.name, "devices": g.meta.devices, "seed": g.meta.seed},
        "ops": [dict({"id": o.id, "op_code": o.op_code, "kind": o.kind, "input_shape_key": o.input_shape_key,
                      "out_bytes": o.out_bytes}, **({} if o.compute_us is None else {"compute_us": o.compute_us}))
                for o in g.ops],
        "edges": [{"src": e.src, "dst": e.dst, "bytes": e.bytes} for e in g.edges],
        "allreduce": [{"id": a.id, "producer_op": a.producer_op, "tensor_bytes": a.tensor_bytes}
                      for a in g.allreduces],
    }
    plain_groups = len(g.groups) == len(g.ops) and all(
        len(x.member_ops) == 1 and x.id in x.member_ops and not x.duplicated_ops for x in g.groups)
    if explicit_state or not plain_groups:
        doc["groups"] = [{"id": x.id, "members": sorted(x.member_ops), "duplicated": sorted(x.duplicated_ops)}
                         for x in g.groups]
    plain_buckets = len(g.buckets) == len(g.allreduces) and all(
        len(b.members) == 1 and b.id in b.members for b in g.buckets)
    if explicit_state or not plain_buckets:
        doc["buckets"] = [{"id": b.id, "members": sorted(b.members)} for b in g.buckets]
    return doc


def _open(path, mode):
    return gzip.open(path, mode + "t", encoding="utf-8") if str(path).endswith(".gz") else open(
        path, mode, encoding="utf-8")


def load_graph(path) -> HloGraph:
    with _open(path, "r") as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise GraphFormatError(f"{path}: not valid JSON") from exc
    return graph_from_doc(doc)


def save_graph(path, g: HloGraph, explicit_state: bool = False) -> None:
    with _open(path, "w") as fh:
        json.dump(graph_to_doc(g, explicit_state), fh, indent=1, sort_keys=True)
        fh.write("\n")


def state_arrays(g: HloGraph):
    """Fusion state of ``g`` as the C-ABI's three int32 arrays with compact,
    order-preserving ids (include/disco_b200.h).  Returns
    (ngid, rgid, bkt, gid_bound, group_ids, bucket_ids)."""
    import numpy as np

    op_index = {o.id: i for i, o in enumerate(sorted(g.ops, key=lambda o: o.id))}
    ar_index = {a.id: i for i, a in enumerate(sorted(g.allreduces, key=lambda a: a.id))}
    gids = sorted(x.id for x in g.groups)
    grank = {gid: i for i, gid in enumerate(gids)}
    V, A = len(op_index), len(ar_index)
    ng = np.full(V, -1, np.int32)
    rg = np.full(V, -1, np.int32)
    for x in g.groups:
        r = grank[x.id]
        for m in x.member_ops:
            if m in x.duplicated_ops:
                rg[op_index[m]] = r
            else:
                ng[op_index[m]] = r
    bids = sorted(b.id for b in g.buckets)
    brank = {b: i for i, b in enumerate(bids)}
    bk = np.full(A, -1, np.int32)
    for b in g.buckets:
        for m in b.members:
            bk[ar_index[m]] = brank[b.id]
    if V and (ng < 0).any():
        raise GraphFormatError("op without a normal group membership")
    if A and (bk < 0).any():
        raise GraphFormatError("AllReduce outside every bucket")
    return ng, rg, bk, max(len(gids), 1), gids, bids


def state_from_arrays(g: HloGraph, ngid, rgid, bkt) -> HloGraph:
    """Inverse of state_arrays for engine-produced states (group ids are the
    engine's compact ids, bucket ids are AllReduce ids of the min member)."""
    ops = sorted(g.ops, key=lambda o: o.id)
    ars = sorted(g.allreduces, key=lambda a: a.id)
    members, dups = {}, {}
    for i, o in enumerate(ops):
        members.setdefault(int(ngid[i]), set()).add(o.id)
        if rgid[i] >= 0:
            members.setdefault(int(rgid[i]), set()).add(o.id)
            dups.setdefault(int(rgid[i]), set()).add(o.id)
    # engine group ids are ranks over op indices; map them back to the
    # reference's convention (a group keeps the smallest id in its history,
    # replica ids count up from the largest op id)
    groups = [FusionGroup(gid, frozenset(m), frozenset(dups.get(gid, ()))) for gid, m in members.items()]
    bmembers = {}
    for i, a in enumerate(ars):
        bmembers.setdefault(int(bkt[i]), []).append(a.id)
    buckets = [(ars[b].id if b < len(ars) else b, sorted(m)) for b, m in bmembers.items()]
    size = {a.id: a.tensor_bytes for a in ars}
    owner = {m: bid for bid, ms in buckets for m in ms}
    new_ars = tuple(AllReduceInstr(a.id, a.producer_op, a.tensor_bytes, owner[a.id]) for a in ars)
    bks = tuple(TensorBucket(bid, tuple(ms), sum(size[m] for m in ms)) for bid, ms in sorted(buckets))
    return HloGraph(g.meta, g.ops, g.edges, new_ars, tuple(sorted(groups, key=lambda x: x.id)), bks)


class ModuleStats(NamedTuple):
    total_compute_us: float
    total_comm_us: float
    op_count: int
    bucket_count: int


def module_stats(g: HloGraph, costs, comm) -> ModuleStats:
    """Exact compute/communication totals from per-group and per-bucket
    durations (graph.py:583-601); builtin sum in group/bucket order, as the
    reference sums them."""
    from .errors import MissingCost

    for gr in g.groups:
        if gr.id not in costs:
            raise MissingCost(f"no duration for group {gr.id}")
    for b in g.buckets:
        if b.id not in comm:
            raise MissingCost(f"no duration for bucket {b.id}")
    return ModuleStats(
        total_compute_us=float(sum(costs[gr.id] for gr in g.groups)),
        total_comm_us=float(sum(comm[b.id] for b in g.buckets)),
        op_count=len(g.groups),
        bucket_count=len(g.buckets),
    )
