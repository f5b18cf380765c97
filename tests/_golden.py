"""Shared helpers for the golden fixtures (tests/golden, made by make_golden.py)."""

import gzip
import json
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read(path):
    full = os.path.join(GOLDEN, path)
    if full.endswith(".gz"):
        with gzip.open(full, "rt") as fh:
            return json.load(fh)
    with open(full) as fh:
        return json.load(fh)


def cases(name):
    return read(f"cases/{name}.cases.json.gz")


def canon_doc(g, sdoc):
    """Canonical (groups, buckets) of a sparse fixture state: ids dropped,
    matching canonical_hash's equality semantics (graph.py:559-580)."""
    op_ids = sorted(o.id for o in g.ops)
    covered, groups = set(), set()
    for _, mem, dup in sdoc["groups"]:
        groups.add((tuple(sorted(mem)), tuple(sorted(dup))))
        covered |= set(mem) - set(dup)
    groups |= {((o,), ()) for o in op_ids if o not in covered}
    cov, buckets = set(), set()
    for _, mem in sdoc["buckets"]:
        buckets.add(tuple(sorted(mem)))
        cov |= set(mem)
    buckets |= {(a.id,) for a in g.allreduces if a.id not in cov}
    return groups, buckets


def canon_arrays(g, ng, rg, bk):
    """Canonical (groups, buckets) of engine arrays (ops / ARs in id order)."""
    op_ids = sorted(o.id for o in g.ops)
    ar_ids = sorted(a.id for a in g.allreduces)
    mem, dup = {}, {}
    for i, o in enumerate(op_ids):
        mem.setdefault(int(ng[i]), []).append(o)
        if rg[i] >= 0:
            mem.setdefault(int(rg[i]), []).append(o)
            dup.setdefault(int(rg[i]), []).append(o)
    groups = {(tuple(sorted(m)), tuple(sorted(dup.get(k, [])))) for k, m in mem.items()}
    b = {}
    for i, a in enumerate(ar_ids):
        b.setdefault(int(bk[i]), []).append(a)
    return groups, {tuple(sorted(m)) for m in b.values()}


def canon_graph(g):
    groups = {(tuple(sorted(x.member_ops)), tuple(sorted(x.duplicated_ops))) for x in g.groups}
    buckets = {tuple(sorted(b.members)) for b in g.buckets}
    return groups, buckets


def graph_with_state(g, sdoc):
    """The candidate graph of a fixture state (same static graph objects)."""
    from paper_2209_12769_b200.graph import FusionGroup, build_graph

    ops = sorted(o.id for o in g.ops)
    covered, groups = set(), []
    for gid, mem, dup in sdoc["groups"]:
        groups.append(FusionGroup(gid, frozenset(mem), frozenset(dup)))
        covered |= set(mem) - set(dup)
    groups += [FusionGroup(o, frozenset([o])) for o in ops if o not in covered]
    cov, buckets = set(), []
    for bid, mem in sdoc["buckets"]:
        buckets.append((bid, mem))
        cov |= set(mem)
    buckets += [(a.id, [a.id]) for a in g.allreduces if a.id not in cov]
    c = build_graph(g.ops, g.edges, [(a.id, a.producer_op, a.tensor_bytes) for a in g.allreduces], groups=groups,
                    buckets=buckets, meta=g.meta)
    # share the static tuples so device handles are reused
    object.__setattr__(c, "ops", g.ops)
    object.__setattr__(c, "edges", g.edges)
    return c
