"""The rewrite primitives (fuse_nondup / fuse_dup / fuse_allreduce,
fusible_pairs / bucket_pairs / neighbors_allreduce, rewrite.py:49-219) through
the native engine, mirroring the reference's own rewrite tests
(test_rewrite.py:35-310).  The structural checks run on the host engine; the
timeline checks need the device simulator."""

import random

import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200.graph import DataEdge, OpNode, build_graph, canonical_hash
from paper_2209_12769_b200.rewrite import OptimizationMethod


def op(i, code="Mul", kind="compute", out=1024, us=10.0):
    return OpNode(id=i, op_code=code, kind=kind, input_shape_key=f"k{i}", out_bytes=out, compute_us=us)


def chain(n, allreduces=()):
    return build_graph([op(i) for i in range(n)], [DataEdge(i, i + 1, 1024) for i in range(n - 1)], allreduces)


def diamond():
    return build_graph([op(i) for i in range(4)],
                       [DataEdge(0, 1, 1024), DataEdge(0, 2, 1024), DataEdge(1, 3, 1024), DataEdge(2, 3, 1024)])


def normal_group_of(g, o):
    return next(x.id for x in g.groups if o in x.member_ops and o not in x.duplicated_ops)


def replica_group_of(g, o):
    return next(x.id for x in g.groups if o in x.duplicated_ops)


def fixed_costs(comm_us=None):
    return P.CostProviders(op_cost=lambda g, gr: sum(g.op(m).compute_us or 0.0 for m in gr.member_ops),
                           comm_cost=lambda g, b: 1.0 if comm_us is None else comm_us[b.id])


def random_dag(rng, n_ops=8, n_tensors=2, p_edge=0.35):
    ops = [op(i, us=round(rng.uniform(1, 40), 1), out=rng.randrange(256, 65536)) for i in range(n_ops)]
    edges = []
    for j in range(1, n_ops):
        preds = [i for i in range(j) if rng.random() < p_edge] or ([rng.randrange(j)] if rng.random() < 0.8 else [])
        edges += [DataEdge(i, j, ops[i].out_bytes) for i in preds]
    ars = [(t, p, 4096 * (t + 1)) for t, p in enumerate(rng.sample(range(n_ops), min(n_tensors, n_ops)))]
    return build_graph(ops, edges, ars)


def test_nondup_chain():
    out = P.fuse_nondup(chain(2), 1, 0)
    assert out.applied and len(out.graph.groups) == 1 and out.graph.groups[0].member_ops == {0, 1}


def test_nondup_rejects_cycle_via_alternate_path():
    g = diamond()
    out = P.fuse_nondup(g, 3, 1)
    assert out.applied
    merged = normal_group_of(out.graph, 3)
    again = P.fuse_nondup(out.graph, merged, 0)
    assert not again.applied and canonical_hash(again.graph) == canonical_hash(out.graph)
    assert P.fuse_nondup(out.graph, merged, 2).applied


def test_nondup_rejects_parameter_member_and_requires_adjacency():
    g = build_graph([op(0, kind="parameter", us=None), op(1)], [DataEdge(0, 1, 10)])
    out = P.fuse_nondup(g, 1, 0)
    assert not out.applied and "parameter" in out.description
    assert not P.fuse_nondup(chain(3), 2, 0).applied


def test_dup_fanout_creates_replica():
    g = build_graph([op(0, us=10.0), op(1, us=20.0), op(2, us=5.0)], [DataEdge(0, 1, 100), DataEdge(0, 2, 100)])
    out = P.fuse_dup(g, 1, 0)
    assert out.applied
    assert frozenset({0, 1}) in {frozenset(x.member_ops) for x in out.graph.groups}
    assert out.graph.group(replica_group_of(out.graph, 0)).duplicated_ops == {0}
    work = sum(out.graph.op(m).compute_us for x in out.graph.groups for m in x.member_ops)
    assert work == 10.0 + 20.0 + 5.0 + 10.0  # the replica is paid for again


def test_dup_single_consumer_degrades_to_nondup():
    g = chain(2)
    out = P.fuse_dup(g, 1, 0)
    assert out.applied and len(out.graph.groups) == 1 and not out.graph.groups[0].duplicated_ops
    assert canonical_hash(out.graph) == canonical_hash(P.fuse_nondup(g, 1, 0).graph)


def test_dup_rejects_predecessor_with_replica_members():
    ops = [op(0, us=10.0), op(1, us=20.0), op(2, us=5.0), op(3, us=5.0)]
    g = build_graph(ops, [DataEdge(0, 1, 100), DataEdge(0, 2, 100), DataEdge(0, 3, 100)])
    first = P.fuse_dup(g, 1, 0)
    assert first.applied
    second = P.fuse_dup(first.graph, normal_group_of(first.graph, 2), replica_group_of(first.graph, 0))
    assert not second.applied


def test_neighbors():
    assert P.neighbors_allreduce(build_graph([op(0), op(1)], [], [(0, 0, 100), (1, 1, 100)]), 0) == set()
    g = chain(2, allreduces=[(0, 0, 100), (1, 1, 100)])
    assert P.neighbors_allreduce(g, 0) == {1} and P.neighbors_allreduce(g, 1) == {0}
    rng = random.Random(23)
    for _ in range(20):  # the relation is symmetric
        g = random_dag(rng, n_ops=rng.randrange(3, 10), n_tensors=rng.randrange(2, 4))
        for b in g.buckets:
            for other in P.neighbors_allreduce(g, b.id):
                assert b.id in P.neighbors_allreduce(g, other)


def test_fuse_allreduce():
    g = chain(2, allreduces=[(0, 0, 300), (1, 1, 200)])
    out = P.fuse_allreduce(g, 0, 1)
    assert out.applied and len(out.graph.buckets) == 1 and out.graph.buckets[0].total_bytes == 500
    assert all(a.bucket == out.graph.buckets[0].id for a in out.graph.allreduces)
    with pytest.raises(P.NotNeighbors):
        P.fuse_allreduce(g, 0, 0)
    with pytest.raises(P.NotNeighbors):
        P.fuse_allreduce(build_graph([op(0), op(1)], [], [(0, 0, 100), (1, 1, 100)]), 0, 1)
    g3 = chain(3, allreduces=[(0, 0, 100), (1, 1, 100), (2, 2, 100)])
    assert P.neighbors_allreduce(g3, 0) == {1}
    out = P.fuse_allreduce(g3, 0, 1)
    merged = next(b.id for b in out.graph.buckets if len(b.members) == 2)
    assert 2 in P.neighbors_allreduce(out.graph, merged)
    out2 = P.fuse_allreduce(out.graph, merged, 2)
    assert out2.applied and len(out2.graph.buckets) == 1 and out2.graph.buckets[0].total_bytes == 300


def test_same_group_tensors_stay_neighbors():
    g = chain(2, allreduces=[(0, 0, 100), (1, 1, 100)])
    fused = P.fuse_nondup(g, 1, 0)
    assert fused.applied and P.neighbors_allreduce(fused.graph, 0) == {1}
    assert len(P.fuse_allreduce(fused.graph, 0, 1).graph.buckets) == 1


def test_update_cannot_fuse_into_its_producer():
    g = build_graph([op(0, us=10.0), op(1, code="ApplyGrad", us=1.0)], [DataEdge(0, 1, 100)], [(0, 0, 1000)])
    out = P.fuse_nondup(g, 1, 0)
    assert not out.applied and "cyclic" in out.description


def test_pairs_match_random_apply_choices():
    """fusible_pairs / bucket_pairs list exactly the choices random_apply draws
    from: one draw with randrange over the list picks the same rewrite."""
    rng = random.Random(3)
    for _ in range(20):
        g = random_dag(rng, n_ops=rng.randrange(4, 10), n_tensors=rng.randrange(2, 4))
        fp = P.fusible_pairs(g)
        if fp:
            seed = rng.randrange(1000)
            r = random.Random(seed)
            pick = fp[r.randrange(len(fp))]
            via_api = P.fuse_nondup(g, *pick)
            via_random = P.random_apply(g, OptimizationMethod.NON_DUPLICATE_FUSION, 1, random.Random(seed))
            assert via_api.applied == via_random.applied
            assert canonical_hash(via_api.graph) == canonical_hash(via_random.graph)


def test_bucket_bytes_conserved_and_work_accounting():
    rng = random.Random(9)
    g = random_dag(rng, n_ops=8, n_tensors=3)
    total = sum(b.total_bytes for b in g.buckets)
    cur = g
    for _ in range(30):
        m = rng.choice(list(OptimizationMethod))
        before = sum(cur.op(x).compute_us for gr in cur.groups for x in gr.member_ops)
        out = P.random_apply(cur, m, 1, rng)
        after = sum(out.graph.op(x).compute_us for gr in out.graph.groups for x in gr.member_ops)
        if m is OptimizationMethod.DUPLICATE_FUSION and out.applied:
            assert after >= before
        else:
            assert after == before
        cur = out.graph
        assert sum(b.total_bytes for b in cur.buckets) == total


# --- timelines on the device -------------------------------------------------

@pytest.mark.gpu
def test_nondup_other_consumer_waits_for_merged_group():
    g = build_graph([op(0, us=10.0), op(1, us=20.0), op(2, us=5.0)], [DataEdge(0, 1, 100), DataEdge(0, 2, 100)])
    out = P.fuse_nondup(g, 1, 0)
    tl = P.simulate(out.graph, fixed_costs())
    merged_end = next(e for gid, _, e in tl.compute_events if gid == normal_group_of(out.graph, 0))
    start2 = next(s for gid, s, _ in tl.compute_events if gid == normal_group_of(out.graph, 2))
    assert start2 == merged_end == 30.0


@pytest.mark.gpu
def test_dup_timelines():
    g = build_graph([op(0, us=10.0), op(1, us=20.0), op(2, us=5.0)], [DataEdge(0, 1, 100), DataEdge(0, 2, 100)])
    out = P.fuse_dup(g, 1, 0)
    tl = P.simulate(out.graph, fixed_costs())
    rep = replica_group_of(out.graph, 0)
    rep_end = next(e for gid, _, e in tl.compute_events if gid == rep)
    assert next(s for gid, s, _ in tl.compute_events if gid == normal_group_of(out.graph, 2)) == rep_end
    assert sum(e - s for _, s, e in tl.compute_events) == 10.0 + 20.0 + 5.0 + 10.0
    # an AllReduce of the duplicated producer starts when the replica finishes
    g2 = build_graph([op(0, us=10.0), op(1, us=20.0)], [DataEdge(0, 1, 100)], [(0, 0, 1000)])
    dup = P.fuse_dup(g2, 1, 0)
    tl2 = P.simulate(dup.graph, fixed_costs(comm_us={0: 15.0}))
    rep2 = replica_group_of(dup.graph, 0)
    rep2_end = next(e for gid, _, e in tl2.compute_events if gid == rep2)
    assert next(s for b, s, _ in tl2.comm_events if b == 0) == rep2_end == 10.0
