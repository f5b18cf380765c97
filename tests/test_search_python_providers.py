"""backtracking_search / exhaustive_search with arbitrary Python CostProviders
(the reference accepts any provider object, search.py:84-225), mirroring the
reference's own search tests (test_search.py:41-215).  The callbacks run in
Python, simulate runs on the device, so these are GPU tests."""

import random

import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
from paper_2209_12769_b200.graph import DataEdge, FusionGroup, OpNode, build_graph, canonical_hash
from paper_2209_12769_b200.rewrite import OptimizationMethod
from paper_2209_12769_b200.search import _host_driven_search

pytestmark = pytest.mark.gpu


def op(i, code="Mul", kind="compute", out=1024, us=10.0):
    return OpNode(id=i, op_code=code, kind=kind, input_shape_key=f"k{i}", out_bytes=out, compute_us=us)


def chain(n):
    return build_graph([op(i) for i in range(n)], [DataEdge(i, i + 1, 1024) for i in range(n - 1)])


def fixed_costs(comm=lambda g, b: 1.0):
    return P.CostProviders(op_cost=lambda g, gr: sum(g.op(m).compute_us or 0.0 for m in gr.member_ops),
                           comm_cost=comm)


def comm_heavy_graph(n_tensors=5, tensor_bytes=64 * 1024):
    ops = [op(i, code="GradW", us=5.0, out=tensor_bytes) for i in range(n_tensors)]
    return build_graph(ops, [DataEdge(i, i + 1, 1024) for i in range(n_tensors - 1)],
                       [(t, t, tensor_bytes) for t in range(n_tensors)])


def test_single_op_graph_unchanged():
    g = chain(1)
    r = P.backtracking_search(g, P.SearchConfig(seed=1, max_unchanged=20), fixed_costs())
    assert canonical_hash(r.best_graph) == canonical_hash(g) and r.best_cost_us == 10.0


def test_allreduce_only_mask_improves_overhead_bound_graph():
    g = comm_heavy_graph()
    cp = fixed_costs(lambda graph, b: 1e-6 * b.total_bytes + 1000.0)
    initial = P.cost(g, cp)
    cfg = P.SearchConfig(alpha=1.1, beta=2, seed=3, max_unchanged=60, methods=(OptimizationMethod.ALLREDUCE_FUSION,))
    r = P.backtracking_search(g, cfg, cp)
    assert r.best_cost_us < initial
    assert len(r.best_graph.buckets) < len(g.buckets) and len(r.best_graph.groups) == len(g.groups)


@pytest.mark.parametrize("name", ["chain24", "residual40", "attention36"])
def test_never_worse_pruning_and_determinism(name):
    g = P.load_workload(name)[0]
    cp = fixed_costs(lambda graph, b: 0.002 * b.total_bytes + 50.0)
    cfg = P.SearchConfig(alpha=1.05, beta=4, seed=5, max_unchanged=60)
    r = P.backtracking_search(g, cfg, cp)
    assert r.best_cost_us <= P.cost(g, cp) + 1e-9
    assert r.best_cost_us >= P.fo_bound(r.best_graph, cp) - 1e-9
    for rec in r.trace:  # what entered the queue respected the bound at its moment
        if rec.enqueued:
            assert rec.cost_us <= cfg.alpha * rec.best_cost_us
    r2 = P.backtracking_search(g, cfg, cp)
    assert r2.trace == r.trace and r2.candidates_evaluated == r.candidates_evaluated


@pytest.mark.parametrize("name", ["chain24", "recurrent30"])
def test_host_driver_equals_native_driver(name):
    """The one-candidate-at-a-time driver reproduces the native lock-stepped
    driver exactly when both score with the same device providers."""
    g, prof, comm, mp, lin = P.load_workload(name)
    cp = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
    cfg = P.SearchConfig(alpha=1.05, beta=6, seed=2, max_unchanged=40)
    a = P.backtracking_search(g, cfg, cp)
    b = _host_driven_search(g, cfg, cp)
    assert (a.steps, a.candidates_evaluated, a.candidates_enqueued) == (b.steps, b.candidates_evaluated,
                                                                         b.candidates_enqueued)
    assert [(t.step, t.action, t.queue_len, t.enqueued) for t in a.trace] == [
        (t.step, t.action, t.queue_len, t.enqueued) for t in b.trace]
    assert [t.cost_us for t in a.trace] == pytest.approx([t.cost_us for t in b.trace], rel=1e-12)


def test_exhaustive_small_cases():
    cp = fixed_costs()
    assert canonical_hash(P.exhaustive_search(chain(1), cp).best_graph) == canonical_hash(chain(1))
    g = chain(2)
    r = P.exhaustive_search(g, cp)
    fused = build_graph(g.ops, g.edges, groups=[FusionGroup(0, frozenset({0, 1}))])
    assert r.best_cost_us == min(P.cost(g, cp), P.cost(fused, cp)) and r.candidates_evaluated == 2
    with pytest.raises(P.LimitExceeded):
        P.exhaustive_search(chain(9), cp)


def test_exhaustive_dominates_backtracking():
    rng = random.Random(5)
    cp = P.oracle_providers(P.HardwareParams(), precision=N.FO_PREC_FP64)
    for seed in range(4):
        n = rng.randrange(4, 8)
        ops = [op(i, code="GradW" if i % 2 else "Mul", us=rng.uniform(2, 30), out=rng.randrange(512, 65536))
               for i in range(n)]
        edges = [DataEdge(i, i + 1, 256) for i in range(n - 1)]
        ars = [(t, 2 * t + 1, 4096 * (t + 1)) for t in range(min(2, n // 2))]
        g = build_graph(ops, edges, ars)
        exact = P.exhaustive_search(g, cp)
        found = P.backtracking_search(g, P.SearchConfig(alpha=1.1, beta=2, seed=seed, max_unchanged=60), cp)
        assert exact.best_cost_us <= found.best_cost_us + 1e-9


def _fig4():
    ops = [op(0, out=4096), op(1, out=4096), op(2, out=4096), op(3, code="ApplyGrad", us=1.0, out=4096)]
    edges = [DataEdge(0, 1, 4096), DataEdge(1, 2, 4096), DataEdge(0, 3, 4096)]
    return build_graph(ops, edges, [(0, 0, 4096), (1, 1, 4096), (2, 2, 4096)])


def _fig4_providers(per_byte, overhead, saving):
    def op_cost(graph, group):
        base = sum(graph.op(m).compute_us or 0.0 for m in group.member_ops)
        return max(0.1, base - saving * (len(group.member_ops) - 1))

    return P.CostProviders(op_cost=op_cost, comm_cost=lambda graph, b: per_byte * b.total_bytes + overhead)


def test_delayed_communication_branch():
    """test_search.py:201-221 (the paper's Fig. 4): comm-dominated costs keep
    the chain unfused; compute savings make fusing win."""
    g = _fig4()
    exact = P.exhaustive_search(g, _fig4_providers(25.0 / 4096, 0.1, 1.0))
    owner = {m: x for x in exact.best_graph.groups for m in x.member_ops if m not in x.duplicated_ops}
    for op_id in (0, 1, 2):
        assert owner[op_id].member_ops == {op_id}
    exact2 = P.exhaustive_search(g, _fig4_providers(1e-5, 0.05, 6.0))
    assert max(len(x.member_ops) for x in exact2.best_graph.groups) >= 3


@pytest.mark.parametrize("name", ["residual40", "bert", "gpt2m"])
def test_python_provider_durations_reach_every_node(name):
    """Regression: host-supplied durations (arbitrary Python providers) must
    reach every schedule node in the block-per-candidate geometry too, so the
    makespan is at least each lane's total work (fo_bound)."""
    g = P.load_workload(name)[0]
    cp = fixed_costs(lambda graph, b: 0.002 * b.total_bytes + 50.0)
    tl = P.simulate(g, cp)
    assert tl.makespan_us >= P.fo_bound(g, cp) - 1e-9
    assert len(tl.comm_events) == len(g.buckets)
    ev = {i: (s, e) for i, s, e in tl.comm_events}
    for b in g.buckets[:20]:  # end = start + duration (rounded at the magnitude of end)
        s0, e0 = ev[b.id]
        assert abs((e0 - s0) - (0.002 * b.total_bytes + 50.0)) <= 1e-12 * max(1.0, e0)
