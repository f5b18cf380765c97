"""Heuristic baselines (search.py:228-302) -- greedy_postorder_fusion and
threshold_allreduce_fusion -- against the unmodified reference's outputs
(tests/golden/baselines.json.gz, sweep_gpt2m.json.gz) and its own unit tests
(test_search.py:222-279).  Without cost providers both run on the host engine
only; the simulated-order threshold scan needs the device simulator."""

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200.graph import DataEdge, OpNode, build_graph

from _golden import canon_doc, canon_graph, graph_with_state, read

MB = 1024 * 1024
NAMES = ["chain24", "residual40", "attention36", "recurrent30", "vgg16", "resnet50", "bert"]


def _doc():
    return read("baselines.json.gz")


def op(i, code="Mul", kind="compute", out=1024, us=10.0):
    return OpNode(id=i, op_code=code, kind=kind, input_shape_key=f"k{i}", out_bytes=out, compute_us=us)


def chain(n):
    return build_graph([op(i) for i in range(n)], [DataEdge(i, i + 1, 1024) for i in range(n - 1)])


def comm_heavy_graph(n_tensors=5, tensor_bytes=64 * 1024):
    ops = [op(i, code="GradW", us=5.0, out=tensor_bytes) for i in range(n_tensors)]
    edges = [DataEdge(i, i + 1, 1024) for i in range(n_tensors - 1)]
    return build_graph(ops, edges, [(t, t, tensor_bytes) for t in range(n_tensors)])


@pytest.mark.parametrize("name", NAMES)
def test_greedy_matches_reference(name):
    g = P.load_workload(name)[0]
    ent = _doc()[name]
    for start in ("unfused", "cand3"):
        x = graph_with_state(g, ent["starts"][start])
        assert canon_graph(P.greedy_postorder_fusion(x)) == canon_doc(g, ent["greedy"][start]), start


@pytest.mark.parametrize("name", NAMES)
def test_threshold_production_order_matches_reference(name):
    g = P.load_workload(name)[0]
    ent = _doc()[name]
    for row in ent["threshold"]:
        x = graph_with_state(g, ent["starts"][row["start"]])
        got = P.threshold_allreduce_fusion(x, row["T"])
        assert canon_graph(got) == canon_doc(g, row["topo"]), (row["start"], row["T"])


def test_greedy_gpt2_matches_reference():
    """The GPT-2-medium greedy parent of the bucket-size sweep (BASELINE configs[3])."""
    g = P.load_workload("gpt2m")[0]
    doc = read("sweep_gpt2m.json.gz")
    assert canon_graph(P.greedy_postorder_fusion(g)) == canon_doc(g, doc["greedy"]["state"])


def test_greedy_fuses_whole_chain():
    out = P.greedy_postorder_fusion(chain(3))
    assert len(out.groups) == 1


def test_greedy_never_crosses_parameter():
    ops = [op(0), op(1, kind="parameter", us=None), op(2)]
    g = build_graph(ops, [DataEdge(0, 1, 10), DataEdge(1, 2, 10)])
    out = P.greedy_postorder_fusion(g)
    owner = {m: x.id for x in out.groups for m in x.member_ops if m not in x.duplicated_ops}
    assert owner[1] != owner[0]
    for x in out.groups:
        if len(x.member_ops) > 1:
            assert all(out.op(m).kind == "compute" for m in x.member_ops)


def test_threshold_no_merges_when_all_large():
    out = P.threshold_allreduce_fusion(comm_heavy_graph(4, 4 * MB), 1 * MB)
    assert len(out.buckets) == 4


def test_threshold_greedy_scan():
    out = P.threshold_allreduce_fusion(comm_heavy_graph(5, 1 * MB), 3 * MB)
    assert sorted(b.total_bytes for b in out.buckets) == [2 * MB, 3 * MB]


def test_threshold_infinite_single_bucket():
    out = P.threshold_allreduce_fusion(comm_heavy_graph(5, 1 * MB), 10**15)
    assert len(out.buckets) == 1 and out.buckets[0].total_bytes == 5 * MB


def test_threshold_rejects_non_positive():
    with pytest.raises(P.InvalidConfig):
        P.threshold_allreduce_fusion(comm_heavy_graph(), 0)


# --- simulated production order (device simulator) -----------------------------


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_threshold_simulated_order_matches_reference(name):
    from paper_2209_12769_b200 import make_cost_providers

    g, prof, comm, mp, lin = P.load_workload(name)
    import paper_2209_12769_b200._native as N

    cp = make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
    ent = _doc()[name]
    for row in ent["threshold"]:
        x = graph_with_state(g, ent["starts"][row["start"]])
        got = P.threshold_allreduce_fusion(x, row["T"], cp)
        assert canon_graph(got) == canon_doc(g, row["sim"]), (row["start"], row["T"])


@pytest.mark.gpu
def test_threshold_with_python_providers():
    cp = P.CostProviders(op_cost=lambda graph, gr: sum(graph.op(m).compute_us for m in gr.member_ops),
                         comm_cost=lambda graph, b: 1.0)
    out = P.threshold_allreduce_fusion(comm_heavy_graph(5, 1 * MB), 3 * MB, cp)
    assert sorted(b.total_bytes for b in out.buckets) == [2 * MB, 3 * MB]


@pytest.mark.gpu
def test_gpt2_sweep_parents_built_natively():
    """BASELINE configs[3] parents produced by this package (not read from the
    fixture): threshold AR fusion of the unfused and of the greedy graph."""
    from paper_2209_12769_b200 import make_cost_providers
    import paper_2209_12769_b200._native as N

    g, prof, comm, mp, lin = P.load_workload("gpt2m")
    cp = make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
    doc = read("sweep_gpt2m.json.gz")
    greedy = P.greedy_postorder_fusion(g)
    for ent in doc["sweep"][::4]:
        a = P.threshold_allreduce_fusion(g, ent["T"], cp)
        b = P.threshold_allreduce_fusion(greedy, ent["T"], cp)
        assert canon_graph(a) == canon_doc(g, ent["ar_only"]["state"]), ent["T"]
        assert canon_graph(b) == canon_doc(g, ent["both"]["state"]), ent["T"]
        np.testing.assert_allclose(P.cost(b, cp), ent["both"]["cost"], rtol=1e-12)


def test_module_stats_matches_reference_semantics():
    g = comm_heavy_graph(3, 1 * MB)
    costs = {x.id: 0.1 * (x.id + 1) for x in g.groups}
    comm = {b.id: 2.5 for b in g.buckets}
    st = P.module_stats(g, costs, comm)
    assert st == (sum(costs[x.id] for x in g.groups), 7.5, 3, 3)
    with pytest.raises(P.MissingCost):
        P.module_stats(g, {}, comm)


@pytest.mark.gpu
def test_report_lines_device_providers():
    from paper_2209_12769_b200 import make_cost_providers
    import paper_2209_12769_b200._native as N

    g, prof, comm, mp, lin = P.load_workload("vgg16")
    cp = make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
    lines = P.report_lines(g, cp, "x")
    assert lines[0] == f"[x] makespan_us {P.cost(g, cp):.6f}"
    assert lines[-1] == f"[x] groups {len(g.groups)} buckets {len(g.buckets)}"
