"""Feature-level estimator API against the unmodified reference
(tests/golden/features.json.gz, made by make_golden.py `features`):
featurize / group_io (estimator.py:157-191, graph.py:181-213) on the host,
predict_fused (estimator.py:462-470) and oracle_time (workloads.py:276-291)
on the device."""

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200.estimator import analytic_model

from _golden import graph_with_state, read

NAMES = ["chain24", "residual40", "attention36", "recurrent30", "vgg16", "resnet50", "bert"]


def _doc():
    return read("features.json.gz")


def _feat(d):
    return P.SubgraphFeatures(op_codes=tuple(d["op_codes"]), compute_us=tuple(d["compute_us"]),
                              in_bytes=tuple(d["in_bytes"]), out_bytes=tuple(d["out_bytes"]),
                              edges=tuple(tuple(e) for e in d["edges"]), member_count=d["member_count"],
                              total_compute_us=d["total_compute_us"], internal_bytes=d["internal_bytes"],
                              external_in_bytes=d["external_in_bytes"], external_out_bytes=d["external_out_bytes"],
                              longest_path_len=d["longest_path_len"])


def _rows(name):
    g, prof, comm, mp, lin = P.load_workload(name)
    for row in _doc()[name]:
        c = graph_with_state(g, row["state"])
        for ent in row["groups"]:
            yield c, c.group(ent["gid"]), ent, (prof, comm, mp, lin)


@pytest.mark.parametrize("name", NAMES)
def test_featurize_matches_reference(name):
    n = 0
    for c, gr, ent, (prof, *_rest) in _rows(name):
        assert P.featurize(c, gr, prof) == _feat(ent["features"]), ent["gid"]
        assert list(P.group_io(c, gr.id)) == ent["io"]
        n += 1
    assert n > 10


def test_featurize_unknown_op_raises():
    g, prof, *_ = P.load_workload("chain24")
    with pytest.raises(P.UnknownOp):
        P.featurize(g, g.groups[0], P.Profile({}))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_predict_fused_matches_reference(name):
    ana = analytic_model(5.0, 1.0 / 1024.0)
    for c, gr, ent, (prof, comm, mp, lin) in _rows(name):
        f = _feat(ent["features"])
        # fp64: MP to 1e-9 (matmul association differs from numpy's), the
        # closed forms to 1e-12
        np.testing.assert_allclose(P.predict_fused(mp, f), ent["mp"], rtol=1e-9, err_msg=f"mp {ent['gid']}")
        np.testing.assert_allclose(P.predict_fused(lin, f), ent["lin"], rtol=1e-12, err_msg=f"lin {ent['gid']}")
        np.testing.assert_allclose(P.predict_fused(ana, f), ent["analytic"], rtol=1e-12, err_msg=f"ana {ent['gid']}")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["residual40", "bert"])
def test_predict_fused_fp32(name):
    import paper_2209_12769_b200._native as N

    for c, gr, ent, (prof, comm, mp, lin) in _rows(name):
        f = _feat(ent["features"])
        np.testing.assert_allclose(P.predict_fused(mp, f, N.FO_PREC_FP32), ent["mp"], rtol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["residual40", "vgg16", "bert"])
def test_predict_fused_equals_scoring_path(name):
    """Feature-level prediction and the simulator's per-group duration are the
    same device computation."""
    import paper_2209_12769_b200._native as N

    g, prof, comm, mp, lin = P.load_workload(name)
    cp = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
    for row in _doc()[name]:
        c = graph_with_state(g, row["state"])
        dur = P.predict_fused_groups(cp, c)
        for gid, want in dur.items():
            got = P.predict_fused(mp, P.featurize(c, c.group(gid), prof))
            np.testing.assert_allclose(got, want, rtol=1e-12, err_msg=str(gid))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_oracle_time_matches_reference(name):
    hws = [P.HardwareParams(), P.HardwareParams(noise=0.05, seed=42)]
    for c, gr, ent, _ in _rows(name):
        for hw, want in zip(hws, ent["oracle"]):
            np.testing.assert_allclose(P.oracle_time(c, gr, hw), want, rtol=1e-12, err_msg=str(gr.id))


@pytest.mark.gpu
def test_predict_fused_shape_mismatch():
    g, prof, comm, mp, lin = P.load_workload("chain24")
    bad = P.EstimatorModel(mp.variant, dict(mp.params, W_emb=np.zeros((3, 3))), mp.vocab, mp.node_norm, None,
                           mp.layers, mp.hidden, mp.out_scale)
    f = P.featurize(g, g.groups[0], prof)
    with pytest.raises(P.DimensionMismatch):
        P.predict_fused(bad, f)


@pytest.mark.gpu
def test_predict_fused_empty_and_edge_free():
    g, prof, comm, mp, lin = P.load_workload("chain24")
    f = P.featurize(g, g.groups[3], prof)
    v = P.predict_fused(mp, f)
    assert v > 0
    ana = analytic_model(5.0, 1.0 / 1024.0)
    f0 = P.SubgraphFeatures((), (), (), (), (), 0, 0.0, 0, 0, 0, 0)
    assert P.predict_fused(ana, f0) == pytest.approx(5.0)


@pytest.mark.parametrize("name", NAMES)
def test_topo_order_matches_reference(name):
    """topo_order (graph.py:536-556) through the native engine (host only)."""
    g = P.load_workload(name)[0]
    for row in _doc()[name]:
        c = graph_with_state(g, row["state"])
        assert P.topo_order(c) == row["topo"]


def test_topo_order_cyclic_contraction_raises():
    from paper_2209_12769_b200.graph import DataEdge, FusionGroup, OpNode, build_graph

    ops = [OpNode(i, "Mul", input_shape_key=f"k{i}", out_bytes=8, compute_us=1.0) for i in range(3)]
    edges = [DataEdge(0, 1, 8), DataEdge(1, 2, 8)]
    g = build_graph(ops, edges, groups=[FusionGroup(0, frozenset([0, 2])), FusionGroup(1, frozenset([1]))])
    with pytest.raises(P.CycleError):
        P.topo_order(g)
    assert P.topo_order(build_graph(ops, edges)) == [0, 1, 2]
