"""Device parity: the CUDA scoring path (C-ABI library) against the reference's
golden vectors and the CPU oracle on the same inputs.  Run on a B200 with
``pytest -m gpu``.

Tolerances: fp32 message-passing estimator <= 1e-4 relative (north star);
fp64 estimator <= 1e-12 relative (different summation order than OpenBLAS);
analytic / hardware-oracle / linear providers and every schedule are fp64
max/+ arithmetic: bit-exact (rel 0) except linear (log1p, 1e-12).
"""

import random

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
from paper_2209_12769_b200.graph import DataEdge, FusionGroup, OpNode, build_graph

from _golden import canon_doc, canon_graph, cases, graph_with_state, read

pytestmark = pytest.mark.gpu

SMALL = ["chain24", "residual40", "attention36", "recurrent30", "vgg16", "resnet50", "bert"]
TOL = {("mp", N.FO_PREC_FP32): 1e-4, ("mp", N.FO_PREC_FP64): 1e-12, ("lin", N.FO_PREC_FP32): 1e-12,
       ("lin", N.FO_PREC_FP64): 1e-12, ("analytic", N.FO_PREC_FP32): 0.0, ("analytic", N.FO_PREC_FP64): 0.0,
       ("oracle", N.FO_PREC_FP32): 0.0, ("oracle", N.FO_PREC_FP64): 0.0}


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)


def providers(name, precision):
    g, prof, comm, mp, lin = P.load_workload(name)
    return g, {
        "mp": P.make_cost_providers(prof, comm, mp, precision=precision),
        "lin": P.make_cost_providers(prof, comm, lin, precision=precision),
        "analytic": P.make_cost_providers(prof, comm, P.analytic_model(5.0, 1 / 1024), precision=precision),
        "oracle": P.oracle_providers(P.HardwareParams(), precision=precision),
    }


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
@pytest.mark.parametrize("name", SMALL + ["gpt2m", "synth50k"])
def test_costs_match_reference(name, precision):
    g, cps = providers(name, precision)
    doc = cases(name)
    graphs = [graph_with_state(g, c["state"]) for c in doc["candidates"]]
    for pname, cp in cps.items():
        got = P.cost_batch(graphs, cp)
        ref = np.array([c["cost"][pname] for c in doc["candidates"]])
        tol = TOL[(pname, precision)]
        np.testing.assert_allclose(got, ref, rtol=tol, atol=0, err_msg=f"{name}/{pname}")
        assert P.cost(g, cp) == pytest.approx(doc["base_cost"][pname], rel=tol, abs=0)


@pytest.mark.parametrize("name", SMALL)
def test_fused_group_predictions_match_predict_fused(name):
    for precision in (N.FO_PREC_FP32, N.FO_PREC_FP64):
        g, cps = providers(name, precision)
        for c in cases(name)["candidates"][:16]:
            cand = graph_with_state(g, c["state"])
            for pname in ("mp", "lin", "analytic", "oracle"):
                pred = P.predict_fused_groups(cps[pname], cand)
                for f in c["fused"]:
                    assert pred[f["id"]] == pytest.approx(f[pname], rel=max(TOL[(pname, precision)], 1e-15))


@pytest.mark.parametrize("name", SMALL)
def test_timelines_match_reference(name):
    g, cps = providers(name, N.FO_PREC_FP64)
    for c in cases(name)["candidates"]:
        if "timeline" not in c:
            continue
        tl = P.simulate(graph_with_state(g, c["state"]), cps["mp"])
        ref = c["timeline"]
        assert [e[0] for e in tl.compute_events] == [e[0] for e in ref["compute"]]
        assert [e[0] for e in tl.comm_events] == [e[0] for e in ref["comm"]]
        for a, b in zip(tl.compute_events + tl.comm_events, [tuple(x) for x in ref["compute"] + ref["comm"]]):
            assert a[1] == pytest.approx(b[1], rel=1e-12, abs=1e-9) and a[2] == pytest.approx(b[2], rel=1e-12, abs=1e-9)
        assert tl.makespan_us == pytest.approx(ref["makespan"], rel=1e-12)


def test_full_batch_against_oracle_and_bounds():
    """BASELINE configs[1] at full size: 4096 ResNet-50 candidates scored in one
    batch; a 512-candidate sample checked against the C oracle, and every
    candidate against the size-independent bounds fo <= cost <= sum (test_simulator.py:112-122)."""
    from oracle.oracle import Oracle, load_workload

    g, cps = providers("resnet50", N.FO_PREC_FP32)
    cp = cps["mp"]
    dg = cp.device_graph(g)
    ng, rg, bk, gb = dg.make_candidates(np.arange(4096, dtype=np.uint64))
    cost, st = dg.score_host(ng, rg, bk, gb, N.FO_PREC_FP32)
    assert (st == 0).all()
    o = Oracle(load_workload("resnet50"), "mp")
    idx = np.arange(0, 4096, 8)
    sts, ref = o.cost_batch(*(np.stack([o.make_candidate(int(i))[j] for i in idx]) for j in range(3)))
    assert (sts == 0).all()
    np.testing.assert_allclose(cost[idx], ref, rtol=1e-4)
    # bounds through the durations the device used
    for k in range(0, 4096, 64):
        st2, dur, G, bad = dg.node_durations_arrays(ng[k], rg[k], bk[k], gb, N.FO_PREC_FP32)
        B = len(set(bk[k].tolist()))
        lo = max(dur[:G].sum(), dur[G:G + B].sum())
        assert lo <= cost[k] * (1 + 1e-12) and cost[k] <= dur[:G + B].sum() * (1 + 1e-12)


def test_device_and_host_entry_points_agree():
    import torch

    g, cps = providers("bert", N.FO_PREC_FP32)
    dg = cps["mp"].device_graph(g)
    ng, rg, bk, gb = dg.make_candidates(np.arange(300, dtype=np.uint64))
    c1, s1 = dg.score_host(ng, rg, bk, gb)
    d = [torch.from_numpy(x).cuda() for x in (ng, rg, bk)]
    c2 = torch.empty(300, dtype=torch.float64, device="cuda")
    s2 = torch.empty(300, dtype=torch.int32, device="cuda")
    dg.score_device(d[0], d[1], d[2], gb, c2, s2)
    torch.cuda.synchronize()
    assert np.array_equal(c1, c2.cpu().numpy()) and np.array_equal(s1, s2.cpu().numpy())


@pytest.mark.parametrize("path", [p for p in __import__("glob").glob(
    __import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "search", "*.search.json.gz"))],
    ids=lambda p: p.split("/")[-1].split(".search")[0])
def test_search_trace_bit_exact(path):
    d = read(path.split("golden/")[1])
    g, cps = providers(d["workload"], N.FO_PREC_FP64)
    cfg = P.SearchConfig(alpha=d["cfg"]["alpha"], beta=d["cfg"]["beta"], max_unchanged=d["cfg"]["max_unchanged"],
                         seed=d["cfg"]["seed"])
    r = P.backtracking_search(g, cfg, cps[d["provider"]])
    assert (r.steps, r.candidates_evaluated, r.candidates_enqueued) == (
        d["steps"], d["candidates_evaluated"], d["candidates_enqueued"])
    assert len(r.trace) == len(d["trace"])
    for a, b in zip(r.trace, d["trace"]):
        assert (a.step, a.action, a.queue_len, a.enqueued) == (b[0], b[1], b[4], b[5])
        assert a.cost_us == pytest.approx(b[2], rel=1e-12) and a.best_cost_us == pytest.approx(b[3], rel=1e-12)
    assert canon_graph(r.best_graph) == canon_doc(g, d["best_state"])
    assert r.best_cost_us == pytest.approx(d["best_cost_us"], rel=1e-12)


@pytest.mark.parametrize("name,prov", [("chain24", "mp"), ("residual40", "analytic"), ("recurrent30", "oracle")])
def test_lockstep_seeds_equal_single_seed_oracle(name, prov):
    """R lock-stepped searches scored in shared batches: each seed's trajectory
    equals the oracle's single-seed Alg. 1 run with that seed."""
    from oracle.oracle import Oracle, load_workload

    g, cps = providers(name, N.FO_PREC_FP64)
    cfg = P.SearchConfig(alpha=1.05, beta=6, max_unchanged=50)
    seeds = list(range(12))
    res = P.lockstep_search(g, cfg, cps[prov], seeds)
    o = Oracle(load_workload(name), prov)
    for s, r in zip(seeds, res):
        ref = o.search(alpha=1.05, beta=6, max_unchanged=50, seed=s)
        assert (r.steps, r.candidates_evaluated, r.candidates_enqueued) == (
            ref["steps"], ref["candidates_evaluated"], ref["candidates_enqueued"])
        assert [(t.step, t.action, t.queue_len, t.enqueued) for t in r.trace] == [
            (t[0], t[1], t[4], t[5]) for t in ref["trace"]]
        np.testing.assert_allclose([t.cost_us for t in r.trace], [t[2] for t in ref["trace"]], rtol=1e-12)


def test_exhaustive_search_matches_reference():
    from paper_2209_12769_b200.graph import graph_from_doc

    for case in read("exhaustive.json.gz"):
        g = graph_from_doc(case["graph"])
        if case["provider"] == "oracle":
            cp = P.oracle_providers(P.HardwareParams())
        else:
            prof = P.Profile({(a, b): v for a, b, v in case["profile"]})
            cp = P.make_cost_providers(prof, P.CommModelParams(0.001, 100.0), P.analytic_model(5.0, 1 / 1024))
        r = P.exhaustive_search(g, cp)
        assert r.candidates_evaluated == case["candidates_evaluated"]
        assert r.steps == case["steps"]
        assert r.best_cost_us == pytest.approx(case["best_cost_us"], rel=1e-12)
        assert canon_graph(r.best_graph) == canon_doc(g, case["best_state"])


# ---- the reference's own simulator tests (test_simulator.py) through the device

def op(i, code="Mul", kind="compute", out=1024, us=10.0, key=None):
    return OpNode(id=i, op_code=code, kind=kind, input_shape_key=key if key is not None else f"k{i}",
                  out_bytes=out, compute_us=us)


def chain(n, us=10.0, out=1024, allreduces=()):
    return build_graph([op(i, us=us, out=out) for i in range(n)], [DataEdge(i, i + 1, out) for i in range(n - 1)],
                       allreduces)


def fixed_costs(op_us=None, comm_us=None):
    def op_cost(g, group):
        return sum((op_us[m] if op_us is not None else (g.op(m).compute_us or 0.0)) for m in group.member_ops)

    def comm_cost(g, bucket):
        return 1.0 if comm_us is None else comm_us[bucket.id]

    return P.CostProviders(op_cost=op_cost, comm_cost=comm_cost)


def test_serial_chain():
    tl = P.simulate(chain(2), fixed_costs(op_us={0: 10.0, 1: 20.0}))
    assert tl.compute_events == ((0, 0.0, 10.0), (1, 10.0, 30.0)) and tl.makespan_us == 30.0


def test_full_overlap_and_update_waits_for_bucket():
    g = build_graph([op(0, us=10.0), op(1, us=20.0)], [], [(0, 0, 1000)])
    tl = P.simulate(g, fixed_costs(comm_us={0: 15.0}))
    assert tl.compute_events == ((0, 0.0, 10.0), (1, 10.0, 30.0)) and tl.comm_events == ((0, 10.0, 25.0),)
    g = build_graph([op(0, us=10.0), op(2, code="ApplyGrad", us=5.0)], [DataEdge(0, 2, 1000)], [(0, 0, 1000)])
    tl = P.simulate(g, fixed_costs(comm_us={0: 15.0}))
    assert tl.comm_events == ((0, 10.0, 25.0),)
    assert next(e for e in tl.compute_events if e[0] == 2) == (2, 25.0, 30.0) and tl.makespan_us == 30.0


def test_comm_fifo_by_ready_time_and_zero_durations():
    g = build_graph([op(0, us=5.0), op(1, us=50.0)], [], [(0, 1, 100), (1, 0, 100)])
    tl = P.simulate(g, fixed_costs(comm_us={0: 10.0, 1: 10.0}))
    assert tl.comm_events[0] == (1, 5.0, 15.0) and tl.comm_events[1] == (0, 55.0, 65.0)
    tl = P.simulate(chain(2), fixed_costs(op_us={0: 0.0, 1: 0.0}))
    assert tl.makespan_us == 0.0 and tl.compute_events == ((0, 0.0, 0.0), (1, 0.0, 0.0))


def test_empty_graph_and_format_timeline():
    assert P.cost(build_graph([], [], []), fixed_costs()) == 0.0
    text = P.format_timeline(P.simulate(build_graph([op(0, us=10.0)], [], [(0, 0, 100)]), fixed_costs(comm_us={0: 4.0})))
    lines = text.strip().splitlines()
    assert lines[0] == "kind id start_us end_us" and lines[1].startswith("compute 0 0.000000")
    assert lines[-1] == "makespan_us 14.000000"


def test_bounds_on_random_graphs():
    rng = random.Random(77)
    for _ in range(60):
        n = rng.randrange(2, 14)
        ops = [op(i, us=round(rng.uniform(1, 40), 1), out=rng.randrange(256, 65536)) for i in range(n)]
        edges = [DataEdge(i, j, 64) for j in range(1, n) for i in range(j) if rng.random() < 0.35]
        ars = [(t, p, 1000) for t, p in enumerate(rng.sample(range(n), min(rng.randrange(0, 4), n)))]
        g = build_graph(ops, edges, ars)
        comm = {b.id: rng.uniform(0.5, 60.0) for b in g.buckets}
        cp = fixed_costs(comm_us=comm)
        c = P.cost(g, cp)
        assert P.fo_bound(g, cp) <= c + 1e-9
        assert c <= sum(o.compute_us for o in ops) + sum(comm.values()) + 1e-9


def test_error_mapping():
    g = chain(1)
    with pytest.raises(ValueError):
        P.simulate(g, P.CostProviders(op_cost=lambda g, gr: -1.0, comm_cost=lambda g, b: 1.0))

    def boom(g, gr):
        raise KeyError("nope")

    with pytest.raises(P.MissingCost):
        P.simulate(g, P.CostProviders(op_cost=boom, comm_cost=lambda g, b: 1.0))
    # fused group with no estimator -> MissingCost (estimator.py:815-818)
    fused = build_graph(chain(2).ops, chain(2).edges, groups=[FusionGroup(0, frozenset({0, 1}))])
    prof = P.Profile({("Mul", "k0"): 10.0, ("Mul", "k1"): 12.0})
    with pytest.raises(P.MissingCost):
        P.cost(fused, P.make_cost_providers(prof, P.CommModelParams(0.0, 1.0), None))
    # missing profile entry -> MissingCost via UnknownOp (simulator.py:45-46)
    with pytest.raises(P.MissingCost):
        P.cost(chain(2), P.make_cost_providers(P.Profile({("Mul", "k0"): 10.0}), P.CommModelParams(0.0, 1.0)))
    # an update op fused into its gradient producer deadlocks -> CycleError (test_rewrite.py:216-224)
    ops = [op(0, us=10.0), op(1, code="ApplyGrad", us=1.0)]
    cyc = build_graph(ops, [DataEdge(0, 1, 100)], [(0, 0, 1000)], groups=[FusionGroup(0, frozenset({0, 1}))])
    with pytest.raises(P.CycleError):
        P.simulate(cyc, P.oracle_providers(P.HardwareParams()))


def test_int16_encoding_matches_int32():
    import torch

    g, cps = providers("resnet50", N.FO_PREC_FP32)
    dg = cps["mp"].device_graph(g)
    ng, rg, bk, gb = dg.make_candidates(np.arange(512, dtype=np.uint64))
    c32, s32 = dg.score_host(ng, rg, bk, gb)
    c16, s16 = dg.score_host(ng.astype(np.int16), rg.astype(np.int16), bk.astype(np.int16), gb)
    assert np.array_equal(c32, c16) and np.array_equal(s32, s16)
    d = [torch.from_numpy(x.astype(np.int16)).cuda() for x in (ng, rg, bk)]
    c = torch.empty(512, dtype=torch.float64, device="cuda")
    s = torch.empty(512, dtype=torch.int32, device="cuda")
    dg.score_device(d[0], d[1], d[2], gb, c, s)
    torch.cuda.synchronize()
    assert np.array_equal(c.cpu().numpy(), c32)


def test_gpt2_sweep_parents_match_reference():
    """BASELINE configs[3]: the bucket-size sweep parents (threshold AR fusion on
    the unfused and on the greedily op-fused GPT-2 graph).  The greedy parent
    holds fused groups of thousands of ops (the large-group second pass)."""
    doc = read("sweep_gpt2m.json.gz")
    for precision in (N.FO_PREC_FP32, N.FO_PREC_FP64):
        g, cps = providers("gpt2m", precision)
        graphs, ref = [graph_with_state(g, doc["greedy"]["state"])], [doc["greedy"]["cost"]]
        for ent in doc["sweep"]:
            for kind in ("ar_only", "both"):
                graphs.append(graph_with_state(g, ent[kind]["state"]))
                ref.append(ent[kind]["cost"])
        got = P.cost_batch(graphs, cps["mp"])
        np.testing.assert_allclose(got, ref, rtol=1e-4 if precision == N.FO_PREC_FP32 else 1e-12)


def test_estimator_memo_is_exact():
    """Memo hits return the very prediction computed for the same member set."""
    g, cps = providers("resnet50", N.FO_PREC_FP32)
    dg = cps["mp"].device_graph(g)
    ng, rg, bk, gb = dg.make_candidates(np.arange(1024, dtype=np.uint64))
    N.lib().fo_memo_enable(dg.h, 0)
    off, _ = dg.score_host(ng, rg, bk, gb)
    N.lib().fo_memo_enable(dg.h, 1)
    N.lib().fo_memo_clear(dg.h, None)
    cold, _ = dg.score_host(ng, rg, bk, gb)
    warm, _ = dg.score_host(ng, rg, bk, gb)
    assert np.array_equal(off, cold) and np.array_equal(off, warm)


def test_batch_best_and_pairs_best():
    import torch

    cost = torch.tensor([5.0, 2.0, 7.0, 2.0, 9.0], dtype=torch.float64, device="cuda")
    st = torch.tensor([0, 0, 0, 0, 0], dtype=torch.int32, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    N.lib().fo_batch_best(N.ptr(cost), N.ptr(st), 5, 100, N.ptr(out), None)
    torch.cuda.synchronize()
    assert out.tolist() == [2.0, 101.0]  # strict <: lowest id among equal costs
    st[1] = 2  # a failed candidate is skipped
    N.lib().fo_batch_best(N.ptr(cost), N.ptr(st), 5, 100, N.ptr(out), None)
    torch.cuda.synchronize()
    assert out.tolist() == [2.0, 103.0]
    pairs = torch.tensor([3.0, 40.0, 1.0, 77.0, 1.0, 12.0, float("inf"), -1.0], dtype=torch.float64, device="cuda")
    N.lib().fo_pairs_best(N.ptr(pairs), 4, N.ptr(out), None)
    torch.cuda.synchronize()
    assert out.tolist() == [1.0, 12.0]


@pytest.mark.parametrize("name", ["resnet50", "bert", "gpt2m"])
def test_delta_scoring_equals_dense(name):
    """Sparse candidates against the resident parent score bit-identically to
    the dense encoding, from the unfused parent and from a fused one (the GPT-2
    greedy sweep parent holds groups of thousands of ops)."""
    import torch

    doc = read("sweep_gpt2m.json.gz") if name == "gpt2m" else None
    for precision in (N.FO_PREC_FP32, N.FO_PREC_FP64):
        g, cps = providers(name, precision)
        dg = cps["mp"].device_graph(g)
        bases = [None]
        if doc is not None:
            from paper_2209_12769_b200.graph import state_arrays

            x = graph_with_state(g, doc["sweep"][3]["both"]["state"])
            bases.append(state_arrays(x)[:3])
        for base in bases:
            seeds = np.arange(300, dtype=np.uint64)
            ng, rg, bk, gb = dg.make_candidates(seeds, base=base)
            dense, st0 = dg.score_host(ng, rg, bk, gb, precision)
            dg.set_parent(*(base if base is not None else (None, None, None)))
            off, chg = dg.make_candidates_delta(seeds, base=base)
            sparse, st1 = dg.score_delta_host(off, chg, precision)
            assert np.array_equal(st0, st1) and np.array_equal(dense, sparse), (name, precision)
            c = torch.empty(len(seeds), dtype=torch.float64, device="cuda")
            s = torch.empty(len(seeds), dtype=torch.int32, device="cuda")
            dg.score_delta_device(torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda(), c, s, precision)
            torch.cuda.synchronize()
            assert np.array_equal(c.cpu().numpy(), dense)


def test_pipelined_delta_submissions_equal_sync():
    """fo_score_delta_submit / fo_score_wait: several batches in flight (two
    slots, so the third submission waits for the first) give the synchronous
    call's results, per batch and in any wait order."""
    import torch

    g, cps = providers("resnet50", N.FO_PREC_FP32)
    dg = cps["mp"].device_graph(g)
    dg.set_parent()
    batches = []
    for b in range(5):
        seeds = np.arange(b * 700, b * 700 + 600 + 37 * b, dtype=np.uint64)
        off, chg = dg.make_candidates_delta(seeds)
        ref, st_ref = dg.score_delta_host(off, chg)
        h = [torch.from_numpy(off).pin_memory(), torch.from_numpy(chg).pin_memory(),
             torch.zeros(len(seeds), dtype=torch.float64).pin_memory(),
             torch.full((len(seeds),), -1, dtype=torch.int32).pin_memory()]
        batches.append((h, ref, st_ref))
    tickets = [dg.score_delta_submit(*(x for x in h), clear_memo=(i % 2 == 0)) for i, (h, _, _) in enumerate(batches)]
    for t in reversed(tickets):
        dg.score_wait(t)
    for h, ref, st_ref in batches:
        assert np.array_equal(h[3].numpy(), st_ref) and np.array_equal(h[2].numpy(), ref)
    # a synchronous call between submissions is ordered with them
    h, ref, _ = batches[0]
    h[2].zero_()
    t = dg.score_delta_submit(*h)
    mid, _ = dg.score_delta_host(h[0].numpy(), h[1].numpy())
    dg.score_wait(t)
    assert np.array_equal(h[2].numpy(), ref) and np.array_equal(mid, ref)
    with pytest.raises(Exception):
        dg.score_wait(10**9)


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
def test_pipelined_bench_batches_on_two_streams_equal_sync(precision):
    """Bench-sized batches (4,096 candidates) submitted back to back: the
    submissions alternate between two compute streams with their own scratch
    and memo tables (each cleared per batch), and every batch equals the
    synchronous call."""
    import torch

    g, cps = providers("resnet50", precision)
    dg = cps["mp"].device_graph(g)
    dg.set_parent()
    batches = []
    for b in range(6):
        off, chg = dg.make_candidates_delta(np.arange(b * 4096, (b + 1) * 4096, dtype=np.uint64))
        ref, st_ref = dg.score_delta_host(off, chg, precision)
        h = [torch.from_numpy(off).pin_memory(), torch.from_numpy(chg).pin_memory(),
             torch.zeros(4096, dtype=torch.float64).pin_memory(), torch.full((4096,), -1, dtype=torch.int32).pin_memory()]
        batches.append((h, ref, st_ref))
    for rep in range(2):
        pending = []
        for h, ref, st_ref in batches:
            h[2].zero_()
            pending.append(dg.score_delta_submit(*h, precision=precision, clear_memo=True))
            if len(pending) == 2:
                dg.score_wait(pending.pop(0))
        for t in pending:
            dg.score_wait(t)
        for h, ref, st_ref in batches:
            assert np.array_equal(h[3].numpy(), st_ref) and np.array_equal(h[2].numpy(), ref)


def test_device_batches_on_scratch_slots_equal_serial():
    """fo_score_delta_slot: device-resident batches on the three scratch slots,
    each on its own stream and running concurrently (memo cleared per batch),
    equal the serial fo_score_delta of the same batch; slot ids are checked."""
    import torch

    g, cps = providers("resnet50", N.FO_PREC_FP32)
    dg = cps["mp"].device_graph(g)
    dg.set_parent()
    batches = []
    for b in range(6):
        off, chg = dg.make_candidates_delta(np.arange(b * 4096, (b + 1) * 4096, dtype=np.uint64))
        batches.append((torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda()))
    refs = []
    for o, c in batches:
        cost = torch.empty(4096, dtype=torch.float64, device="cuda")
        st = torch.empty(4096, dtype=torch.int32, device="cuda")
        dg.score_delta_device(o, c, cost, st)
        torch.cuda.synchronize()
        refs.append((cost.cpu(), st.cpu()))
    streams = [torch.cuda.Stream() for _ in range(N.SUBMIT_SLOTS)]
    outs = [(torch.empty(4096, dtype=torch.float64, device="cuda"), torch.empty(4096, dtype=torch.int32, device="cuda"))
            for _ in batches]
    for i, (o, c) in enumerate(batches):
        k = i % N.SUBMIT_SLOTS
        dg.score_delta_slot(k, o, c, outs[i][0], outs[i][1], stream=streams[k].cuda_stream, clear_memo=True)
    torch.cuda.synchronize()
    for (cost, st), (rc, rs) in zip(outs, refs):
        assert torch.equal(cost.cpu(), rc) and torch.equal(st.cpu(), rs)
    with pytest.raises(Exception):
        dg.score_delta_slot(N.SUBMIT_SLOTS, *batches[0], *outs[0])


def test_delta_scoring_rejects_bad_input():
    g, cps = providers("vgg16", N.FO_PREC_FP32)
    dg = cps["mp"].device_graph(g)
    dg.set_parent()
    off = np.array([0, 1], np.int32)
    cost, st = dg.score_delta_host(off, np.array([[2 * dg.V + dg.A, 0]], np.int32))
    assert st[0] == N.FO_INVALID_ARG


@pytest.mark.parametrize("name", ["chain24", "residual40", "attention36", "vgg16", "resnet50", "bert"])
def test_hw_oracle_jitter_matches_reference(name):
    """oracle_providers with noise > 0: the reference's blake2b content-key
    jitter (workloads.py:254-291) reproduced on the device, per candidate cost
    and per group duration."""
    doc = read("jitter.json.gz")[name]
    g = P.load_workload(name)[0]
    cs = {c["i"]: c for c in cases(name)["candidates"]}
    for ent in doc:
        hw = P.HardwareParams(noise=ent["noise"], seed=ent["seed"])
        cp = P.oracle_providers(hw, precision=N.FO_PREC_FP64)
        graphs = [graph_with_state(g, cs[r["i"]]["state"]) for r in ent["rows"]]
        got = P.cost_batch(graphs, cp)
        ref = np.array([r["cost"] for r in ent["rows"]])
        np.testing.assert_allclose(got, ref, rtol=1e-15, atol=0)
        for r, x in zip(ent["rows"], graphs):
            if "groups" not in r:
                continue
            groups, _ = cp.node_durations(x)
            for gid, d in r["groups"]:
                assert groups[gid] == d, (name, ent["seed"], r["i"], gid)


def test_hw_oracle_jitter_is_deterministic_and_bounded():
    """test_workloads.py:134-145: jitter is a pure function of group content and
    stays within [1 - noise, 1 + noise] of the noise-free time."""
    g = P.load_workload("vgg16")[0]
    base = P.oracle_providers(P.HardwareParams(noise=0.0), precision=N.FO_PREC_FP64)
    noisy = P.oracle_providers(P.HardwareParams(noise=0.05, seed=77), precision=N.FO_PREC_FP64)
    a, _ = noisy.node_durations(g)
    b, _ = noisy.node_durations(g)
    c, _ = base.node_durations(g)
    assert a == b
    for gid, d in c.items():
        assert abs(a[gid] - d) <= 0.05 * d + 1e-12


@pytest.mark.parametrize("name", ["vgg16", "bert"])
def test_speculative_search_equals_plain(name, monkeypatch):
    """One-step speculation (FO_SEARCH_SPEC) changes only how many device round
    trips a search takes: traces, counters and results are identical."""
    g, cps = providers(name, N.FO_PREC_FP64)
    cfg = P.SearchConfig(alpha=1.05, beta=10, max_unchanged=60 if name == "bert" else 200)
    out = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("FO_SEARCH_SPEC", mode)
        res = P.lockstep_search(g, cfg, cps["mp"], [0, 1, 2])
        out[mode] = [(r.steps, r.candidates_evaluated, r.candidates_enqueued, r.best_cost_us,
                      [(t.step, t.action, t.cost_us, t.best_cost_us, t.queue_len, t.enqueued) for t in r.trace])
                     for r in res]
    assert out["0"] == out["1"]


def test_delta_scoring_needs_parent_and_handles_empty():
    g, prof, comm, mp, lin = P.load_workload("chain24")
    dg = P.make_cost_providers(prof, comm, mp).device_graph(g)  # fresh handle: no parent yet
    with pytest.raises(P.GraphFormatError):
        dg.score_delta_host(np.array([0, 0], np.int32), np.zeros((0, 2), np.int32))
    dg.set_parent()
    cost, st = dg.score_delta_host(np.zeros(1, np.int32), np.zeros((0, 2), np.int32))  # K = 0
    assert cost.shape == (0,)
    base, _ = dg.score_delta_host(np.array([0, 0], np.int32), np.zeros((0, 2), np.int32))  # the parent itself
    ng, rg, bk, vb, _, _ = __import__("paper_2209_12769_b200.graph", fromlist=["x"]).state_arrays(g)
    ref, _ = dg.score_host(ng[None], rg[None], bk[None], vb)
    assert base[0] == ref[0] and base[0] > 0


# ---- the reference's estimator known answers (test_estimator.py:101-139, :351-418)

KB = 1024


def _two_op_worked_example():
    """test_estimator.py:101-118: external 10 KB input -> op 1 (raw 100 us,
    50 KB out) -> op 2 (raw 200 us, 20 KB out); launch 5 us, 1 us per KB."""
    ops = [op(0, code="Src", out=10 * KB, us=1.0, key="src"), op(1, code="Mul", out=50 * KB, us=100.0, key="m1"),
           op(2, code="Mul", out=20 * KB, us=200.0, key="m2")]
    g = build_graph(ops, [DataEdge(0, 1, 10 * KB), DataEdge(1, 2, 50 * KB)])
    prof = P.Profile({("Src", "src"): 16.0, ("Mul", "m1"): 165.0, ("Mul", "m2"): 275.0})
    return g, prof


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
def test_analytic_worked_example(precision):
    g, prof = _two_op_worked_example()
    cp = P.make_cost_providers(prof, P.CommModelParams(0.0, 1.0), P.analytic_model(5.0, 1.0 / KB), precision)
    fused = build_graph(g.ops, g.edges, groups=[FusionGroup(0, frozenset({0})), FusionGroup(1, frozenset({1, 2}))])
    # unfused 165 + 275 = 440; fused keeps the 50 KB tensor on chip: 300 + 5 + 30 = 335
    assert P.predict_fused_groups(cp, fused)[1] == pytest.approx(335.0, rel=1e-12)
    # a singleton group is the profile lookup itself (estimator.py:810-814)
    assert cp.node_durations(g)[0][1] == 165.0


def _zero_mp_model(vocab=("Mul", "<other>"), hidden=4, layers=2, c3=1.7):
    feat = 6 + len(vocab)
    p = {"W_emb": np.zeros((hidden, feat)), "W_r": np.zeros((hidden, hidden)), "A1": np.zeros((hidden, hidden)),
         "c1": np.zeros(hidden), "A2": np.zeros((hidden, hidden)), "c2": np.zeros(hidden), "a3": np.zeros(hidden),
         "c3": np.array(c3)}
    for layer in range(1, layers + 1):
        p[f"W_{layer}"] = np.zeros((hidden, hidden))
    return P.EstimatorModel(P.EstimatorVariant.MESSAGE_PASSING, p, vocab=vocab, layers=layers, hidden=hidden)


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
def test_mp_zero_weights_constant_output(precision):
    """test_estimator.py:376-382: all-zero weights give softplus(c3) for any group."""
    rng = random.Random(6)
    expected = float(np.logaddexp(0, 1.7))
    for _ in range(5):
        n = rng.randrange(3, 9)
        g = build_graph([op(i, code=rng.choice(["Mul", "Conv2D"]), us=rng.uniform(1, 50)) for i in range(n)],
                        [DataEdge(i, i + 1, 64) for i in range(n - 1)])
        prof = P.Profile({(o.op_code, o.input_shape_key): o.compute_us for o in g.ops})
        cp = P.make_cost_providers(prof, P.CommModelParams(0.0, 1.0), _zero_mp_model(), precision)
        fused = build_graph(g.ops, g.edges, groups=[FusionGroup(0, frozenset(range(n)))])
        assert P.predict_fused_groups(cp, fused)[0] == pytest.approx(expected, rel=1e-6 if precision == N.FO_PREC_FP32 else 1e-15)


def test_mp_dimension_mismatch():
    """test_estimator.py:413-418: a W_emb that does not match the feature width
    raises DimensionMismatch for fused groups."""
    g, prof = _two_op_worked_example()
    m = _zero_mp_model(vocab=("Mul", "<other>"))
    m.params["W_emb"] = np.zeros((4, 99))
    cp = P.make_cost_providers(prof, P.CommModelParams(0.0, 1.0), m)
    fused = build_graph(g.ops, g.edges, groups=[FusionGroup(0, frozenset({0})), FusionGroup(1, frozenset({1, 2}))])
    with pytest.raises(P.DimensionMismatch):
        P.cost(fused, cp)


def test_graph_beyond_16bit_nodes_matches_oracle():
    """A 70,000-op graph: schedule nodes exceed the 16-bit fast paths (ring
    buffers, shared-memory arena), so the 32-bit event loop runs; costs match
    the oracle under the hardware-oracle provider."""
    from oracle.oracle import Oracle, Workload
    from paper_2209_12769_b200.graph import graph_to_doc

    n = 70000
    ops = [op(i, code="GradW" if i % 70 == 0 else "Mul", us=1.0 + (i % 7)) for i in range(n)]
    edges = [DataEdge(i, i + 1, 256) for i in range(n - 1)] + [DataEdge(i, i + 3, 64) for i in range(0, n - 3, 5)]
    ars = [(t, 70 * t, 4096 + t) for t in range(n // 70)]
    g = build_graph(ops, edges, ars)
    hw = P.HardwareParams()
    cp = P.oracle_providers(hw, precision=N.FO_PREC_FP64)
    dg = cp.device_graph(g)
    ng, rg, bk, gb = dg.make_candidates(np.arange(3, dtype=np.uint64))
    got, st = dg.score_host(ng, rg, bk, gb, N.FO_PREC_FP64)
    assert (st == 0).all()
    o = Oracle(Workload("big", graph_to_doc(g), {}, (hw.comm_params.C, hw.comm_params.D), {}, {}), "oracle")
    for k in range(3):
        _, ref = o.cost(ng[k], rg[k], bk[k])
        assert got[k] == pytest.approx(ref, rel=1e-12)


@pytest.mark.parametrize("name", ["residual40", "vgg16", "resnet50", "bert", "gpt2m"])
def test_block_and_warp_geometries_agree(name, monkeypatch):
    """The block-per-candidate and warp-per-candidate geometries (FO_TEAM)
    give bit-identical costs and statuses for every provider, with the
    shared-memory arena on and off, and the jittered oracle."""
    g, cps = providers(name, N.FO_PREC_FP64)
    cps = dict(cps)
    cps["oracle_noise"] = P.oracle_providers(P.HardwareParams(noise=0.1, seed=3), precision=N.FO_PREC_FP64)
    K = 200
    for pname, cp in cps.items():
        dg = cp.device_graph(g)
        ng, rg, bk, gb = dg.make_candidates(np.arange(K, dtype=np.uint64))
        out = {}
        for team in ("0", "1"):
            for arena in ("0", "1"):
                monkeypatch.setenv("FO_TEAM", team)
                monkeypatch.setenv("FO_SIM_SMEM", arena)
                out[(team, arena)] = dg.score_host(ng, rg, bk, gb, N.FO_PREC_FP64)
        ref = out[("0", "0")]
        for key, (c, s) in out.items():
            assert np.array_equal(s, ref[1]) and np.array_equal(c, ref[0]), (name, pname, key)


def test_per_round_driver_equals_native_run():
    """The per-round path (fo_search_round, used with a time budget and by the
    sharded exchange every M rounds) walks the same trajectories as
    fo_search_run, speculation included; a tiny budget stops early."""
    g, cps = providers("chain24", N.FO_PREC_FP64)
    seeds = [0, 1, 2, 3]
    base = P.SearchConfig(alpha=1.05, beta=6, max_unchanged=40)
    native = P.LockstepSearch(g, base, cps["mp"], seeds).run()
    timed = P.SearchConfig(alpha=1.05, beta=6, max_unchanged=40, time_budget_s=600.0)
    rounds = P.LockstepSearch(g, timed, cps["mp"], seeds).run()
    for a, b in zip(native, rounds):
        assert (a.steps, a.candidates_evaluated, a.candidates_enqueued, a.best_cost_us) == (
            b.steps, b.candidates_evaluated, b.candidates_enqueued, b.best_cost_us)
        assert a.trace == b.trace
    short = P.LockstepSearch(g, P.SearchConfig(alpha=1.05, beta=6, max_unchanged=40, time_budget_s=0.0),
                             cps["mp"], seeds).run()
    for a, b in zip(native, short):
        assert b.steps <= 1 and b.best_cost_us >= a.best_cost_us


def _bench_batch(precision):
    """bench.py's headline batch, built exactly as bench.py builds it: the
    unfused parent resident on the device (set_parent()), 4,096 sparse
    candidates from make_candidates_delta(seeds 0..4095, beta 10)."""
    g, cps = providers("resnet50", precision)
    dg = cps["mp"].device_graph(g)
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(4096, dtype=np.uint64), beta=10)
    return g, dg, off, chg


def _score_delta_on_device(dg, off, chg, precision, memo=True):
    import torch

    N.lib().fo_memo_enable(dg.h, 1 if memo else 0)
    try:
        N.lib().fo_memo_clear(dg.h, N.C.c_void_p(torch.cuda.current_stream().cuda_stream))
        c = torch.empty(len(off) - 1, dtype=torch.float64, device="cuda")
        s = torch.empty(len(off) - 1, dtype=torch.int32, device="cuda")
        dg.score_delta_device(torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda(), c, s, precision)
        torch.cuda.synchronize()
        return c.cpu().numpy(), s.cpu().numpy()
    finally:
        N.lib().fo_memo_enable(dg.h, 1)


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
def test_benchmarked_path_matches_oracle_and_reference(precision):
    """The exact path behind bench.py's headline number: fo_score_delta at
    K = 4,096 (warp-per-candidate geometry), the estimator memo on and
    emptied once per batch, and the pipelined fo_score_delta_submit /
    fo_score_wait that the e2e figure times.  All 4,096 costs against the C
    oracle (fp32 <= 1e-4, fp64 <= 1e-12 relative), the first 48 against the
    reference's own costs (tests/golden/cases/resnet50), and the geometry
    asserted so the test cannot silently run the block path."""
    import torch
    from oracle.oracle import Oracle, load_workload

    g, dg, off, chg = _bench_batch(precision)
    geo = np.zeros(4, np.int32)
    assert N.lib().fo_score_geometry(dg.h, 4096, precision, N.ptr(geo)) == 0
    assert geo[0] == 0, "K = 4,096 must take the warp-per-candidate geometry"
    cost, st = _score_delta_on_device(dg, off, chg, precision)
    assert (st == 0).all()
    o = Oracle(load_workload("resnet50"), "mp" if precision == N.FO_PREC_FP32 else "mp")
    sts, ref = o.cost_batch(*(np.stack([o.make_candidate(i)[j] for i in range(4096)]) for j in range(3)))
    assert (sts == 0).all()
    tol = TOL[("mp", precision)]
    np.testing.assert_allclose(cost, ref, rtol=tol, atol=0)
    gold = np.array([c["cost"]["mp"] for c in cases("resnet50")["candidates"]])
    np.testing.assert_allclose(cost[:len(gold)], gold, rtol=tol, atol=0)
    # the e2e leg: the same batch through host buffers, two submissions in flight
    h = [torch.from_numpy(off).pin_memory(), torch.from_numpy(chg).pin_memory()]
    outs = [(torch.zeros(4096, dtype=torch.float64).pin_memory(), torch.full((4096,), -1, dtype=torch.int32).pin_memory())
            for _ in range(2)]
    tickets = [dg.score_delta_submit(h[0], h[1], c, s, precision, clear_memo=True) for c, s in outs]
    for t in tickets:
        dg.score_wait(t)
    for c, s in outs:
        assert (s.numpy() == 0).all() and np.array_equal(c.numpy(), cost)


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
def test_estimator_memo_changes_no_cost_on_the_bench_batch(precision):
    """The memo keys a prediction by a 128-bit member-set hash with no member
    check on a hit.  On the benchmarked batch (4,096 candidates, ~2,900
    distinct fused member sets) memo-on and memo-off scoring agree bit for
    bit -- any collision would show as a differing cost -- and the host
    restatement of the two hashes finds no colliding pair of distinct sets."""
    g, dg, off, chg = _bench_batch(precision)
    on, s1 = _score_delta_on_device(dg, off, chg, precision, memo=True)
    off_, s2 = _score_delta_on_device(dg, off, chg, precision, memo=False)
    assert (s1 == 0).all() and (s2 == 0).all()
    assert np.array_equal(on, off_)
    sets = _fused_member_sets(dg, off, chg)
    hashes = {}
    for m in sets:
        h = _memo_hash(m)
        assert hashes.setdefault(h, m) == m, f"memo hash collision: {m} vs {hashes[h]}"


def _fused_member_sets(dg, off, chg):
    V, A = dg.V, dg.A
    base = np.concatenate([np.arange(V), -np.ones(V), np.arange(A)]).astype(np.int64)
    out = set()
    for k in range(len(off) - 1):
        st = base.copy()
        c = chg[off[k]:off[k + 1]]
        st[c[:, 0]] = c[:, 1]
        mem = {}
        for v in range(V):
            mem.setdefault(int(st[v]), []).append(v)
            if st[V + v] >= 0:
                mem.setdefault(int(st[V + v]), []).append(v)
        out |= {tuple(sorted(m)) for m in mem.values() if len(m) > 1}
    return out


_M64 = (1 << 64) - 1


def _smix(x):
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _memo_hash(members):
    """Host restatement of set_hash (score.cu): two commutative 64-bit sums."""
    a = sum(_smix(2 * m + 1) for m in members) & _M64
    b = sum(_smix(((m << 32) ^ 0x5BD1E995) & _M64) for m in members) & _M64
    n = len(members)
    return _smix((a + n) & _M64) | 1, _smix(b ^ ((n * 0xFF51AFD7ED558CCD) & _M64))
