"""The CPU oracle (oracle/fo_oracle.c) pinned against golden vectors produced
by the unmodified reference (tests/golden/make_golden.py).  CPU-only."""

import glob
import gzip
import json
import os

import pytest

from oracle.oracle import Oracle, PyRandom, load_workload

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SMALL = ["chain24", "residual40", "attention36", "recurrent30", "vgg16", "resnet50", "bert"]
PROVIDERS = ["mp", "lin", "analytic", "oracle"]


def _cases(name):
    with gzip.open(os.path.join(GOLDEN, "cases", f"{name}.cases.json.gz"), "rt") as fh:
        return json.load(fh)


def test_rng_matches_cpython_random():
    with open(os.path.join(GOLDEN, "rng.json")) as fh:
        d = json.load(fh)
    for s, seq in d["randint_0_10"].items():
        r = PyRandom(int(s))
        assert [r.randint(0, 10) for _ in seq] == seq
    for s, seq in d["getrandbits32"].items():
        r = PyRandom(int(s))
        assert [r.getrandbits(32) for _ in seq] == seq
    for s, seq in d["randrange"].items():
        r = PyRandom(int(s))
        assert [[k, r.randrange(k)] for k, _ in seq] == seq


@pytest.mark.parametrize("name", SMALL + ["gpt2m", "synth50k"])
@pytest.mark.parametrize("prov", PROVIDERS)
def test_oracle_costs_match_reference(name, prov):
    wl = load_workload(name)
    cases = _cases(name)
    o = Oracle(wl, prov)
    ng, rg, bk = o.g.default_state()
    st, c = o.cost(ng, rg, bk)
    assert st == 0 and c == pytest.approx(cases["base_cost"][prov], rel=1e-12)
    for cand in cases["candidates"]:
        ng, rg, bk = o.g.state_from_doc(cand["state"])
        st, c = o.cost(ng, rg, bk)
        assert st == 0
        assert c == pytest.approx(cand["cost"][prov], rel=1e-12)


@pytest.mark.parametrize("name", SMALL)
def test_oracle_group_predictions_match_reference(name):
    wl = load_workload(name)
    cases = _cases(name)
    for prov in PROVIDERS:
        o = Oracle(wl, prov)
        for cand in cases["candidates"][:16]:
            ng, rg, bk = o.g.state_from_doc(cand["state"])
            n, gid, bid, dur, io = o.node_durations(ng, rg, bk)
            assert n > 0
            pos = {int(g): i for i, g in enumerate(gid)}
            for f in cand["fused"]:
                i = pos[f["id"]]
                assert dur[i] == pytest.approx(f[prov], rel=1e-12)
                assert list(io[i]) == f["io"]


@pytest.mark.parametrize("name", SMALL)
def test_oracle_timelines_match_reference(name):
    wl = load_workload(name)
    o = Oracle(wl, "mp")
    for cand in _cases(name)["candidates"]:
        if "timeline" not in cand:
            continue
        st, mk, comp, comm = o.cost(*o.g.state_from_doc(cand["state"]), timeline=True)
        tl = cand["timeline"]
        assert [e[0] for e in comp] == [e[0] for e in tl["compute"]]
        assert [e[0] for e in comm] == [e[0] for e in tl["comm"]]
        for a, b in zip(comp + comm, tl["compute"] + tl["comm"]):
            assert a[1] == pytest.approx(b[1], rel=1e-12, abs=1e-9)
            assert a[2] == pytest.approx(b[2], rel=1e-12, abs=1e-9)
        assert mk == pytest.approx(tl["makespan"], rel=1e-12)


@pytest.mark.parametrize("name", SMALL + ["gpt2m"])
def test_oracle_candidate_generation_bit_exact(name):
    wl = load_workload(name)
    o = Oracle(wl, "mp")
    for cand in _cases(name)["candidates"]:
        ng, rg, bk = o.make_candidate(cand["i"])
        assert o.g.state_to_doc(ng, rg, bk) == cand["state"]


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "search", "*.search.json.gz"))),
                         ids=lambda p: os.path.basename(p).split(".search")[0])
def test_oracle_search_trace_bit_exact(path):
    with gzip.open(path, "rt") as fh:
        d = json.load(fh)
    o = Oracle(load_workload(d["workload"]), d["provider"])
    cfg = d["cfg"]
    r = o.search(alpha=cfg["alpha"], beta=cfg["beta"], max_unchanged=cfg["max_unchanged"], seed=cfg["seed"])
    assert r["status"] == 0
    assert (r["steps"], r["candidates_evaluated"], r["candidates_enqueued"]) == (
        d["steps"], d["candidates_evaluated"], d["candidates_enqueued"])
    assert len(r["trace"]) == len(d["trace"])
    for a, b in zip(r["trace"], d["trace"]):
        assert (a[0], a[1], a[4], a[5]) == (b[0], b[1], b[4], b[5])
        assert a[2] == pytest.approx(b[2], rel=1e-12)
        assert a[3] == pytest.approx(b[3], rel=1e-12)
    assert o.g.state_to_doc(*r["best_state"]) == d["best_state"]
    assert r["best_cost_us"] == pytest.approx(d["best_cost_us"], rel=1e-12)
