"""CPU-only checks of the product library: it loads, exports every symbol the
public header declares, and its host-side batch-expand engine reproduces the
reference's candidates bit-exactly.  No device compute is called here."""

import ctypes
import os
import random
import re

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
from paper_2209_12769_b200.rewrite import ALL_METHODS, engine_graph

from _golden import canon_arrays, canon_doc, canon_graph, cases, read

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = ["chain24", "residual40", "attention36", "recurrent30", "vgg16", "resnet50", "bert"]


def test_library_exports_every_header_symbol():
    with open(os.path.join(ROOT, "include", "disco_b200.h")) as fh:
        text = fh.read()
    declared = set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(fo_\w+)\s*\(", text, re.M))
    assert len(declared) >= 18
    lib = ctypes.CDLL(N.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    bound = {s[0] for s in N.SIGNATURES}
    assert declared == bound, declared ^ bound


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setattr(N, "LIB_PATH", "/nonexistent/libdiscob200.so")
    with pytest.raises(ImportError):
        N.lib()


@pytest.mark.parametrize("name", SMALL + ["gpt2m"])
def test_engine_candidates_bit_exact(name):
    g = P.load_workload(name)[0]
    cs = cases(name)["candidates"]
    ng, rg, bk, vb = P.make_candidates(g, [c["i"] for c in cs])
    assert vb == 2 * len(g.ops) + 2
    for k, c in enumerate(cs):
        assert canon_arrays(g, ng[k], rg[k], bk[k]) == canon_doc(g, c["state"]), c["i"]


@pytest.mark.parametrize("name", ["chain24", "attention36", "vgg16"])
def test_random_apply_dropin_drives_python_random(name):
    """random_apply(g, method, n, rng) consumes a random.Random exactly like the
    reference: chaining it as the golden generator did reproduces every candidate."""
    g = P.load_workload(name)[0]
    for c in cases(name)["candidates"][:12]:
        rng = random.Random(c["i"])
        cur = g
        for m in ALL_METHODS:
            n = rng.randint(0, 10)
            cur = P.random_apply(cur, m, n, rng).graph
        assert canon_graph(cur) == canon_doc(g, c["state"])


def test_random_apply_zero_and_single_op_are_noops():
    g = P.build_graph([P.OpNode(0, "Mul", input_shape_key="k0", out_bytes=1024, compute_us=10.0)])
    for m in ALL_METHODS:
        out = P.random_apply(g, m, 5, random.Random(0))
        assert not out.applied and out.graph is g


def test_state_hash_equality_semantics():
    g = P.load_workload("resnet50")[0]
    dg = engine_graph(g)
    seeds = np.arange(200)
    ng, rg, bk, _ = dg.make_candidates(seeds)
    h = dg.state_hash(ng, rg, bk)
    canon = [canon_arrays(g, ng[k], rg[k], bk[k]) for k in range(len(seeds))]
    for i in range(len(seeds)):
        for j in range(i + 1, len(seeds)):
            assert (h[i] == h[j]) == (canon[i] == canon[j])
    # relabelled ids: a monotone shift of group ids hashes the same
    ng2, rg2 = ng[3] * 3 + 7, np.where(rg[3] >= 0, rg[3] * 3 + 7, -1)
    assert dg.state_hash(ng2, rg2, bk[3])[0] == h[3]


def test_candidate_generation_threads_deterministic():
    g = P.load_workload("bert")[0]
    a = P.make_candidates(g, range(64), n_threads=1)
    b = P.make_candidates(g, range(64), n_threads=8)
    for x, y in zip(a[:3], b[:3]):
        assert np.array_equal(x, y)


def test_exhaustive_closure_sizes_match_reference():
    """BFS closure of the three rewrites (search.py:158-225): the number of
    distinct reachable states equals the reference's candidates_evaluated."""
    from paper_2209_12769_b200.graph import graph_from_doc, state_arrays
    from paper_2209_12769_b200.rewrite import expand_all

    for case in read("exhaustive.json.gz"):
        if case["provider"] != "oracle":
            continue
        g = graph_from_doc(case["graph"])
        dg = engine_graph(g)
        ng, rg, bk, _, _, _ = state_arrays(g)
        seen = {int(dg.state_hash(ng, rg, bk)[0])}
        frontier = [(ng, rg, bk)]
        while frontier:
            nxt = []
            for s in frontier:
                cn, cr, cb = expand_all(g, *s)
                if len(cn) == 0:
                    continue
                for i, h in enumerate(dg.state_hash(cn, cr, cb)):
                    if int(h) not in seen:
                        seen.add(int(h))
                        nxt.append((cn[i], cr[i], cb[i]))
            frontier = nxt
        assert len(seen) == case["candidates_evaluated"]


def test_graph_json_round_trip(tmp_path):
    g = P.load_workload("vgg16")[0]
    p = tmp_path / "g.json"
    P.save_graph(p, g, explicit_state=True)
    h = P.load_graph(p)
    assert P.canonical_hash(h) == P.canonical_hash(g)
    assert canon_graph(h) == canon_graph(g)


def test_state_arrays_round_trip():
    from paper_2209_12769_b200.graph import state_arrays, state_from_arrays

    g = P.load_workload("attention36")[0]
    ng, rg, bk, _ = P.make_candidates(g, [11])
    c = state_from_arrays(g, ng[0], rg[0], bk[0])
    assert canon_graph(c) == canon_arrays(g, ng[0], rg[0], bk[0])
    n2, r2, b2, _, _, _ = state_arrays(c)
    assert canon_arrays(g, n2, r2, b2) == canon_graph(c)


def test_host_only_handle_refuses_device_work():
    g = P.load_workload("chain24")[0]
    dg = engine_graph(g)
    if dg.device >= 0:
        pytest.skip("a device is present")
    ng, rg, bk, vb = dg.make_candidates([1, 2])
    with pytest.raises(P.DeviceError):
        dg.score_host(ng, rg, bk, vb)
    off = np.zeros(3, np.int32)
    chg = np.zeros((0, 2), np.int32)
    cost, st = np.zeros(2), np.zeros(2, np.int32)
    with pytest.raises(P.DeviceError):
        dg.score_delta_submit(off, chg, cost, st)
    with pytest.raises(P.DeviceError):
        dg.score_wait(0)


def test_score_delta_submit_validates_host_buffers():
    """The pipelined submission writes into the caller's buffers after it
    returns, so it refuses anything it could not write safely: wrong dtypes,
    short or non-contiguous buffers, a changes array that does not cover
    offsets[K] (before any device work, so this runs on a host-only handle)."""
    g = P.load_workload("chain24")[0]
    dg = engine_graph(g)
    off = np.array([0, 1, 2], np.int32)
    chg = np.zeros((2, 2), np.int32)
    cost, st = np.zeros(2), np.zeros(2, np.int32)
    with pytest.raises(TypeError):
        dg.score_delta_submit(off, chg, cost.astype(np.float32), st)
    with pytest.raises(TypeError):
        dg.score_delta_submit(off, chg, cost, st.astype(np.int64))
    with pytest.raises(ValueError):
        dg.score_delta_submit(off, chg, cost, st[:1])
    with pytest.raises(ValueError):
        dg.score_delta_submit(off, chg, np.zeros(4)[::2], st)
    with pytest.raises(ValueError):
        dg.score_delta_submit(off, chg[:1], cost, st)
    with pytest.raises(TypeError):
        dg.score_delta_submit(off.astype(np.int64), chg, cost, st)


@pytest.mark.parametrize("name", SMALL + ["gpt2m"])
def test_incremental_engine_matches_full_rebuild(name, monkeypatch):
    """The incremental engine (Inc) draws, accepts and labels exactly like the
    full-rebuild engine (FO_ENGINE=full), also from deep base states."""
    g = P.load_workload(name)[0]
    dg = engine_graph(g)
    base = None
    rounds = 3 if name == "gpt2m" else 4
    for rnd in range(rounds):
        seeds = np.arange(rnd * 1000, rnd * 1000 + 96, dtype=np.uint64)
        monkeypatch.delenv("FO_ENGINE", raising=False)
        a = dg.make_candidates(seeds, 30, 7, base, 4)
        monkeypatch.setenv("FO_ENGINE", "full")
        b = dg.make_candidates(seeds, 30, 7, base, 4)
        for x, y in zip(a[:3], b[:3]):
            assert np.array_equal(x, y), (name, rnd)
        base = (a[0][rnd].copy(), a[1][rnd].copy(), a[2][rnd].copy())


def _ranked(ng, rg):
    ids = np.unique(np.concatenate([ng, rg[rg >= 0]]))
    r = {int(x): i for i, x in enumerate(ids)}
    return (np.array([r[int(x)] for x in ng], np.int32),
            np.array([r[int(x)] if x >= 0 else -1 for x in rg], np.int32))


@pytest.mark.parametrize("name", ["vgg16", "resnet50", "bert", "gpt2m"])
def test_delta_candidates_reconstruct_dense(name):
    """fo_make_candidates_delta = fo_make_candidates as (index, value) changes
    against the id-ranked base, for the unfused base and a fused one."""
    g = P.load_workload(name)[0]
    dg = engine_graph(g)
    V, A = dg.V, dg.A
    seeds = np.arange(64, dtype=np.uint64)
    first = dg.make_candidates(np.array([7], np.uint64))
    for base in (None, (first[0][0], first[1][0], first[2][0])):
        ng, rg, bk, _ = dg.make_candidates(seeds, base=base)
        off, chg = dg.make_candidates_delta(seeds, base=base)
        if base is None:
            b = np.concatenate([np.arange(V), -np.ones(V), np.arange(A)]).astype(np.int32)
        else:
            bn, br = _ranked(base[0], base[1])
            b = np.concatenate([bn, br, base[2]]).astype(np.int32)
        for k in range(len(seeds)):
            x = b.copy()
            c = chg[off[k]:off[k + 1]]
            assert len(np.unique(c[:, 0])) == len(c)
            x[c[:, 0]] = c[:, 1]
            assert np.array_equal(x, np.concatenate([ng[k], rg[k], bk[k]])), (name, k)


def test_delta_candidates_edge_cases():
    g = P.load_workload("chain24")[0]
    dg = engine_graph(g)
    off, chg = dg.make_candidates_delta(np.zeros(0, np.uint64))
    assert off.tolist() == [0] and chg.shape == (0, 2)
    off, chg = dg.make_candidates_delta(np.arange(5, dtype=np.uint64), beta=0)  # n = 0 rewrites: no changes
    assert off.tolist() == [0] * 6
