"""The reference arm of bench.py: the UNMODIFIED reference package `fuseopt`
(pure Python + numpy), installed once into baseline/_ref with

    python -m pip install --no-index --no-build-isolation --no-deps \\
        --find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>

and timed on the host cores through its own public API, exactly the unit of
work SURVEY.md 8(d) names: ``cost(HloGraph(...fresh object...), cp)`` with
``cp = make_cost_providers(profile, comm, model)`` (simulator.py:143-145,
estimator.py:801-824), so the _Index contraction, featurize, the numpy MP
forward and the heap event loop are all inside the timed call.

Bench infrastructure only: the product never imports this module or
baseline/_ref.  The candidate sample is the reference's own candidates
(tests/golden/cases/<config>.cases.json.gz: seeds 0.. of the same random
batch the GPU arm scores), rebuilt as reference graphs, and every one is
checked against its stored reference cost before any timing.
"""

from __future__ import annotations

import gzip
import json
import os
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF = os.path.join(HERE, "_ref")

_STATE = None  # (graphs, cp, cost) of this process


def available() -> bool:
    return os.path.isfile(os.path.join(REF, "fuseopt", "__init__.py"))


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _json(path):
    if path.endswith(".gz"):
        with gzip.open(path, "rt") as fh:
            return json.load(fh)
    with open(path) as fh:
        return json.load(fh)


def load(config: str):
    """The reference's graph, providers and candidate graphs for `config`,
    through the reference's own loaders (graph_from_doc, load_profile,
    load_params, load_model, build_graph)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from fuseopt import cost, make_cost_providers
    from fuseopt.comm import load_params
    from fuseopt.estimator import load_model, load_profile
    from fuseopt.graph import FusionGroup, build_graph, graph_from_doc

    wl = os.path.join(ROOT, "workloads")
    base = os.path.join(wl, config)
    g = graph_from_doc(_json(base + ".graph.json.gz"))
    src = config
    if os.path.exists(base + ".model_from.json"):
        src = _json(base + ".model_from.json")["model_from"]
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "profile.json")
        with open(p, "w") as fh:
            json.dump(_json(base + ".profile.json.gz"), fh)
        profile = load_profile(p)
        m = os.path.join(tmp, "model.json")
        with open(m, "w") as fh:
            json.dump(_json(os.path.join(wl, src + ".mp.model.json.gz")), fh)
        model = load_model(m)
    comm = load_params(base + ".comm.json")
    cp = make_cost_providers(profile, comm, model)

    cases = _json(os.path.join(ROOT, "tests", "golden", "cases", f"{config}.cases.json.gz"))["candidates"]
    ops = sorted(o.id for o in g.ops)
    graphs, expect = [], []
    for c in cases:
        st = c["state"]
        covered, groups = set(), []
        for gid, mem, dup in st["groups"]:
            groups.append(FusionGroup(gid, frozenset(mem), frozenset(dup)))
            covered |= set(mem) - set(dup)
        groups += [FusionGroup(o, frozenset([o])) for o in ops if o not in covered]
        cov, buckets = set(), []
        for bid, mem in st["buckets"]:
            buckets.append((bid, mem))
            cov |= set(mem)
        buckets += [(a.id, [a.id]) for a in g.allreduces if a.id not in cov]
        graphs.append(build_graph(g.ops, g.edges, [(a.id, a.producer_op, a.tensor_bytes) for a in g.allreduces],
                                  groups=groups, buckets=buckets, meta=g.meta))
        expect.append(c["cost"]["mp"])
    return graphs, cp, cost, expect


def _fresh(HloGraph, c):
    # a new object per call: the lazily cached _Index (graph.py:288-290) is
    # rebuilt, as for every new candidate in the reference's search
    return HloGraph(c.meta, c.ops, c.edges, c.allreduces, c.groups, c.buckets)


def _init(config):
    global _STATE
    graphs, cp, cost, _ = load(config)
    from fuseopt.graph import HloGraph

    _STATE = (graphs, cp, cost, HloGraph)


def _score(idx):
    graphs, cp, cost, HloGraph = _STATE
    for i in idx:
        cost(_fresh(HloGraph, graphs[i % len(graphs)]), cp)
    return len(idx)


def check(config: str) -> int:
    """Every sample candidate's reference cost equals the stored golden
    (same code, same inputs); returns the sample size."""
    graphs, cp, cost, expect = load(config)
    for c, e in zip(graphs, expect):
        got = cost(c, cp)
        if got != e:
            raise AssertionError(f"reference arm: cost {got!r} != golden {e!r}")
    return len(graphs)


class Pool:
    """`n` worker processes (spawned: no CUDA state crosses), each holding the
    reference's graphs and providers; step(k) scores k fresh candidates,
    cycling the sample, split evenly over the workers."""

    def __init__(self, config: str, n: int):
        import multiprocessing as mp

        self.n = n
        self.pool = mp.get_context("spawn").Pool(n, initializer=_init, initargs=(config,))
        self.pool.map(_score, [[0]] * n)  # warm every worker

    def step(self, k: int) -> int:
        chunks = [list(range(w, k, self.n)) for w in range(self.n)]
        return sum(self.pool.map(_score, chunks, chunksize=1))

    def close(self):
        self.pool.close()
        self.pool.join()


def rate_one_core(config: str, budget_s: float):
    """cost() per second on this process's one core (the reference as is)."""
    _init(config)
    n0 = len(_STATE[0])
    _score(range(2))  # warm-up
    n, t0 = 0, time.perf_counter()
    while True:
        n += _score(range(n, n + 4))
        dt = time.perf_counter() - t0
        if dt >= budget_s:
            break
    return n / dt, n, dt, n0


def rate_pool(config: str, n_procs: int, budget_s: float):
    pool = Pool(config, n_procs)
    try:
        k = 4 * n_procs
        pool.step(k)
        n, t0 = 0, time.perf_counter()
        while True:
            n += pool.step(k)
            dt = time.perf_counter() - t0
            if dt >= budget_s:
                break
    finally:
        pool.close()
    return n / dt, n, dt
