"""Golden-vector generator: runs the UNMODIFIED reference `fuseopt` package
(pure Python, importable in the build container from /root/reference/pkg/src)
and writes the fixtures the oracle and the CUDA path are pinned against.

This script is test infrastructure.  It is the only file in the repo that
imports the reference, and it only ever runs in the build container
(/root/reference does not exist on the GPU box); its outputs are committed.

Usage:  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [section ...]
Sections: workloads rng cases search exhaustive sweep baselines jitter acceptance features
(default: the first five)

Inputs follow SURVEY.md section 8(d) / BASELINE.md section 3:
  * graphs   gen_workload(WorkloadSpec(family, V, A, seed=0))      (workloads.py:131)
  * profile  make_profile(g, HardwareParams())                       (workloads.py:307)
  * MP model train(gen_training_samples(g, 256, (1, min(50, V)), hw, seed=0),
                   TrainConfig(epochs=0, seed=0), MESSAGE_PASSING)   (estimator.py:623)
  * candidate i: rng = random.Random(i); accumulating random_apply for
    (nondup, dup, ar), each with n = rng.randint(0, 10)              (rewrite.py:222)
"""

from __future__ import annotations

import gzip
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

from fuseopt import (  # noqa: E402
    EstimatorVariant,
    HardwareParams,
    OptimizationMethod,
    SearchConfig,
    TrainConfig,
    WorkloadSpec,
    backtracking_search,
    build_graph,
    canonical_hash,
    cost,
    featurize,
    gen_training_samples,
    gen_workload,
    make_cost_providers,
    make_profile,
    oracle_providers,
    predict_fused,
    random_apply,
    simulate,
    train,
)
from fuseopt.comm import CommModelParams, save_params  # noqa: E402
from fuseopt.estimator import analytic_model, save_model, save_profile  # noqa: E402
from fuseopt.graph import DataEdge, OpNode, graph_to_doc  # noqa: E402

OUT = HERE
WL = os.path.join(os.path.dirname(os.path.dirname(HERE)), "workloads")  # inputs: <repo>/workloads

# name -> (family, V, A, comm C, comm D, model source)
CONFIGS = {
    # VGG-16 proxy, 8 workers: C = 2(N-1)/(N*B), N=8, B=12,500 B/us
    "vgg16": ("chain", 144, 32, 2 * 7 / (8 * 12500.0), 100.0, None),
    "resnet50": ("residual", 672, 161, None, None, None),
    "bert": ("attention", 760, 199, None, None, None),
    "gpt2m": ("attention", 5000, 292, None, None, "bert"),
    "synth50k": ("residual", 50000, 1000, None, None, "resnet50"),
}
SMALL = {
    "chain24": ("chain", 24, 4, None, None, None),
    "residual40": ("residual", 40, 6, None, None, None),
    "attention36": ("attention", 36, 5, None, None, None),
    "recurrent30": ("recurrent", 30, 5, None, None, None),
}

METHODS = (
    OptimizationMethod.NON_DUPLICATE_FUSION,
    OptimizationMethod.DUPLICATE_FUSION,
    OptimizationMethod.ALLREDUCE_FUSION,
)


def _dump_gz(path, doc):
    with gzip.open(path, "wt", encoding="utf-8") as fh:
        json.dump(doc, fh, sort_keys=True, separators=(",", ":"))


def _dump(path, doc):
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, sort_keys=True, separators=(",", ":"))
        fh.write("\n")


def make_candidate(g, i, beta=10):
    """Candidate i of a random batch."""
    rng = random.Random(i)
    cur = g
    for m in METHODS:
        n = rng.randint(0, beta)
        cur = random_apply(cur, m, n, rng).graph
    return cur


def state_doc(g):
    """Sparse fusion state: only non-trivial groups/buckets."""
    groups = []
    for gr in g.groups:
        trivial = len(gr.member_ops) == 1 and gr.id in gr.member_ops and not gr.duplicated_ops
        if not trivial:
            groups.append([gr.id, sorted(gr.member_ops), sorted(gr.duplicated_ops)])
    buckets = []
    for b in g.buckets:
        if not (len(b.members) == 1 and b.id in b.members):
            buckets.append([b.id, sorted(b.members)])
    return {"groups": groups, "buckets": buckets}


def _write_workload(name, family, V, A, C, D, model_src, hw):
    t0 = time.time()
    g = gen_workload(WorkloadSpec(family, V, A, seed=0), hw)
    profile, _ = make_profile(g, hw)
    comm = CommModelParams(C=C, D=D) if C is not None else hw.comm_params
    base = os.path.join(WL, name)
    _dump_gz(base + ".graph.json.gz", graph_to_doc(g))
    tmp = base + ".tmp"
    save_profile(tmp, profile)
    with open(tmp) as fh:
        _dump_gz(base + ".profile.json.gz", json.load(fh))
    save_params(base + ".comm.json", comm)
    if model_src is None:
        samples = gen_training_samples(g, 256, (1, min(50, V)), hw, seed=0)
        mp = train(samples, TrainConfig(epochs=0, seed=0), EstimatorVariant.MESSAGE_PASSING)
        save_model(tmp, mp)
        with open(tmp) as fh:
            _dump_gz(base + ".mp.model.json.gz", json.load(fh))
        lin = train(samples, TrainConfig(epochs=0, seed=0), EstimatorVariant.LINEAR_FEATURES)
        save_model(base + ".lin.model.json", lin)
    else:
        meta = {"model_from": model_src}
        _dump(base + ".model_from.json", meta)
    os.remove(tmp)
    print(f"workload {name}: V={len(g.ops)} E={len(g.edges)} A={len(g.allreduces)} "
          f"in {time.time() - t0:.1f}s", flush=True)


def section_workloads(names=None):
    os.makedirs(WL, exist_ok=True)
    hw = HardwareParams()
    table = dict(CONFIGS)
    table.update(SMALL)
    for name, (family, V, A, C, D, src) in table.items():
        if names and name not in names:
            continue
        _write_workload(name, family, V, A, C, D, src, hw)


# ---------------------------------------------------------------------------
# loading back (shared with the case/search sections)


def load_workload(name):
    from fuseopt.comm import load_params
    from fuseopt.estimator import load_model, load_profile
    from fuseopt.graph import graph_from_doc

    base = os.path.join(WL, name)
    with gzip.open(base + ".graph.json.gz", "rt") as fh:
        g = graph_from_doc(json.load(fh))
    tmp = f"/tmp/_golden_{os.getpid()}.json"
    with gzip.open(base + ".profile.json.gz", "rt") as fh:
        doc = json.load(fh)
    with open(tmp, "w") as fh:
        json.dump(doc, fh)
    profile = load_profile(tmp)
    comm = load_params(base + ".comm.json")
    src = name
    if os.path.exists(base + ".model_from.json"):
        with open(base + ".model_from.json") as fh:
            src = json.load(fh)["model_from"]
    sbase = os.path.join(WL, src)
    with gzip.open(sbase + ".mp.model.json.gz", "rt") as fh:
        doc = json.load(fh)
    with open(tmp, "w") as fh:
        json.dump(doc, fh)
    mp = load_model(tmp)
    lin = load_model(sbase + ".lin.model.json")
    os.remove(tmp)
    return g, profile, comm, mp, lin


def providers(profile, comm, mp, lin):
    hw = HardwareParams()
    return {
        "mp": make_cost_providers(profile, comm, mp),
        "lin": make_cost_providers(profile, comm, lin),
        "analytic": make_cost_providers(profile, comm, analytic_model(5.0, 1.0 / 1024.0)),
        "oracle": oracle_providers(hw),
    }


# ---------------------------------------------------------------------------
# RNG golden sequences (CPython random.Random; search.py:88,119; rewrite.py:250)


def section_rng():
    out = {"randint_0_10": {}, "randrange": {}, "getrandbits32": {}}
    for seed in [0, 1, 2, 7, 42, 1234, 2**32 + 5, 10**12 + 3]:
        r = random.Random(seed)
        out["randint_0_10"][str(seed)] = [r.randint(0, 10) for _ in range(64)]
        r = random.Random(seed)
        out["getrandbits32"][str(seed)] = [r.getrandbits(32) for _ in range(16)]
        r = random.Random(seed)
        seq = []
        for k in [1, 2, 3, 5, 7, 8, 17, 100, 1000, 65537, 2**31 - 1]:
            seq.append([k, r.randrange(k)])
        for k in range(1, 200):
            seq.append([k, r.randrange(k)])
        out["randrange"][str(seed)] = seq
    _dump(os.path.join(OUT, "rng.json"), out)
    print("rng done", flush=True)


# ---------------------------------------------------------------------------
# Scoring cases: candidates + reference costs + per-fused-group predictions


def _case(name, g, profile, comm, mp, lin, n_cand, n_timeline):
    cps = providers(profile, comm, mp, lin)
    cands = []
    t0 = time.time()
    for i in range(n_cand):
        c = make_candidate(g, i)
        fresh = build_graph(
            c.ops, c.edges,
            [(ar.id, ar.producer_op, ar.tensor_bytes) for ar in c.allreduces],
            groups=c.groups,
            buckets=[(b.id, b.members) for b in c.buckets],
            meta=c.meta,
        )
        rec = {"i": i, "state": state_doc(c), "hash_of_parent_equal": canonical_hash(c) == canonical_hash(g)}
        rec["cost"] = {k: cost(fresh, cp) for k, cp in cps.items()}
        fused = []
        for gr in c.groups:
            if len(gr.member_ops) > 1:
                f = featurize(c, gr, profile)
                fused.append({
                    "id": gr.id,
                    "members": sorted(gr.member_ops),
                    "mp": predict_fused(mp, f),
                    "lin": predict_fused(lin, f),
                    "analytic": predict_fused(analytic_model(5.0, 1.0 / 1024.0), f),
                    "oracle": cps["oracle"].op_cost(c, gr),
                    "io": [f.internal_bytes, f.external_in_bytes, f.external_out_bytes],
                    "longest": f.longest_path_len,
                })
        rec["fused"] = fused
        if i < n_timeline:
            tl = simulate(fresh, cps["mp"])
            rec["timeline"] = {
                "compute": [list(e) for e in tl.compute_events],
                "comm": [list(e) for e in tl.comm_events],
                "makespan": tl.makespan_us,
            }
        cands.append(rec)
    base_cost = {k: cost(g, cp) for k, cp in cps.items()}
    doc = {"workload": name, "base_cost": base_cost, "candidates": cands}
    _dump_gz(os.path.join(OUT, "cases", f"{name}.cases.json.gz"), doc)
    print(f"cases {name}: {n_cand} candidates in {time.time() - t0:.1f}s", flush=True)


CASE_COUNTS = {
    "chain24": (64, 8), "residual40": (64, 8), "attention36": (64, 8), "recurrent30": (64, 8),
    "vgg16": (64, 4), "resnet50": (48, 4), "bert": (48, 4), "gpt2m": (48, 1), "synth50k": (16, 0),
}


def section_cases(names=None):
    os.makedirs(os.path.join(OUT, "cases"), exist_ok=True)
    for name, (n, nt) in CASE_COUNTS.items():
        if names and name not in names:
            continue
        g, profile, comm, mp, lin = load_workload(name)
        _case(name, g, profile, comm, mp, lin, n, nt)


# ---------------------------------------------------------------------------
# Search traces (search.py:84-155)


SEARCHES = [
    # (workload, provider, cfg kwargs)
    ("chain24", "mp", dict(alpha=1.05, beta=4, seed=0, max_unchanged=60)),
    ("chain24", "oracle", dict(alpha=1.05, beta=4, seed=1, max_unchanged=60)),
    ("residual40", "mp", dict(alpha=1.05, beta=10, seed=2, max_unchanged=80)),
    ("residual40", "analytic", dict(alpha=1.1, beta=5, seed=3, max_unchanged=80)),
    ("attention36", "mp", dict(alpha=1.05, beta=10, seed=4, max_unchanged=80)),
    ("attention36", "lin", dict(alpha=1.05, beta=6, seed=5, max_unchanged=80)),
    ("recurrent30", "oracle", dict(alpha=1.02, beta=3, seed=6, max_unchanged=80)),
    ("recurrent30", "mp", dict(alpha=1.2, beta=10, seed=7, max_unchanged=80)),
    ("vgg16", "mp", dict()),  # reference defaults (BASELINE config 0)
    ("bert", "mp", dict(seed=0, max_unchanged=60)),
    ("bert", "mp", dict(), "default"),  # reference defaults (BASELINE config 2, one seed)
]


def section_search(only=None):
    os.makedirs(os.path.join(OUT, "search"), exist_ok=True)
    for wl, prov, kw, *suffix in SEARCHES:
        tag = f"{wl}.{prov}.s{kw.get('seed', 0)}" + "".join("." + x for x in suffix)
        if only and tag not in only and wl not in only:
            continue
        g, profile, comm, mp, lin = load_workload(wl)
        cp = providers(profile, comm, mp, lin)[prov]
        cfg = SearchConfig(**kw)
        t0 = time.time()
        res = backtracking_search(g, cfg, cp)
        wall = time.time() - t0
        doc = {
            "workload": wl, "provider": prov,
            "cfg": {"alpha": cfg.alpha, "beta": cfg.beta, "max_unchanged": cfg.max_unchanged, "seed": cfg.seed},
            "best_cost_us": res.best_cost_us, "steps": res.steps,
            "candidates_evaluated": res.candidates_evaluated,
            "candidates_enqueued": res.candidates_enqueued,
            "best_state": state_doc(res.best_graph),
            "trace": [[r.step, r.action, r.cost_us, r.best_cost_us, r.queue_len, r.enqueued] for r in res.trace],
            "wall_s": wall,
        }
        _dump_gz(os.path.join(OUT, "search", f"{tag}.search.json.gz"), doc)
        print(f"search {tag}: steps={res.steps} evals={res.candidates_evaluated} "
              f"best={res.best_cost_us:.3f} in {wall:.1f}s", flush=True)


def section_exhaustive(_=None):
    """exhaustive_search (search.py:158-225) on small graphs, hardware-oracle
    and analytic providers; mirrors test_exhaustive_dominates_backtracking."""
    from fuseopt import exhaustive_search

    out = []
    rng = random.Random(5)
    hw = HardwareParams()
    for seed in range(8):
        spec = WorkloadSpec(family=["chain", "residual", "attention", "recurrent"][seed % 4],
                            op_count=rng.randrange(4, 9), tensor_count=rng.randrange(0, 3), seed=seed)
        g = gen_workload(spec, hw)
        profile, _ = make_profile(g, hw)
        for prov_name, cp in (("oracle", oracle_providers(hw)),
                              ("analytic", make_cost_providers(profile, hw.comm_params, analytic_model(5.0, 1 / 1024)))):
            res = exhaustive_search(g, cp)
            out.append({"graph": graph_to_doc(g), "profile": [[k[0], k[1], v] for k, v in sorted(profile.times.items())],
                        "provider": prov_name, "best_cost_us": res.best_cost_us,
                        "candidates_evaluated": res.candidates_evaluated, "steps": res.steps,
                        "best_state": state_doc(res.best_graph)})
    _dump_gz(os.path.join(OUT, "exhaustive.json.gz"), out)
    print(f"exhaustive: {len(out)} cases", flush=True)


def section_sweep(_=None):
    """BASELINE configs[3]: GPT-2-medium proxy, tensor-fusion bucket-size sweep.
    Parents = threshold_allreduce_fusion(g, T, cp) and the same on
    greedy_postorder_fusion(g) (search.py:228-302; the compare verb's "both"
    row, cli.py:378-383) for T = 2^k, k = 16..28, with their reference costs."""
    from fuseopt import greedy_postorder_fusion, threshold_allreduce_fusion

    g, profile, comm, mp, lin = load_workload("gpt2m")
    cp = make_cost_providers(profile, comm, mp)
    t0 = time.time()
    greedy = greedy_postorder_fusion(g)
    print(f"greedy done in {time.time() - t0:.0f}s", flush=True)
    out = {"greedy": {"state": state_doc(greedy), "cost": cost(greedy, cp)}, "sweep": []}
    for k in range(16, 29):
        T = 2 ** k
        a = threshold_allreduce_fusion(g, T, cp)
        b = threshold_allreduce_fusion(greedy, T, cp)
        out["sweep"].append({"T": T, "ar_only": {"state": state_doc(a), "cost": cost(a, cp)},
                             "both": {"state": state_doc(b), "cost": cost(b, cp)}})
        print(f"sweep T=2^{k}: {time.time() - t0:.0f}s", flush=True)
        _dump_gz(os.path.join(OUT, "sweep_gpt2m.json.gz"), out)


def section_baselines(names=None):
    """Heuristic baselines (search.py:228-302) on the small configs: the greedy
    post-order op fusion, threshold AllReduce fusion without cost providers
    (contracted production order) and with the MP providers (simulated start
    order), each from the unfused graph, from the greedy result and from a
    random-batch candidate (which holds replica groups)."""
    from fuseopt import greedy_postorder_fusion, threshold_allreduce_fusion

    out = {}
    for name in list(SMALL) + ["vgg16", "resnet50", "bert"]:
        if names and name not in names:
            continue
        t0 = time.time()
        g, profile, comm, mp, lin = load_workload(name)
        cp = make_cost_providers(profile, comm, mp)
        starts = {"unfused": g, "cand3": make_candidate(g, 3)}
        greedy = {k: greedy_postorder_fusion(x) for k, x in starts.items()}
        ent = {"greedy": {k: state_doc(x) for k, x in greedy.items()}, "threshold": []}
        starts["greedy"] = greedy["unfused"]
        for T in (64 * 1024, 4 * 1024 * 1024, 256 * 1024 * 1024):
            for k, x in starts.items():
                ent["threshold"].append({"T": T, "start": k, "topo": state_doc(threshold_allreduce_fusion(x, T)),
                                         "sim": state_doc(threshold_allreduce_fusion(x, T, cp))})
        ent["starts"] = {k: state_doc(x) for k, x in starts.items()}
        out[name] = ent
        print(f"baselines {name}: {time.time() - t0:.0f}s", flush=True)
        _dump_gz(os.path.join(OUT, "baselines.json.gz"), out)


def section_jitter(names=None):
    """oracle_providers with noise > 0 (workloads.py:254-291): candidate costs
    and per-group durations under the reference's blake2b jitter."""
    out = {}
    for name in ["chain24", "residual40", "attention36", "vgg16", "resnet50", "bert"]:
        if names and name not in names:
            continue
        g = load_workload(name)[0]
        ent = []
        for noise, seed in ((0.05, 42), (0.3, 7)):
            hw = HardwareParams(noise=noise, seed=seed)
            cp = oracle_providers(hw)
            rows = []
            for i in range(10):
                c = make_candidate(g, i)
                row = {"i": i, "cost": cost(c, cp)}
                if i < 2:
                    row["groups"] = [[gr.id, cp.op_cost(c, gr)] for gr in c.groups]
                rows.append(row)
            ent.append({"noise": noise, "seed": seed, "rows": rows})
        out[name] = ent
        print(f"jitter {name}", flush=True)
    _dump_gz(os.path.join(OUT, "jitter.json.gz"), out)


def section_acceptance(names=None):
    """The reference's acceptance criteria 1-3 inputs (test_acceptance.py:59-149):
    generated workloads with their oracle-provider costs / bounds, and the
    small criterion-2 workloads with their exhaustive optimum."""
    from fuseopt import exhaustive_search, fo_bound
    from fuseopt.workloads import FAMILIES

    hw = HardwareParams()
    cp = oracle_providers(hw)
    rng = random.Random(0)
    c1 = []
    for i in range(1000):
        spec = WorkloadSpec(family=FAMILIES[i % 4], op_count=rng.randrange(10, 201), tensor_count=rng.randrange(0, 31),
                            seed=i)
        g = gen_workload(spec, hw)
        total = sum(cp.op_cost(g, gr) for gr in g.groups) + sum(cp.comm_cost(g, b) for b in g.buckets)
        c1.append({"i": i, "graph": graph_to_doc(g), "cost": cost(g, cp), "fo_bound": fo_bound(g, cp),
                   "total": total})
    rng = random.Random(0)
    c2 = []
    for k in range(50):
        spec = WorkloadSpec(family=FAMILIES[k % 4], op_count=rng.randrange(4, 9), tensor_count=rng.randrange(0, 4),
                            seed=k)
        g = gen_workload(spec, hw)
        c2.append({"k": k, "graph": graph_to_doc(g), "exact": exhaustive_search(g, cp).best_cost_us})
    # criteria 8 / 9 (test_acceptance.py:250-322): the two generated graphs
    g8 = gen_workload(WorkloadSpec(family="recurrent", op_count=40, tensor_count=10, min_tensor_bytes=8 * 1024,
                                   max_tensor_bytes=64 * 1024, seed=21))
    g9 = gen_workload(WorkloadSpec(family="attention", op_count=100, tensor_count=12, seed=33))
    _dump_gz(os.path.join(OUT, "acceptance.json.gz"), {"criterion1": c1, "criterion2": c2,
                                                      "criterion8": graph_to_doc(g8), "criterion9": graph_to_doc(g9)})
    print(f"acceptance: {len(c1)} + {len(c2)} workloads", flush=True)


def section_features(names=None):
    """featurize / predict_fused / oracle_time per fused group (estimator.py:157-191,
    :462-470; workloads.py:276-291) on random candidates, plus group_io."""
    from fuseopt.graph import group_io
    from fuseopt.workloads import oracle_time

    out = {}
    for name in ["chain24", "residual40", "attention36", "recurrent30", "vgg16", "resnet50", "bert"]:
        if names and name not in names:
            continue
        g, profile, comm, mp, lin = load_workload(name)
        ana = analytic_model(5.0, 1.0 / 1024.0)
        hws = [HardwareParams(), HardwareParams(noise=0.05, seed=42)]
        rows = []
        from fuseopt.search import greedy_postorder_fusion

        for i in range(5):
            c = make_candidate(g, i) if i < 4 else greedy_postorder_fusion(g)
            fused = [gr for gr in c.groups if len(gr.member_ops) > 1]
            fused = fused[:25] if i < 4 else sorted(fused, key=lambda x: (-len(x.member_ops), x.id))[:12]
            singles = [gr for gr in c.groups if len(gr.member_ops) == 1][:3]
            grs = []
            for gr in fused + singles:
                f = featurize(c, gr, profile)
                io = group_io(c, gr.id)
                grs.append({"gid": gr.id, "io": [io.internal_bytes, io.external_in_bytes, io.external_out_bytes],
                            "features": {"op_codes": list(f.op_codes), "compute_us": list(f.compute_us),
                                         "in_bytes": list(f.in_bytes), "out_bytes": list(f.out_bytes),
                                         "edges": [list(e) for e in f.edges], "member_count": f.member_count,
                                         "total_compute_us": f.total_compute_us,
                                         "internal_bytes": f.internal_bytes,
                                         "external_in_bytes": f.external_in_bytes,
                                         "external_out_bytes": f.external_out_bytes,
                                         "longest_path_len": f.longest_path_len},
                            "mp": predict_fused(mp, f), "lin": predict_fused(lin, f),
                            "analytic": predict_fused(ana, f),
                            "oracle": [oracle_time(c, gr, hw) for hw in hws]})
            from fuseopt.graph import topo_order

            rows.append({"i": i, "state": state_doc(c), "groups": grs, "topo": topo_order(c)})
        out[name] = rows
        print(f"features {name}", flush=True)
    _dump_gz(os.path.join(OUT, "features.json.gz"), out)


def main(argv):
    sections = [a for a in argv if a in ("workloads", "rng", "cases", "search", "exhaustive", "sweep", "baselines", "jitter", "acceptance", "features")]
    names = [a for a in argv if a not in sections]
    if not sections:
        sections = ["workloads", "rng", "cases", "search", "exhaustive"]
    for s in sections:
        {"workloads": section_workloads, "rng": lambda _: section_rng(), "exhaustive": section_exhaustive,
         "sweep": section_sweep, "baselines": section_baselines, "jitter": section_jitter,
         "acceptance": section_acceptance, "features": section_features,
         "cases": section_cases, "search": section_search}[s](names or None)


if __name__ == "__main__":
    main(sys.argv[1:])
