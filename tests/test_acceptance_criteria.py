"""The reference's acceptance criteria 1-3 (test_acceptance.py:59-149) on this
package: generated workloads (the reference's own generator, committed as
fixtures by make_golden.py's acceptance section) scored and searched on the
device under the hardware-oracle providers."""

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
from paper_2209_12769_b200.graph import graph_from_doc

from _golden import read

pytestmark = pytest.mark.gpu


def _cp():
    return P.oracle_providers(P.HardwareParams(), precision=N.FO_PREC_FP64)


def test_criterion_01_simulator_bounds():
    """fo_bound <= cost <= sum of all durations, and the reference's values."""
    cp = _cp()
    for w in read("acceptance.json.gz")["criterion1"]:
        g = graph_from_doc(w["graph"])
        c = P.cost(g, cp)
        lo = P.fo_bound(g, cp)
        assert lo <= c + 1e-9 and c <= w["total"] + 1e-9, w["i"]
        assert c == pytest.approx(w["cost"], rel=1e-12) and lo == pytest.approx(w["fo_bound"], rel=1e-12)


def test_criteria_02_03_oracle_equivalence_and_search_invariants():
    """Criterion 2: 20 searches per small workload never go below the
    exhaustive optimum and reach it within 5 % on >= 45 of 50 workloads.
    Criterion 3 on every run: never worse than the start, every enqueue within
    alpha * best, best cost not below its fo_bound."""
    cp = _cp()
    hits, runs = 0, 0
    for w in read("acceptance.json.gz")["criterion2"]:
        g = graph_from_doc(w["graph"])
        k = w["k"]
        exact = P.exhaustive_search(g, cp)
        assert exact.best_cost_us == pytest.approx(w["exact"], rel=1e-12), k
        initial = P.cost(g, cp)
        cfg = P.SearchConfig(alpha=1.1, beta=2, max_unchanged=60)
        # the 20 seeds k*100+i of the reference test, lock-stepped in one driver
        res = P.lockstep_search(g, cfg, cp, [k * 100 + i for i in range(20)])
        best = np.inf
        for r in res:
            runs += 1
            assert r.best_cost_us >= exact.best_cost_us - 1e-9, "found below optimum"
            assert r.best_cost_us <= initial + 1e-9
            assert all(t.cost_us <= cfg.alpha * t.best_cost_us + 1e-9 for t in r.trace if t.enqueued)
            assert r.best_cost_us >= P.fo_bound(r.best_graph, cp) - 1e-9
            best = min(best, r.best_cost_us)
        hits += best / exact.best_cost_us <= 1.05 + 1e-12
    assert runs == 1000
    assert hits >= 45, f"only {hits}/50 within 5%"


def _cp_c8():
    hw = P.HardwareParams(comm_params=P.CommModelParams(C=0.0008, D=400.0))
    return P.oracle_providers(hw, precision=N.FO_PREC_FP64)


def _checked(results, g, cp, cfg):
    initial = P.cost(g, cp)
    for r in results:
        assert r.best_cost_us <= initial + 1e-9
        assert all(t.cost_us <= cfg.alpha * t.best_cost_us + 1e-9 for t in r.trace if t.enqueued)
    return results


def test_criterion_08_ablation_direction():
    """Median best cost is non-increasing as methods are added."""
    from paper_2209_12769_b200.rewrite import OptimizationMethod as M

    g = graph_from_doc(read("acceptance.json.gz")["criterion8"])
    cp = _cp_c8()
    masks = [(M.NON_DUPLICATE_FUSION,), (M.NON_DUPLICATE_FUSION, M.DUPLICATE_FUSION),
             (M.NON_DUPLICATE_FUSION, M.DUPLICATE_FUSION, M.ALLREDUCE_FUSION)]
    medians = []
    for mask in masks:
        cfg = P.SearchConfig(alpha=1.05, beta=10, max_unchanged=100, methods=mask)
        res = _checked(P.lockstep_search(g, cfg, cp, list(range(10))), g, cp, cfg)
        medians.append(float(np.median([r.best_cost_us for r in res])))
    assert medians[0] >= medians[1] - 1e-9 and medians[1] >= medians[2] - 1e-9


def test_criterion_09_alpha_beta_tradeoff():
    """A looser alpha costs more evaluations and finds no worse; a larger beta
    (more rewrites per step) needs fewer evaluations."""
    g = graph_from_doc(read("acceptance.json.gz")["criterion9"])
    cp = _cp_c8()

    def sweep(alpha, beta, max_unchanged):
        cfg = P.SearchConfig(alpha=alpha, beta=beta, max_unchanged=max_unchanged)
        res = _checked(P.lockstep_search(g, cfg, cp, list(range(10))), g, cp, cfg)
        return float(np.median([r.best_cost_us for r in res])), float(np.median([r.candidates_evaluated for r in res]))

    cost_tight, evals_tight = sweep(1.0, 10, 200)
    cost_loose, evals_loose = sweep(1.1, 10, 200)
    assert cost_loose <= cost_tight + 1e-9 and evals_loose > evals_tight
    _, evals_beta1 = sweep(1.05, 1, 100)
    _, evals_beta30 = sweep(1.05, 30, 100)
    assert evals_beta30 < evals_beta1
