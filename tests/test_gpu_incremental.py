"""The incremental sparse-candidate kernel (csrc/score_inc.cuh) against the
general kernel: every cost and status identical, bit for bit, on the bench
batch, on every workload, from unfused and from deep (fused, replicated)
parents, in fp32 and fp64.  Mode 2 (no fallback) shows how many candidates
the incremental kernel scored itself."""

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)


def _handle(name, precision):
    g, prof, comm, mp, lin = P.load_workload(name)
    return g, P.make_cost_providers(prof, comm, mp, precision=precision).device_graph(g)


def _score(dg, off, chg, precision, mode, memo=True):
    import torch

    N.lib().fo_set_delta_mode(dg.h, mode)
    N.lib().fo_memo_enable(dg.h, 1 if memo else 0)
    try:
        N.lib().fo_memo_clear(dg.h, N.C.c_void_p(torch.cuda.current_stream().cuda_stream))  # stream-ordered
        K = len(off) - 1
        c = torch.empty(K, dtype=torch.float64, device="cuda")
        s = torch.empty(K, dtype=torch.int32, device="cuda")
        dg.score_delta_device(torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda(), c, s, precision)
        torch.cuda.synchronize()
        return c.cpu().numpy(), s.cpu().numpy()
    finally:
        N.lib().fo_set_delta_mode(dg.h, 1)
        N.lib().fo_memo_enable(dg.h, 1)


def _check(dg, off, chg, precision, min_inc_share):
    ref, st_ref = _score(dg, off, chg, precision, 0)
    got, st = _score(dg, off, chg, precision, 1)
    assert np.array_equal(st, st_ref)
    assert np.array_equal(got, ref), f"max diff {np.max(np.abs(got - ref))}"
    only, st_only = _score(dg, off, chg, precision, 2)
    handled = st_only != 101
    assert handled.mean() >= min_inc_share, f"incremental kernel scored only {handled.mean():.3f}"
    assert np.array_equal(only[handled], ref[handled]) and np.array_equal(st_only[handled], st_ref[handled])
    return handled.mean()


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
@pytest.mark.parametrize("name,K", [("resnet50", 4096), ("bert", 2048), ("vgg16", 2048), ("chain24", 512),
                                    ("residual40", 512), ("attention36", 512), ("recurrent30", 512),
                                    ("gpt2m", 512)])
def test_incremental_equals_general_from_unfused_parent(name, K, precision):
    g, dg = _handle(name, precision)
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64), beta=10)
    _check(dg, off, chg, precision, 0.99)


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
@pytest.mark.parametrize("name", ["resnet50", "bert", "attention36", "residual40", "recurrent30", "vgg16"])
def test_incremental_equals_general_from_deep_parents(name, precision):
    """Parents several rounds deep (fused groups, replicas, merged buckets):
    every slot kind, vanishing groups and rank changes get exercised."""
    g, dg = _handle(name, precision)
    base = None
    for rnd in range(4):
        ng, rg, bk, _ = dg.make_candidates(np.arange(rnd * 7919, rnd * 7919 + 8, dtype=np.uint64), beta=10, base=base)
        base = (ng[rnd % 8], rg[rnd % 8], bk[rnd % 8])
        dg.set_parent(*base)
        off, chg = dg.make_candidates_delta(np.arange(1000 * rnd, 1000 * rnd + 768, dtype=np.uint64), beta=10,
                                            base=base)
        _check(dg, off, chg, precision, 0.95)


def test_incremental_plan_follows_parent_and_model_changes():
    """A new parent (fo_set_parent) or cost model rebuilds the plan."""
    g, prof, comm, mp, lin = P.load_workload("bert")
    cp = P.make_cost_providers(prof, comm, mp)
    dg = cp.device_graph(g)
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(256, dtype=np.uint64))
    a, _ = _score(dg, off, chg, N.FO_PREC_FP32, 1)
    ng, rg, bk, _ = dg.make_candidates(np.array([5], dtype=np.uint64))
    dg.set_parent(ng[0], rg[0], bk[0])
    off2, chg2 = dg.make_candidates_delta(np.arange(256, dtype=np.uint64), base=(ng[0], rg[0], bk[0]))
    b, sb = _score(dg, off2, chg2, N.FO_PREC_FP32, 1)
    b0, sb0 = _score(dg, off2, chg2, N.FO_PREC_FP32, 0)
    assert np.array_equal(b, b0) and np.array_equal(sb, sb0)
    dg.set_parent()
    a2, _ = _score(dg, off, chg, N.FO_PREC_FP32, 1)
    assert np.array_equal(a, a2)


def test_incremental_hands_back_invalid_and_oversized_candidates():
    """Out-of-range ids, duplicate indices and more changes than the fast path
    holds are handed to the general kernel, which reports them as before."""
    g, dg = _handle("resnet50", N.FO_PREC_FP32)
    dg.set_parent()
    V, A = dg.V, dg.A
    off, chg = dg.make_candidates_delta(np.arange(8, dtype=np.uint64))
    cands = [chg[off[k]:off[k + 1]] for k in range(8)]
    cands.append(np.array([[0, 2 * V + 5]], np.int32))              # group id out of range
    cands.append(np.array([[2 * V, A + 3]], np.int32))               # bucket id out of range
    big = np.array([[2 * V + a, 0] for a in range(1, 71)], np.int32)  # 70 changes: ARs 1..70 into bucket 0
    cands.append(big)
    off2 = np.concatenate([[0], np.cumsum([len(c) for c in cands])]).astype(np.int32)
    chg2 = np.concatenate(cands).astype(np.int32)
    ref, st_ref = _score(dg, off2, chg2, N.FO_PREC_FP32, 0)
    got, st = _score(dg, off2, chg2, N.FO_PREC_FP32, 1)
    assert np.array_equal(st, st_ref) and np.array_equal(got, ref)
    assert st[8] == N.FO_INVALID_ARG and st[9] == N.FO_INVALID_ARG
    _, st_only = _score(dg, off2, chg2, N.FO_PREC_FP32, 2)
    assert (st_only[8:] >= 101).all() and (st_only[:8] < 101).all()  # 101+: handed back (110 + reason in mode 2)


def test_plan_built_under_a_phase_stop_is_still_exact():
    """The measurement hook (fo_set_phase_stop) must not leak into the plan:
    a plan first built while a phase stop is set still carries the parent's
    full durations."""
    g, dg = _handle("vgg16", N.FO_PREC_FP32)
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(512, dtype=np.uint64))
    ref, _ = _score(dg, off, chg, N.FO_PREC_FP32, 0)
    g2, dg2 = _handle("vgg16", N.FO_PREC_FP32)
    dg2.set_parent()
    N.lib().fo_set_phase_stop(dg2.h, 1)
    _score(dg2, off, chg, N.FO_PREC_FP32, 1)  # plan built here
    N.lib().fo_set_phase_stop(dg2.h, 0)
    got, _ = _score(dg2, off, chg, N.FO_PREC_FP32, 1)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("precision", [N.FO_PREC_FP32, N.FO_PREC_FP64])
@pytest.mark.parametrize("name,K", [("resnet50", 4096), ("bert", 1024), ("vgg16", 1024)])
def test_event_loop_fast_forward_is_exact_and_used(name, K, precision, monkeypatch):
    """Candidates start their event loop from the parent's last snapshot
    before the first touched node becomes ready: same costs as the general
    kernel and as the incremental kernel started at level 0, and most
    candidates do fast-forward."""
    g, dg = _handle(name, precision)
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
    ref, st_ref = _score(dg, off, chg, precision, 0)
    stats = np.zeros(6, np.int64)
    N.lib().fo_inc_stats(dg.h, precision, N.ptr(stats))  # reset
    only, st_only = _score(dg, off, chg, precision, 2)
    N.lib().fo_inc_stats(dg.h, precision, N.ptr(stats))
    handled = st_only < 101
    assert handled.mean() >= 0.95
    assert np.array_equal(only[handled], ref[handled]) and np.array_equal(st_only[handled], st_ref[handled])
    loops, ff, skipped, iters, nsnap = (int(x) for x in stats[:5])
    assert nsnap > 0 and iters > 0 and loops >= handled.sum()
    assert ff >= 0.3 * loops, stats
    assert 0 < skipped <= ff * iters
    monkeypatch.setenv("FO_INC_NO_SNAP", "1")
    dg.set_parent()  # the plan is rebuilt without the parent-loop record
    got0, st0 = _score(dg, off, chg, precision, 1)
    N.lib().fo_inc_stats(dg.h, precision, N.ptr(stats))
    assert stats[4] == 0
    assert np.array_equal(got0, ref) and np.array_equal(st0, st_ref)
