"""Bench lines for BASELINE.json configs[3] and [4] (the headline bench.py line
is configs[1]).

  python tools/bench_configs.py gpt2-sweep [--batch 256]
      GPT-2-medium proxy (V=5000): the 13 bucket-size thresholds x {AR-only,
      greedy op fusion + AR} parents, built by this package's
      greedy_postorder_fusion / threshold_allreduce_fusion and checked against
      the reference's own (tests/golden/sweep_gpt2m.json.gz), each scored and
      then used as the parent of a random-candidate batch.
  python tools/bench_configs.py synth50k [--batch 8192]
      synthetic 50k-op DAG: one round of random candidates per GPU
      (64k per round on 8 GPUs = 8192 per GPU).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def timed_score(dg, ng, rg, bk, gb, prec, reps=5):
    """Dense candidates resident on the device; memo emptied before each rep."""
    import ctypes

    import numpy as np
    import torch

    from paper_2209_12769_b200 import _native as N

    d = [torch.from_numpy(x).cuda() for x in (ng, rg, bk)]
    K = ng.shape[0]
    cost = torch.empty(K, dtype=torch.float64, device="cuda")
    st = torch.empty(K, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    dg.score_device(d[0], d[1], d[2], gb, cost, st, prec)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        N.lib().fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dg.score_device(d[0], d[1], d[2], gb, cost, st, prec)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return cost.cpu().numpy(), st.cpu().numpy(), float(np.median(ts))


def timed_score_delta(dg, off, chg, prec, reps=5):
    """Sparse candidates against the handle's resident parent (fo_score_delta)."""
    import ctypes

    import numpy as np
    import torch

    from paper_2209_12769_b200 import _native as N

    K = len(off) - 1
    d_off, d_chg = torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda()
    cost = torch.empty(K, dtype=torch.float64, device="cuda")
    st = torch.empty(K, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    dg.score_delta_device(d_off, d_chg, cost, st, prec)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        N.lib().fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dg.score_delta_device(d_off, d_chg, cost, st, prec)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return cost.cpu().numpy(), st.cpu().numpy(), float(np.median(ts))


def gpt2_sweep(args):
    import numpy as np
    import torch

    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N
    from _golden import graph_with_state, read

    torch.cuda.set_device(0)
    prec = N.FO_PREC_FP64 if args.precision == "fp64" else N.FO_PREC_FP32
    g, prof, comm, mp, lin = P.load_workload("gpt2m")
    cp = P.make_cost_providers(prof, comm, mp, precision=prec)
    cp64 = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)  # decision-exact parents
    dg = cp.device_graph(g)
    sweep = read("sweep_gpt2m.json.gz")
    rows, worst, total_c, total_ms, gen_s, total_ms_dense = [], 0.0, 0, 0.0, 0.0, 0.0
    from paper_2209_12769_b200.graph import state_arrays
    from _golden import canon_doc, canon_graph

    # parents built by this package (greedy op fusion, then the threshold scan
    # in simulated production order); the reference's parents are the check
    t0 = time.perf_counter()
    greedy = P.greedy_postorder_fusion(g)
    parents_s = time.perf_counter() - t0
    match = canon_graph(greedy) == canon_doc(g, sweep["greedy"]["state"])
    for ent in sweep["sweep"]:
        t0 = time.perf_counter()
        built = {"ar_only": P.threshold_allreduce_fusion(g, ent["T"], cp64),
                 "both": P.threshold_allreduce_fusion(greedy, ent["T"], cp64)}
        parents_s += time.perf_counter() - t0
        for kind in ("ar_only", "both"):
            parent = built[kind]
            match &= canon_graph(parent) == canon_doc(g, ent[kind]["state"])
            c_dev = P.cost(parent, cp)
            rel = abs(c_dev - ent[kind]["cost"]) / ent[kind]["cost"]
            worst = max(worst, rel)
            ng0, rg0, bk0, _, _, _ = state_arrays(parent)
            t0 = time.perf_counter()
            dg.set_parent(ng0, rg0, bk0)  # the parent stays resident; candidates are its changes
            off, chg = dg.make_candidates_delta(np.arange(args.batch, dtype=np.uint64), base=(ng0, rg0, bk0))
            gen_s += time.perf_counter() - t0
            ng, rg, bk, gb = dg.make_candidates(np.arange(args.batch, dtype=np.uint64), base=(ng0, rg0, bk0))
            c2, st2, ms_d = timed_score(dg, ng, rg, bk, gb, prec, reps=3)
            # sparse while the changes are fewer bytes than the dense ids (a
            # duplicated giant group of a greedy parent rewrites thousands)
            sparse = 8 * float(off[-1]) / args.batch < (2 * dg.V + dg.A)  # at most a quarter of int32 ids
            if sparse:
                cost, st, ms = timed_score_delta(dg, off, chg, prec)
            else:
                cost, st, ms = c2, st2, ms_d
            assert (st == 0).all() and np.array_equal(c2, cost)
            total_c += args.batch
            total_ms += ms
            total_ms_dense += ms_d
            rows.append({"T": ent["T"], "parent": kind, "parent_cost_us": c_dev, "ref_parent_cost_us": ent[kind]["cost"],
                         "batch_best_us": float(cost.min()), "batch_ms": ms, "encoding": "sparse" if sparse else "dense",
                         "changes_per_candidate": float(off[-1]) / args.batch})
    line = {"metric": "fusion candidates scored/sec (GNN est.+sim)", "config": "gpt2m bucket-size sweep",
            "value": total_c / (total_ms / 1e3), "unit": "candidates/s", "n_gpus": 1,
            "encoding": "per parent: sparse changes vs the resident parent, dense ids when the changes are larger",
            "value_dense_int32": total_c / (total_ms_dense / 1e3),
            "thresholds": len(sweep["sweep"]), "batch_per_parent": args.batch, "parents": len(rows),
            "parent_cost_max_rel_err_vs_reference": worst, "parents_match_reference": bool(match),
            "parents_build_s": parents_s, "candidate_generation_s": gen_s,
            "best": min(rows, key=lambda r: r["batch_best_us"]), "rows": rows}
    print(json.dumps(line))


def synth50k(args):
    import numpy as np
    import torch

    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N

    torch.cuda.set_device(0)
    prec = N.FO_PREC_FP32
    g, prof, comm, mp, lin = P.load_workload("synth50k")
    cp = P.make_cost_providers(prof, comm, mp, precision=prec)
    dg = cp.device_graph(g)
    # every candidate distinct (the incremental engine: ~0.5 ms per candidate
    # per thread at 50k ops), in the sparse form the round is scored in
    nd = min(args.distinct, args.batch)
    t0 = time.perf_counter()
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(nd, dtype=np.uint64), beta=args.beta)
    gen_s = time.perf_counter() - t0
    if nd < args.batch:  # tile the distinct set to the round size
        reps_ = (args.batch + nd - 1) // nd
        sizes = np.diff(off)
        sizes = np.tile(sizes, reps_)[: args.batch]
        chg = np.concatenate([chg] * reps_)[: int(sizes.sum())]
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    cost, st, ms = timed_score_delta(dg, off, chg, prec, reps=3)
    # the same round with dense int32 encodings, for comparison
    V, A = dg.V, dg.A
    base = np.concatenate([np.arange(V), -np.ones(V), np.arange(A)]).astype(np.int32)
    dense = np.tile(base, (args.batch, 1))
    for k in range(args.batch):
        c = chg[off[k]:off[k + 1]]
        dense[k, c[:, 0]] = c[:, 1]
    c2, st2, ms_dense = timed_score(dg, np.ascontiguousarray(dense[:, :V]), np.ascontiguousarray(dense[:, V:2 * V]),
                                    np.ascontiguousarray(dense[:, 2 * V:]), 2 * V + 2, prec, reps=3)
    assert np.array_equal(c2, cost) and np.array_equal(st2, st)
    line = {"metric": "fusion candidates scored/sec (GNN est.+sim)", "config": "synthetic 50k-op DAG, one round",
            "value": args.batch / (ms / 1e3), "unit": "candidates/s", "n_gpus": 1, "batch": args.batch,
            "beta": args.beta, "ms_per_round": ms, "encoding": "sparse changes vs resident parent",
            "changes_per_candidate": float(off[-1]) / args.batch, "bytes_per_candidate_sparse": 8 * float(off[-1]) / args.batch + 4,
            "bytes_per_candidate_dense": 4 * (2 * V + A), "ms_per_round_dense_int32": ms_dense,
            "candidate_generation_s": gen_s, "distinct_candidates": nd,
            "statuses": {str(k): int(v) for k, v in zip(*np.unique(st, return_counts=True))},
            "best_us": float(cost[st == 0].min()) if (st == 0).any() else None}
    if args.check > 0:
        from oracle.oracle import Oracle, load_workload

        o = Oracle(load_workload("synth50k"), "mp")
        t1 = time.perf_counter()
        errs = []
        for i in range(args.check):
            s_, c = o.cost(*o.make_candidate(i, args.beta))
            errs.append(abs(c - cost[i]) / c)
        line["oracle_check"] = {"candidates": args.check, "max_rel_err": max(errs),
                                "oracle_s_per_candidate": (time.perf_counter() - t1) / args.check}
    print(json.dumps(line))


def synth50k_sharded(args):
    """BASELINE configs[4] on N GPUs of one box (torchrun): rank r scores its
    own `batch` candidates (seeds r*batch..), then the round's best (cost,
    candidate id) is exchanged (device argmin, 16-byte all-gather, argmin over
    the pairs).  Time = max over ranks of the device-timed round."""
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N

    ws, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    prec = N.FO_PREC_FP32
    g, prof, comm, mp, lin = P.load_workload("synth50k")
    dg = P.make_cost_providers(prof, comm, mp, precision=prec).device_graph(g)
    B = args.batch
    t0 = time.perf_counter()
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(rank * B, (rank + 1) * B, dtype=np.uint64), beta=args.beta,
                                        n_threads=max(1, (os.cpu_count() or 1) // local_ws))
    gen_s = time.perf_counter() - t0
    d_off, d_chg = torch.from_numpy(off).to(dev), torch.from_numpy(chg).to(dev)
    cost = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    pair = torch.empty(2, dtype=torch.float64, device=dev)
    gathered = torch.empty(2 * ws, dtype=torch.float64, device=dev)
    final = torch.empty(2, dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream()
    cs = ctypes.c_void_p(s.cuda_stream)

    def round_():
        dg.score_delta_device(d_off, d_chg, cost, st, prec, s.cuda_stream)
        N.lib().fo_batch_best(N.ptr(cost), N.ptr(st), B, rank * B, N.ptr(pair), cs)
        dist.all_gather_into_tensor(gathered, pair)
        N.lib().fo_pairs_best(N.ptr(gathered), ws, N.ptr(final), cs)

    round_()
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        N.lib().fo_memo_clear(dg.h, cs)
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        round_()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = torch.tensor([float(np.median(ts)), gen_s], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    best = final.cpu().numpy()
    if rank == 0:
        print(json.dumps({"metric": "fusion candidates scored/sec (GNN est.+sim)",
                          "config": "synthetic 50k-op DAG, one round, candidates sharded over GPUs",
                          "value": B * ws / (float(t[0]) / 1e3), "unit": "candidates/s", "n_gpus": ws,
                          "candidates_per_round": B * ws, "ms_per_round_max_over_ranks": float(t[0]),
                          "candidate_generation_s_max": float(t[1]), "best": {"cost_us": float(best[0]),
                                                                            "candidate": int(best[1])},
                          "scaling": "weak"}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["gpt2-sweep", "synth50k"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--beta", type=int, default=10)
    ap.add_argument("--check", type=int, default=2)
    ap.add_argument("--distinct", type=int, default=8192)
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    a = ap.parse_args()
    if a.what == "synth50k" and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        a.batch = a.batch or 8192
        synth50k_sharded(a)
    elif a.what == "gpt2-sweep":
        a.batch = a.batch or 256
        gpt2_sweep(a)
    else:
        a.batch = a.batch or 8192
        synth50k(a)
