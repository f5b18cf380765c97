"""Search benchmark (BASELINE.json configs[0] and [2]): Alg. 1 backtracking
search with reference defaults, R lock-stepped seeds per GPU, frontier
(seed set) sharded across ranks with the per-round best (cost, seed)
exchanged over NCCL.  Reports candidates evaluated per second and search
wall time, next to the oracle port's single-thread search on the same seeds.

  python tools/bench_search.py --config vgg16 --seeds 1
  torchrun --nproc-per-node N tools/bench_search.py --config bert --seeds 16
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="vgg16")
    ap.add_argument("--seeds", type=int, default=1, help="lock-stepped seeds per GPU")
    ap.add_argument("--max-unchanged", type=int, default=1000)
    ap.add_argument("--alpha", type=float, default=1.05)
    ap.add_argument("--beta", type=int, default=10)
    ap.add_argument("--precision", default="fp64")
    ap.add_argument("--oracle-seeds", type=int, default=1, help="seeds re-run on the CPU oracle (rank 0)")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--exchange", default="round", help="round (the per-round exchange) | end (once) | N (every N rounds)")
    ap.add_argument("--lag", type=int, default=0, help="exchanges in flight (0: ShardedSearch's default)")
    args = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N
    from paper_2209_12769_b200.parallel import ShardedSearch

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    prec = N.FO_PREC_FP64 if args.precision == "fp64" else N.FO_PREC_FP32
    g, prof, comm, mp, lin = P.load_workload(args.config)
    cp = P.make_cost_providers(prof, comm, mp, precision=prec)
    cfg = P.SearchConfig(alpha=args.alpha, beta=args.beta, max_unchanged=args.max_unchanged)
    seeds = list(range(args.seeds * ws))
    cp.device_graph(g)  # build the handle outside the timed region
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    local_ws = int(os.environ.get("LOCAL_WORLD_SIZE", str(ws)))
    threads = args.threads or max(1, (os.cpu_count() or 1) // local_ws)  # no oversubscription across ranks
    sh = ShardedSearch(g, cfg, cp, seeds, rank, ws, precision=prec, n_threads=threads)
    if args.lag > 0:
        sh.lag = args.lag
    every = 1 if args.exchange == "round" else (None if args.exchange == "end" else int(args.exchange))
    best_cost, best_seed = sh.run(dev, exchange_every=every)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    # per-seed counters straight from the native search (no graph reconstruction)
    cnt = [sh.s.counters(r) for r in range(len(sh.local_seeds))] if sh.s else []
    bests = sh.s.best_costs() if sh.s else []
    local_evals = sum(c[1] for c in cnt)
    local_steps = max((c[0] for c in cnt), default=0)
    tm = sh.s.timing()
    t = torch.tensor([wall, local_evals, tm["device_ms"], tm["expand_ms"], tm["scored"]], dtype=torch.float64,
                     device=dev)
    if ws > 1:
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        wall_max = float(mx[0])
    else:
        wall_max = float(t[0])
    total_evals = int(t[1])
    line = None
    if rank == 0:
        line = {
            "metric": "search: candidates evaluated/sec and search wall time", "config": args.config,
            "n_gpus": ws, "seeds_total": len(seeds), "seeds_per_gpu": args.seeds, "precision": args.precision,
            "search_cfg": {"alpha": args.alpha, "beta": args.beta, "max_unchanged": args.max_unchanged},
            "wall_s": wall_max, "candidates_evaluated": total_evals, "cand_per_s": total_evals / wall_max,
            "rounds": sh.s.rounds if sh.s else 0, "max_steps_one_seed": local_steps,
            "best_cost_us": best_cost, "best_seed": int(best_seed),
            "rank0_device_ms": tm["device_ms"], "rank0_expand_ms": tm["expand_ms"], "rank0_scored": tm["scored"],
            "host_threads": os.cpu_count(), "exchange": args.exchange, "lag": sh.lag,
            "exchanges": len(sh.best_history),
        }
        if args.oracle_seeds > 0:
            from oracle.oracle import Oracle, load_workload

            o = Oracle(load_workload(args.config), "mp")
            ev, tt, match = 0, 0.0, True
            for s in range(min(args.oracle_seeds, len(cnt))):
                t1 = time.perf_counter()
                r = o.search(alpha=args.alpha, beta=args.beta, max_unchanged=args.max_unchanged, seed=s)
                tt += time.perf_counter() - t1
                ev += r["candidates_evaluated"]
                match &= (r["steps"], r["candidates_evaluated"], r["candidates_enqueued"]) == cnt[s][:3]
                match &= abs(r["best_cost_us"] - bests[s]) <= 1e-9 * r["best_cost_us"]
            line["oracle_port_1thread"] = {"seeds": min(args.oracle_seeds, len(cnt)), "wall_s": tt,
                                           "cand_per_s": ev / tt, "trajectories_match": bool(match)}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
