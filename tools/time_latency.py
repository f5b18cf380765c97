"""Latency of small batches (search-round sized), memo cleared per call.

usage: time_latency.py [fp32|fp64] cfg:K [cfg:K ...]
FO_TEAM=0/1 is toggled per measurement (warp-per-candidate vs block-per-candidate).
"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N

args = sys.argv[1:]
prec = N.FO_PREC_FP64
if args and args[0] in ("fp32", "fp64"):
    prec = N.FO_PREC_FP32 if args.pop(0) == "fp32" else N.FO_PREC_FP64
specs = args or ["bert:1"]
torch.cuda.set_device(0)
s = torch.cuda.current_stream()
cache = {}
for spec in specs:
    cfg, K = spec.split(":")
    K = int(K)
    if cfg not in cache:
        g, prof, comm, mp, lin = P.load_workload(cfg)
        cp = P.make_cost_providers(prof, comm, mp, precision=prec)
        cache[cfg] = cp.device_graph(g)
    dg = cache[cfg]
    ng, rg, bk, gb = dg.make_candidates(np.arange(K, dtype=np.uint64))
    d = [torch.from_numpy(x).cuda() for x in (ng, rg, bk)]
    cost = torch.empty(K, dtype=torch.float64, device="cuda")
    st = torch.empty(K, dtype=torch.int32, device="cuda")
    out = {"config": cfg, "K": K}
    ref = None
    for team in ("0", "1"):
        os.environ["FO_TEAM"] = team
        ts = []
        for i in range(23):
            N.lib().fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dg.score_device(d[0], d[1], d[2], gb, cost, st, prec)
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        c = cost.cpu().numpy().copy()
        if ref is None:
            ref = c
        else:
            out["same_costs"] = bool(np.array_equal(ref, c))
        out[f"ms_team{team}"] = round(float(np.median(ts)), 4)
        for ph in (1, 2):  # phase stops: after the contraction, after the estimator
            N.lib().fo_set_phase_stop(dg.h, ph)
            tp = []
            for i in range(13):
                N.lib().fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                dg.score_device(d[0], d[1], d[2], gb, cost, st, prec)
                b.record()
                torch.cuda.synchronize()
                if i >= 3:
                    tp.append(a.elapsed_time(b))
            N.lib().fo_set_phase_stop(dg.h, 0)
            out[f"ms_team{team}_stop{ph}"] = round(float(np.median(tp)), 4)
    os.environ.pop("FO_TEAM", None)
    print(json.dumps(out), flush=True)
