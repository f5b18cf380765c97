"""Per-phase latency of small batches (search-round sized), memo cleared per
call: K1 (contract), K1+K2 (estimate), full (simulate), via fo_set_phase_stop.

usage: time_latency_phases.py [fp32|fp64] cfg:K [cfg:K ...]
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
    for ph, name in ((1, "k1"), (2, "k1k2"), (0, "full")):
        N.lib().fo_set_phase_stop(dg.h, ph)
        ts = []
        for i in range(43):
            N.lib().fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            dg.score_device(d[0], d[1], d[2], gb, cost, st, prec)
            b.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(a.elapsed_time(b))
        out[f"ms_{name}"] = round(float(np.median(ts)), 4)
    N.lib().fo_set_phase_stop(dg.h, 0)
    print(json.dumps(out), flush=True)
