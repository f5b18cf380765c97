"""Host-side cost of one asynchronous scoring launch (fo_score), by batch size."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "bert"
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfg)
cp = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
dg = cp.device_graph(g)
for K in (3, 48, 300, 700, 4096):
    ng, rg, bk, gb = dg.make_candidates(np.arange(K, dtype=np.uint64))
    d = [torch.from_numpy(x).cuda() for x in (ng, rg, bk)]
    cost = torch.empty(K, dtype=torch.float64, device="cuda"); st = torch.empty(K, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): dg.score_device(d[0], d[1], d[2], gb, cost, st, N.FO_PREC_FP64, s)
    torch.cuda.synchronize()
    host, tot = [], []
    for _ in range(20):
        t0 = time.perf_counter(); dg.score_device(d[0], d[1], d[2], gb, cost, st, N.FO_PREC_FP64, s); t1 = time.perf_counter()
        torch.cuda.synchronize(); t2 = time.perf_counter()
        host.append((t1 - t0) * 1e3); tot.append((t2 - t0) * 1e3)
    print(json.dumps({"config": cfg, "K": K, "launch_host_ms": round(float(np.median(host)), 4), "total_ms": round(float(np.median(tot)), 4)}))
