"""Time the score kernel on a config batch (CUDA events, L2 flushed), for A/B of builds."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
prec = N.FO_PREC_FP64 if (len(sys.argv) > 3 and sys.argv[3] == "fp64") else N.FO_PREC_FP32
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfg)
cp = P.make_cost_providers(prof, comm, mp, precision=prec)
dg = cp.device_graph(g)
ng, rg, bk, gb = dg.make_candidates(np.arange(K, dtype=np.uint64))
d = [torch.from_numpy(x).cuda() for x in (ng, rg, bk)]
cost = torch.empty(K, dtype=torch.float64, device="cuda"); st = torch.empty(K, dtype=torch.int32, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for _ in range(3): dg.score_device(d[0], d[1], d[2], gb, cost, st, prec)
ts = []
for _ in range(10):
    flush.zero_()
    N.lib().fo_memo_clear(dg.h, __import__("ctypes").c_void_p(torch.cuda.current_stream().cuda_stream))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); dg.score_device(d[0], d[1], d[2], gb, cost, st, prec); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ref = cost.cpu().numpy()
print(json.dumps({"lib": os.environ.get("FO_LIB_PATH", "default"), "config": cfg, "K": K, "prec": int(prec),
                  "ms_median": float(np.median(ts)), "ms_min": float(min(ts)), "cand_per_s": K / (float(np.median(ts)) / 1e3),
                  "max_status": int(st.max()), "cost_sum": float(ref.sum())}))
