"""Minimal driver for ncu: score one batch of candidates a few times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
prec = N.FO_PREC_FP64 if (len(sys.argv) > 3 and sys.argv[3] == "fp64") else N.FO_PREC_FP32
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfg)
cp = P.make_cost_providers(prof, comm, mp, precision=prec)
dg = cp.device_graph(g)
delta = os.environ.get("FO_PROF_ENCODING", "delta") == "delta"  # bench.py's default encoding
cost = torch.empty(K, dtype=torch.float64, device="cuda"); st = torch.empty(K, dtype=torch.int32, device="cuda")
if delta:
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
    d_off, d_chg = torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda()
else:
    ng, rg, bk, gb = dg.make_candidates(np.arange(K, dtype=np.uint64))
    d = [torch.from_numpy(x).cuda() for x in (ng, rg, bk)]
for _ in range(reps):
    if os.environ.get("FO_PROF_MEMO_CLEAR", "1") == "1":  # batch-local memo, as bench.py
        N.lib().fo_memo_clear(dg.h, None)
    if delta:
        dg.score_delta_device(d_off, d_chg, cost, st, prec)
    else:
        dg.score_device(d[0], d[1], d[2], gb, cost, st, prec)
torch.cuda.synchronize()
print("ok", float(cost.mean()), int(st.max()))
