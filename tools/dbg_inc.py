"""One sparse batch through one mode / phase stop (debugging aid):
python tools/dbg_inc.py CONFIG K MODE STOP [MEMO]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
cfg, K, mode, stop = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
memo = int(sys.argv[5]) if len(sys.argv) > 5 else 1
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfg)
dg = P.make_cost_providers(prof, comm, mp).device_graph(g)
dg.set_parent()
off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
N.lib().fo_set_delta_mode(dg.h, mode)
N.lib().fo_memo_enable(dg.h, memo)
N.lib().fo_set_phase_stop(dg.h, stop)
c = torch.empty(K, dtype=torch.float64, device="cuda"); s = torch.empty(K, dtype=torch.int32, device="cuda")
for rep in range(2):
    dg.score_delta_device(torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda(), c, s, N.FO_PREC_FP32)
    torch.cuda.synchronize()
    print(cfg, K, "mode", mode, "stop", stop, "memo", memo, "rep", rep, "status", dict(zip(*np.unique(s.cpu().numpy(), return_counts=True))), float(c.sum()), flush=True)
