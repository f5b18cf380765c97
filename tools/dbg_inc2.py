import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
cfg, K, memo = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfg)
dg = P.make_cost_providers(prof, comm, mp).device_graph(g)
dg.set_parent()
off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
def run(mode):
    N.lib().fo_set_delta_mode(dg.h, mode); N.lib().fo_memo_enable(dg.h, memo)
    N.lib().fo_memo_clear(dg.h, N.C.c_void_p(torch.cuda.current_stream().cuda_stream))
    c = torch.empty(K, dtype=torch.float64, device="cuda"); s = torch.empty(K, dtype=torch.int32, device="cuda")
    dg.score_delta_device(torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda(), c, s, N.FO_PREC_FP32)
    torch.cuda.synchronize()
    return c.cpu().numpy(), s.cpu().numpy()
ref, sr = run(0)
for rep in range(3):
    got, sg = run(2)
    bad = np.nonzero((got != ref) & (sg == 0))[0]
    print("rep", rep, "statuses", dict(zip(*np.unique(sg, return_counts=True))), "wrong", len(bad), bad[:10].tolist(), flush=True)
# per-candidate: number of changes and fused groups
nchg = np.diff(off)
print("nchg of wrong:", nchg[bad[:10]].tolist(), "nchg of right:", nchg[:10].tolist())
ng, rg, bk, gb = dg.make_candidates(np.arange(K, dtype=np.uint64))
def nfused(k):
    from collections import Counter
    c = Counter(ng[k].tolist()) + Counter(x for x in rg[k].tolist() if x >= 0)
    return sum(1 for v in c.values() if v > 1), max(c.values())
print("fused(wrong):", [nfused(k) for k in bad[:10]], "fused(right0..9):", [nfused(k) for k in range(10)])
