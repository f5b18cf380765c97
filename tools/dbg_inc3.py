import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload("bert")
dg = P.make_cost_providers(prof, comm, mp).device_graph(g)
def run(off, chg, mode):
    N.lib().fo_set_delta_mode(dg.h, mode)
    N.lib().fo_memo_clear(dg.h, N.C.c_void_p(torch.cuda.current_stream().cuda_stream))
    K = len(off) - 1
    c = torch.empty(K, dtype=torch.float64, device="cuda"); s = torch.empty(K, dtype=torch.int32, device="cuda")
    dg.score_delta_device(torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda(), c, s, N.FO_PREC_FP32)
    torch.cuda.synchronize()
    return c.cpu().numpy(), s.cpu().numpy()
dg.set_parent()
off, chg = dg.make_candidates_delta(np.arange(256, dtype=np.uint64))
a, _ = run(off, chg, 1); a0, _ = run(off, chg, 0); a2x, _ = run(off, chg, 2)
print("fresh: inc vs general wrong", np.nonzero(a != a0)[0].tolist(), "mode2 wrong", np.nonzero(a2x != a0)[0].tolist())
ng, rg, bk, _ = dg.make_candidates(np.array([5], dtype=np.uint64))
dg.set_parent(ng[0], rg[0], bk[0])
off2, chg2 = dg.make_candidates_delta(np.arange(256, dtype=np.uint64), base=(ng[0], rg[0], bk[0]))
b, _ = run(off2, chg2, 1); b0, _ = run(off2, chg2, 0)
print("deep: wrong", np.nonzero(b != b0)[0].tolist())
dg.set_parent()
c1, s1 = run(off, chg, 1); c0, _ = run(off, chg, 0); c2, s2 = run(off, chg, 2)
print("back: inc wrong", np.nonzero(c1 != c0)[0].tolist(), "mode2", np.nonzero((c2 != c0) & (s2 == 0))[0].tolist(), dict(zip(*np.unique(s2, return_counts=True))))
print("a0 == c0", np.array_equal(a0, c0))
