"""A/B of the sparse-candidate kernels on one batch: general (mode 0) vs
incremental (mode 1), whole kernel and the phase stops (1: after setup/K1,
2: after K2), L2 flushed and memo emptied before every launch, CUDA events."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N

cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
prec = N.FO_PREC_FP64 if (len(sys.argv) > 3 and sys.argv[3] == "fp64") else N.FO_PREC_FP32
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfg)
dg = P.make_cost_providers(prof, comm, mp, precision=prec).device_graph(g)
dg.set_parent()
off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
d_off, d_chg = torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda()
cost = torch.empty(K, dtype=torch.float64, device="cuda")
st = torch.empty(K, dtype=torch.int32, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()


def timed(mode, phase, reps=15):
    N.lib().fo_set_delta_mode(dg.h, mode)
    N.lib().fo_set_phase_stop(dg.h, phase)
    ts = []
    for i in range(reps + 3):
        flush.zero_()
        N.lib().fo_memo_clear(dg.h, N.C.c_void_p(s.cuda_stream))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        dg.score_delta_device(d_off, d_chg, cost, st, prec, s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    N.lib().fo_set_phase_stop(dg.h, 0)
    return statistics.median(ts)


out = {"config": cfg, "K": K, "prec": "fp64" if prec else "fp32"}
for mode in (0, 1, 2):
    out[f"mode{mode}"] = {f"stop{p}": round(timed(mode, p), 4) for p in (1, 2, 0)}
N.lib().fo_set_delta_mode(dg.h, 2)
timed(2, 0, 1)
out["handled_by_inc"] = float((st.cpu().numpy() != 101).mean())
N.lib().fo_set_delta_mode(dg.h, 1)
print(json.dumps(out))
