"""K2 time per estimator arithmetic (FFMA / TF32 / 3xTF32 tensor cores) on the
bench batch, memo off (every fused group estimated) and on: the incremental
path's phase stops 1 (setup) and 2 (+ estimator kernel), CUDA events, L2
flushed and memo emptied before every launch."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "resnet50"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfg)
dg = P.make_cost_providers(prof, comm, mp).device_graph(g)
dg.set_parent()
off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
d_off, d_chg = torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda()
cost = torch.empty(K, dtype=torch.float64, device="cuda"); st = torch.empty(K, dtype=torch.int32, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()
def timed(phase, reps=15):
    N.lib().fo_set_phase_stop(dg.h, phase)
    ts = []
    for i in range(reps + 3):
        flush.zero_(); N.lib().fo_memo_clear(dg.h, N.C.c_void_p(s.cuda_stream))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s); dg.score_delta_device(d_off, d_chg, cost, st, N.FO_PREC_FP32, s.cuda_stream); e1.record(s)
        torch.cuda.synchronize()
        if i >= 3: ts.append(e0.elapsed_time(e1))
    N.lib().fo_set_phase_stop(dg.h, 0)
    return statistics.median(ts)
out = {"config": cfg, "K": K}
for memo in (0, 1):
    N.lib().fo_memo_enable(dg.h, memo)
    for mode, label in ((0, "ffma"), (1, "tf32"), (2, "3xtf32")):
        N.lib().fo_set_estimator_arith(dg.h, mode)
        t1, t2, t0 = timed(1), timed(2), timed(0)
        out[f"memo{memo}/{label}"] = {"k2_ms": round(t2 - t1, 4), "total_ms": round(t0, 4)}
print(json.dumps(out))
