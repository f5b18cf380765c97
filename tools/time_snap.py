"""A/B of the event-loop fast-forward (parent snapshots, score_kernel_inc_k3)
on one batch: the incremental kernel with and without snapshots
(FO_INC_NO_SNAP, read when the plan is built), the general kernel beside
them, costs compared bit for bit.  L2 flushed and memo emptied before every
launch, CUDA events."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["resnet50", "bert", "vgg16"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
prec = N.FO_PREC_FP64 if (len(sys.argv) > 3 and sys.argv[3] == "fp64") else N.FO_PREC_FP32
torch.cuda.set_device(0)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream()

for cfg in cfgs:
    g, prof, comm, mp, lin = P.load_workload(cfg)
    dg = P.make_cost_providers(prof, comm, mp, precision=prec).device_graph(g)
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
    d_off, d_chg = torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda()
    cost = torch.empty(K, dtype=torch.float64, device="cuda")
    st = torch.empty(K, dtype=torch.int32, device="cuda")

    def timed(mode, phase=0, reps=15):
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
        return statistics.median(ts), cost.cpu().numpy().copy(), st.cpu().numpy().copy()

    out = {"config": cfg, "K": K, "prec": "fp64" if prec else "fp32"}
    t0, c0, s0 = timed(0)
    os.environ["FO_INC_NO_SNAP"] = "1"
    dg.set_parent()  # rebuilds the plan without the parent-loop record
    tn, cn, sn = timed(1)
    tn2, _, _ = timed(1, 2)
    del os.environ["FO_INC_NO_SNAP"]
    dg.set_parent()
    ts_, cs, ss = timed(1)
    ts2, _, _ = timed(1, 2)
    N.lib().fo_inc_stats(dg.h, prec, N.ptr(np.zeros(6, np.int64)))  # reset
    _, cd, sd = timed(2, reps=1)
    stats = np.zeros(6, np.int64)
    N.lib().fo_inc_stats(dg.h, prec, N.ptr(stats))
    out["event_loops"], out["fast_forwarded"], out["iters_skipped"] = int(stats[0]), int(stats[1]), int(stats[2])
    out["parent_iters"], out["snapshots"], out["snap_every"] = int(stats[3]), int(stats[4]), int(stats[5])
    out["skipped_share"] = round(stats[2] / max(1, stats[0] * stats[3]), 4)
    out["general_ms"] = round(t0, 4)
    out["inc_nosnap_ms"] = round(tn, 4)
    out["inc_snap_ms"] = round(ts_, 4)
    out["k3_nosnap_ms"] = round(tn - tn2, 4)
    out["k3_snap_ms"] = round(ts_ - ts2, 4)
    out["bitexact_snap_vs_general"] = bool(np.array_equal(cs.view(np.int64), c0.view(np.int64)) and np.array_equal(ss, s0))
    out["bitexact_nosnap_vs_general"] = bool(np.array_equal(cn.view(np.int64), c0.view(np.int64)) and np.array_equal(sn, s0))
    out["handled_by_inc"] = float((sd < 101).mean())
    N.lib().fo_set_delta_mode(dg.h, 1)
    print(json.dumps(out), flush=True)
