"""A/B of the second-pass geometry (FO_RETRY_TEAM) on the GPT-2 greedy parents."""
import os, sys, time, json, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
from paper_2209_12769_b200.graph import state_arrays
from _golden import read, graph_with_state
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload("gpt2m")
doc = read("sweep_gpt2m.json.gz")
s = torch.cuda.current_stream()
for prec in (N.FO_PREC_FP32, N.FO_PREC_FP64):
    cp = P.make_cost_providers(prof, comm, mp, precision=prec)
    dg = cp.device_graph(g)
    b = state_arrays(graph_with_state(g, doc["sweep"][0]["both"]["state"]))[:3]
    ng, rg, bk, gb = dg.make_candidates(np.arange(512, dtype=np.uint64), base=b)
    d = [torch.from_numpy(x).cuda() for x in (ng, rg, bk)]
    out = {}
    for mode in ("0", "1", "0", "1"):
        os.environ["FO_RETRY_TEAM"] = mode
        cost = torch.empty(512, dtype=torch.float64, device="cuda"); st = torch.empty(512, dtype=torch.int32, device="cuda")
        dg.score_device(d[0], d[1], d[2], gb, cost, st, prec); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            N.lib().fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); dg.score_device(d[0], d[1], d[2], gb, cost, st, prec); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        c = cost.cpu().numpy()
        out.setdefault(mode, c)
        rel = float(np.max(np.abs(c - out["0"]) / np.abs(out["0"])))
        print(json.dumps({"prec": prec, "retry_team": mode, "ms": [round(t, 2) for t in ts], "max_status": int(st.max()),
                          "max_rel_vs_warp": rel}), flush=True)
