"""A/B of the speculative search driver (FO_SEARCH_SPEC) in one process."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
cfgname = sys.argv[1] if len(sys.argv) > 1 else "bert"
seeds_list = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,4,16").split(",")]
torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload(cfgname)
cp = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
cp.device_graph(g)
cfg = P.SearchConfig()
for R in seeds_list:
    for rep in range(2):
        for mode in ("0", "1"):
            os.environ["FO_SEARCH_SPEC"] = mode
            t = time.perf_counter()
            s = P.LockstepSearch(g, cfg, cp, list(range(R)))
            res = s.run()
            wall = time.perf_counter() - t
            tm = s.timing()
            ev = sum(r.candidates_evaluated for r in res)
            print(json.dumps({"config": cfgname, "seeds": R, "spec": mode, "wall_s": round(wall, 4), "evaluated": ev,
                              "device_ms": round(tm["device_ms"], 1), "expand_ms": round(tm["expand_ms"], 1),
                              "scored": tm["scored"]}), flush=True)
