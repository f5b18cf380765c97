"""Single-seed Alg. 1 search latency on a warm handle: the search run three
times (first run builds everything), wall time per run, device time per round
and host expand per round (fo_search_timing)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N

torch.cuda.set_device(0)
for cfgname in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["vgg16", "bert"]):
    g, prof, comm, mp, lin = P.load_workload(cfgname)
    cp = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP64)
    cfg = P.SearchConfig(alpha=1.05, beta=10, max_unchanged=1000)
    cp.device_graph(g)
    for rep in range(3):
        t0 = time.perf_counter()
        res = P.backtracking_search(g, cfg, cp)
        dt = time.perf_counter() - t0
        print(f"{cfgname} run {rep}: {dt*1e3:.1f} ms  best {res.best_cost_us:.3f}  steps {res.steps}  evaluated {res.candidates_evaluated}", flush=True)
