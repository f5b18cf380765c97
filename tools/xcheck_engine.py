import sys
import os, sys, time, numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2209_12769_b200 as P
from paper_2209_12769_b200.rewrite import engine_graph
def both(dg, seeds, beta, base, nt=8, mask=7):
    os.environ.pop("FO_ENGINE", None)
    t=time.perf_counter(); a = dg.make_candidates(seeds, beta, mask, base, nt); ta=time.perf_counter()-t
    os.environ["FO_ENGINE"]="full"
    t=time.perf_counter(); b = dg.make_candidates(seeds, beta, mask, base, nt); tb=time.perf_counter()-t
    os.environ.pop("FO_ENGINE", None)
    bad = [k for k in range(len(seeds)) if not all(np.array_equal(x[k], y[k]) for x, y in zip(a[:3], b[:3]))]
    return a, bad, ta, tb
tot=0
for name in ["chain24","residual40","attention36","recurrent30","vgg16","resnet50","bert"]:
    g = P.load_workload(name)[0]; dg = engine_graph(g)
    base = None
    for rnd in range(6):
        a, bad, ta, tb = both(dg, np.arange(rnd*1000, rnd*1000+200, dtype=np.uint64), 30, base)
        tot += len(bad)
        if bad: print(name, rnd, "BAD", bad[:5])
        k = rnd % 64
        base = (a[0][k].copy(), a[1][k].copy(), a[2][k].copy())
    print(name, "ok so far; last inc/full", round(ta,3), round(tb,3), flush=True)
for name in ["gpt2m", "synth50k"]:
    g = P.load_workload(name)[0]; dg = engine_graph(g)
    n = 128 if name == "gpt2m" else 32
    a, bad, ta, tb = both(dg, np.arange(n, dtype=np.uint64), 10, None)
    tot += len(bad)
    print(name, "bad", len(bad), f"inc {ta:.3f}s full {tb:.3f}s for {n}", flush=True)
print("TOTAL BAD", tot)
