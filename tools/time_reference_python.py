"""Time the unmodified reference (fuseopt, pure Python) on ResNet-50 proxy
candidates, here in the build container: (i) one core as-is, (ii) all cores
with multiprocessing.Pool over the candidate list.
Candidates are materialised first (generation is timed separately), each
score is cost() on a fresh HloGraph as the survey prescribes.

  PYTHONPATH=/root/reference/pkg/src python tools/time_reference_python.py [n]
"""
import json
import multiprocessing as mp
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "tests", "golden"))

_G = None


def _init():
    global _G
    import make_golden as mg

    g, profile, comm, mpm, lin = mg.load_workload("resnet50")
    _G = (g, mg.make_cost_providers(profile, comm, mpm))


def _score(state):
    from fuseopt import HloGraph, cost

    g, cp = _G
    c = HloGraph(g.meta, g.ops, g.edges, state[2], state[0], state[1])
    return cost(c, cp)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    import make_golden as mg

    _init()
    g, cp = _G
    t0 = time.time()
    cands = [mg.make_candidate(g, i) for i in range(n)]
    gen = time.time() - t0
    states = [(c.groups, c.buckets, c.allreduces) for c in cands]
    t0 = time.time()
    for s in states:
        _score(s)
    one = time.time() - t0
    cores = os.cpu_count() or 1
    with mp.Pool(cores, initializer=_init) as pool:
        t0 = time.time()
        pool.map(_score, states * 2, chunksize=4)
        many = time.time() - t0
    print(json.dumps({"reference": "fuseopt (unmodified, pure Python)", "config": "resnet50", "candidates": n,
                      "generation_s_per_candidate": gen / n, "score_1_core_cand_per_s": n / one,
                      "score_all_cores_cand_per_s": 2 * n / many, "cores": cores,
                      "host": "build container (no GPU); the GPU box's host cores differ"}))


if __name__ == "__main__":
    main()
