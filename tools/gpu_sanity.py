"""Quick device-vs-golden check used during development (run under gpurun)."""
import gzip, json, sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N
from paper_2209_12769_b200.graph import build_graph, FusionGroup
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

def golden_graph(g, sdoc):
    ops = sorted(o.id for o in g.ops)
    covered = set(); groups = []
    for gid, mem, dup in sdoc["groups"]:
        groups.append(FusionGroup(gid, frozenset(mem), frozenset(dup)))
        covered |= set(mem) - set(dup)
    groups += [FusionGroup(o, frozenset([o])) for o in ops if o not in covered]
    cov = set(); buckets = []
    for bid, mem in sdoc["buckets"]:
        buckets.append((bid, mem)); cov |= set(mem)
    buckets += [(a.id, [a.id]) for a in g.allreduces if a.id not in cov]
    return build_graph(g.ops, g.edges, [(a.id, a.producer_op, a.tensor_bytes) for a in g.allreduces],
                       groups=groups, buckets=buckets, meta=g.meta)

names = sys.argv[1:] or ["chain24","residual40","attention36","recurrent30","vgg16","resnet50","bert","gpt2m","synth50k"]
for name in names:
    g, prof, comm, mp, lin = P.load_workload(name)
    cases = json.load(gzip.open(f"{ROOT}/tests/golden/cases/{name}.cases.json.gz","rt"))
    provs = {"mp": P.make_cost_providers(prof, comm, mp), "lin": P.make_cost_providers(prof, comm, lin),
             "analytic": P.make_cost_providers(prof, comm, P.analytic_model(5.0, 1/1024)),
             "oracle": P.oracle_providers(P.HardwareParams())}
    graphs = [golden_graph(g, c["state"]) for c in cases["candidates"]]
    for pname, cp in provs.items():
        for prec in (N.FO_PREC_FP32, N.FO_PREC_FP64):
            cp.precision = prec
            t = time.time()
            c = P.cost_batch(graphs, cp)
            ref = np.array([x["cost"][pname] for x in cases["candidates"]])
            err = np.max(np.abs(c - ref) / np.abs(ref))
            nexact = int(np.sum(c == ref))
            print(f"{name:12s} {pname:8s} prec={prec} maxrel={err:.3e} exact={nexact}/{len(ref)} {time.time()-t:.2f}s", flush=True)
    # timeline check
    cp = provs["mp"]; cp.precision = N.FO_PREC_FP64
    for c, gg in zip(cases["candidates"], graphs):
        if "timeline" not in c: continue
        tl = P.simulate(gg, cp)
        ok = [e[0] for e in tl.compute_events] == [e[0] for e in c["timeline"]["compute"]] and \
             [e[0] for e in tl.comm_events] == [e[0] for e in c["timeline"]["comm"]]
        print(f"{name} timeline {c['i']} ids_ok={ok} mk={tl.makespan_us} ref={c['timeline']['makespan']}", flush=True)
