"""Break the bench's e2e step (fo_memo_clear + fo_score_delta_host) into parts:
host wall per call of each piece, ResNet-50 4,096 sparse candidates."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N

torch.cuda.set_device(0)
g, prof, comm, mp, lin = P.load_workload("resnet50")
cp = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP32)
dg = cp.device_graph(g)
dg.set_parent()
K = 4096
off, chg = dg.make_candidates_delta(np.arange(K, dtype=np.uint64))
h_off = torch.from_numpy(off).pin_memory()
h_chg = torch.from_numpy(chg).pin_memory()
h_cost = torch.empty(K, dtype=torch.float64).pin_memory()
h_st = torch.empty(K, dtype=torch.int32).pin_memory()
L = N.lib()


def clear():
    L.fo_memo_clear(dg.h, None)


def score():
    assert L.fo_score_delta_host(dg.h, N.ptr(h_off), N.ptr(h_chg), K, N.FO_PREC_FP32, N.ptr(h_cost), N.ptr(h_st)) == 0


def timeit(fn, n=50, sync=True):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
        if sync:
            torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


print("memo_clear+score ms", round(timeit(lambda: (clear(), score())), 4))
print("score only (warm memo) ms", round(timeit(score), 4))
print("memo_clear only ms", round(timeit(clear), 4))
d_off, d_chg = h_off.cuda(), h_chg.cuda()
cost = torch.empty(K, dtype=torch.float64, device="cuda")
st = torch.empty(K, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()


def dev():
    L.fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
    dg.score_delta_device(d_off, d_chg, cost, st, N.FO_PREC_FP32, s.cuda_stream)


print("device memo_clear+score (host wall, sync) ms", round(timeit(dev), 4))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
ts = []
for i in range(20):
    ev[0].record()
    L.fo_memo_clear(dg.h, ctypes.c_void_p(s.cuda_stream))
    ev[1].record()
    dg.score_delta_device(d_off, d_chg, cost, st, N.FO_PREC_FP32, s.cuda_stream)
    ev[2].record()
    torch.cuda.synchronize()
    ts.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
print("device-timed memset / kernel ms", np.median(np.array(ts), axis=0).round(4).tolist())
