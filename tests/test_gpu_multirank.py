"""The multi-GPU exchange on a real device with two ranks: ShardedSearch (per
round through round(), in blocks through run(exchange_every=M), and once at
the end) and bench.py's per-step chain fo_batch_best -> all-gather ->
fo_pairs_best.  Both ranks share cuda:0 over gloo (NCCL refuses two ranks on
one GPU; bench.py's N > 1 runs take the NCCL path).  The global results must
equal one process scoring / searching everything."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _search_worker(rank, world, port, q, mode):
    import sys

    sys.path.insert(0, ROOT)
    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N
    from paper_2209_12769_b200.parallel import ShardedSearch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, prof, comm, mpm, lin = P.load_workload("residual40")
        cp = P.make_cost_providers(prof, comm, mpm, precision=N.FO_PREC_FP64)
        cfg = P.SearchConfig(alpha=1.05, beta=10, max_unchanged=80)
        sh = ShardedSearch(g, cfg, cp, list(range(6)), rank, world)
        if mode == "round":
            while sh.round("cpu") > 0:
                pass
            res = sh.best_history[-1]
        elif mode == "block":
            res = sh.run("cpu", exchange_every=7)
        else:
            res = sh.run("cpu", exchange_every=None)
        q.put((rank, res, len(sh.best_history)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["round", "block", "end"])
def test_sharded_search_two_ranks_equals_lockstep(mode):
    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N

    torch.cuda.set_device(0)
    g, prof, comm, mpm, lin = P.load_workload("residual40")
    cp = P.make_cost_providers(prof, comm, mpm, precision=N.FO_PREC_FP64)
    cfg = P.SearchConfig(alpha=1.05, beta=10, max_unchanged=80)
    ref = P.lockstep_search(g, cfg, cp, list(range(6)))
    best = min(range(6), key=lambda r: (ref[r].best_cost_us, r))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_search_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out[0][1] == out[1][1] and out[0][2] == out[1][2]
    assert out[0][1] == (ref[best].best_cost_us, float(best))


def _chain_worker(rank, world, port, q):
    import ctypes
    import sys

    sys.path.insert(0, ROOT)
    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, prof, comm, mpm, lin = P.load_workload("resnet50")
        dg = P.make_cost_providers(prof, comm, mpm).device_graph(g)
        dg.set_parent()
        K = 1024
        off, chg = dg.make_candidates_delta(np.arange(rank * K, (rank + 1) * K, dtype=np.uint64))
        cost = torch.empty(K, dtype=torch.float64, device="cuda")
        st = torch.empty(K, dtype=torch.int32, device="cuda")
        s = torch.cuda.current_stream()
        dg.score_delta_device(torch.from_numpy(off).cuda(), torch.from_numpy(chg).cuda(), cost, st, N.FO_PREC_FP32,
                              s.cuda_stream)
        pair = torch.empty(2, dtype=torch.float64, device="cuda")
        N.lib().fo_batch_best(N.ptr(cost), N.ptr(st), K, rank * K, N.ptr(pair), ctypes.c_void_p(s.cuda_stream))
        gathered = torch.empty(world * 2, dtype=torch.float64)
        dist.all_gather_into_tensor(gathered, pair.cpu())
        g_dev = gathered.cuda()
        final = torch.empty(2, dtype=torch.float64, device="cuda")
        N.lib().fo_pairs_best(N.ptr(g_dev), world, N.ptr(final), ctypes.c_void_p(s.cuda_stream))
        torch.cuda.synchronize()
        q.put((rank, tuple(final.cpu().tolist()), cost.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_bench_exchange_chain_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_chain_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted((q.get(timeout=300) for _ in procs), key=lambda x: x[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    allc = np.concatenate([out[0][2], out[1][2]])
    j = int(np.argmin(allc))  # first minimum: the lowest global id among ties (search.py:124)
    assert out[0][1] == out[1][1] == (float(allc[j]), float(j))


def _nccl_worker(rank, world, port, q, seeds, every):
    import sys

    sys.path.insert(0, ROOT)
    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N
    from paper_2209_12769_b200.parallel import ShardedSearch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    try:
        g, prof, comm, mpm, lin = P.load_workload("residual40")
        cp = P.make_cost_providers(prof, comm, mpm, precision=N.FO_PREC_FP64)
        cfg = P.SearchConfig(alpha=1.05, beta=10, max_unchanged=80)
        sh = ShardedSearch(g, cfg, cp, seeds, rank, world)
        sh.lag = 3
        res = sh.run(torch.device("cuda", rank), exchange_every=every)
        q.put((rank, res, len(sh.best_history)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("seeds,every", [(list(range(6)), 1), (list(range(5)), 3), ([2], 1)])
def test_native_nccl_exchange_two_gpus(seeds, every):
    """ShardedSearch over NCCL on two GPUs: the per-round exchange runs natively
    (fo_xchg); both ranks post the same number of exchanges and return the
    single-process answer (also when rank 1 has no seeds)."""
    import paper_2209_12769_b200 as P
    from paper_2209_12769_b200 import _native as N

    torch.cuda.set_device(0)
    g, prof, comm, mpm, lin = P.load_workload("residual40")
    cp = P.make_cost_providers(prof, comm, mpm, precision=N.FO_PREC_FP64)
    cfg = P.SearchConfig(alpha=1.05, beta=10, max_unchanged=80)
    ref = P.lockstep_search(g, cfg, cp, seeds)
    best = min(range(len(seeds)), key=lambda r: (ref[r].best_cost_us, r))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q, seeds, every)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert out[0][2] == out[1][2] and out[0][2] >= 1
    assert out[0][1] == out[1][1] == (ref[best].best_cost_us, float(best))
