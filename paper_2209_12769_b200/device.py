"""Device handles: one ``fo_graph`` (include/disco_b200.h) per static graph and
cost-provider configuration, plus the state encoding that crosses the C-ABI."""

from __future__ import annotations

import ctypes as C
import math
import threading

import numpy as np

from . import _native as N
from .errors import DeviceError, _raise
from .graph import KIND_CODE, HloGraph, state_arrays


def current_device() -> int:
    """CUDA device of the calling rank, or -1 (host-only handle: the native
    batch-expand engine works, every device entry point raises)."""
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return -1


def _host_array(x, dtype, name, ndim, writable=False):
    """A host buffer that can cross the C-ABI by pointer: numpy arrays or CPU
    torch tensors of exactly ``dtype``, C-contiguous (no silent copy -- the
    library writes into / reads from this very memory asynchronously)."""
    try:
        import torch

        if isinstance(x, torch.Tensor):
            if x.device.type != "cpu":
                raise ValueError(f"{name} must be a host buffer, got a {x.device} tensor")
            x = x.numpy()
    except ImportError:
        pass
    if not isinstance(x, np.ndarray):
        raise TypeError(f"{name} must be a numpy array or a CPU tensor")
    if x.dtype != dtype:
        raise TypeError(f"{name} must be {np.dtype(dtype).name}, got {x.dtype}")
    if x.ndim != ndim or not x.flags.c_contiguous:
        raise ValueError(f"{name} must be a C-contiguous {ndim}-D array")
    if writable and not x.flags.writeable:
        raise ValueError(f"{name} must be writable")
    return x


class StaticArrays:
    """A graph's static part in build_graph order (graph.py:314-316)."""

    def __init__(self, g: HloGraph, op_time=None):
        ops = sorted(g.ops, key=lambda o: o.id)
        self.op_ids = [o.id for o in ops]
        self.op_index = {o.id: i for i, o in enumerate(ops)}
        ars = sorted(g.allreduces, key=lambda a: a.id)
        self.ar_ids = [a.id for a in ars]
        self.ar_index = {a.id: i for i, a in enumerate(ars)}
        edges = sorted(g.edges, key=lambda e: (e.src, e.dst))
        self.V, self.E, self.A = len(ops), len(edges), len(ars)
        self.op_kind = np.array([KIND_CODE.get(o.kind, 0) for o in ops], np.int32)
        self.op_out = np.array([o.out_bytes for o in ops], np.int64)
        self.op_prof = np.array([math.nan if op_time is None else op_time(o) for o in ops], np.float64)
        self.op_compute = np.array([math.nan if o.compute_us is None else float(o.compute_us) for o in ops],
                                   np.float64)
        self.e_src = np.array([self.op_index[e.src] for e in edges], np.int32)
        self.e_dst = np.array([self.op_index[e.dst] for e in edges], np.int32)
        self.e_bytes = np.array([e.bytes for e in edges], np.int64)
        self.ar_prod = np.array([self.op_index[a.producer_op] for a in ars], np.int32)
        self.ar_bytes = np.array([a.tensor_bytes for a in ars], np.int64)
        self.op_codes = [o.op_code for o in ops]
        # _group_content_key fragments (workloads.py:267-273), for the jittered oracle
        self.op_keys = [f"{o.op_code}:{o.input_shape_key}:{o.compute_us}" for o in ops]

    def desc(self):
        d = N.GraphDesc()
        d.n_ops, d.n_edges, d.n_allreduces = self.V, self.E, self.A
        d.op_kind = N.tptr(self.op_kind, C.c_int32)
        d.op_out_bytes = N.tptr(self.op_out, C.c_int64)
        d.op_profile_us = N.tptr(self.op_prof, C.c_double)
        d.op_compute_us = N.tptr(self.op_compute, C.c_double)
        d.edge_src = N.tptr(self.e_src, C.c_int32)
        d.edge_dst = N.tptr(self.e_dst, C.c_int32)
        d.edge_bytes = N.tptr(self.e_bytes, C.c_int64)
        d.ar_producer = N.tptr(self.ar_prod, C.c_int32)
        d.ar_bytes = N.tptr(self.ar_bytes, C.c_int64)
        return d


class DeviceGraph:
    """An ``fo_graph`` handle with its cost model installed."""

    def __init__(self, g: HloGraph, cost_model_fn, op_time=None, device=None):
        self.static = StaticArrays(g, op_time)
        self.V, self.E, self.A = self.static.V, self.static.E, self.static.A
        self.device = current_device() if device is None else device
        self._lock = threading.Lock()
        L = N.lib()
        h = C.c_void_p()
        st = L.fo_graph_create(C.byref(self.static.desc()), self.device, C.byref(h))
        _raise(st, "fo_graph_create", N.last_error())
        self.h = h
        self._keep = []
        self._inflight = {}  # ticket -> host buffers of a pipelined submission
        cm = cost_model_fn(self.static, self._keep)
        st = L.fo_graph_set_cost_model(self.h, C.byref(cm))
        _raise(st, "fo_graph_set_cost_model", N.last_error())

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                N.lib().fo_graph_destroy(h)
            except Exception:
                pass

    # -- scoring -------------------------------------------------------------
    def score_host(self, ng, rg, bk, gid_bound, precision=N.FO_PREC_FP32):
        """cost() of K candidates held in host arrays [K, V] / [K, A]; int16
        arrays take the half-width path (fo_score_host_i16)."""
        i16 = np.asarray(ng).dtype == np.int16
        dt = np.int16 if i16 else np.int32
        ng = np.ascontiguousarray(ng, dt)
        rg = np.ascontiguousarray(rg, dt)
        bk = np.ascontiguousarray(bk, dt)
        K = ng.shape[0] if ng.ndim == 2 else (bk.shape[0] if bk.ndim == 2 else 1)
        cost = np.zeros(K, np.float64)
        status = np.zeros(K, np.int32)
        fn = N.lib().fo_score_host_i16 if i16 else N.lib().fo_score_host
        st = fn(self.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), K, int(gid_bound), precision, N.ptr(cost), N.ptr(status))
        _raise(st, "fo_score_host", N.last_error())
        return cost, status

    def score_device(self, ng, rg, bk, gid_bound, cost, status, precision=N.FO_PREC_FP32, stream=None):
        """Asynchronous scoring of device-resident candidates (torch tensors)."""
        K = int(cost.shape[0])
        if stream is None:
            import torch

            stream = torch.cuda.current_stream().cuda_stream
        import torch

        fn = N.lib().fo_score_i16 if ng.dtype == torch.int16 else N.lib().fo_score
        st = fn(self.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), K, int(gid_bound), precision, N.ptr(cost), N.ptr(status),
                C.c_void_p(stream))
        _raise(st, "fo_score", N.last_error())

    def simulate_arrays(self, ng, rg, bk, gid_bound, durations=None, precision=N.FO_PREC_FP32):
        V, A = self.V, self.A
        c_id = np.zeros(2 * V + 1, np.int32)
        c_s = np.zeros(2 * V + 1)
        c_e = np.zeros(2 * V + 1)
        b_id = np.zeros(A + 1, np.int32)
        b_s = np.zeros(A + 1)
        b_e = np.zeros(A + 1)
        nc, nb, bad = C.c_int32(), C.c_int32(), C.c_int32(-1)
        mk = C.c_double()
        dur = None
        if durations is not None:
            dur = np.zeros(2 * V + A + 2, np.float64)
            dur[: len(durations)] = durations
        st = N.lib().fo_simulate(self.h, N.ptr(np.ascontiguousarray(ng, np.int32)),
                                 N.ptr(np.ascontiguousarray(rg, np.int32)),
                                 N.ptr(np.ascontiguousarray(bk, np.int32)), int(gid_bound), precision, N.ptr(dur),
                                 N.ptr(c_id), N.ptr(c_s), N.ptr(c_e), C.byref(nc), N.ptr(b_id), N.ptr(b_s),
                                 N.ptr(b_e), C.byref(nb), C.byref(mk), C.byref(bad))
        n1, n2 = nc.value, nb.value
        return st, mk.value, (c_id[:n1], c_s[:n1], c_e[:n1]), (b_id[:n2], b_s[:n2], b_e[:n2]), bad.value

    def node_durations_arrays(self, ng, rg, bk, gid_bound, precision=N.FO_PREC_FP32):
        dur = np.zeros(2 * self.V + self.A + 2)
        G, bad = C.c_int32(), C.c_int32(-1)
        st = N.lib().fo_node_durations(self.h, N.ptr(np.ascontiguousarray(ng, np.int32)),
                                       N.ptr(np.ascontiguousarray(rg, np.int32)),
                                       N.ptr(np.ascontiguousarray(bk, np.int32)), int(gid_bound), precision,
                                       N.ptr(dur), C.byref(G), C.byref(bad))
        return st, dur, G.value, bad.value

    # -- native batch-expand ----------------------------------------------------
    def make_candidates(self, seeds, beta=10, methods_mask=7, base=None, n_threads=0):
        seeds = np.ascontiguousarray(seeds, np.uint64)
        K = len(seeds)
        ng = np.zeros((K, self.V), np.int32)
        rg = np.zeros((K, self.V), np.int32)
        bk = np.zeros((K, self.A), np.int32)
        vb = C.c_int32()
        b0 = (None, None, None) if base is None else tuple(np.ascontiguousarray(x, np.int32) for x in base)
        st = N.lib().fo_make_candidates(self.h, N.ptr(b0[0]), N.ptr(b0[1]), N.ptr(b0[2]), N.ptr(seeds), K, beta,
                                        methods_mask, n_threads, N.ptr(ng), N.ptr(rg), N.ptr(bk), C.byref(vb))
        _raise(st, "fo_make_candidates", N.last_error())
        return ng, rg, bk, vb.value

    # -- sparse (delta) candidates against a resident parent -----------------------
    def set_parent(self, ng=None, rg=None, bk=None):
        """Make (ng, rg, bk) -- any ids; None = unfused default -- the resident
        parent of sparse candidates (fo_set_parent)."""
        b0 = (None, None, None) if ng is None else tuple(np.ascontiguousarray(x, np.int32) for x in (ng, rg, bk))
        st = N.lib().fo_set_parent(self.h, N.ptr(b0[0]), N.ptr(b0[1]), N.ptr(b0[2]))
        _raise(st, "fo_set_parent", N.last_error())

    def make_candidates_delta(self, seeds, beta=10, methods_mask=7, base=None, n_threads=0):
        """make_candidates' batch as changes against the base: (offsets[K+1],
        changes[n, 2] of (index, value) over ngid | rgid | bkt)."""
        seeds = np.ascontiguousarray(seeds, np.uint64)
        K = len(seeds)
        b0 = (None, None, None) if base is None else tuple(np.ascontiguousarray(x, np.int32) for x in base)
        off = np.zeros(K + 1, np.int32)
        cap = max(64, 48 * K)
        for _ in range(2):
            chg = np.zeros((cap, 2), np.int32)
            st = N.lib().fo_make_candidates_delta(self.h, N.ptr(b0[0]), N.ptr(b0[1]), N.ptr(b0[2]), N.ptr(seeds), K,
                                                  beta, methods_mask, n_threads, N.ptr(off), N.ptr(chg), cap)
            if st == 0 or int(off[K]) <= cap:
                break
            cap = int(off[K])
        _raise(st, "fo_make_candidates_delta", N.last_error())
        return off, chg[: int(off[K])]

    def score_delta_host(self, offsets, changes, precision=N.FO_PREC_FP32):
        """cost() of sparse candidates held in host arrays (fo_score_delta_host)."""
        off = np.ascontiguousarray(offsets, np.int32)
        chg = np.ascontiguousarray(changes, np.int32)
        K = len(off) - 1
        cost = np.zeros(K, np.float64)
        status = np.zeros(K, np.int32)
        st = N.lib().fo_score_delta_host(self.h, N.ptr(off), N.ptr(chg), K, precision, N.ptr(cost), N.ptr(status))
        _raise(st, "fo_score_delta_host", N.last_error())
        return cost, status

    def score_delta_submit(self, offsets, changes, cost, status, precision=N.FO_PREC_FP32, clear_memo=False):
        """Pipelined fo_score_delta_host: enqueue one batch of sparse candidates
        held in host arrays (pinned for overlap) and return a ticket; four
        batches may be in flight, on four compute streams.  `cost` (float64) / `status` (int32), host,
        length >= K, are written once score_wait(ticket) returns.  The handle
        keeps references to all four buffers until then."""
        import ctypes

        offsets_a = _host_array(offsets, np.int32, "offsets", ndim=1)
        K = offsets_a.shape[0] - 1
        if K < 0:
            raise ValueError("offsets must hold K + 1 entries")
        changes_a = _host_array(changes, np.int32, "changes", ndim=2)
        n = int(offsets_a[K])
        if changes_a.shape[1] != 2 or changes_a.shape[0] < n:
            raise ValueError(f"changes must have shape (offsets[K], 2) = ({n}, 2), got {changes_a.shape}")
        cost_a = _host_array(cost, np.float64, "cost", ndim=1, writable=True)
        status_a = _host_array(status, np.int32, "status", ndim=1, writable=True)
        if cost_a.shape[0] < K or status_a.shape[0] < K:
            raise ValueError(f"cost / status must hold K = {K} entries")
        t = ctypes.c_int64(-1)
        st = N.lib().fo_score_delta_submit(self.h, N.ptr(offsets_a), N.ptr(changes_a), K, precision,
                                           int(bool(clear_memo)), N.ptr(cost_a), N.ptr(status_a), ctypes.byref(t))
        _raise(st, "fo_score_delta_submit", N.last_error())
        # the device copies read / write these until score_wait: keep them alive
        self._inflight[t.value] = (offsets, changes, cost, status, offsets_a, changes_a, cost_a, status_a)
        return t.value

    def score_wait(self, ticket):
        try:
            _raise(N.lib().fo_score_wait(self.h, int(ticket)), "fo_score_wait", N.last_error())
        finally:
            self._inflight.pop(int(ticket), None)

    def score_delta_device(self, offsets, changes, cost, status, precision=N.FO_PREC_FP32, stream=None):
        """Asynchronous scoring of device-resident sparse candidates (torch tensors)."""
        import torch

        K = int(cost.shape[0])
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        st = N.lib().fo_score_delta(self.h, N.ptr(offsets), N.ptr(changes), K, precision, N.ptr(cost), N.ptr(status),
                                    C.c_void_p(stream))
        _raise(st, "fo_score_delta", N.last_error())

    def score_delta_slot(self, slot, offsets, changes, cost, status, precision=N.FO_PREC_FP32, stream=None,
                         clear_memo=False):
        """score_delta_device on scratch set `slot` (fo_score_delta_slot):
        batches on different slots may run at once on different streams."""
        import torch

        K = int(cost.shape[0])
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        st = N.lib().fo_score_delta_slot(self.h, int(slot), N.ptr(offsets), N.ptr(changes), K, precision,
                                         int(bool(clear_memo)), N.ptr(cost), N.ptr(status), C.c_void_p(stream))
        _raise(st, "fo_score_delta_slot", N.last_error())

    def state_hash(self, ng, rg, bk):
        ng = np.ascontiguousarray(np.atleast_2d(ng), np.int32)
        rg = np.ascontiguousarray(np.atleast_2d(rg), np.int32)
        bk = np.ascontiguousarray(bk, np.int32).reshape(ng.shape[0], -1)
        out = np.zeros(ng.shape[0], np.uint64)
        st = N.lib().fo_state_hash(self.h, N.ptr(ng), N.ptr(rg), N.ptr(bk), ng.shape[0], N.ptr(out))
        _raise(st, "fo_state_hash", N.last_error())
        return out

    # -- HloGraph conveniences ----------------------------------------------------
    def encode(self, g: HloGraph):
        return state_arrays(g)
