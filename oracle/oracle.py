"""ctypes front-end of the CPU oracle (fo_oracle.c).

TEST INFRASTRUCTURE ONLY: the parity checker and the CPU baseline.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  The product package never does.

States are given with REFERENCE ids: ``ngid[v]`` is the id of op v's normal
group, ``rgid[v]`` its replica group id or -1, ``bkt[a]`` the bucket id of
AllReduce a (ops and AllReduces indexed in ascending id order, exactly as
``build_graph`` sorts them, graph.py:314-316).
"""

from __future__ import annotations

import ctypes as C
import gzip
import json
import math
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libfo_oracle.so")
GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")

STATUS = {0: "OK", 1: "CYCLE", 2: "MISSING_COST", 3: "NEGATIVE_DURATION", 4: "DIM_MISMATCH", 5: "INVALID_ARG"}
KINDS = {"compute": 0, "parameter": 1, "control": 2}
PROV_PROFILE, PROV_HW_ORACLE = 0, 1
VAR_NONE, VAR_ANALYTIC, VAR_LINEAR, VAR_MP = -1, 0, 1, 2
METHODS = ("nondup", "dup", "ar")


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


P = C.POINTER


class GraphDesc(C.Structure):
    _fields_ = [("V", C.c_int32), ("E", C.c_int32), ("A", C.c_int32),
                ("op_kind", P(C.c_int32)), ("op_out_bytes", P(C.c_int64)),
                ("op_prof", P(C.c_double)), ("op_compute", P(C.c_double)), ("op_slot", P(C.c_int32)),
                ("e_src", P(C.c_int32)), ("e_dst", P(C.c_int32)), ("e_bytes", P(C.c_int64)),
                ("ar_prod", P(C.c_int32)), ("ar_bytes", P(C.c_int64))]


class Model(C.Structure):
    _fields_ = [("provider", C.c_int32), ("variant", C.c_int32),
                ("comm_C", C.c_double), ("comm_D", C.c_double), ("launch", C.c_double), ("mem", C.c_double),
                ("layers", C.c_int32), ("hidden", C.c_int32), ("feat_dim", C.c_int32),
                ("W_emb", P(C.c_double)), ("W_layer", P(C.c_double)), ("W_r", P(C.c_double)),
                ("A1", P(C.c_double)), ("c1", P(C.c_double)), ("A2", P(C.c_double)), ("c2", P(C.c_double)),
                ("a3", P(C.c_double)), ("c3", C.c_double),
                ("node_mean", P(C.c_double)), ("node_std", P(C.c_double)),
                ("lin_w", P(C.c_double)), ("lin_b", C.c_double),
                ("agg_mean", P(C.c_double)), ("agg_std", P(C.c_double)), ("out_scale", C.c_double)]


class Timeline(C.Structure):
    _fields_ = [("c_id", P(C.c_int32)), ("c_start", P(C.c_double)), ("c_end", P(C.c_double)), ("n_c", C.c_int32),
                ("b_id", P(C.c_int32)), ("b_start", P(C.c_double)), ("b_end", P(C.c_double)), ("n_b", C.c_int32)]


class SearchCfg(C.Structure):
    _fields_ = [("alpha", C.c_double), ("beta", C.c_int32), ("max_unchanged", C.c_int32),
                ("methods_mask", C.c_int32), ("seed", C.c_uint64), ("max_steps", C.c_int64)]


class TraceRec(C.Structure):
    _fields_ = [("step", C.c_int32), ("method", C.c_int8), ("cost", C.c_double), ("best", C.c_double),
                ("queue_len", C.c_int32), ("enqueued", C.c_int8)]


class Rng(C.Structure):
    _fields_ = [("mt", C.c_uint32 * 624), ("mti", C.c_int)]


def _declare(L):
    vp = C.c_void_p
    L.orc_prepare.restype = vp
    L.orc_prepare.argtypes = [P(GraphDesc)]
    L.orc_free.argtypes = [vp]
    L.orc_cost.restype = C.c_int
    L.orc_cost.argtypes = [vp, P(Model), vp, vp, vp, P(C.c_double), P(Timeline), P(C.c_int32)]
    L.orc_cost_batch.argtypes = [vp, P(Model), vp, vp, vp, C.c_int32, vp, vp]
    L.orc_node_durations.restype = C.c_int
    L.orc_node_durations.argtypes = [vp, P(Model), vp, vp, vp, vp, vp, vp, P(C.c_int32), vp]
    L.orc_rng_seed.argtypes = [P(Rng), C.c_uint64]
    L.orc_rng_getrandbits.restype = C.c_uint32
    L.orc_rng_getrandbits.argtypes = [P(Rng), C.c_int]
    L.orc_rng_randbelow.restype = C.c_uint32
    L.orc_rng_randbelow.argtypes = [P(Rng), C.c_uint32]
    L.orc_rng_size.restype = C.c_int32
    L.orc_random_apply.restype = C.c_int
    L.orc_random_apply.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, P(Rng)]
    L.orc_make_candidate.argtypes = [vp, C.c_uint64, C.c_int, vp, vp, vp]
    L.orc_state_hash.restype = C.c_uint64
    L.orc_state_hash.argtypes = [vp, vp, vp, vp]
    L.orc_search.restype = C.c_int
    L.orc_search.argtypes = [vp, P(Model), P(SearchCfg), vp, vp, vp, P(C.c_double), vp, P(TraceRec), C.c_int64]
    assert L.orc_rng_size() == C.sizeof(Rng)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _dptr(a, ct):
    return a.ctypes.data_as(P(ct))


# ---------------------------------------------------------------------------
# fixture loading (the reference's JSON formats: graph.py:626-743,
# estimator.py:72-92, :739-794, comm.py:116-127)


def _read_json(path):
    if path.endswith(".gz"):
        with gzip.open(path, "rt", encoding="utf-8") as fh:
            return json.load(fh)
    with open(path, "r", encoding="utf-8") as fh:
        return json.load(fh)


@dataclass
class Workload:
    name: str
    graph: dict
    profile: dict  # (op_code, shape) -> us
    comm: tuple
    mp: dict
    lin: dict


WORKLOADS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "workloads")


def load_workload(name, root=WORKLOADS) -> Workload:
    base = os.path.join(root, name)
    graph = _read_json(base + ".graph.json.gz")
    prof = _read_json(base + ".profile.json.gz")
    profile = {(e["op_code"], e["input_shape_key"]): float(e["time_us"]) for e in prof["entries"]}
    comm = _read_json(base + ".comm.json")
    src = name
    if os.path.exists(base + ".model_from.json"):
        src = _read_json(base + ".model_from.json")["model_from"]
    sbase = os.path.join(root, src)
    mp = _read_json(sbase + ".mp.model.json.gz")
    lin = _read_json(sbase + ".lin.model.json")
    return Workload(name, graph, profile, (float(comm["C"]), float(comm["D"])), mp, lin)


class StaticGraph:
    """Arrays of a graph document in build_graph order (graph.py:302-340)."""

    def __init__(self, doc: dict, profile: dict, vocab=()):
        ops = sorted(doc.get("ops", []), key=lambda o: int(o["id"]))
        self.op_ids = np.array([int(o["id"]) for o in ops], dtype=np.int64)
        self.op_index = {int(o["id"]): i for i, o in enumerate(ops)}
        self.V = len(ops)
        edges = sorted(((int(e["src"]), int(e["dst"]), int(e.get("bytes", 0))) for e in doc.get("edges", [])),
                       key=lambda t: (t[0], t[1]))
        ars = sorted((int(a["id"]), int(a["producer_op"]), int(a["tensor_bytes"])) for a in doc.get("allreduce", []))
        self.E, self.A = len(edges), len(ars)
        self.ar_ids = np.array([a[0] for a in ars], dtype=np.int64)
        self.ar_index = {a[0]: i for i, a in enumerate(ars)}
        self.op_kind = np.array([KINDS[o.get("kind", "compute")] for o in ops], dtype=np.int32)
        self.op_out = np.array([int(o.get("out_bytes", 0)) for o in ops], dtype=np.int64)
        self.op_prof = np.array([profile.get((o["op_code"], o.get("input_shape_key", "")), math.nan) for o in ops],
                                dtype=np.float64)
        self.op_compute = np.array([math.nan if o.get("compute_us") is None else float(o["compute_us"]) for o in ops],
                                   dtype=np.float64)
        slot = {c: i for i, c in enumerate(vocab)}
        other = slot.get("<other>", len(vocab) - 1 if vocab else 0)
        self.op_slot = np.array([slot.get(o["op_code"], other) for o in ops], dtype=np.int32)
        self.e_src = np.array([self.op_index[e[0]] for e in edges], dtype=np.int32)
        self.e_dst = np.array([self.op_index[e[1]] for e in edges], dtype=np.int32)
        self.e_bytes = np.array([e[2] for e in edges], dtype=np.int64)
        self.ar_prod = np.array([self.op_index[a[1]] for a in ars], dtype=np.int32)
        self.ar_bytes = np.array([a[2] for a in ars], dtype=np.int64)
        self.doc = doc

    def desc(self):
        d = GraphDesc()
        d.V, d.E, d.A = self.V, self.E, self.A
        d.op_kind = _dptr(self.op_kind, C.c_int32)
        d.op_out_bytes = _dptr(self.op_out, C.c_int64)
        d.op_prof = _dptr(self.op_prof, C.c_double)
        d.op_compute = _dptr(self.op_compute, C.c_double)
        d.op_slot = _dptr(self.op_slot, C.c_int32)
        d.e_src = _dptr(self.e_src, C.c_int32)
        d.e_dst = _dptr(self.e_dst, C.c_int32)
        d.e_bytes = _dptr(self.e_bytes, C.c_int64)
        d.ar_prod = _dptr(self.ar_prod, C.c_int32)
        d.ar_bytes = _dptr(self.ar_bytes, C.c_int64)
        return d

    # -- states with reference ids -------------------------------------------
    def default_state(self):
        ng = self.op_ids.astype(np.int32).copy()
        rg = np.full(self.V, -1, dtype=np.int32)
        bk = self.ar_ids.astype(np.int32).copy()
        return ng, rg, bk

    def state_from_doc(self, sdoc):
        """Sparse fixture state (make_golden.state_doc) -> arrays."""
        ng, rg, bk = self.default_state()
        for gid, members, dups in sdoc["groups"]:
            dset = set(dups)
            for m in members:
                i = self.op_index[m]
                if m in dset:
                    rg[i] = gid
                else:
                    ng[i] = gid
        for bid, members in sdoc["buckets"]:
            for m in members:
                bk[self.ar_index[m]] = bid
        return ng, rg, bk

    def state_to_doc(self, ng, rg, bk):
        groups = {}
        for i in range(self.V):
            groups.setdefault(int(ng[i]), [[], []])[0].append(int(self.op_ids[i]))
            if rg[i] >= 0:
                g = groups.setdefault(int(rg[i]), [[], []])
                g[0].append(int(self.op_ids[i]))
                g[1].append(int(self.op_ids[i]))
        out_g = []
        for gid in sorted(groups):
            mem, dup = groups[gid]
            if not (len(mem) == 1 and mem[0] == gid and not dup):
                out_g.append([gid, sorted(mem), sorted(dup)])
        buckets = {}
        for a in range(self.A):
            buckets.setdefault(int(bk[a]), []).append(int(self.ar_ids[a]))
        out_b = [[bid, sorted(m)] for bid, m in sorted(buckets.items()) if not (len(m) == 1 and m[0] == bid)]
        return {"groups": out_g, "buckets": out_b}


def _model_params(doc):
    return {k: np.asarray(v["data"], dtype=np.float64).reshape(v["shape"]) for k, v in doc["params"].items()}


class Oracle:
    """One graph + one cost-provider configuration.

    provider: "mp" | "lin" | "analytic" | "oracle" | "none"
    """

    def __init__(self, wl: Workload, provider: str = "mp", analytic=(5.0, 1.0 / 1024.0), hw=(5.0, 1.0 / 1024.0),
                 comm: Optional[tuple] = None):
        self.wl = wl
        mdoc = wl.mp if provider == "mp" else wl.lin if provider == "lin" else None
        vocab = tuple(mdoc.get("vocab", [])) if mdoc else ()
        self.g = StaticGraph(wl.graph, wl.profile, vocab)
        L = lib()
        self._desc = self.g.desc()
        self.h = L.orc_prepare(C.byref(self._desc))
        self._keep = []
        m = Model()
        m.comm_C, m.comm_D = comm if comm is not None else wl.comm
        m.provider = PROV_PROFILE
        if provider == "oracle":
            m.provider = PROV_HW_ORACLE
            m.variant = VAR_NONE
            m.launch, m.mem = hw
            m.comm_C, m.comm_D = comm if comm is not None else (0.001, 100.0)  # HardwareParams().comm_params
        elif provider == "analytic":
            m.variant = VAR_ANALYTIC
            m.launch, m.mem = analytic
        elif provider == "none":
            m.variant = VAR_NONE
        elif provider == "lin":
            m.variant = VAR_LINEAR
            p = _model_params(mdoc)
            w = np.ascontiguousarray(p["w"])
            self._keep.append(w)
            m.lin_w = _dptr(w, C.c_double)
            m.lin_b = float(p["b"])
            if mdoc.get("agg_norm"):
                am = np.asarray(mdoc["agg_norm"]["mean"], dtype=np.float64)
                asd = np.asarray(mdoc["agg_norm"]["std"], dtype=np.float64)
                self._keep += [am, asd]
                m.agg_mean, m.agg_std = _dptr(am, C.c_double), _dptr(asd, C.c_double)
            m.out_scale = float(mdoc["hyper"].get("out_scale", 1.0))
        elif provider == "mp":
            m.variant = VAR_MP
            p = _model_params(mdoc)
            h = int(mdoc["hyper"]["hidden"])
            L_ = int(mdoc["hyper"]["layers"])
            m.layers, m.hidden = L_, h
            m.feat_dim = p["W_emb"].shape[1]
            wl_ = np.ascontiguousarray(np.stack([p[f"W_{i}"] for i in range(1, L_ + 1)]))
            arrs = {k: np.ascontiguousarray(p[k]) for k in ("W_emb", "W_r", "A1", "c1", "A2", "c2", "a3")}
            self._keep += [wl_] + list(arrs.values())
            m.W_layer = _dptr(wl_, C.c_double)
            for k, a in arrs.items():
                setattr(m, k, _dptr(a, C.c_double))
            m.c3 = float(p["c3"])
            if mdoc.get("node_norm"):
                nm = np.asarray(mdoc["node_norm"]["mean"], dtype=np.float64)
                ns = np.asarray(mdoc["node_norm"]["std"], dtype=np.float64)
                self._keep += [nm, ns]
                m.node_mean, m.node_std = _dptr(nm, C.c_double), _dptr(ns, C.c_double)
            m.out_scale = float(mdoc["hyper"].get("out_scale", 1.0))
        else:
            raise ValueError(provider)
        self.model = m

    def __del__(self):
        try:
            lib().orc_free(self.h)
        except Exception:
            pass

    def cost(self, ng, rg, bk, timeline=False):
        L = lib()
        c = C.c_double()
        bad = C.c_int32()
        tl = None
        if timeline:
            V, A = self.g.V, self.g.A
            bufs = [np.zeros(2 * V + 1, np.int32), np.zeros(2 * V + 1), np.zeros(2 * V + 1),
                    np.zeros(A + 1, np.int32), np.zeros(A + 1), np.zeros(A + 1)]
            tl = Timeline(_dptr(bufs[0], C.c_int32), _dptr(bufs[1], C.c_double), _dptr(bufs[2], C.c_double), 0,
                          _dptr(bufs[3], C.c_int32), _dptr(bufs[4], C.c_double), _dptr(bufs[5], C.c_double), 0)
        st = L.orc_cost(self.h, C.byref(self.model), _ptr(np.ascontiguousarray(ng, np.int32)),
                        _ptr(np.ascontiguousarray(rg, np.int32)), _ptr(np.ascontiguousarray(bk, np.int32)),
                        C.byref(c), C.byref(tl) if tl is not None else None, C.byref(bad))
        if not timeline:
            return st, c.value
        comp = [(int(bufs[0][i]), float(bufs[1][i]), float(bufs[2][i])) for i in range(tl.n_c)]
        comm = [(int(bufs[3][i]), float(bufs[4][i]), float(bufs[5][i])) for i in range(tl.n_b)]
        return st, c.value, comp, comm

    def cost_batch(self, ng, rg, bk):
        K = ng.shape[0]
        out = np.zeros(K)
        st = np.zeros(K, np.int32)
        lib().orc_cost_batch(self.h, C.byref(self.model), _ptr(np.ascontiguousarray(ng, np.int32)),
                             _ptr(np.ascontiguousarray(rg, np.int32)), _ptr(np.ascontiguousarray(bk, np.int32)),
                             K, _ptr(out), _ptr(st))
        return st, out

    def node_durations(self, ng, rg, bk):
        V, A = self.g.V, self.g.A
        gid = np.zeros(2 * V + 1, np.int32)
        bid = np.zeros(A + 1, np.int32)
        dur = np.zeros(2 * V + A + 1)
        io = np.zeros(3 * (2 * V + 1), np.int64)
        G = C.c_int32()
        n = lib().orc_node_durations(self.h, C.byref(self.model), _ptr(np.ascontiguousarray(ng, np.int32)),
                                     _ptr(np.ascontiguousarray(rg, np.int32)),
                                     _ptr(np.ascontiguousarray(bk, np.int32)), _ptr(gid), _ptr(bid), _ptr(dur),
                                     C.byref(G), _ptr(io))
        G = G.value
        return n, gid[:G].copy(), bid.copy(), dur.copy(), io[: 3 * G].reshape(G, 3).copy()

    def make_candidate(self, seed, beta=10):
        ng, rg, bk = self.g.default_state()
        lib().orc_make_candidate(self.h, seed, beta, _ptr(ng), _ptr(rg), _ptr(bk))
        return ng, rg, bk

    def state_hash(self, ng, rg, bk):
        return lib().orc_state_hash(self.h, _ptr(np.ascontiguousarray(ng, np.int32)),
                                    _ptr(np.ascontiguousarray(rg, np.int32)),
                                    _ptr(np.ascontiguousarray(bk, np.int32)))

    def search(self, alpha=1.05, beta=10, max_unchanged=1000, seed=0, methods=("nondup", "dup", "ar"),
               max_steps=0, trace_cap=1 << 20, state=None):
        ng, rg, bk = state if state is not None else self.g.default_state()
        ng, rg, bk = ng.copy(), rg.copy(), bk.copy()
        cfg = SearchCfg(alpha, beta, max_unchanged, sum(1 << METHODS.index(m) for m in methods), seed, max_steps)
        best = C.c_double()
        counters = np.zeros(4, np.int64)
        trace = (TraceRec * trace_cap)()
        st = lib().orc_search(self.h, C.byref(self.model), C.byref(cfg), _ptr(ng), _ptr(rg), _ptr(bk),
                              C.byref(best), _ptr(counters), trace, trace_cap)
        n = int(min(counters[3], trace_cap))
        recs = [(trace[i].step, METHODS[trace[i].method], trace[i].cost, trace[i].best, trace[i].queue_len,
                 bool(trace[i].enqueued)) for i in range(n)]
        return {"status": st, "best_cost_us": best.value, "steps": int(counters[0]),
                "candidates_evaluated": int(counters[1]), "candidates_enqueued": int(counters[2]),
                "trace": recs, "best_state": (ng, rg, bk)}


class PyRandom:
    """CPython random.Random(seed) restated over the oracle's MT19937."""

    def __init__(self, seed: int):
        self.r = Rng()
        lib().orc_rng_seed(C.byref(self.r), seed)

    def getrandbits(self, k):
        return lib().orc_rng_getrandbits(C.byref(self.r), k)

    def randrange(self, n):
        return lib().orc_rng_randbelow(C.byref(self.r), n)

    def randint(self, a, b):
        return a + lib().orc_rng_randbelow(C.byref(self.r), b - a + 1)
