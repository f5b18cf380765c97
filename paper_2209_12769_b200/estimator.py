"""Cost providers backed by the device path.

``make_cost_providers`` and ``oracle_providers`` return objects that still
satisfy the reference's ``CostProviders`` protocol (op_cost / comm_cost
callables, simulator.py:28-35) and additionally carry the device configuration
used by simulate / cost / cost_batch / backtracking_search.

Model and profile files use the reference's formats (estimator.py:72-92,
:739-794; comm.py:116-127).
"""

from __future__ import annotations

import ctypes as C
import gzip
import json
import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Mapping, Optional

import numpy as np

from . import _native as N
from .comm import CommModelParams
from .errors import GraphFormatError, MissingCost, UnknownOp, _raise
from .graph import KIND_PARAMETER, HloGraph, state_arrays

OTHER_OP_CODE = "<other>"


@dataclass(frozen=True)
class Profile:
    """Measured per-op times keyed by (op_code, input_shape_key)."""

    times: Mapping

    def __post_init__(self) -> None:
        for key, value in self.times.items():
            if not value > 0:
                raise ValueError(f"profiled time for {key} must be > 0")


def lookup(profile: Profile, op) -> float:
    """Exact-match lookup (estimator.py:63-69)."""
    try:
        return profile.times[(op.op_code, op.input_shape_key)]
    except KeyError:
        raise UnknownOp(f"no profile entry for {(op.op_code, op.input_shape_key)}") from None


def _read(path):
    op = gzip.open if str(path).endswith(".gz") else open
    with op(path, "rt", encoding="utf-8") as fh:
        return json.load(fh)


def load_profile(path) -> Profile:
    doc = _read(path)
    try:
        return Profile({(str(e["op_code"]), str(e["input_shape_key"])): float(e["time_us"]) for e in doc["entries"]})
    except (KeyError, TypeError) as exc:
        raise GraphFormatError(f"{path}: bad profile document") from exc


class EstimatorVariant(Enum):
    ANALYTIC = "analytic"
    LINEAR_FEATURES = "linear_features"
    MESSAGE_PASSING = "message_passing"


@dataclass
class EstimatorModel:
    variant: EstimatorVariant
    params: dict
    vocab: tuple = ()
    node_norm: Optional[tuple] = None
    agg_norm: Optional[tuple] = None
    layers: int = 6
    hidden: int = 32
    out_scale: float = 1.0


def analytic_model(launch_overhead_us: float, mem_us_per_byte: float) -> EstimatorModel:
    return EstimatorModel(EstimatorVariant.ANALYTIC, {"launch_overhead_us": np.array(float(launch_overhead_us)),
                                                      "mem_us_per_byte": np.array(float(mem_us_per_byte))})


def model_from_doc(doc: dict) -> EstimatorModel:
    try:
        if doc["format_version"] != 1:
            raise GraphFormatError("unsupported model format version")
        params = {k: np.array(v["data"], np.float64).reshape(v["shape"]) for k, v in doc["params"].items()}

        def norm(key):
            b = doc.get(key)
            return None if b is None else (np.array(b["mean"], np.float64), np.array(b["std"], np.float64))

        return EstimatorModel(EstimatorVariant(doc["variant"]), params, tuple(doc.get("vocab", [])), norm("node_norm"),
                              norm("agg_norm"), int(doc["hyper"]["layers"]), int(doc["hyper"]["hidden"]),
                              float(doc["hyper"].get("out_scale", 1.0)))
    except (KeyError, TypeError, ValueError) as exc:
        raise GraphFormatError(f"bad model document: {exc}") from exc


def load_model(path) -> EstimatorModel:
    return model_from_doc(_read(path))


def _vocab_slots(model: EstimatorModel, op_codes):
    slot = {c: i for i, c in enumerate(model.vocab)}
    other = slot.get(OTHER_OP_CODE, len(model.vocab) - 1 if model.vocab else 0)
    return np.array([slot.get(c, other) for c in op_codes], np.int32)


class DeviceCostProviders:
    """A CostProviders drop-in whose durations are computed on the B200.

    kind: "profile" (make_cost_providers) or "hw_oracle" (oracle_providers).
    precision: FO_PREC_FP32 (throughput) or FO_PREC_FP64 (decision-exact).
    """

    def __init__(self, kind, profile=None, comm_params=None, model=None, hw=None, precision=N.FO_PREC_FP32):
        self.kind = kind
        self.profile = profile
        self.comm_params = comm_params
        self.model = model
        self.hw = hw
        self.precision = precision
        self._graphs = {}

    # -- device handle cache keyed by the static graph ------------------------
    def device_graph(self, g: HloGraph):
        from .device import DeviceGraph

        ar_key = tuple((a.id, a.producer_op, a.tensor_bytes) for a in g.allreduces)
        key = (id(g.ops), id(g.edges), ar_key)
        ent = self._graphs.get(key)
        if ent is None:  # same static content under new tuples (e.g. build_graph copies)
            ckey = ("content", hash(g.ops), hash(g.edges), ar_key)
            ent = self._graphs.get(ckey)
            if ent is not None and ent[1] == g.ops and ent[2] == g.edges:
                self._graphs[key] = (ent[0], g.ops, g.edges)
                return ent[0]
        if ent is None:
            op_time = None
            if self.kind == "profile":
                times = self.profile.times

                def op_time(o):
                    return times.get((o.op_code, o.input_shape_key), math.nan)

            dg = DeviceGraph(g, self._cost_model, op_time)
            ent = (dg, g.ops, g.edges)  # keep ops/edges alive so ids stay unique
            self._graphs[key] = ent
            self._graphs[("content", hash(g.ops), hash(g.edges), ar_key)] = ent
        return ent[0]

    def _cost_model(self, static, keep):
        cm = N.CostModel()
        if self.kind == "hw_oracle":
            hw = self.hw
            cm.provider = N.FO_PROVIDER_HW_ORACLE
            cm.variant = N.FO_EST_NONE
            cm.comm_C, cm.comm_D = hw.comm_params.C, hw.comm_params.D
            cm.launch_us, cm.mem_us_per_byte = hw.launch_overhead_us, hw.mem_us_per_byte
            if hw.noise != 0:  # jitter keys (workloads.py:254-273)
                frags = [k.encode() for k in static.op_keys]
                off = np.zeros(len(frags) + 1, np.int64)
                off[1:] = np.cumsum([len(f) for f in frags])
                blob = b"".join(frags) or b"\0"
                prefix = f"{hw.seed}|".encode()
                keep += [off, blob, prefix]
                cm.hw_noise = float(hw.noise)
                cm.hw_key_prefix, cm.hw_key_prefix_len = prefix, len(prefix)
                cm.op_key_bytes = blob
                cm.op_key_off = N.tptr(off, C.c_int64)
            return cm
        cm.provider = N.FO_PROVIDER_PROFILE
        cm.comm_C, cm.comm_D = self.comm_params.C, self.comm_params.D
        m = self.model
        if m is None:
            cm.variant = N.FO_EST_NONE
            return cm
        cm.out_scale = float(m.out_scale)
        if m.variant is EstimatorVariant.ANALYTIC:
            cm.variant = N.FO_EST_ANALYTIC
            cm.launch_us = float(m.params["launch_overhead_us"])
            cm.mem_us_per_byte = float(m.params["mem_us_per_byte"])
            return cm
        if m.variant is EstimatorVariant.LINEAR_FEATURES:
            w = np.asarray(m.params["w"], np.float64).ravel()
            if w.shape != (12,):
                cm.variant = N.FO_EST_INVALID
                return cm
            p = np.concatenate([w, [float(m.params["b"])]]).astype(np.float64)
            keep.append(p)
            cm.variant = N.FO_EST_LINEAR
            cm.params, cm.n_params = N.tptr(p, C.c_double), 13
            if m.agg_norm is not None:
                mean = np.ascontiguousarray(m.agg_norm[0], np.float64)
                std = np.ascontiguousarray(m.agg_norm[1], np.float64)
                keep += [mean, std]
                cm.norm_mean, cm.norm_std = N.tptr(mean, C.c_double), N.tptr(std, C.c_double)
            return cm
        # message passing (estimator.py:363-389)
        h, L = int(m.hidden), int(m.layers)
        p = m.params
        F = 6 + len(m.vocab)
        try:
            shapes_ok = p["W_emb"].shape == (h, F) and all(p[f"W_{i}"].shape == (h, h) for i in range(1, L + 1))
        except KeyError:
            shapes_ok = False
        if not shapes_ok:
            cm.variant = N.FO_EST_INVALID
            return cm
        flat = np.concatenate([np.asarray(p["W_emb"]).ravel()] + [np.asarray(p[f"W_{i}"]).ravel()
                                                                   for i in range(1, L + 1)] +
                              [np.asarray(p[k]).ravel() for k in ("W_r", "A1", "c1", "A2", "c2", "a3")] +
                              [np.asarray(p["c3"]).ravel()]).astype(np.float64)
        slots = _vocab_slots(m, static.op_codes)
        keep += [flat, slots]
        cm.variant = N.FO_EST_MESSAGE_PASSING
        cm.layers, cm.hidden, cm.feat_dim = L, h, F
        cm.op_vocab_slot = N.tptr(slots, C.c_int32)
        cm.params, cm.n_params = N.tptr(flat, C.c_double), flat.size
        if m.node_norm is not None:
            mean = np.ascontiguousarray(m.node_norm[0], np.float64)
            std = np.ascontiguousarray(m.node_norm[1], np.float64)
            keep += [mean, std]
            cm.norm_mean, cm.norm_std = N.tptr(mean, C.c_double), N.tptr(std, C.c_double)
        return cm

    # -- the reference's callback protocol (simulator.py:28-35) ------------------
    def node_durations(self, g: HloGraph):
        """Durations of every group (id order) and bucket (id order)."""
        dg = self.device_graph(g)
        ng, rg, bk, vb, gids, bids = state_arrays(g)
        st, dur, G, bad = dg.node_durations_arrays(ng, rg, bk, vb, self.precision)
        if st:
            node = ("g", gids[bad]) if 0 <= bad < len(gids) else ("b", bids[bad - len(gids)]) if bad >= 0 else None
            _raise(st, f"no duration for {node[0]} {node[1]}" if node else "duration", N.last_error())
        return dict(zip(gids, dur[:G])), dict(zip(bids, dur[G:G + len(bids)]))

    def op_cost(self, g: HloGraph, group) -> float:
        if self.kind == "profile" and len(group.member_ops) == 1:  # estimator.py:810-814
            op = g.op(next(iter(group.member_ops)))
            return 0.0 if op.kind == KIND_PARAMETER else lookup(self.profile, op)
        if self.kind == "profile" and self.model is None:
            raise MissingCost(f"group {group.id} is fused and no fused-op estimator was provided")
        return float(self.node_durations(g)[0][group.id])

    def comm_cost(self, g: HloGraph, bucket) -> float:
        cp = self.comm_params if self.kind == "profile" else self.hw.comm_params
        return cp.C * bucket.total_bytes + cp.D


def make_cost_providers(profile: Profile, comm_params: CommModelParams, model: Optional[EstimatorModel] = None,
                        precision: int = N.FO_PREC_FP32) -> DeviceCostProviders:
    """Profile lookups for original ops, the device estimator for fused groups,
    the linear comm model for buckets (estimator.py:801-824)."""
    return DeviceCostProviders("profile", profile=profile, comm_params=comm_params, model=model, precision=precision)


def predict_fused_groups(cp: DeviceCostProviders, g: HloGraph, gids=None) -> dict:
    """predict_fused (estimator.py:462-470) for the fused groups of ``g``,
    computed by the device estimator."""
    groups, _ = cp.node_durations(g)
    want = set(gids) if gids is not None else {x.id for x in g.groups if len(x.member_ops) > 1}
    return {k: v for k, v in groups.items() if k in want}
