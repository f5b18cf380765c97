"""simulate / cost / fo_bound with the reference's signatures
(simulator.py:53-166), executed by the device kernel (csrc/score.cu).

Any ``CostProviders`` works: device providers (make_cost_providers,
oracle_providers) compute durations on the device; plain Python callbacks are
evaluated here in node order with the reference's error rules
(simulator.py:38-50) and their durations are handed to the device event loop.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as N
from .errors import MissingCost, _raise
from .graph import HloGraph, state_arrays


@dataclass(frozen=True)
class Timeline:
    compute_events: tuple
    comm_events: tuple
    makespan_us: float


@dataclass(frozen=True)
class CostProviders:
    op_cost: Callable
    comm_cost: Callable


def _is_device(cp) -> bool:
    from .estimator import DeviceCostProviders

    return isinstance(cp, DeviceCostProviders)


_plain = None


def _plain_providers():
    """Device handle factory for externally supplied durations."""
    global _plain
    if _plain is None:
        from .comm import CommModelParams
        from .estimator import DeviceCostProviders, Profile

        _plain = DeviceCostProviders("profile", profile=Profile({}), comm_params=CommModelParams(0.0, 0.0))
    return _plain


def _duration(cp, g, kind, ident) -> float:
    try:
        value = cp.op_cost(g, g.group(ident)) if kind == "g" else cp.comm_cost(g, g.bucket(ident))
    except KeyError as exc:
        raise MissingCost(f"no duration for {kind} {ident}") from exc
    value = float(value)
    if value < 0:
        raise ValueError(f"negative duration {value} for {kind} {ident}")
    if value != value:  # NaN: no schedule order exists (every comparison is false)
        raise ValueError(f"NaN duration for {kind} {ident}")
    return value


def _node_name(bad, gids, bids):
    if bad is None or bad < 0:
        return "schedule"
    return f"g {gids[bad]}" if bad < len(gids) else f"b {bids[bad - len(gids)]}"


def simulate(g: HloGraph, cp) -> Timeline:
    """Two-lane schedule of ``g`` (simulator.py:53-140) on the device."""
    ng, rg, bk, vb, gids, bids = state_arrays(g)
    if _is_device(cp):
        dg = cp.device_graph(g)
        st, mk, comp, comm, bad = dg.simulate_arrays(ng, rg, bk, vb, None, cp.precision)
    else:
        durs = [_duration(cp, g, "g", x) for x in gids] + [_duration(cp, g, "b", b) for b in bids]
        dg = _plain_providers().device_graph(g)
        st, mk, comp, comm, bad = dg.simulate_arrays(ng, rg, bk, vb, np.array(durs, np.float64))
    if st:
        if st == N.FO_CYCLE:
            _raise(st, "schedule deadlocked; dependency structure is cyclic")
        _raise(st, f"no duration for {_node_name(bad, gids, bids)}", N.last_error())
    c = tuple((gids[int(i)], float(s), float(e)) for i, s, e in zip(*comp))
    b = tuple((bids[int(i)], float(s), float(e)) for i, s, e in zip(*comm))
    return Timeline(c, b, float(mk))


def cost(g: HloGraph, cp) -> float:
    """End-to-end iteration time of the candidate graph (simulator.py:143-145)."""
    if not _is_device(cp):
        return simulate(g, cp).makespan_us
    ng, rg, bk, vb, gids, bids = state_arrays(g)
    c, st = cp.device_graph(g).score_host(ng[None], rg[None], bk[None], vb, cp.precision)
    if st[0]:
        return simulate(g, cp).makespan_us  # re-run for the detailed error
    return float(c[0])


def cost_batch(graphs: Sequence[HloGraph], cp) -> np.ndarray:
    """cost() of many candidates of the same static graph in one device batch."""
    if not graphs:
        return np.zeros(0)
    if not _is_device(cp):
        return np.array([cost(x, cp) for x in graphs])
    enc = [state_arrays(x) for x in graphs]
    vb = max(e[3] for e in enc)
    ng = np.stack([e[0] for e in enc])
    rg = np.stack([e[1] for e in enc])
    bk = np.stack([e[2] for e in enc])
    c, st = cp.device_graph(graphs[0]).score_host(ng, rg, bk, vb, cp.precision)
    for i in np.nonzero(st)[0]:
        simulate(graphs[int(i)], cp)  # raises the reference's exception
    return c


def fo_bound(g: HloGraph, cp) -> float:
    """max(total compute, total comm) ignoring dependencies (simulator.py:148-153)."""
    if _is_device(cp):
        groups, buckets = cp.node_durations(g)
        total_c = sum(groups[x] for x in sorted(groups))
        total_b = sum(buckets[b] for b in sorted(buckets))
        return max(total_c, total_b)
    total_c = sum(_duration(cp, g, "g", x.id) for x in g.groups)
    total_b = sum(_duration(cp, g, "b", b.id) for b in g.buckets)
    return max(total_c, total_b)


def format_timeline(tl: Timeline) -> str:
    """One event per line sorted by start, makespan footer (simulator.py:156-166)."""
    rows = sorted([("compute", i, s, e) for i, s, e in tl.compute_events] +
                  [("comm", i, s, e) for i, s, e in tl.comm_events], key=lambda r: (r[2], r[0], r[1]))
    out = ["kind id start_us end_us"] + [f"{k} {i} {s:.6f} {e:.6f}" for k, i, s, e in rows]
    out.append(f"makespan_us {tl.makespan_us:.6f}")
    return "\n".join(out) + "\n"


def report_lines(g: HloGraph, cp, label: str) -> list:
    """The compare/report verb's per-graph summary (cli.py:227-238): makespan,
    fo_bound and module totals, from one device simulate and one device
    durations pass."""
    from .graph import module_stats

    tl = simulate(g, cp)
    if _is_device(cp):
        costs, comms = cp.node_durations(g)
    else:
        costs = {gr.id: cp.op_cost(g, gr) for gr in g.groups}
        comms = {b.id: cp.comm_cost(g, b) for b in g.buckets}
    stats = module_stats(g, costs, comms)
    return [
        f"[{label}] makespan_us {tl.makespan_us:.6f}",
        f"[{label}] fo_bound_us {fo_bound(g, cp):.6f}",
        f"[{label}] total_compute_us {stats.total_compute_us:.6f}",
        f"[{label}] total_comm_us {stats.total_comm_us:.6f}",
        f"[{label}] groups {stats.op_count} buckets {stats.bucket_count}",
    ]
