"""The hardware-oracle cost providers (workloads.py:53-74, :276-304 of the
reference) on the device, and loading of the committed synthetic workload
inputs (workloads/ at the repository root: graphs, profiles, comm params and
random-init estimator models made by the reference's own gen_workload /
make_profile / train, see tests/golden/make_golden.py).  They are inputs, not
expected outputs: the expected outputs live under tests/golden."""

from __future__ import annotations

import os
from dataclasses import dataclass, field

from . import _native as N
from .comm import CommModelParams, load_params
from .errors import InvalidConfig
from .estimator import DeviceCostProviders, load_model, load_profile
from .graph import load_graph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURES = os.path.join(ROOT, "workloads")

# BASELINE.json configs -> fixture names
CONFIGS = {
    "vgg16": "VGG-16 data-parallel training graph, 8 simulated workers (chain, V=144, A=32)",
    "resnet50": "ResNet-50 training graph proxy (residual, V=672, A=161)",
    "bert": "BERT-base training graph proxy (attention, V=760, A=199)",
    "gpt2m": "GPT-2 medium training graph proxy (attention, V=5000, A=292)",
    "synth50k": "synthetic 50k-op DAG (residual, V=50000, A=1000)",
}


@dataclass(frozen=True)
class HardwareParams:
    launch_overhead_us: float = 5.0
    mem_us_per_byte: float = 1.0 / 1024.0
    compute_rates: dict = field(default_factory=dict)
    comm_params: CommModelParams = CommModelParams(C=0.001, D=100.0)
    noise: float = 0.0
    seed: int = 0

    def __post_init__(self) -> None:
        if self.launch_overhead_us <= 0 or self.mem_us_per_byte <= 0:
            raise InvalidConfig("launch overhead and memory rate must be > 0")
        if not (0 <= self.noise <= 0.5):
            raise InvalidConfig("noise fraction must lie in [0, 0.5]")


def oracle_providers(hw: HardwareParams, precision: int = N.FO_PREC_FP32) -> DeviceCostProviders:
    """Ground-truth providers: member compute + one launch + memory traffic of
    externally moved bytes per group (workloads.py:276-291), linear comm.
    With noise > 0 every group's time carries the reference's deterministic
    blake2b jitter of its content key (workloads.py:254-273), on the device."""
    return DeviceCostProviders("hw_oracle", hw=hw, precision=precision)


_ORACLES: dict = {}


def oracle_time(g, group, hw: HardwareParams) -> float:
    """Ground-truth execution time of one group of ``g`` (workloads.py:276-291),
    computed by the device hardware oracle in fp64; providers are cached per
    HardwareParams so repeated calls reuse one device handle per graph."""
    key = (hw.launch_overhead_us, hw.mem_us_per_byte, hw.comm_params.C, hw.comm_params.D, hw.noise, hw.seed)
    cp = _ORACLES.get(key)
    if cp is None:
        if len(_ORACLES) >= 8:
            _ORACLES.clear()
        cp = _ORACLES[key] = oracle_providers(hw, precision=N.FO_PREC_FP64)
    return cp.op_cost(g, group)


def load_workload(name: str, root: str = FIXTURES):
    """(graph, profile, comm params, MP model, linear model) of a fixture."""
    import json

    base = os.path.join(root, name)
    g = load_graph(base + ".graph.json.gz")
    profile = load_profile(base + ".profile.json.gz")
    comm = load_params(base + ".comm.json")
    src = name
    if os.path.exists(base + ".model_from.json"):
        with open(base + ".model_from.json") as fh:
            src = json.load(fh)["model_from"]
    sbase = os.path.join(root, src)
    mp = load_model(sbase + ".mp.model.json.gz")
    lin = load_model(sbase + ".lin.model.json")
    return g, profile, comm, mp, lin
