"""The tensor-core option for the FP32 message-passing transforms (north
star: "tensor cores only if the result stays within tolerance, otherwise
FP32 FFMA").  Every fused-group prediction of the reference's golden
candidates and every cost of a batch are compared with the FP64 oracle for
the three arithmetics; the measured errors are written to
gpurun_out/tensorcore_error.json (DESIGN.md records the decision).  Only
3xTF32 is held to the 1e-4 tolerance: plain TF32 is expected to break it."""

import json
import os

import numpy as np
import pytest

import paper_2209_12769_b200 as P
from paper_2209_12769_b200 import _native as N

from _golden import cases, graph_with_state

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _device():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    torch.cuda.set_device(0)


def _errors(name, mode):
    from oracle.oracle import Oracle, load_workload

    g, prof, comm, mp, lin = P.load_workload(name)
    cp = P.make_cost_providers(prof, comm, mp, precision=N.FO_PREC_FP32)
    dg = cp.device_graph(g)
    N.lib().fo_set_estimator_arith(dg.h, mode)
    N.lib().fo_memo_clear(dg.h, None)
    doc = cases(name)
    group_err = 0.0
    for c in doc["candidates"]:
        pred = P.predict_fused_groups(cp, graph_with_state(g, c["state"]))
        for f in c["fused"]:
            group_err = max(group_err, abs(pred[f["id"]] - f["mp"]) / f["mp"])
    dg.set_parent()
    off, chg = dg.make_candidates_delta(np.arange(1024, dtype=np.uint64))
    N.lib().fo_memo_clear(dg.h, None)
    cost, st = dg.score_delta_host(off, chg, N.FO_PREC_FP32)
    assert (st == 0).all()
    o = Oracle(load_workload(name), "mp")
    sts, ref = o.cost_batch(*(np.stack([o.make_candidate(i)[j] for i in range(1024)]) for j in range(3)))
    cost_err = float(np.max(np.abs(cost - ref) / ref))
    N.lib().fo_set_estimator_arith(dg.h, 0)
    return group_err, cost_err


def test_tensor_core_arithmetic_against_fp64():
    out = {}
    for name in ("resnet50", "bert"):
        for mode, label in ((0, "fp32_ffma"), (1, "tf32_tensor_core"), (2, "3xtf32_tensor_core")):
            ge, ce = _errors(name, mode)
            out[f"{name}/{label}"] = {"max_rel_err_fused_group_vs_reference": ge, "max_rel_err_cost_vs_oracle": ce}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "tensorcore_error.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    for name in ("resnet50", "bert"):
        assert out[f"{name}/fp32_ffma"]["max_rel_err_fused_group_vs_reference"] <= 1e-4
        assert out[f"{name}/3xtf32_tensor_core"]["max_rel_err_fused_group_vs_reference"] <= 1e-4
        assert out[f"{name}/3xtf32_tensor_core"]["max_rel_err_cost_vs_oracle"] <= 1e-4
