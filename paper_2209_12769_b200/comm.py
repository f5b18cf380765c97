"""AllReduce time model consumed by the simulator: T = C * bytes + D
(comm.py:20-49 of the reference).  On the device this is one fp64 multiply
and add per bucket inside the scoring kernel."""

from __future__ import annotations

import json
from dataclasses import dataclass

from .errors import GraphFormatError


@dataclass(frozen=True)
class CommModelParams:
    C: float  # microseconds per byte
    D: float  # fixed per-AllReduce overhead, microseconds

    def __post_init__(self) -> None:
        if self.C < 0 or self.D < 0:
            raise ValueError("C and D must be non-negative")


def predict(params: CommModelParams, nbytes: float) -> float:
    if nbytes < 0:
        raise ValueError("bytes must be >= 0")
    return params.C * nbytes + params.D


def load_params(path) -> CommModelParams:
    with open(path, "r", encoding="utf-8") as fh:
        doc = json.load(fh)
    if not isinstance(doc, dict) or set(doc) != {"C", "D"}:
        raise GraphFormatError(f"{path}: expected a two-field document {{'C','D'}}")
    return CommModelParams(C=float(doc["C"]), D=float(doc["D"]))


def save_params(path, params: CommModelParams) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        json.dump({"C": params.C, "D": params.D}, fh, sort_keys=True)
        fh.write("\n")
