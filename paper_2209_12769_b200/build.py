"""Builds the in-tree C-ABI library for sm_100a:
paper_2209_12769_b200/_build/libdiscob200.so (CUDA kernels + C-ABI + native
batch-expand/search engine).  Runs on a CPU-only host: nvcc cross-compiles."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_build")
OUT = os.path.join(OUT_DIR, "libdiscob200.so")
SOURCES = ["score.cu", "capi.cu", "engine.cpp", "xchg.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # schedule arithmetic must stay plain IEEE add/mul (bit-exact vs the reference)
    "-Xcompiler", "-fPIC,-fopenmp,-O3",
]
HEADERS = [os.path.join(CSRC, "fo_internal.h"), os.path.join(CSRC, "score_inc.cuh"),
           os.path.join(os.path.dirname(HERE), "include", "disco_b200.h")]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "disco_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in [src, *HEADERS])


def build(force: bool = False, verbose: bool = False) -> str:
    """Per-source objects (rebuilt when the source or a shared header changed),
    then one shared library."""
    if not force and not needs_build():
        return OUT
    os.makedirs(OUT_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(OUT_DIR, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        if force or _stale(obj, path):
            cmd = [nvcc, *NVCC_FLAGS, "-c", path, "-o", obj + ".tmp"]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            os.replace(obj + ".tmp", obj)
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", OUT + ".tmp", "-lgomp", "-ldl"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
