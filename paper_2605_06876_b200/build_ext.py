"""Build the in-tree CUDA extension ``libadps.so`` for sm_100a.

Each ``csrc/*.cu`` is compiled with nvcc (``-gencode arch=compute_100a,
code=sm_100a -lineinfo -O3``), then linked into one shared library with the
CUDA runtime linked statically.  Files whose fp64 arithmetic decides integer
outputs (maps thresholds, select, child init, merge) are compiled with
``-fmad=false`` so no multiply-add is contracted behind numpy's back; the
render keeps FMA.

Usage:  python -m paper_2605_06876_b200.build_ext   (or __graft_entry__.build())
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libadps.so")
BUILD = os.path.join(ROOT, "build", "adps")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "-I", os.path.join(ROOT, "include")]
NO_FMA = {"attribution.cu", "tile_warp.cu", "normals.cu", "split.cu", "merge.cu", "plan.cu"}
SOURCES = ["attribution.cu", "tile_warp.cu", "normals.cu", "split.cu", "merge.cu", "render.cu", "plan.cu"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj: str, deps: list) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "adps.h"))
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(obj)
        if not force and not _stale(obj, [path] + headers):
            continue
        flags = ARCH + COMMON + (["-fmad=false"] if src in NO_FMA else [])
        cmd = [nvcc()] + flags + ["-c", path, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    if force or _stale(LIB, objs):
        # export only the C ABI (adps_* symbols carry default visibility via extern "C")
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
