"""ctypes wrapper of oracle/render_oracle.c -- TEST/BASELINE INFRASTRUCTURE ONLY.

``build()`` compiles it with gcc (-O2, IEEE, no fast-math) into
oracle/liboracle_render.so; ``render(g, cam)`` mirrors
``adpsplit_oracle.render`` for large scenes (the numpy one loops in Python
per splat).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "render_oracle.c")
LIB = os.path.join(HERE, "liboracle_render.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.run(["gcc", "-O2", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC",
                        "-o", LIB, SRC, "-lm"], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        lib = C.CDLL(LIB)
        p = C.c_void_p
        lib.oracle_render.argtypes = [C.c_int64, p, p, p, p, p, p, C.c_int, p, p, p, p]
        lib.oracle_render.restype = C.c_int
        _lib = lib
    return _lib


def render(g, cam_row, background=(0.0, 0.0, 0.0)):
    """(image H x W x 3 fp64, dominant H x W int64) of oracle Gaussians ``g``."""
    lib = _load()
    cam = np.ascontiguousarray(cam_row, dtype=np.float64)
    w, h = int(cam[16]), int(cam[17])
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (g.mu, g.scale, g.rot, g.opacity, g.sh_dc)]
    k = g.sh_rest.shape[1]
    rest = np.ascontiguousarray(g.sh_rest, dtype=np.float64) if k else None
    bg = np.ascontiguousarray(background, dtype=np.float64)
    img = np.empty((h, w, 3))
    dom = np.empty((h, w), dtype=np.int64)
    ptr = lambda a: a.ctypes.data_as(C.c_void_p) if a is not None else None  # noqa: E731
    rc = lib.oracle_render(len(g), *[ptr(a) for a in arrs], ptr(rest), k, ptr(cam), ptr(bg), ptr(img), ptr(dom))
    if rc != 0:
        raise MemoryError("oracle_render failed")
    return img, dom
