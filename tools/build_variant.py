"""Build a dev variant of libadps.so with extra -D flags for one source (dev tool).

usage: python tools/build_variant.py NAME SOURCE.cu[,OTHER.cu] -DFOO=1 ...
writes paper_2605_06876_b200/_variants/libadps_NAME.so; select it with ADPS_LIB=...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import build_ext as B  # noqa: E402

name, srcs, defs = sys.argv[1], sys.argv[2].split(","), sys.argv[3:]
B.build()
out_dir = os.path.join(B.HERE, "_variants")
os.makedirs(out_dir, exist_ok=True)
objs = []
for s in B.SOURCES:
    obj = os.path.join(B.BUILD, s.replace(".cu", ".o"))
    if s in srcs:
        obj = os.path.join(B.BUILD, f"{name}_{s.replace('.cu', '.o')}")
        flags = B.ARCH + B.COMMON + (["-fmad=false"] if s in B.NO_FMA else []) + defs
        subprocess.run([B.nvcc()] + flags + ["-c", os.path.join(B.CSRC, s), "-o", obj], check=True)
    objs.append(obj)
lib = os.path.join(out_dir, f"libadps_{name}.so")
subprocess.run([B.nvcc()] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs, check=True)
print(lib)
