"""One attribution render of a bench config's views bracketed by cudaProfilerStart/Stop (dev tool)."""
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config3"
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 4
wl = S.CONFIGS[name]
ini, cams, _, _ = dataclasses.replace(wl, stats_mode="uniform").build()   # the stats are not used
plan = op.Plan("cuda:0")
g = op.GaussianTensors.from_numpy(*ini.arrays(), device="cuda")
img, dom = plan.render(g, cams[:nv])
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
plan.render(g, cams[:nv], out=(img, dom))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok", img.shape)
