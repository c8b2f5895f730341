"""One densify step of a bench config bracketed by cudaProfilerStart/Stop (dev tool).

ncu --profile-from-start off ... python tools/profile_step.py [config3] [--timing]
captures exactly the launches of one warm step (renders resident, as bench.py).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402
from paper_2605_06876_b200.types import AdpSplitConfig  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
name = args[0] if args else "config3"
wl = S.CONFIGS[name]
plan = op.Plan("cuda:0")
_d = wl.build_device(plan)
ini, cams, (ga, den) = _d["ini"], _d["cams"], _d["stats"]
g, gt_img, img, dom = _d["g"], _d["gt_img"], _d["img"], _d["dom"]
cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
ga_t, den_t = torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda")
if "--timing" in sys.argv:   # stage-timing mode: one tile launch over all views (no pipelining), as bench's breakdown
    plan.set_timing(True)


def step():
    return op.densify_step(g, ini.extent, cams, gt_img, ga_t, den_t, cfg, np.random.default_rng(0),
                           renders=(img, dom), plan=plan, view_ids=list(range(len(cams))))


for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
res = step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("deferred tiles", plan.deferred_tiles(), "counts", res.counts)
for k, name in ((7, "tile_pairs"), (8, "gates"), (9, "gates_passed")):
    print(name, plan.get_param(k))
