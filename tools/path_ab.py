"""Step time (CUDA events, warm) under each tile CCL path at a bench config (dev tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402
from paper_2605_06876_b200.types import AdpSplitConfig  # noqa: E402

wl = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config3"]
plan = op.Plan("cuda:0")
d = wl.build_device(plan)
ini, cams, (ga, den) = d["ini"], d["cams"], d["stats"]
ga_t, den_t = torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda")
cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
vids = list(range(len(cams)))


def step():
    return op.densify_step(d["g"], ini.extent, cams, d["gt_img"], ga_t, den_t, cfg, np.random.default_rng(0),
                           renders=(d["img"], d["dom"]), plan=plan, view_ids=vids)


for rep in range(2):
    for path in (0, 3, 2):
        plan.set_tile_path(path)
        for _ in range(3):
            r = step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            r = step()
        e1.record()
        torch.cuda.synchronize()
        print(f"path {path}: {e0.elapsed_time(e1) / 10:.3f} ms/step  n_regions {r.counts['n_regions']}")
plan.set_tile_path(0)
