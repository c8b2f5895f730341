"""Sweep the attribution pipeline (view chunks x input-pass residency) at a bench config (dev tool)."""
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


def step():
    return op.densify_step(d["g"], ini.extent, cams, d["gt_img"], ga_t, den_t, cfg, np.random.default_rng(0),
                           renders=(d["img"], d["dom"]), plan=plan, view_ids=list(range(len(cams))))


e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for chunks in (1, 2, 4, 8, 16):
    for bps in (0, 6, 4, 3, 2):
        plan.lib.adps_set_param(plan._h, 10, chunks)
        plan.lib.adps_set_param(plan._h, 11, bps)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            step()
        e1.record()
        torch.cuda.synchronize()
        print(f"chunks {chunks:2d} input blocks/SM {bps}: {e0.elapsed_time(e1) / 10:.4f} ms/step", flush=True)
