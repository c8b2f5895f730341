"""Merge-gate statistics of one config-3 step (dev tool; needs a -DADPS_MERGE_STATS=1 build via ADPS_LIB)."""
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
cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
r = op.densify_step(d["g"], ini.extent, cams, d["gt_img"], torch.as_tensor(ga, device="cuda"),
                    torch.as_tensor(den, device="cuda"), cfg, np.random.default_rng(0), renders=(d["img"], d["dom"]),
                    plan=plan, view_ids=list(range(len(cams))))
pp = r.report_arrays["cand_proposals"].cpu().numpy()
print("counts", r.counts)
print("tile pairs", plan.get_param(7), "gates", plan.get_param(8), "passed", plan.get_param(9))
print("proposals: total", int(pp.sum()), "max", int(pp.max()), ">32:", int((pp > 32).sum()), "sum over >32:", int(pp[pp > 32].sum()))
