"""How many pixels would a 16-bit (bfloat-like, truncated) raw-error cache leave
ambiguous against the view's thresholds (dev probe for a 2 B/px cache)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import _abi  # noqa: E402
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402
from paper_2605_06876_b200.types import AdpSplitConfig  # noqa: E402

wl = S.CONFIGS["config3"]
plan = op.Plan("cuda:0")
d = wl.build_device(plan)
ini, cams, (ga, den) = d["ini"], d["cams"], d["stats"]
nv = 8
cfg = AdpSplitConfig(v_views=nv, n_max=wl.n_max)
img, dom, gt = d["img"][:nv].contiguous(), d["dom"][:nv].contiguous(), d["gt_img"][:nv].contiguous()
plan.phase1(d["g"], ini.extent, torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda"), cfg,
            cams[:nv], img, gt, dom)
lo_p, n_lo, _ = plan.buffer(_abi.BUF_LO)
th_p, n_th, _ = plan.buffer(_abi.BUF_THRESHOLDS)
lo = torch.empty(n_lo, dtype=torch.float64, device="cuda")
th = torch.empty(n_th, dtype=torch.float64, device="cuda")
op._copy_device(lo, lo_p, 8 * n_lo, plan.device)
op._copy_device(th, th_p, 8 * n_th, plan.device)
L = n_th // n_lo
raw = (img.double() - gt.double()).abs()
raw = (raw[..., 0] + raw[..., 1]) + raw[..., 2]
f32 = raw.float()   # round to nearest; RZ differs by at most one ulp, fine for a rate estimate
b16 = f32.view(torch.int32) >> 16
for bits, name in ((16, "top 16 bits (7-bit mantissa)"), (20, "top 20 bits (11-bit mantissa)")):
    sh = 32 - bits
    b = f32.view(torch.int32) >> sh
    amb = torch.zeros_like(b, dtype=torch.bool)
    for v in range(nv):
        for k in range(L):
            X = float(lo[v] + th[v * L + k])
            xb = int(np.array([X], dtype=np.float32).view(np.int32)[0]) >> sh
            amb[v] |= b[v] == xb
    print(f"{name}: ambiguous pixel fraction {amb.float().mean().item():.5f}")
