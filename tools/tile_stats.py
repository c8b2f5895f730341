"""Tile-level statistics of the attribution CCL at a bench config (dev tool): how
many 32x32 tiles hold candidate pixels, keyed pixels (eroded metric & candidate),
keyed rows and runs -- the work the tile kernels see."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402
from paper_2605_06876_b200.types import AdpSplitConfig  # noqa: E402

wl = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config3"]
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 8
plan = op.Plan("cuda:0")
d = wl.build_device(plan)
ini, cams, (ga, den) = d["ini"], d["cams"], d["stats"]
cfg = AdpSplitConfig(v_views=nv, n_max=wl.n_max)
V, H, W = nv, wl.height, wl.width
m = torch.zeros(V, H, W, dtype=torch.uint8, device="cuda")
b = torch.zeros_like(m)
plan.set_debug_maps(m, b)
img, dom, gt = d["img"][:nv].contiguous(), d["dom"][:nv].contiguous(), d["gt_img"][:nv].contiguous()
plan.phase1(d["g"], ini.extent, torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda"), cfg,
            cams[:nv], img, gt, dom)
plan.set_debug_maps(None, None)
g = ga / den
cls = torch.as_tensor((g >= cfg.tau_g) & (ini.scale.max(1) > cfg.tau_s * ini.extent), device="cuda")
dl = dom.long()
cand = torch.zeros_like(dl, dtype=torch.bool)
ok = dl >= 0
cand[ok] = cls[dl[ok]]
keyed = (m > 0) & cand
key = torch.where(keyed, dl * 4 + b.long(), torch.full_like(dl, -1))
Hp, Wp = (H + 31) // 32 * 32, (W + 31) // 32 * 32
pad = torch.full((V, Hp, Wp), -1, dtype=torch.long, device="cuda")
pad[:, :H, :W] = key
t = pad.view(V, Hp // 32, 32, Wp // 32, 32).permute(0, 1, 3, 2, 4)   # V, ty, tx, 32, 32
kt = t >= 0
cand_pad = torch.zeros((V, Hp, Wp), dtype=torch.bool, device="cuda")
cand_pad[:, :H, :W] = cand
ct = cand_pad.view(V, Hp // 32, 32, Wp // 32, 32).permute(0, 1, 3, 2, 4)
starts = kt.clone()
starts[..., 1:] &= ~((t[..., 1:] == t[..., :-1]) & kt[..., :-1])
runs = starts.sum((-1, -2)).float()
tiles = runs.numel()
print(f"{wl.name}: {nv} views, {tiles} tiles")
print("pixels: candidate-dominated %.3f, metric %.3f, keyed %.3f" % (cand.float().mean(), (m > 0).float().mean(),
                                                                   keyed.float().mean()))
print("tiles with a candidate pixel %.3f, with a keyed pixel %.3f" % (ct.any(-1).any(-1).float().mean(),
                                                                    kt.any(-1).any(-1).float().mean()))
kr = kt.any(-1).sum(-1).float()
has = kt.any(-1).any(-1)
print("keyed tiles: mean keyed rows %.1f, mean runs %.1f, p99 runs %.0f, >192 runs %d" % (
    kr[has].mean(), runs[has].mean(), torch.quantile(runs[has], 0.99), int((runs > 192).sum())))
