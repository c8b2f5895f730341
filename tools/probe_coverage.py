"""Dev probe: fraction of candidate-dominated pixels, 32-px words and 32x32 tiles at config 3 (how much of the tile CCL could be skipped)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2605_06876_b200 import operator as op, synth as S
from paper_2605_06876_b200.types import AdpSplitConfig
wl = S.CONFIGS["config3"]
plan = op.Plan("cuda:0")
_d = wl.build_device(plan)
ini, cams, (ga, den) = _d["ini"], _d["cams"], _d["stats"]
g, img, dom = _d["g"], _d["img"], _d["dom"]
cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
arr = ini.arrays()
scale = np.asarray(arr[1]).reshape(-1, 3)
gg = np.where(den > 0, ga / np.where(den > 0, den, 1), 0)
cls = np.where(gg >= cfg.tau_g, np.where(scale.max(1) > cfg.tau_s * ini.extent, 1, 2), 0)
cand = torch.as_tensor(cls == 1, device="cuda")
d = dom.long()
c = torch.zeros_like(d, dtype=torch.bool)
ok = d >= 0
c[ok] = cand[d[ok]]
V, H, W = c.shape
print("candidate pixel fraction", c.float().mean().item())
Wp = (W + 31) // 32 * 32
cp = torch.zeros(V, H, Wp, dtype=torch.bool, device="cuda"); cp[:, :, :W] = c
words = cp.view(V, H, Wp // 32, 32).any(-1)
print("words with a candidate", words.float().mean().item())
w = words.float().unsqueeze(1)
nb = torch.nn.functional.max_pool2d(w, 3, 1, 1).squeeze(1) > 0
print("words with a candidate in the 3x3 word neighbourhood", nb.float().mean().item())
t = cp[:, : H // 32 * 32, :].view(V, H // 32, 32, Wp // 32, 32).any(-1).any(2)
print("32x32 tiles with a candidate", t.float().mean().item())
