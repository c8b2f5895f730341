"""cProfile of the host side of densify_step at a bench config (dev tool): where the
Python/ctypes time goes between and around the kernels (us per step, by own time)."""
import cProfile
import os
import pstats
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


for _ in range(3):
    step()
torch.cuda.synchronize()
K = 200
pr = cProfile.Profile()
pr.enable()
for _ in range(K):
    step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
rows = sorted(st.stats.items(), key=lambda kv: -kv[1][2])
for (fn, line, name), (cc, nc, tt, ct, callers) in rows[:45]:
    print(f"{tt / K * 1e6:9.1f} us/step own  {ct / K * 1e6:9.1f} cum  calls/step {nc / K:5.1f}  {os.path.basename(fn)}:{line}({name})")
