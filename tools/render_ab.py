"""Per-view render time (CUDA events) of the two binnings on a bench config (dev tool)."""
import dataclasses
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config3"
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 16
wl = S.CONFIGS[name]
ini, cams, _, _ = dataclasses.replace(wl, stats_mode="uniform").build()
g = op.GaussianTensors.from_numpy(*ini.arrays(), device="cuda")
ref = None
for fast in (False, True, False, True):
    plan = op.Plan("cuda:0")
    plan.set_render_binning(fast)
    img, dom = plan.render(g, cams[:nv])
    torch.cuda.synchronize()
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.render(g, cams[:nv], out=(img, dom))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / nv)
    same = None
    if ref is None:
        ref = (img.clone(), dom.clone())
    else:
        same = bool(torch.equal(img, ref[0]) and torch.equal(dom, ref[1]))
    import hashlib
    h = hashlib.md5(img.cpu().numpy().tobytes() + dom.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"fast={fast} ms/view={min(ts):.4f} (runs {', '.join(f'{t:.4f}' for t in ts)}) identical={same} md5={h}")
