"""Host-side timing of one densify step (dev helper): where does wall time go?"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2605_06876_b200 import operator as op, synth as S
from paper_2605_06876_b200.types import AdpSplitConfig

wl = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config3"]
plan = op.Plan("cuda:0")
_d = wl.build_device(plan)
ini, cams, (ga, den) = _d["ini"], _d["cams"], _d["stats"]
g, gt_img, img, dom = _d["g"], _d["gt_img"], _d["img"], _d["dom"]
ga_t, den_t = torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda")
cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
vids = list(range(len(cams)))
for it in range(6):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    rng = np.random.default_rng((0, 0))
    cams_v = cams
    counts = plan.phase1(g, ini.extent, ga_t, den_t, cfg, cams_v, img, gt_img, dom)
    t.append(time.perf_counter())
    nf = counts["n_fallback"]
    normals_np = rng.standard_normal(6 * nf)
    t.append(time.perf_counter())
    normals = torch.as_tensor(normals_np, dtype=torch.float64, device="cuda")
    t.append(time.perf_counter())
    out = op.GaussianTensors.empty(counts["n_out"], 0, "cuda")
    index_map = torch.empty(counts["n_out"], dtype=torch.int64, device="cuda")
    plan.phase2(g, normals, out, index_map)
    t.append(time.perf_counter())
    ra = plan.report_arrays(counts["n_split"], counts["n_clone"])
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print(f"phase1 {d[0]:.3f} normals({6*nf}) {d[1]:.3f} h2d {d[2]:.3f} alloc+phase2 {d[3]:.3f} report+sync {d[4]:.3f} total {sum(d):.3f} ms")
