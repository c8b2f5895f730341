"""Host cost of the densify_step prologue operations, one by one (dev tool)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import operator as op, synth as S
from paper_2605_06876_b200.types import AdpSplitConfig
F32, F64 = torch.float32, torch.float64
wl = S.CONFIGS['config3']
plan = op.Plan('cuda:0')
d = wl.build_device(plan)
cams = d['cams']; g = d['g']; gt = d['gt_img']; img, dom = d['img'], d['dom']
ga = torch.as_tensor(d['stats'][0], device='cuda'); den = torch.as_tensor(d['stats'][1], device='cuda')
cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
vids = list(range(len(cams)))
dev = plan.device
def t(name, fn, n=2000):
    fn()
    t0 = time.perf_counter()
    for _ in range(n): fn()
    print(f"{name:40s} {(time.perf_counter()-t0)/n*1e6:8.2f} us")
t('camera_rows', lambda: op.camera_rows(cams))
cr = op.camera_rows(cams)
t('cams[view_ids]', lambda: cr[vids])
t('_gather_views', lambda: op._gather_views(gt, vids, dev))
t('ga.to().contiguous()', lambda: ga.to(dev, F64).contiguous())
t('img.to().contiguous()', lambda: img.to(dev, F32).contiguous())
t('dom.to().contiguous()', lambda: dom.to(dev, torch.int32).contiguous())
t('config_struct', lambda: op.config_struct(cfg))
t('g.abi()', lambda: g.abi())
t('_check_inputs', lambda: plan._check_inputs(ga, den, img, gt, dom))
t('_stream()', lambda: plan._stream())
t('rng default_rng', lambda: np.random.default_rng(0))
r = np.random.default_rng(0)
t('bitgen.state', lambda: r.bit_generator.state)
t('torch.empty(10000,int64)', lambda: torch.empty(10000, dtype=torch.int64, device=dev))
t('GaussianTensors.empty', lambda: op.GaussianTensors.empty(1300000, 0, dev))
