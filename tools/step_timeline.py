"""Host/GPU timeline of one warm densify step (dev helper): where does the GPU idle?

Wraps the Plan methods densify_step calls with host timestamps and CUDA events
on the plan's stream, then prints each call's host span and the GPU time
between consecutive marks.  Gaps where the host runs while the GPU waits show
up as host spans that end with a synchronisation.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402
from paper_2605_06876_b200.types import AdpSplitConfig  # noqa: E402

wl = S.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "config3"]
plan = op.Plan("cuda:0")
_d = wl.build_device(plan)
ini, cams, (ga, den) = _d["ini"], _d["cams"], _d["stats"]
g, gt_img, img, dom = _d["g"], _d["gt_img"], _d["img"], _d["dom"]
ga_t, den_t = torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda")
cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
marks = []


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record(torch.cuda.current_stream())
    marks.append((name, time.perf_counter(), e))


def wrap(obj, name):
    f = getattr(obj, name)

    def w(*a, **k):
        mark(name + ">")
        r = f(*a, **k)
        mark(name + "<")
        return r
    setattr(obj, name, w)


for n in ("phase1_begin", "phase1_end", "phase2", "report_arrays", "normals_pcg64", "capacity", "phase1_end_emit"):
    if hasattr(plan, n):
        wrap(plan, n)


def step():
    return op.densify_step(g, ini.extent, cams, gt_img, ga_t, den_t, cfg, np.random.default_rng(0),
                           renders=(img, dom), plan=plan, view_ids=list(range(len(cams))),
                           one_sync=os.environ.get("ADPS_TWO_CALL", "0") != "1")


for _ in range(3):
    step()
for it in range(3):
    torch.cuda.synchronize()
    marks.clear()
    mark("start")
    step()
    mark("end")
    torch.cuda.synchronize()
    t0, e0 = marks[0][1], marks[0][2]
    print(f"--- step {it}: gpu {e0.elapsed_time(marks[-1][2]):.3f} ms, host {(marks[-1][1] - t0) * 1e3:.3f} ms")
    for (n0, h0, ev0), (n1, h1, ev1) in zip(marks, marks[1:]):
        print(f"  {n0:>16s} -> {n1:<16s} host {(h1 - h0) * 1e3:7.3f} ms   gpu {ev0.elapsed_time(ev1):7.3f} ms")
