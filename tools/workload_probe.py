"""Workload probe (GPU): for synthetic variants of a BASELINE config, the measured
depth complexity (GT and init renders), the split/clone/fallback/reset shares
and the step's region/proposal counts -- used to choose the benchmark workload.

  python tools/workload_probe.py config3 ms=0.5,lf=0.06,mode=weighted ...
"""
import dataclasses
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402
from paper_2605_06876_b200.types import AdpSplitConfig  # noqa: E402


def variant(base, spec):
    kw = dict(x.split("=") for x in spec.split(",")) if spec else {}
    ms, ml = float(kw.get("ms", 1)), float(kw.get("ml", 1))
    return dataclasses.replace(base, size_factor=base.size_factor * ms,
                               large_range=(base.large_range[0] * ml, base.large_range[1] * ml),
                               large_frac=float(kw.get("lf", base.large_frac)),
                               stats_mode=kw.get("mode", base.stats_mode),
                               weight_floor=float(kw.get("floor", base.weight_floor)),
                               p_split=float(kw.get("ps", base.p_split)))


def main():
    base = S.CONFIGS[sys.argv[1]]
    plan = op.Plan("cuda:0")
    for spec in sys.argv[2:] or [""]:
        wl = variant(base, spec)
        t0 = time.time()
        d = wl.build_device(plan)
        ga, den = d["stats"]
        cfg = AdpSplitConfig(v_views=len(d["cams"]), n_max=wl.n_max)
        vids = list(range(len(d["cams"])))
        args = (d["g"], d["ini"].extent, d["cams"], d["gt_img"], torch.as_tensor(ga, device="cuda"),
                torch.as_tensor(den, device="cuda"), cfg)
        for _ in range(2):
            res = op.densify_step(*args, np.random.default_rng(0), renders=(d["img"], d["dom"]), plan=plan,
                                  view_ids=vids)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            res = op.densify_step(*args, np.random.default_rng(0), renders=(d["img"], d["dom"]), plan=plan,
                                  view_ids=vids)
        e1.record()
        torch.cuda.synchronize()
        c = res.counts
        ns = max(c["n_split"], 1)
        pp = res.report_arrays["cand_proposals"].cpu().numpy()
        print(json.dumps(dict(spec=spec, rho=wl.rho, dc_gt=round(d["dc_gt"], 2), dc_init=round(d["dc_init"], 2),
                              n=d["g"].n, n_split=c["n_split"], n_clone=c["n_clone"],
                              fallback_share=c["n_fallback"] / ns, reset_share=c["n_reset"] / ns,
                              adaptive_share=(ns - c["n_fallback"] - c["n_reset"]) / ns,
                              n_regions=c["n_regions"], n_proposals=c["n_proposals"], n_children=c["n_children"],
                              props_max=int(pp.max()) if len(pp) else 0, ms_per_step=e0.elapsed_time(e1) / 5,
                              setup_s=round(time.time() - t0, 1))), flush=True)
        del d, res


if __name__ == "__main__":
    main()
