"""Stage-isolated parity at the BASELINE configs.

The same GPU attribution (image, dominant) and GT images go into the CUDA step
(through the C ABI) and into the CPU oracle, which is pinned to the reference's
golden vectors (tests/test_oracle_golden.py).  Every integer output is compared
exactly -- the region table (candidate, view, band, first pixel, int64 pixel
moments), per-candidate case, regions_per_view, proposals, N_i, merge_edges,
clones, resets, index_map, child_parent and insert offsets -- and the child
parameters within the float tolerance; near-threshold candidates (merge gates
within 1e-9 of gamma_d, |t*| ~ 0, extent ties, degenerate eigenspaces) are
counted and reported (PARITY_REPORT), their rows excluded from the float check.

  config2: 100k Gaussians, all 16 views of 800x800
  config3: 1.2M Gaussians, 4 of the 64 views of 1237x822 (views 0, 16, 32, 48),
           every parent merged
  config4: 3M Gaussians, 2 of the 128 views of 1297x840 (views 0, 64)
  config5: 8M Gaussians, 2 of its 256 views (views 0, 128)

Run on a B200:  PARITY_REPORT=gpurun_out/parity.json python -m pytest tests -m gpu -q
"""

import numpy as np
import pytest

import parity as PA
from oracle import adpsplit_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def op():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2605_06876_b200 import operator
    return operator


def _stage_isolated(op, name, views, cap_huge=None):
    import torch
    from paper_2605_06876_b200 import _abi
    from paper_2605_06876_b200 import synth as S
    from paper_2605_06876_b200.types import AdpSplitConfig
    wl = S.CONFIGS[name]
    plan = op.Plan("cuda:0")
    if cap_huge is not None:
        plan.set_param(_abi.PARAM_CAP_HUGE, cap_huge)
        assert plan.get_param(_abi.PARAM_CAP_HUGE) == cap_huge
    d = wl.build_device(plan)
    ini, cams, (ga, den) = d["ini"], d["cams"], d["stats"]
    cams_k = cams[views]
    idx = torch.as_tensor(views, device="cuda")
    img, dom, gt = d["img"].index_select(0, idx), d["dom"].index_select(0, idx), d["gt_img"].index_select(0, idx)
    del d
    # the k cameras are the step's camera list and v_views = k: both sides sample all of
    # them with the same Generator call (ref/adc.py:161) and then draw the same normals
    cfg = AdpSplitConfig(v_views=len(views), n_max=wl.n_max)
    gres = op.densify_step(op.GaussianTensors.from_numpy(*ini.arrays(), device="cuda"), ini.extent, cams_k, gt,
                           torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda"), cfg,
                           np.random.default_rng(11), renders=(img, dom), plan=plan)
    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    cam_objs = [O.Cam.from_row(r) for r in cams_k]
    renders = {k: (img[k].double().cpu().numpy(), dom[k].long().cpu().numpy()) for k in range(len(views))}
    gts = {k: gt[k].double().cpu().numpy() for k in range(len(views))}
    ores = O.adpsplit_step(g, ini.extent, cam_objs, gts, ga, den, cfg, np.random.default_rng(11), renders=renders)
    np.testing.assert_array_equal(PA.gpu_regions(plan), PA.oracle_regions(ores, list(range(len(views)))))
    flagged = PA.flag_candidates(ores, g, cam_objs, cfg)
    st = PA.compare_step(gres, ores, flagged, g)
    c = gres.counts
    assert plan.check_guards() == (0, 0)   # no write past any plan buffer
    assert c["n_regions"] == sum(len(r) for r in ores.regions.values())
    assert c["n_fallback"] == sum(r.fallback for r in ores.candidates)
    assert c["n_reset"] == len(ores.reset_indices)
    c["max_groups"] = max((len(v) for v in ores.all_groups.values()), default=0)   # before the cap
    return st, c


def test_config2_all_views_stage_isolated(op):
    st, c = _stage_isolated(op, "config2", list(range(16)))
    assert st["mismatched"] == 0, st
    assert c["n_regions"] > 1000 and c["n_children"] > 100, c


def test_config3_view_subset_stage_isolated(op):
    st, c = _stage_isolated(op, "config3", [0, 16, 32, 48])
    assert st["mismatched"] == 0, st
    assert c["n_regions"] > 1000 and c["n_children"] > 100, c


def test_cap_cluster_selection_stage_isolated(op):
    """Every parent with more than 64 merged groups through the cap's
    thread-block-cluster selection (the path of config 3's background parent
    with thousands of groups at 64 views): same results as the oracle."""
    st, c = _stage_isolated(op, "config3", [0, 16, 32, 48], cap_huge=64)
    assert st["mismatched"] == 0, st
    assert c["max_groups"] > 64, c   # the cluster path ran
    assert c["n_children"] > 100, c


def test_config4_view_subset_stage_isolated(op):
    st, c = _stage_isolated(op, "config4", [0, 64])
    assert st["mismatched"] == 0, st
    assert c["n_regions"] > 1000 and c["n_children"] > 100, c


def test_config5_view_subset_stage_isolated(op):
    st, c = _stage_isolated(op, "config5", [0, 128])
    assert st["mismatched"] == 0, st
    assert c["n_regions"] > 1000 and c["n_children"] > 100, c
