"""GPU render depth order: the fast path (32-bit depth keys, a fix-up of equal
keys, no host synchronisation between views) gives the same images, dominant
maps, epilogue outputs and workload statistics as the 64-bit sort of the fp64
depths, including the views whose pairs exceed the tile sort's capacity and
the depth runs too long for the fix-up (both rendered again by the host).

Run on a B200:  python -m pytest tests -m gpu -q
"""

import numpy as np
import pytest

import golden_io
import parity as PA
from oracle import adpsplit_oracle as O

pytestmark = pytest.mark.gpu

DATA, META = golden_io.load()


@pytest.fixture(scope="module")
def op():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2605_06876_b200 import operator
    return operator


def _both(op, g, cams, bg=(0.0, 0.0, 0.0), cap=None):
    """(image, dominant, plan) with the fast path (optionally from a pair
    capacity of `cap`) and with the 64-bit sort, on fresh plans."""
    from paper_2605_06876_b200 import _abi
    out = []
    for fast in (True, False):
        plan = op.Plan("cuda:0")
        plan.set_render_binning(fast)
        if fast and cap is not None:
            plan.set_param(_abi.PARAM_RENDER_PAIR_CAP, cap)
        img, dom = plan.render(g, cams, bg=bg)
        out.append((img.cpu().numpy(), dom.cpu().numpy(), plan))
    return out


@pytest.mark.parametrize("c", range(12))
def test_fast_depth_order_golden_renders(op, c):
    g, _ = golden_io.scene(DATA, f"render__{c}__scene")
    (i1, d1, _), (i0, d0, _) = _both(op, PA.to_tensors(PA.oracle_gaussians_f32(g)), DATA[f"render__{c}__cam"],
                                     bg=(0.1, 0.2, 0.3))
    np.testing.assert_array_equal(i1, i0)
    np.testing.assert_array_equal(d1, d0)


def test_fast_depth_order_baseline_views_and_overflow(op):
    """Config 2's 16 views, bit-identical; then the same from a 10-pair
    capacity (every view exceeds it, the capacity grows, the views are redone)."""
    import dataclasses
    from paper_2605_06876_b200 import _abi
    from paper_2605_06876_b200 import synth as S
    wl = S.CONFIGS["config2"]
    ini, cams, _, _ = dataclasses.replace(wl, stats_mode="uniform").build()
    g = op.GaussianTensors.from_numpy(*ini.arrays(), device="cuda")
    (i1, d1, _), (i0, d0, _) = _both(op, g, cams)
    np.testing.assert_array_equal(i1, i0)
    np.testing.assert_array_equal(d1, d0)
    (i2, d2, p2), _ = _both(op, g, cams[:3], cap=10)
    np.testing.assert_array_equal(i2, i0[:3])
    np.testing.assert_array_equal(d2, d0[:3])
    assert p2.get_param(_abi.PARAM_RENDER_PAIR_CAP) > 10


def _sheet(n, rng, x_decreasing=False):
    """n Gaussians on the plane z = 1 over a 16 x 16 image."""
    x = np.sort(rng.uniform(-0.3, 0.3, n))[::-1] if x_decreasing else rng.uniform(-0.3, 0.3, n)
    mu = np.c_[x, rng.uniform(-0.3, 0.3, n), np.ones(n)]
    return O.Gaussians(mu, np.full((n, 3), 0.04), np.tile([1.0, 0, 0, 0], (n, 1)), rng.uniform(0.2, 0.9, n),
                       rng.normal(0, 0.5, (n, 3)))


@pytest.mark.parametrize("case", ["sub_float_reversed", "equal_depths_short", "equal_depths_long"])
def test_fast_depth_order_equal_keys(op, case):
    """Depths that one float cannot tell apart: 40 distinct doubles within a
    few float ulps, the indices in reverse depth order (the fix-up reorders
    them); 200 and 600 identical depths (index order; the 600-run is longer
    than the fix-up and takes the 64-bit sort).  Same images as the 64-bit
    sort and as the oracle."""
    rng = np.random.default_rng(5)
    R = np.eye(3)
    if case == "sub_float_reversed":
        # a camera turned by 1e-6 rad: depths 3 + 1e-6 x, a few float ulps for
        # 40 Gaussians, increasing in x while the index decreases in x
        a = 1e-6
        R = np.array([[np.cos(a), 0, np.sin(a)], [0, 1, 0], [-np.sin(a), 0, np.cos(a)]])
        g = _sheet(40, rng, x_decreasing=True)
    else:
        g = _sheet(200 if case == "equal_depths_short" else 600, rng)
    cam = O.Cam(R, np.array([0, 0, -2.0]), 20.0, 20.0, 7.5, 7.5, 16, 16)
    g = PA.oracle_gaussians_f32(g)
    (i1, d1, _), (i0, d0, _) = _both(op, PA.to_tensors(g), cam.row()[None])
    np.testing.assert_array_equal(i1, i0)
    np.testing.assert_array_equal(d1, d0)
    img_o, dom_o, best, second = O.render(g, cam, with_weights=True)
    assert np.abs(i1[0].astype(np.float64) - img_o).max() < 2e-5
    tie = (best - second) <= PA.EPS_TIE * np.maximum(best, 1e-30)
    assert not ((d1[0] != dom_o) & ~tie).any()


def test_fast_depth_order_epilogue_and_stats(op):
    """The fused epilogue's step and the workload statistics (blending weights,
    contributions) do not depend on the depth-order path."""
    import torch
    from paper_2605_06876_b200 import synth as S
    from paper_2605_06876_b200.types import AdpSplitConfig
    wl = S.CONFIGS["config2"]
    res = {}
    for fast in (True, False):
        plan = op.Plan("cuda:0")
        plan.set_render_binning(fast)
        d = wl.build_device(plan)
        g, cams = d["g"], d["cams"]
        ga, den = (torch.as_tensor(x, device="cuda") for x in d["stats"])
        cfg = AdpSplitConfig(v_views=len(cams) // 2, n_max=wl.n_max)
        r = op.densify_step(g, d["ini"].extent, cams, d["gt_img"], ga, den, cfg, np.random.default_rng(3),
                            plan=plan, fused=True)
        out = dict(r.gaussians.numpy())
        out.update(index_map=r.index_map.cpu().numpy(), img=d["img"].cpu().numpy(), dom=d["dom"].cpu().numpy(),
                   weight=d["weight"].cpu().numpy() if hasattr(d["weight"], "cpu") else np.asarray(d["weight"]),
                   dc=np.array([d["dc_init"], d["dc_gt"]]))
        res[fast] = (r.counts, out)
    assert res[True][0] == res[False][0]
    for k in res[False][1]:
        if k == "weight":   # float atomics: summation order varies between runs
            np.testing.assert_allclose(res[True][1][k], res[False][1][k], rtol=1e-5, atol=1e-30, err_msg=k)
        else:
            np.testing.assert_array_equal(res[True][1][k], res[False][1][k], err_msg=k)
