"""CPU-side checks: the C-ABI library loads and exports every symbol the header
declares; ctypes struct layouts match; host logic (types mirror, view
sampling, RNG stream contract, synthetic workloads) behaves like the reference."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "adps.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"ADPS_API\s+[\w\s\*]+?\b(adps_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2605_06876_b200 import _abi
    lib = _abi.load()
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_abi.EXPORTS)
    assert lib.adps_abi_version() == _abi.ABI_VERSION == 3


def test_struct_layouts():
    from paper_2605_06876_b200 import _abi
    assert C.sizeof(_abi.Gaussians) == 6 * 8 + 8
    assert C.sizeof(_abi.Config) == 8 + 6 * 4 + 6 * 8
    assert C.sizeof(_abi.Counts) == 13 * 8 + 8
    assert _abi.Config.gamma_d.offset == 32


def test_no_gpu_operator_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2605_06876_b200 import operator as op
    with pytest.raises(RuntimeError, match="CUDA"):
        op.Plan()


def test_types_mirror_reference_validation():
    from paper_2605_06876_b200 import types as T
    with pytest.raises(T.InvariantError):
        T.Gaussian3D(mu=[0, 0, 0], scale=[0.1, 0.1, 0.1], rot=[1, 0, 0, 0.1], opacity=0.5, sh_dc=[0, 0, 0])
    with pytest.raises(T.InvariantError):
        T.Gaussian3D(mu=[0, 0, 0], scale=[0.1, 0.0, 0.1], rot=[1, 0, 0, 0], opacity=0.5, sh_dc=[0, 0, 0])
    with pytest.raises(T.InvariantError):
        T.AdpSplitConfig(tau_l1=1.0)
    with pytest.raises(KeyError):
        T.AdpSplitConfig().with_overrides({"nope": 1})
    cfg = T.AdpSplitConfig()
    assert (cfg.tau_l1, cfg.r_erode, cfg.m_min, cfg.l_bands, cfg.n_max, cfg.v_views) == (0.1, 2, 5, 3, 19, 20)
    s = T.DensifyStats(np.array([1.0, 2.0]), np.array([0.0, 4.0]))
    assert s.g().tolist() == [0.0, 0.5]


def test_view_sampling_matches_reference_rng_use():
    from oracle import adpsplit_oracle as O
    from paper_2605_06876_b200.operator import sample_views
    a = sample_views(20, 6, np.random.default_rng(3))
    b = O.sample_views(20, 6, np.random.default_rng(3))
    c = sorted(np.random.default_rng(3).choice(20, size=6, replace=False))
    assert a == b == [int(x) for x in c]
    with pytest.raises(ValueError):
        sample_views(2, 5, np.random.default_rng(0))


def test_fallback_normals_are_chunk_invariant():
    """Drawing 6F normals at once == 3 per child in candidate order (ref/adc.py:97)."""
    r1, r2 = np.random.default_rng(11), np.random.default_rng(11)
    a = r1.standard_normal(6 * 5)
    b = np.concatenate([r2.standard_normal(3) for _ in range(10)])
    np.testing.assert_array_equal(a, b)


def test_synthetic_workload_counts():
    from paper_2605_06876_b200 import synth as S
    import dataclasses
    ini, cams, (ga, den), gt = dataclasses.replace(S.CONFIGS["config2"], stats_mode="uniform").build()
    assert ini.n == S.CONFIGS["config2"].n_gt // 2 + 1 and cams.shape == (16, 18)
    split = (ga / den >= 2e-4) & (ini.scale.max(1) > 0.01 * ini.extent)
    assert abs(split.sum() - S.CONFIGS["config2"].p_split * ini.n) < 2
    # the dominance-weighted draw: p_S * N candidates, the heavy ones first
    w = np.zeros(ini.n)
    large = np.flatnonzero(ini.scale.max(1) > 0.01 * ini.extent)
    w[large[: len(large) // 10]] = 1000.0
    ga2, den2 = S.synth_stats_weighted(ini.scale, ini.extent, 2e-4, 0.01, 0.01, 0.02, w, 0.0, 0)
    split2 = np.flatnonzero((ga2 / den2 >= 2e-4) & (ini.scale.max(1) > 0.01 * ini.extent))
    assert abs(len(split2) - 0.01 * ini.n) < 2
    assert set(split2) <= set(large[: len(large) // 10]) or len(split2) > len(large) // 10
    # fp32-representable parameters
    assert np.array_equal(ini.mu, ini.mu.astype(np.float32).astype(np.float64))


def test_c_render_matches_numpy_oracle():
    import golden_io
    from oracle import adpsplit_oracle as O
    from oracle import c_render
    c_render.build()
    data, _ = golden_io.load()
    for c in range(12):
        g, _ = golden_io.scene(data, f"render__{c}__scene")
        cam = data[f"render__{c}__cam"][0]
        img, dom = c_render.render(g, cam)
        img_o, dom_o = O.render(g, O.Cam.from_row(cam))
        assert np.abs(img - img_o).max() < 1e-12
        np.testing.assert_array_equal(dom, dom_o)
