"""GPU parity: the CUDA operator (through the C ABI) vs the CPU oracle.

Run on a B200:  python -m pytest tests -m gpu -q
"""

import numpy as np
import pytest

import golden_io
import parity as PA
from oracle import adpsplit_oracle as O

pytestmark = pytest.mark.gpu

DATA, META = golden_io.load()
STEP_TAGS = sorted(META["step"])


@pytest.fixture(scope="module")
def op():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2605_06876_b200 import operator
    return operator


@pytest.fixture(scope="module")
def plan(op):
    p = op.Plan("cuda:0")
    p.set_debug_records(True)
    return p


def _golden_step_inputs(tag):
    g, extent = golden_io.scene(DATA, f"step__{tag}__in")
    g = PA.oracle_gaussians_f32(g)
    cams = golden_io.cams(DATA, f"step__{tag}__cams")
    rows = DATA[f"step__{tag}__cams"]
    gts = PA.f32(DATA[f"step__{tag}__gt"])
    m = META["step"][tag]
    return g, extent, cams, rows, gts, golden_io.Cfg(m["cfg"]), m["seed"]


# --------------------------------------------------------------------- render
@pytest.mark.parametrize("c", range(12))
def test_render_matches_oracle(op, plan, c):
    g, _ = golden_io.scene(DATA, f"render__{c}__scene")
    g = PA.oracle_gaussians_f32(g)
    cam = golden_io.cams(DATA, f"render__{c}__cam")[0]
    img_o, dom_o, best, second = O.render(g, cam, with_weights=True)
    t = PA.to_tensors(g)
    img, dom = plan.render(t, DATA[f"render__{c}__cam"])
    img = img[0].double().cpu().numpy()
    dom = dom[0].long().cpu().numpy()
    assert np.abs(img - img_o).max() < 2e-5
    tie = (best - second) <= PA.EPS_TIE * np.maximum(best, 1e-30)
    assert not ((dom != dom_o) & ~tie).any()


def test_render_empty_and_behind_camera(op, plan):
    g = O.Gaussians([[0, 0, -10.0]], [[0.1] * 3], [[1, 0, 0, 0]], [0.5], [[0, 0, 0]])
    cam = O.Cam(np.eye(3), np.array([0, 0, -3.0]), 20.0, 20.0, 7.5, 7.5, 16, 16)
    img, dom = plan.render(PA.to_tensors(g), cam.row()[None], bg=(0.1, 0.2, 0.3))
    assert (dom.cpu().numpy() == -1).all()
    np.testing.assert_allclose(img[0, 0, 0].cpu().numpy(), [0.1, 0.2, 0.3], rtol=1e-6)


# ----------------------------------------------------------------------- maps
@pytest.mark.parametrize("c", range(24))
def test_maps_bit_exact(op, plan, c):
    """Eroded metric map and bands equal compute_maps on identical fp32 inputs."""
    import torch
    cfg = dict(META["maps"][c])
    rendered = PA.f32(DATA[f"maps__{c}__rendered"])
    gt = PA.f32(DATA[f"maps__{c}__gt"])
    h, w = rendered.shape[:2]
    want = O.compute_maps(rendered, gt, cfg)
    g = O.Gaussians([[0, 0, 0.0]], [[0.1] * 3], [[1, 0, 0, 0]], [0.5], [[0, 0, 0]])
    cam = O.Cam(np.eye(3), np.array([0, 0, -3.0]), 20.0, 20.0, (w - 1) / 2, (h - 1) / 2, w, h)
    full = dict(tau_l1=0.1, r_erode=2, m_min=5, l_bands=3, n_max=19, v_views=1, gamma_d=2.0,
                gamma_c=0.15, tau_g=2e-4, tau_s=0.01, eta=1.6, eps=1e-9)
    full.update(cfg)
    m = torch.zeros(1, h, w, dtype=torch.uint8, device="cuda")
    b = torch.zeros(1, h, w, dtype=torch.uint8, device="cuda")
    plan.set_debug_maps(m, b)
    try:
        dev = "cuda"
        img = torch.as_tensor(rendered[None], dtype=torch.float32, device=dev)
        gtt = torch.as_tensor(gt[None], dtype=torch.float32, device=dev)
        dom = torch.full((1, h, w), -1, dtype=torch.int32, device=dev)
        plan.phase1(PA.to_tensors(g), 1.0, torch.zeros(1, dtype=torch.float64, device=dev),
                    torch.ones(1, dtype=torch.float64, device=dev), full, cam.row()[None], img, gtt, dom)
    finally:
        plan.set_debug_maps(None, None)
    np.testing.assert_array_equal(m[0].cpu().numpy().astype(bool), want.m)
    np.testing.assert_array_equal(b[0].cpu().numpy().astype(np.int64), want.b)


# ------------------------------------------------------------------ partition
def _injected_partition(op, plan, e, dom, n_gauss, l_bands, m_min, cands, tau=0.1, r_erode=1, deferred=None,
                        e2=None):
    """Run phase 1 with error map e injected exactly (raw = e, lo = 0, hi = 1;
    raw = e + e2 in fp64 when a second channel e2 is given).

    Both CCL paths run (block kernel for every tile, then the warp kernel with
    its deferred tiles) and must agree bit for bit; returns (warp path, oracle)."""
    import torch
    h, w = e.shape
    e = e.astype(np.float32)
    e.flat[0], e.flat[-1] = 0.0, 1.0
    rendered = np.zeros((h, w, 3), np.float32)
    rendered[..., 0] = e
    if e2 is not None:
        e2 = e2.astype(np.float32)
        e2.flat[0], e2.flat[-1] = 0.0, 0.0
        rendered[..., 1] = e2
    gt = np.zeros((h, w, 3), np.float32)
    rng = np.random.default_rng(0)
    g = O.Gaussians(rng.uniform(-0.2, 0.2, (n_gauss, 3)), np.full((n_gauss, 3), 0.3),
                    np.tile([1.0, 0, 0, 0], (n_gauss, 1)), np.full(n_gauss, 0.5), np.zeros((n_gauss, 3)))
    cam = O.Cam(np.eye(3), np.array([0, 0, -3.0]), 1.2 * w, 1.2 * w, (w - 1) / 2, (h - 1) / 2, w, h)
    ga = np.full(n_gauss, 1e-6)
    ga[cands] = 1.0
    cfg = dict(tau_l1=tau, r_erode=r_erode, m_min=m_min, l_bands=l_bands, n_max=19, v_views=1, gamma_d=2.0,
               gamma_c=0.15, tau_g=2e-4, tau_s=0.01, eta=1.6, eps=1e-9)
    dev = "cuda"
    got_by_path = []
    # block CCL; warp CCL recomputing / caching the raw error; bit-plane warp CCL (l_bands <= 4),
    # fused and with the separate words pass
    for path, raw in ((1, 1), (0, 0), (2, 1), (0, 1), (3, 1)):
        plan.set_tile_path(path)
        plan.set_raw_cache(raw)
        try:
            plan.phase1(PA.to_tensors(g), 1.0, torch.as_tensor(ga, device=dev),
                        torch.ones(n_gauss, dtype=torch.float64, device=dev), cfg, cam.row()[None],
                        torch.as_tensor(rendered[None], device=dev), torch.as_tensor(gt[None], device=dev),
                        torch.as_tensor(dom[None].astype(np.int32), device=dev))
        finally:
            plan.set_tile_path(0)
            plan.set_raw_cache(1)
        got_by_path.append(PA.gpu_regions(plan))
        if path == 0 and deferred is not None:
            assert (plan.deferred_tiles() > 0) == deferred, plan.deferred_tiles()
    np.testing.assert_array_equal(got_by_path[1], got_by_path[0], err_msg="warp CCL != block CCL")
    np.testing.assert_array_equal(got_by_path[2], got_by_path[0], err_msg="cached-raw warp CCL != block CCL")
    np.testing.assert_array_equal(got_by_path[3], got_by_path[0], err_msg="bit-plane warp CCL != block CCL")
    np.testing.assert_array_equal(got_by_path[4], got_by_path[0], err_msg="words-pass warp CCL != block CCL")
    got = got_by_path[3]
    maps = O.compute_maps(rendered.astype(np.float64), gt.astype(np.float64), cfg)
    is_c = np.zeros(n_gauss, bool)
    is_c[cands] = True
    regs = O.partition(maps, dom, is_c, m_min, view=0)
    fake = O.StepResult(None, 0, 0, None, [], [], [], [0], 0, regions={0: regs})
    want = PA.oracle_regions(fake, [0])
    return got, want


@pytest.mark.parametrize("seed", range(8))
def test_partition_random_blocky(op, plan, seed):
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(40, 140)), int(rng.integers(40, 140))
    n = 6
    dom = np.kron(rng.integers(-1, n, (h // 3 + 1, w // 3 + 1)), np.ones((3, 3), np.int64))[:h, :w]
    e = rng.uniform(0, 1, (h, w))
    e[rng.uniform(size=(h, w)) < 0.3] = 0.05
    got, want = _injected_partition(op, plan, e, dom, n, int(rng.integers(1, 4)), int(rng.integers(1, 5)),
                                    [0, 2, 3, 5])
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("shape", [(64, 64), (97, 131), (33, 33), (1, 200), (200, 1)])
def test_partition_snakes_cross_tiles(op, plan, shape):
    """Long thin components crossing many 32x32 tile borders (8-connectivity)."""
    h, w = shape
    e = np.full((h, w), 0.9)
    dom = np.full((h, w), 1, np.int64)
    yy, xx = np.mgrid[0:h, 0:w]
    dom[(xx + yy) % 7 == 0] = 0          # diagonal stripes of another candidate
    dom[(xx * 3 + yy) % 11 == 0] = -1
    got, want = _injected_partition(op, plan, e, dom, 2, 1, 1, [0, 1])
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("l_bands", [1, 3, 6])
@pytest.mark.parametrize("r_erode", [1, 2, 3, 4])
@pytest.mark.parametrize("seed", range(3))
def test_partition_erosion_both_paths(op, plan, seed, r_erode, l_bands):
    """Warp CCL (r <= 3: erosion masks with halo columns; L <= 4 and the general
    band loop) vs block CCL (r = 4) vs oracle."""
    rng = np.random.default_rng(100 + seed)
    h, w = int(rng.integers(30, 170)), int(rng.integers(30, 170))
    n = 5
    dom = np.kron(rng.integers(-1, n, (h // 4 + 1, w // 4 + 1)), np.ones((4, 4), np.int64))[:h, :w]
    e = np.kron(rng.uniform(0, 1, (h // 2 + 1, w // 2 + 1)), np.ones((2, 2)))[:h, :w]
    e[rng.uniform(size=(h, w)) < 0.05] = 0.01
    got, want = _injected_partition(op, plan, e, dom, n, l_bands, int(rng.integers(1, 4)),
                                    [0, 1, 3, 4], r_erode=r_erode)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("seed", range(3))
def test_partition_fp32_cache_near_thresholds(op, plan, seed):
    """Raw errors within one fp32 ulp of the metric threshold and a band edge:
    the bit-plane path's fp32 (round-toward-zero) raw cache cannot decide those
    compares and must redo them exactly in fp64 (same bits as the block CCL)."""
    rng = np.random.default_rng(300 + seed)
    h, w = 70, 90
    dom = np.kron(rng.integers(-1, 4, (h // 2 + 1, w // 2 + 1)), np.ones((2, 2), np.int64))[:h, :w]
    base = np.where(rng.uniform(size=(h, w)) < 0.5, np.float32(0.099999994), np.float32(0.39999998))
    e = base.astype(np.float32)
    e2 = rng.uniform(0.0, 4e-8, (h, w)).astype(np.float32)   # raw = e + e2 straddles the thresholds
    got, want = _injected_partition(op, plan, e, dom, 4, 3, 1, [0, 1, 2], e2=e2)
    np.testing.assert_array_equal(got, want)
    assert len(want) > 0


@pytest.mark.parametrize("shape", [(64, 64), (70, 45)])
def test_partition_deferred_tiles(op, plan, shape):
    """Tiles with more than 256 runs (alternating candidates) go to the block CCL."""
    h, w = shape
    yy, xx = np.mgrid[0:h, 0:w]
    dom = ((xx + (yy // 2)) % 2).astype(np.int64)     # runs of length 1, diagonal links
    dom[:, w // 2:] = 0                              # right half: one big component
    e = np.full((h, w), 0.9)
    got, want = _injected_partition(op, plan, e, dom, 2, 1, 1, [0, 1], deferred=True)
    np.testing.assert_array_equal(got, want)


def test_partition_spiral(op, plan):
    n = 150
    e = np.full((n, n), 0.02)
    dom = np.zeros((n, n), np.int64)
    x, y, dx, dy = 0, 0, 1, 0
    lo_x, hi_x, lo_y, hi_y = 0, n - 1, 2, n - 1
    for _ in range(n * n):
        e[y, x] = 0.8
        nx, ny = x + dx, y + dy
        if not (lo_x <= nx <= hi_x and lo_y - 2 <= ny <= hi_y):
            if dx == 1: hi_x -= 2
            elif dy == 1: hi_y -= 2
            elif dx == -1: lo_x += 2
            else: lo_y += 2
            dx, dy = -dy, dx
            nx, ny = x + dx, y + dy
            if not (0 <= nx < n and 0 <= ny < n) or hi_x < lo_x:
                break
        x, y = nx, ny
    got, want = _injected_partition(op, plan, e, dom, 1, 2, 2, [0])
    np.testing.assert_array_equal(got, want)


# ----------------------------------------------------------------------- step
@pytest.mark.parametrize("tag", STEP_TAGS)
def test_step_stage_isolated(op, plan, tag):
    """Same (image, dominant) into both: integers exact, floats within tolerance."""
    import torch
    g, extent, cams, rows, gts, cfg, seed = _golden_step_inputs(tag)
    views = O.sample_views(len(cams), cfg.v_views, np.random.default_rng(seed))
    img, dom = plan.render(PA.to_tensors(g), rows[views])
    renders_np = {v: (img[k].double().cpu().numpy(), dom[k].long().cpu().numpy()) for k, v in enumerate(views)}
    gres = op.densify_step(PA.to_tensors(g), extent, rows, torch.as_tensor(gts, dtype=torch.float32, device="cuda"),
                           torch.as_tensor(DATA[f"step__{tag}__grad_accum"], device="cuda"),
                           torch.as_tensor(DATA[f"step__{tag}__denom"], device="cuda"), cfg,
                           np.random.default_rng(seed), renders=(img, dom), plan=plan)
    ores = O.adpsplit_step(g, extent, cams, gts, DATA[f"step__{tag}__grad_accum"],
                           DATA[f"step__{tag}__denom"], cfg, np.random.default_rng(seed), renders=renders_np)
    np.testing.assert_array_equal(PA.gpu_regions(plan), PA.oracle_regions(ores, views))
    flagged = PA.flag_candidates(ores, g, cams, cfg)
    st = PA.compare_step(gres, ores, flagged, g)
    assert st["mismatched"] == 0


@pytest.mark.parametrize("tag", STEP_TAGS)
def test_step_end_to_end(op, plan, tag):
    """GPU render + step vs the oracle's fp64 render + step, near-threshold classes excluded."""
    import torch
    g, extent, cams, rows, gts, cfg, seed = _golden_step_inputs(tag)
    gres = op.densify_step(PA.to_tensors(g), extent, rows, torch.as_tensor(gts, dtype=torch.float32, device="cuda"),
                           torch.as_tensor(DATA[f"step__{tag}__grad_accum"], device="cuda"),
                           torch.as_tensor(DATA[f"step__{tag}__denom"], device="cuda"), cfg,
                           np.random.default_rng(seed), plan=plan)
    views = gres.view_ids
    weights, renders_o = {}, {}
    for v in views:
        img_o, dom_o, best, second = O.render(g, cams[v], with_weights=True)
        weights[v] = (best, second)
        renders_o[v] = (img_o, dom_o)
    ores = O.adpsplit_step(g, extent, cams, gts, DATA[f"step__{tag}__grad_accum"],
                           DATA[f"step__{tag}__denom"], cfg, np.random.default_rng(seed), renders=renders_o)
    img, dom = plan.render(PA.to_tensors(g), rows[views])
    gpu_r = {v: (img[k].double().cpu().numpy(), dom[k].long().cpu().numpy()) for k, v in enumerate(views)}
    assert PA.unexplained_dominance(ores, gpu_r, weights) == 0
    flagged = PA.flag_candidates(ores, g, cams, cfg) | PA.flag_end_to_end(ores, gpu_r, gts, cfg, weights)
    PA.compare_step(gres, ores, flagged, g)


def test_reference_api_drop_in(op):
    """adpsplit_step(scene, cameras, gt_images, stats, cfg, rng) with the mirror types."""
    from paper_2605_06876_b200 import types as T
    tag = "blobs"
    g, extent = golden_io.scene(DATA, f"step__{tag}__in")
    cams = [T.Camera(r_c2w=r[:9].reshape(3, 3), center=r[9:12], f_x=r[12], f_y=r[13], p_x=r[14], p_y=r[15],
                     width=int(r[16]), height=int(r[17])) for r in DATA[f"step__{tag}__cams"]]
    gs = [T.Gaussian3D(mu=g.mu[i], scale=g.scale[i], rot=g.rot[i], opacity=g.opacity[i], sh_dc=g.sh_dc[i])
          for i in range(len(g))]
    scene = T.Scene(gaussians=list(gs), extent=extent)
    m = META["step"][tag]
    cfg = T.AdpSplitConfig(**{k: v for k, v in m["cfg"].items()})
    stats = T.DensifyStats(DATA[f"step__{tag}__grad_accum"].copy(), DATA[f"step__{tag}__denom"].copy())
    scene, rep = op.adpsplit_step(scene, cams, list(DATA[f"step__{tag}__gt"]), stats, cfg,
                                  np.random.default_rng(m["seed"]))
    want = m["report"]
    assert rep.count_after == want["count_after"] == len(scene.gaussians)
    assert rep.clones == want["clones"] and rep.sampled_views == want["sampled_views"]
    assert [(r.index, r.fallback, r.reset, r.children_inserted) for r in rep.candidates] == \
        [(r["index"], r["fallback"], r["reset"], r["children_inserted"]) for r in want["candidates"]]
    for new_i, old_i in enumerate(rep.index_map):
        if old_i >= 0:
            assert scene.gaussians[new_i] is gs[old_i]
    with pytest.raises(ValueError):
        op.adpsplit_step(T.Scene(gaussians=list(gs), extent=extent), cams[:2], [], stats,
                         cfg.with_overrides({"v_views": 5}), np.random.default_rng(0))


# ------------------------------------------------------------ larger sizes
def test_select_and_scans_large(op, plan):
    """Split/clone lists and offsets over millions of Gaussians (multi-tile scans)."""
    import torch
    n = 3_000_001
    rng = np.random.default_rng(7)
    scale = rng.uniform(0.001, 0.03, (n, 3)).astype(np.float32)
    ga = rng.uniform(0, 4e-4, n)
    den = np.where(rng.uniform(size=n) < 0.1, 0.0, rng.integers(1, 3, n).astype(np.float64))
    g = O.Gaussians(rng.uniform(-1, 1, (n, 3)), scale, np.tile([1.0, 0, 0, 0], (n, 1)), np.full(n, 0.5),
                    np.zeros((n, 3)))
    w = h = 8
    cam = O.Cam(np.eye(3), np.array([0, 0, -3.0]), 10.0, 10.0, 3.5, 3.5, w, h)
    cfg = dict(tau_l1=0.1, r_erode=2, m_min=5, l_bands=3, n_max=19, v_views=1, gamma_d=2.0, gamma_c=0.15,
               tau_g=2e-4, tau_s=0.01, eta=1.6, eps=1e-9)
    dev = "cuda"
    z = torch.zeros(1, h, w, 3, dtype=torch.float32, device=dev)
    counts = plan.phase1(PA.to_tensors(g), 1.0, torch.as_tensor(ga, device=dev), torch.as_tensor(den, device=dev),
                         cfg, cam.row()[None], z, z, torch.full((1, h, w), -1, dtype=torch.int32, device=dev))
    split, clone = O.select(ga, den, scale.astype(np.float64), 2e-4, 0.01)
    ra = plan.report_arrays(counts["n_split"], counts["n_clone"])
    np.testing.assert_array_equal(ra["cand_index"].cpu().numpy(), split)
    np.testing.assert_array_equal(ra["clone_index"].cpu().numpy(), clone)
    assert (ra["cand_case"].cpu().numpy() == 1).all()      # nothing dominant -> all fallback
    assert counts["n_keep"] == n - len(split)
    assert counts["n_out"] == n - len(split) + 2 * len(split) + len(clone)


def test_render_medium_vs_c_oracle(op, plan):
    """20k Gaussians, non-multiple-of-16 image: GPU render vs the C restatement."""
    from oracle import c_render
    from paper_2605_06876_b200 import synth as S
    wl = S.Workload("t", 40_000, 2, 210, 150, 0.05, 0.02, 0.02 * np.sqrt(2.4e6 / 4e4),
                    large_range=(0.005 * np.sqrt(60), 0.01 * np.sqrt(60)))
    ini, cams, _, _ = wl.build(seed=3)
    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    img, dom = plan.render(PA.to_tensors(g), cams)
    for v in range(len(cams)):
        io, do = c_render.render(g, cams[v])
        ig = img[v].double().cpu().numpy()
        dg = dom[v].long().cpu().numpy()
        assert np.abs(ig - io).max() < 1e-4
        assert (dg != do).mean() < 1e-3      # near-ties only (fp32 vs fp64 weights)


@pytest.mark.parametrize("seed", [0, 1])
def test_synthetic_step_stage_isolated(op, plan, seed):
    """Paper-default cfg on a 8k-Gaussian synthetic scene, 3 of 5 views, 160x112 px."""
    import torch
    from paper_2605_06876_b200 import synth as S
    sf = np.sqrt(2.4e6 / 16000)
    wl = S.Workload("t", 16_000, 5, 160, 112, 0.2, 0.05, 0.02 * sf, large_range=(0.005 * sf, 0.01 * sf))
    ini, cams, (ga, den), gts = wl.build(seed=seed)
    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    gt_g = O.Gaussians(gts.mu, gts.scale, gts.rot, gts.opacity, gts.sh_dc)
    gt_img, _ = plan.render(PA.to_tensors(gt_g), cams)
    cfg = golden_io.Cfg(dict(tau_l1=0.1, r_erode=2, m_min=5, l_bands=3, n_max=19, v_views=3, gamma_d=2.0,
                             gamma_c=0.15, tau_g=2e-4, tau_s=0.01, eta=1.6, eps=1e-9))
    views = O.sample_views(len(cams), 3, np.random.default_rng(seed))
    img, dom = plan.render(PA.to_tensors(g), cams[views])
    gres = op.densify_step(PA.to_tensors(g), ini.extent, cams, gt_img, torch.as_tensor(ga, device="cuda"),
                           torch.as_tensor(den, device="cuda"), cfg, np.random.default_rng(seed),
                           renders=(img, dom), plan=plan)
    gts_np = {v: gt_img[v].double().cpu().numpy() for v in range(len(cams))}
    renders_np = {v: (img[k].double().cpu().numpy(), dom[k].long().cpu().numpy()) for k, v in enumerate(views)}
    cam_objs = [O.Cam.from_row(r) for r in cams]
    ores = O.adpsplit_step(g, ini.extent, cam_objs, gts_np, ga, den, cfg, np.random.default_rng(seed),
                           renders=renders_np)
    np.testing.assert_array_equal(PA.gpu_regions(plan), PA.oracle_regions(ores, views))
    flagged = PA.flag_candidates(ores, g, cam_objs, cfg)
    st = PA.compare_step(gres, ores, flagged, g)
    assert st["mismatched"] == 0
    assert gres.counts["n_regions"] > 50 and gres.counts["n_children"] > 20


@pytest.mark.parametrize("tag", ["paper0", "paper2", "desk3", "blobs"])
def test_large_merge_path_matches_warp_path(op, plan, tag):
    """Routing every parent through the grid-wide pair-tile merge gives the oracle's result."""
    import torch
    g, extent, cams, rows, gts, cfg, seed = _golden_step_inputs(tag)
    views = O.sample_views(len(cams), cfg.v_views, np.random.default_rng(seed))
    img, dom = plan.render(PA.to_tensors(g), rows[views])
    renders_np = {v: (img[k].double().cpu().numpy(), dom[k].long().cpu().numpy()) for k, v in enumerate(views)}
    plan.set_large_threshold(0)
    try:
        gres = op.densify_step(PA.to_tensors(g), extent, rows, torch.as_tensor(gts, dtype=torch.float32,
                               device="cuda"), torch.as_tensor(DATA[f"step__{tag}__grad_accum"], device="cuda"),
                               torch.as_tensor(DATA[f"step__{tag}__denom"], device="cuda"), cfg,
                               np.random.default_rng(seed), renders=(img, dom), plan=plan)
    finally:
        plan.set_large_threshold(32)
    ores = O.adpsplit_step(g, extent, cams, gts, DATA[f"step__{tag}__grad_accum"],
                           DATA[f"step__{tag}__denom"], cfg, np.random.default_rng(seed), renders=renders_np)
    st = PA.compare_step(gres, ores, PA.flag_candidates(ores, g, cams, cfg), g)
    assert st["mismatched"] == 0


def test_large_merge_path_synthetic(op, plan):
    """A parent with hundreds of proposals (multi-tile gate matrix) vs the oracle."""
    import torch
    from paper_2605_06876_b200 import synth as S
    sf = np.sqrt(2.4e6 / 16000)
    wl = S.Workload("t", 16_000, 6, 192, 128, 0.3, 0.05, 0.02 * sf, large_range=(0.005 * sf, 0.01 * sf))
    ini, cams, (ga, den), gts = wl.build(seed=5)
    ga[-1] = 1.0                      # the cover Gaussian: many regions in every view
    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    gt_g = O.Gaussians(gts.mu, gts.scale, gts.rot, gts.opacity, gts.sh_dc)
    gt_img, _ = plan.render(PA.to_tensors(gt_g), cams)
    cfg = golden_io.Cfg(dict(tau_l1=0.1, r_erode=1, m_min=2, l_bands=3, n_max=19, v_views=6, gamma_d=2.0,
                             gamma_c=0.15, tau_g=2e-4, tau_s=0.01, eta=1.6, eps=1e-9))
    views = list(range(6))
    img, dom = plan.render(PA.to_tensors(g), cams)
    plan.set_large_threshold(16)
    try:
        gres = op.densify_step(PA.to_tensors(g), ini.extent, cams, gt_img, torch.as_tensor(ga, device="cuda"),
                               torch.as_tensor(den, device="cuda"), cfg, np.random.default_rng(1),
                               renders=(img, dom), plan=plan)
    finally:
        plan.set_large_threshold(32)
    props = gres.report_arrays["cand_proposals"].cpu().numpy()
    assert props.max() > 64 and (props > 16).sum() >= 3, (props.max(), (props > 16).sum())
    gts_np = {v: gt_img[v].double().cpu().numpy() for v in views}
    renders_np = {v: (img[v].double().cpu().numpy(), dom[v].long().cpu().numpy()) for v in views}
    cam_objs = [O.Cam.from_row(r) for r in cams]
    ores = O.adpsplit_step(g, ini.extent, cam_objs, gts_np, ga, den, cfg, np.random.default_rng(1),
                           renders=renders_np)
    st = PA.compare_step(gres, ores, PA.flag_candidates(ores, g, cam_objs, cfg), g)
    assert st["mismatched"] == 0


def _step_digest(op, plan, res):
    r = plan.regions()
    d = {}
    order = np.lexsort((r["minpix"].cpu().numpy(), r["band"].cpu().numpy(), r["view_pos"].cpu().numpy(),
                        r["candidate"].cpu().numpy()))
    for k in ("candidate", "view_pos", "band", "minpix", "moments", "valid"):
        d[f"reg_{k}"] = r[k].cpu().numpy()[order]
    d.update({k: res.report_arrays[k].cpu().numpy() for k in res.report_arrays})
    d.update({f"out_{k}": v for k, v in res.gaussians.numpy().items()})
    d["index_map"] = res.index_map.cpu().numpy()
    return d


@pytest.mark.parametrize("cfg_name", ["config2"])
def test_determinism_at_scale(op, cfg_name):
    """Two runs of the same step are bitwise identical at BASELINE size."""
    import torch
    from paper_2605_06876_b200 import synth as S
    from paper_2605_06876_b200.types import AdpSplitConfig
    wl = S.CONFIGS[cfg_name]
    plan = op.Plan("cuda:0")
    d = wl.build_device(plan)
    ini, cams, (ga, den) = d["ini"], d["cams"], d["stats"]
    g, gt_img, img, dom = d["g"], d["gt_img"], d["img"], d["dom"]
    cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
    digests = []
    # block CCL / recomputed raw / no bit planes / words pass / phase 2 as its own call: same bits
    for path, raw, one_sync in ((0, 1, True), (0, 1, True), (1, 1, True), (0, 0, True), (2, 1, True),
                                (3, 1, True), (0, 1, False)):
        plan.set_tile_path(path)
        plan.set_raw_cache(raw)
        res = op.densify_step(g, ini.extent, cams, gt_img, torch.as_tensor(ga, device="cuda"),
                              torch.as_tensor(den, device="cuda"), cfg, np.random.default_rng(0),
                              renders=(img, dom), plan=plan, view_ids=list(range(len(cams))), one_sync=one_sync)
        digests.append((res.counts, _step_digest(op, plan, res)))
    plan.set_tile_path(0)
    plan.set_raw_cache(1)
    for counts, dg in digests[1:]:
        assert counts == digests[0][0]
        for k in dg:
            np.testing.assert_array_equal(dg[k], digests[0][1][k], err_msg=k)
    # population accounting and index_map structure
    c = digests[0][0]
    rep = res.report()
    assert c["n_out"] == c["n_keep"] + c["n_inserted"] + c["n_clone"]
    kept = rep.index_map[rep.index_map >= 0]
    assert (np.diff(kept) > 0).all() and len(kept) == c["n_keep"]
    assert all(r.children_inserted <= wl.n_max for r in rep.candidates)


@pytest.mark.parametrize("parent_shard", [True, False])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lockstep_matches_single_gpu(op, world, parent_shard):
    """The view-sharded C-ABI flow (phase1_begin on each rank's views, flag
    reduction, refresh, local records, import of the concatenation, merge)
    gives the single-plan result bit for bit -- all ranks run in one process
    (sharded.run_lockstep) since the test box has one GPU."""
    import torch
    from paper_2605_06876_b200 import sharded as SH
    from paper_2605_06876_b200 import synth as S
    from paper_2605_06876_b200.types import AdpSplitConfig
    wl = S.CONFIGS["config2"]
    base = op.Plan("cuda:0")
    d = wl.build_device(base)
    ini, cams, (ga, den) = d["ini"], d["cams"], d["stats"]
    g, gt_img, img, dom = d["g"], d["gt_img"], d["img"], d["dom"]
    cfg = AdpSplitConfig(v_views=len(cams), n_max=wl.n_max)
    vids = list(range(len(cams)))
    ga_t, den_t = torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda")
    rng1 = np.random.default_rng(5)
    single = op.densify_step(g, ini.extent, cams, gt_img, ga_t, den_t, cfg, rng1, renders=(img, dom), plan=base,
                             view_ids=vids)
    want = _step_digest(op, base, single)
    exs = [SH.GpuExecutor(g, ini.extent, cams, gt_img, ga_t, den_t, cfg, np.random.default_rng(5),
                          renders=(img, dom), plan=op.Plan("cuda:0"), view_ids=vids, world=world, rank=r,
                          parent_shard=parent_shard)
           for r in range(world)]
    results = SH.run_lockstep(exs, len(vids))
    assert single.counts["n_fallback"] > 0
    for r, (ex, res) in enumerate(zip(exs, results)):
        drop = ("n_partials",)   # tile-border fragments: a per-rank diagnostic
        assert {k: v for k, v in res.counts.items() if k not in drop} == \
            {k: v for k, v in single.counts.items() if k not in drop}, r
        got = _step_digest(op, ex.plan, res)
        for k in want:
            np.testing.assert_array_equal(got[k], want[k], err_msg=f"rank {r}: {k}")
        assert ex.rng.bit_generator.state == rng1.bit_generator.state


# ------------------------------------------------- next rows: vanilla ADC, remaps
@pytest.mark.parametrize("n_children", [2, 3])
@pytest.mark.parametrize("tag", ["blobs", "desk0", "paper1"])
def test_vanilla_densify_matches_oracle(op, tag, n_children):
    """vanilla_densify (ref/adc.py:248-280) on the device vs the oracle: layout,
    index_map and clones exact; children within float tolerance; the Generator
    advanced exactly as numpy's."""
    import torch
    g, extent, cams, rows, gts, cfg, seed = _golden_step_inputs(tag)
    ga, den = DATA[f"step__{tag}__grad_accum"], DATA[f"step__{tag}__denom"]
    plan = op.Plan("cuda:0")
    rng_g, rng_o = np.random.default_rng(seed), np.random.default_rng(seed)
    res = op.vanilla_densify_step(PA.to_tensors(g), extent, torch.as_tensor(ga, device="cuda"),
                                  torch.as_tensor(den, device="cuda"), cfg, n_children, rng_g, plan=plan)
    want = O.vanilla_densify(g, extent, ga, den, cfg, n_children, rng_o)
    assert res.counts["n_out"] == want.count_after
    np.testing.assert_array_equal(res.index_map.cpu().numpy(), want.index_map)
    got = res.gaussians.numpy()
    w = PA.oracle_gaussians_f32(want.gaussians)
    np.testing.assert_allclose(got["mu"], w.mu, rtol=2e-6, atol=1e-7)
    np.testing.assert_allclose(got["scale"], w.scale, rtol=2e-6)
    np.testing.assert_array_equal(got["opacity"], w.opacity.astype(np.float32))
    rep = res.report()
    assert [c.index for c in rep.candidates] == [c.index for c in want.candidates]
    assert rep.clones == want.clones
    assert rng_g.bit_generator.state == rng_o.bit_generator.state


@pytest.mark.parametrize("tag", ["desk0", "paper1"])
def test_remap_stats_matches_oracle(op, plan, tag):
    """remap_stats (ref/adc.py:283-296) and the trainer's moment remap
    (ref/harness.py:285-295) through the step's index_map, on the device."""
    import torch
    g, extent, cams, rows, gts, cfg, seed = _golden_step_inputs(tag)
    ga, den = DATA[f"step__{tag}__grad_accum"], DATA[f"step__{tag}__denom"]
    views = O.sample_views(len(cams), cfg.v_views, np.random.default_rng(seed))
    img, dom = plan.render(PA.to_tensors(g), rows[views])
    res = op.densify_step(PA.to_tensors(g), extent, rows, torch.as_tensor(gts, dtype=torch.float32, device="cuda"),
                          torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda"), cfg,
                          np.random.default_rng(seed), renders=(img, dom), plan=plan)
    rep = res.report()
    ga2, den2 = op.remap_stats(plan, res, torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda"))
    want_g, want_d = O.remap_stats(ga, den, rep.index_map, rep.reset_indices, rep.clones)
    np.testing.assert_array_equal(ga2.cpu().numpy(), want_g)
    np.testing.assert_array_equal(den2.cpu().numpy(), want_d)
    # optimizer moments: [n, 3] rows, reset candidates zeroed, clone sources carried
    m = np.random.default_rng(1).normal(size=(len(ga), 3)).astype(np.float32)
    got = op.remap_rows(res.index_map, torch.as_tensor(m, device="cuda"), plan.reset_flags(include_clones=False))
    want = np.zeros((len(rep.index_map), 3), np.float32)
    reset = set(rep.reset_indices)
    for new_i, old_i in enumerate(rep.index_map):
        if old_i >= 0 and old_i not in reset:
            want[new_i] = m[old_i]
    np.testing.assert_array_equal(got.cpu().numpy(), want)


def test_reference_api_vanilla_and_remap(op):
    """vanilla_densify(scene, stats, cfg, n, rng) and remap_stats(stats, report)
    with the mirror types, against the oracle's restatements."""
    from paper_2605_06876_b200 import types as T
    tag = "desk3"
    g, extent = golden_io.scene(DATA, f"step__{tag}__in")
    gs = [T.Gaussian3D(mu=g.mu[i], scale=g.scale[i], rot=g.rot[i], opacity=g.opacity[i], sh_dc=g.sh_dc[i])
          for i in range(len(g))]
    scene = T.Scene(gaussians=list(gs), extent=extent)
    m = META["step"][tag]
    cfg = T.AdpSplitConfig(**{k: v for k, v in m["cfg"].items()})
    ga, den = DATA[f"step__{tag}__grad_accum"].copy(), DATA[f"step__{tag}__denom"].copy()
    stats = T.DensifyStats(ga, den)
    rng = np.random.default_rng(7)
    scene, rep = op.vanilla_densify(scene, stats, cfg, 3, rng)
    want = O.vanilla_densify(g, extent, ga, den, golden_io.Cfg(m["cfg"]), 3, np.random.default_rng(7))
    assert rep.count_after == want.count_after == len(scene.gaussians)
    np.testing.assert_array_equal(rep.index_map, want.index_map)
    assert rep.clones == want.clones
    assert all(r.fallback and r.children_inserted == 3 for r in rep.candidates)
    got = np.array([np.asarray(x.mu) for x in scene.gaussians])
    np.testing.assert_allclose(got, want.gaussians.mu, rtol=1e-6, atol=1e-6)
    st2 = op.remap_stats_ref(stats, rep)
    wg, wd = O.remap_stats(ga, den, want.index_map, [], want.clones)
    np.testing.assert_array_equal(st2.grad_accum, wg)
    np.testing.assert_array_equal(st2.denom, wd)



# ------------------------------------------------------------- degenerate steps
def _tiny_step_inputs(n, seed=0, w=9, h=7, views=2):
    rng = np.random.default_rng(seed)
    g = O.Gaussians(rng.uniform(-0.3, 0.3, (n, 3)), rng.uniform(0.05, 0.2, (n, 3)),
                    np.tile([1.0, 0, 0, 0], (n, 1)), rng.uniform(0.5, 0.9, n), rng.uniform(-1, 1, (n, 3)))
    g = PA.oracle_gaussians_f32(g)
    cams = [O.Cam(np.eye(3), np.array([0.1 * v, 0, -2.0]), 1.0 * w, 1.0 * w, (w - 1) / 2, (h - 1) / 2, w, h)
            for v in range(views)]
    gts = PA.f32(rng.uniform(0, 1, (views, h, w, 3)))
    return g, cams, gts


@pytest.mark.parametrize("case", ["empty", "no_candidates", "tiny_image", "all_split"])
def test_degenerate_steps_match_oracle(op, plan, case):
    """N = 0, no split/clone candidate, a 9x7 image, every Gaussian a candidate."""
    import torch
    n = 0 if case == "empty" else 12
    g, cams, gts = _tiny_step_inputs(n)
    rows = np.stack([c.row() for c in cams])
    ga = np.full(n, 1.0) if case == "all_split" else (np.zeros(n) if case == "no_candidates" else
                                                     np.random.default_rng(3).uniform(0, 1e-3, n))
    den = np.ones(n)
    cfg = golden_io.Cfg(dict(tau_l1=0.1, r_erode=2, m_min=1, l_bands=3, n_max=4, v_views=2, gamma_d=2.0,
                             gamma_c=0.15, tau_g=2e-4, tau_s=0.01 if case != "all_split" else 1e-9, eta=1.6,
                             eps=1e-9))
    views = O.sample_views(len(cams), cfg.v_views, np.random.default_rng(1))
    if n:
        img, dom = plan.render(PA.to_tensors(g), rows[views])
    else:
        img = torch.zeros((len(views), 7, 9, 3), device="cuda")
        dom = torch.full((len(views), 7, 9), -1, dtype=torch.int32, device="cuda")
    res = op.densify_step(PA.to_tensors(g), 1.0, rows, torch.as_tensor(gts, device="cuda"),
                          torch.as_tensor(ga, device="cuda"), torch.as_tensor(den, device="cuda"), cfg,
                          np.random.default_rng(1), renders=(img, dom), plan=plan)
    renders = {v: (img[k].double().cpu().numpy(), dom[k].long().cpu().numpy()) for k, v in enumerate(views)}
    want = O.adpsplit_step(g, 1.0, cams, gts, ga, den, cfg, np.random.default_rng(1), renders=renders)
    assert res.counts["n_out"] == want.count_after
    np.testing.assert_array_equal(res.index_map.cpu().numpy(), want.index_map)
    rep = res.report()
    assert [(c.index, c.fallback, c.reset, c.children_inserted) for c in rep.candidates] == \
        [(c.index, c.fallback, c.reset, c.children_inserted) for c in want.candidates]
    if case == "no_candidates":
        assert res.counts["n_out"] == n and res.counts["n_split"] == 0


def test_wrong_dtypes_are_rejected(op, plan):
    """Raw pointers cross the C ABI: a float64 image or int64 dominant map must raise, not be misread."""
    import torch
    g, cams, gts = _tiny_step_inputs(4)
    rows = np.stack([c.row() for c in cams])
    img = torch.zeros((1, 7, 9, 3), dtype=torch.float64, device="cuda")
    dom = torch.full((1, 7, 9), -1, dtype=torch.int32, device="cuda")
    gt = torch.zeros((1, 7, 9, 3), dtype=torch.float32, device="cuda")
    ga, den = torch.zeros(4, dtype=torch.float64, device="cuda"), torch.ones(4, dtype=torch.float64, device="cuda")
    cfg = dict(tau_l1=0.1, r_erode=2, m_min=1, l_bands=3, n_max=4, v_views=1, gamma_d=2.0, gamma_c=0.15,
               tau_g=2e-4, tau_s=0.01, eta=1.6, eps=1e-9)
    with pytest.raises(ValueError):
        plan.phase1(PA.to_tensors(g), 1.0, ga, den, cfg, rows[:1], img, gt, dom)
    with pytest.raises(ValueError):
        plan.phase1(PA.to_tensors(g), 1.0, ga, den, cfg, rows[:1], img.float(), gt, dom.long())
