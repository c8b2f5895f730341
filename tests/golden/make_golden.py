"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the reference is importable there, not on the GPU
box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``adpsplit`` from /root/reference/pkg/src (read-only), runs each
stage and whole ``adpsplit_step`` calls on small seeded inputs, and writes
``tests/golden/golden_v1.npz``.  The oracle is pinned against these vectors in
tests/test_oracle_golden.py; the GPU path is then checked against the oracle.

Case families (reference symbols, file:line under pkg/src/adpsplit):
  render    raster.render                         raster.py:136-157
  maps      error_partition.compute_maps          error_partition.py:86-91
  part      error_partition.partition+region_stats error_partition.py:94-158
  child     child_init.init_child                 child_init.py:110-140
  merge     cross_view_merge.merge_groups+cap      cross_view_merge.py:72-116
  step      adc.adpsplit_step                     adc.py:143-245
  vanilla   adc.vanilla_densify (n = 2, 3)        adc.py:248-280
  remap     adc.remap_stats after each step       adc.py:283-296
  accum     adc.accumulate_stats                  adc.py:73-79
  prune     harness._prune                        harness.py:320-340
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from adpsplit import adc, raster  # noqa: E402
from adpsplit.child_init import init_child, optimal_t, pixel_ray  # noqa: E402
from adpsplit.cross_view_merge import cap_children, merge_groups  # noqa: E402
from adpsplit.child_init import ChildProposal  # noqa: E402
from adpsplit.error_partition import (  # noqa: E402
    ErrorMaps, ErrorRegion, band_map, compute_maps, partition, region_stats)
from adpsplit import harness  # noqa: E402
from adpsplit.harness import desk_config, init_from_gt, synth_scene  # noqa: E402
from adpsplit.raster import GradOutput  # noqa: E402
from adpsplit.scene import (  # noqa: E402
    AdpSplitConfig, Camera, Gaussian3D, Scene, covariance, rgb_to_dc)

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_v1.npz")
store: dict = {}
meta: dict = {}


def put(key, arr):
    store[key] = np.asarray(arr)


def scene_arrays(scene):
    gs = scene.gaussians
    k = max((len(g.sh_rest) for g in gs), default=0)
    rest = np.zeros((len(gs), k, 3))
    for i, g in enumerate(gs):
        for j, c in enumerate(g.sh_rest):
            rest[i, j] = c
    return dict(mu=np.array([g.mu for g in gs]), scale=np.array([g.scale for g in gs]),
                rot=np.array([g.rot for g in gs]), opacity=np.array([g.opacity for g in gs]),
                sh_dc=np.array([g.sh_dc for g in gs]), sh_rest=rest)


def put_scene(prefix, scene):
    for k, v in scene_arrays(scene).items():
        put(f"{prefix}__{k}", v)
    put(f"{prefix}__extent", scene.extent)


def cam_rows(cams):
    return np.array([np.concatenate([c.r_c2w.ravel(), c.center,
                                     [c.f_x, c.f_y, c.p_x, c.p_y, c.width, c.height]])
                     for c in cams])


def rand_quat(rng):
    q = rng.standard_normal(4)
    return q / np.linalg.norm(q)


def rand_gaussian(rng, mu_range=0.5, scale=(0.05, 0.5), sh_k=0):
    return Gaussian3D(mu=rng.uniform(-mu_range, mu_range, 3), scale=rng.uniform(*scale, 3),
                      rot=rand_quat(rng), opacity=rng.uniform(0.2, 0.995),
                      sh_dc=rgb_to_dc(rng.uniform(0.1, 0.9, 3)),
                      sh_rest=tuple(rng.normal(0, 0.2, 3) for _ in range(sh_k)))


def look_cam(rng, w, h, dist=3.0, f=None):
    ang = rng.uniform(0, 2 * np.pi)
    elev = rng.uniform(-0.6, 0.9)
    eye = dist * np.array([np.cos(ang) * np.cos(elev), np.sin(ang) * np.cos(elev), np.sin(elev)])
    fwd = -eye / np.linalg.norm(eye)
    down0 = np.array([0.0, 0.0, -1.0])
    right = np.cross(down0, fwd)
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    f = f or rng.uniform(0.8, 1.4) * min(w, h)
    return Camera(r_c2w=np.stack([right, down, fwd], axis=1), center=eye, f_x=f,
                  f_y=f * rng.uniform(0.9, 1.1), p_x=(w - 1) / 2 + rng.uniform(-1, 1),
                  p_y=(h - 1) / 2 + rng.uniform(-1, 1), width=w, height=h)


# --------------------------------------------------------------------- render
def gen_render():
    rng = np.random.default_rng(101)
    n_cases = 0
    for c in range(12):
        w, h = int(rng.integers(12, 33)), int(rng.integers(12, 33))
        sh_k = [0, 0, 3, 8, 15][c % 5]
        n = int(rng.integers(3, 30))
        scene = Scene([rand_gaussian(rng, sh_k=sh_k) for _ in range(n)], extent=1.0)
        if c == 7:  # duplicated Gaussian: exact depth tie -> index order
            scene.gaussians.append(scene.gaussians[0])
        cam = look_cam(rng, w, h)
        out = raster.render(scene, cam, np.zeros(3))
        put_scene(f"render__{c}__scene", scene)
        put(f"render__{c}__cam", cam_rows([cam]))
        put(f"render__{c}__image", out.image)
        put(f"render__{c}__dominant", out.dominant_map)
        n_cases += 1
    meta["render"] = n_cases


# ----------------------------------------------------------------------- maps
def gen_maps():
    rng = np.random.default_rng(202)
    cfgs = []
    for c in range(24):
        h, w = int(rng.integers(4, 21)), int(rng.integers(4, 21))
        a = rng.uniform(0, 1, (h, w, 3))
        b = a.copy()
        blob = rng.uniform(0, 1, (h, w)) > rng.uniform(0.2, 0.8)
        b[blob] += rng.uniform(-0.6, 0.6, (int(blob.sum()), 3))
        if c == 0:
            b = a.copy()                       # hi == lo branch
        cfg = dict(tau_l1=float(rng.choice([0.1, 0.25, 0.05])), r_erode=int(c % 5),
                   l_bands=int(rng.integers(1, 5)))
        m = compute_maps(a, b, AdpSplitConfig(**cfg))
        put(f"maps__{c}__rendered", a)
        put(f"maps__{c}__gt", b)
        put(f"maps__{c}__e", m.e)
        put(f"maps__{c}__m", m.m)
        put(f"maps__{c}__b", m.b)
        cfgs.append(cfg)
    meta["maps"] = cfgs


# ------------------------------------------------------------------ partition
def gen_partition():
    rng = np.random.default_rng(303)
    specs = []
    for c in range(40):
        h, w = int(rng.integers(6, 33)), int(rng.integers(6, 33))
        e = rng.uniform(0, 1, (h, w))
        m = (e > 0.1) & (rng.uniform(0, 1, (h, w)) > rng.uniform(0.0, 0.5))
        n_ids = int(rng.integers(1, 6))
        dom = rng.integers(-1, n_ids, (h, w))
        if c % 3 == 0:  # blocky dominance like a real render
            dom = np.kron(rng.integers(-1, n_ids, (h // 4 + 1, w // 4 + 1)),
                          np.ones((4, 4), dtype=np.int64))[:h, :w]
        l_bands = int(rng.integers(1, 4))
        b = band_map(e, 0.1, l_bands)
        cands = sorted(set(int(x) for x in rng.choice(n_ids, size=int(rng.integers(1, n_ids + 1)),
                                                      replace=False)))
        m_min = int(rng.integers(1, 6))
        gt = rng.uniform(0, 1, (h, w, 3))
        regs = partition(ErrorMaps(e=e, m=m, b=b), dom, cands, m_min, view=c)
        rows = []
        pix = []
        for r in regs:
            region_stats(r, gt)
            rows.append([r.candidate, r.band, r.area,
                         int((r.pixels[:, 1] * w + r.pixels[:, 0]).min())])
            pix.append(r.pixels)
        put(f"part__{c}__m", m)
        put(f"part__{c}__dom", dom)
        put(f"part__{c}__b", b)
        put(f"part__{c}__gt", gt)
        put(f"part__{c}__rows", np.array(rows, dtype=np.int64).reshape(-1, 4))
        put(f"part__{c}__pixels", np.concatenate(pix) if pix else np.zeros((0, 2), np.int64))
        put(f"part__{c}__centroid", np.array([r.centroid for r in regs]).reshape(-1, 2))
        put(f"part__{c}__e1", np.array([r.e1 for r in regs]).reshape(-1, 2))
        put(f"part__{c}__sigma", np.array([[r.sigma1, r.sigma2] for r in regs]).reshape(-1, 2))
        put(f"part__{c}__gt_rgb", np.array([r.gt_rgb for r in regs]).reshape(-1, 3))
        specs.append(dict(cands=cands, m_min=m_min, l_bands=l_bands))
    meta["part"] = specs


# ---------------------------------------------------------------------- child
def gen_child():
    rng = np.random.default_rng(404)
    cfg = AdpSplitConfig()
    rows = []
    for c in range(200):
        w, h = int(rng.integers(12, 40)), int(rng.integers(12, 40))
        cam = look_cam(rng, w, h)
        parent = Gaussian3D(mu=rng.uniform(-0.4, 0.4, 3), scale=rng.uniform(0.02, 0.5, 3),
                            rot=rand_quat(rng), opacity=rng.uniform(0.1, 0.9),
                            sh_dc=np.zeros(3))
        if c % 17 == 5:   # parent behind the camera -> t* <= 0
            parent = Gaussian3D(mu=cam.center - 2.0 * cam.forward, scale=parent.scale,
                                rot=parent.rot, opacity=parent.opacity, sh_dc=np.zeros(3))
        e1 = rng.standard_normal(2)
        e1 /= np.linalg.norm(e1)
        if c % 11 == 0:
            e1 = np.array([1.0, 0.0]) if c % 2 else np.array([0.0, 1.0])
        s1 = rng.uniform(0.5, 8.0)
        s2 = rng.uniform(0.5, s1)
        reg = ErrorRegion(candidate=0, view=0, pixels=np.zeros((1, 2), np.int64), area=7,
                          band=0, centroid=rng.uniform([0, 0], [w - 1, h - 1]), e1=e1,
                          e2=np.array([-e1[1], e1[0]]), sigma1=s1, sigma2=s2,
                          gt_rgb=rng.uniform(0, 1, 3))
        if c % 23 == 3:
            reg.e2 = reg.e1.copy()             # parallel-axis fallback branch
        o, d, nrm = pixel_ray(cam, *reg.centroid)
        t = optimal_t(parent.mu, covariance(parent), o, d, cfg.eps)
        ch = init_child(parent, 0, reg, cam, cfg)
        ok = ch is not None
        rows.append(np.concatenate([
            parent.mu, parent.scale, parent.rot, [parent.opacity], cam_rows([cam])[0],
            reg.centroid, reg.e1, reg.e2, [reg.sigma1, reg.sigma2], reg.gt_rgb, [t, ok],
            ch.mu if ok else np.zeros(3), ch.rot.ravel() if ok else np.zeros(9),
            ch.scale if ok else np.zeros(3)]))
    put("child__rows", np.array(rows))
    meta["child_layout"] = ("mu3 scale3 rot4 o1 cam18 centroid2 e1_2 e2_2 sig2 rgb3 t1 ok1 "
                            "cmu3 crot9 cscale3")


# ---------------------------------------------------------------------- merge
def gen_merge():
    rng = np.random.default_rng(505)
    specs = []
    for c in range(150):
        n = int(rng.integers(1, 14))
        props = []
        base = rng.uniform(-0.3, 0.3, 3)
        for k in range(n):
            q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            if np.linalg.det(q) < 0:
                q[:, 0] = -q[:, 0]
            props.append(ChildProposal(
                mu=base + rng.normal(0, rng.choice([0.02, 0.1, 0.3]), 3), rot=q,
                scale=rng.uniform(0.02, 0.3, 3), opacity=0.6,
                rgb=rng.uniform(0.3, 0.7, 3) if c % 4 else np.full(3, 0.5) + rng.normal(0, 0.03, 3),
                parent=0, view=k % 4, region_area=9))
        if c % 10 == 0 and n > 2:
            props[2] = props[1]                  # identical pair, degenerate eigenspaces
        gd, gc = float(rng.choice([2.0, 1.0, 4.0])), float(rng.choice([0.15, 0.05, 1.0]))
        n_max = int(rng.integers(1, 8))
        groups = merge_groups(props, gd, gc)
        capped = cap_children(groups, n_max)
        put(f"merge__{c}__mu", np.array([p.mu for p in props]))
        put(f"merge__{c}__rot", np.array([p.rot for p in props]))
        put(f"merge__{c}__scale", np.array([p.scale for p in props]))
        put(f"merge__{c}__rgb", np.array([p.rgb for p in props]))
        put(f"merge__{c}__g_mu", np.array([g.merged_mu for g in groups]))
        put(f"merge__{c}__g_cov", np.array([g.merged_cov for g in groups]))
        put(f"merge__{c}__g_rgb", np.array([g.merged_rgb for g in groups]))
        put(f"merge__{c}__g_ext", np.array([g.extent for g in groups]))
        put(f"merge__{c}__cap_order", np.array([groups.index(g) for g in capped]))
        specs.append(dict(gamma_d=gd, gamma_c=gc, n_max=n_max,
                          members=[list(map(int, g.members)) for g in groups]))
    meta["merge"] = specs


def gen_merge_large():
    """Proposal lists of 30-300 (the oracle's prefiltered union-find path)."""
    rng = np.random.default_rng(909)
    specs = []
    for c in range(10):
        n = int(rng.integers(30, 300))
        props = []
        centers = rng.uniform(-0.3, 0.3, (int(rng.integers(2, 12)), 3))
        for k in range(n):
            q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
            if np.linalg.det(q) < 0:
                q[:, 0] = -q[:, 0]
            props.append(ChildProposal(
                mu=centers[k % len(centers)] + rng.normal(0, rng.choice([0.01, 0.05, 0.2]), 3), rot=q,
                scale=rng.uniform(0.01, 0.1, 3), opacity=0.6,
                rgb=np.full(3, 0.5) + rng.normal(0, 0.05, 3), parent=0, view=k % 4, region_area=9))
        gd, gc = float(rng.choice([2.0, 1.0, 4.0])), float(rng.choice([0.15, 0.05, 1.0]))
        groups = merge_groups(props, gd, gc)
        put(f"mergeL__{c}__mu", np.array([p.mu for p in props]))
        put(f"mergeL__{c}__rot", np.array([p.rot for p in props]))
        put(f"mergeL__{c}__scale", np.array([p.scale for p in props]))
        put(f"mergeL__{c}__rgb", np.array([p.rgb for p in props]))
        put(f"mergeL__{c}__g_mu", np.array([g.merged_mu for g in groups]))
        put(f"mergeL__{c}__g_cov", np.array([g.merged_cov for g in groups]))
        specs.append(dict(gamma_d=gd, gamma_c=gc, members=[list(map(int, g.members)) for g in groups]))
    meta["merge_large"] = specs


# ----------------------------------------------------------------------- step
def report_dict(rep):
    return dict(count_before=rep.count_before, count_after=rep.count_after,
                clones=[int(i) for i in rep.clones],
                candidates=[dict(index=int(r.index), regions_per_view=[int(x) for x in r.regions_per_view],
                                 proposals=int(r.proposals), merged=int(r.merged),
                                 children_inserted=int(r.children_inserted),
                                 fallback=bool(r.fallback), reset=bool(r.reset))
                            for r in rep.candidates],
                sampled_views=[int(v) for v in rep.sampled_views], merge_edges=int(rep.merge_edges),
                reset_indices=[int(i) for i in rep.reset_indices])


def run_step(tag, scene, cams, gts, stats, cfg, seed):
    put_scene(f"step__{tag}__in", scene)
    put(f"step__{tag}__cams", cam_rows(cams))
    put(f"step__{tag}__gt", np.array(gts))
    put(f"step__{tag}__grad_accum", stats.grad_accum)
    put(f"step__{tag}__denom", stats.denom)
    # capture the renders adpsplit_step makes (for stage-isolated replays)
    captured = {}
    orig = adc.render

    def spy(sc, cam, bg):
        out = orig(sc, cam, bg)
        captured[id(cam)] = out
        return out

    adc.render = spy
    try:
        new_scene, rep = adc.adpsplit_step(scene, cams, gts, stats, cfg, np.random.default_rng(seed))
    finally:
        adc.render = orig
    for v in rep.sampled_views:
        put(f"step__{tag}__img{v}", captured[id(cams[v])].image)
        put(f"step__{tag}__dom{v}", captured[id(cams[v])].dominant_map)
    put_scene(f"step__{tag}__out", new_scene)
    put(f"step__{tag}__index_map", rep.index_map)
    # remap_stats (ref/adc.py:283-296) of this step's report on the step's input stats
    rs = adc.remap_stats(stats, rep)
    put(f"remap__{tag}__grad_accum", rs.grad_accum)
    put(f"remap__{tag}__denom", rs.denom)
    cfgd = {f: getattr(cfg, f) for f in cfg.__dataclass_fields__}
    meta.setdefault("step", {})[tag] = dict(cfg=cfgd, seed=seed, report=report_dict(rep))


def _g(**kw):
    base = dict(mu=[0, 0, 0.5], scale=[0.2, 0.2, 0.2], rot=[1, 0, 0, 0], opacity=0.8,
                sh_dc=rgb_to_dc([0.7, 0.3, 0.3]))
    base.update(kw)
    return Gaussian3D(**base)


def _simple_cam(width=24, height=24, f=30.0, dist=2.0):
    return Camera(r_c2w=np.eye(3), center=np.array([0.0, 0.0, -dist]), f_x=f, f_y=f,
                  p_x=(width - 1) / 2.0, p_y=(height - 1) / 2.0, width=width, height=height)


def gen_steps():
    # (a) the two-blob setup of tests/test_adc.py:122-139, plus bystanders
    cams = [_simple_cam() for _ in range(3)]
    gt_scene = Scene([_g(mu=[-0.25, 0, 0.3], scale=[0.08] * 3, sh_dc=rgb_to_dc([0.9, 0.2, 0.2])),
                      _g(mu=[0.25, 0, 0.3], scale=[0.08] * 3, sh_dc=rgb_to_dc([0.2, 0.2, 0.9]))],
                     extent=1.0)
    gts = [raster.render(gt_scene, c, np.zeros(3)).image for c in cams]
    coarse = Scene([_g(mu=[0, 0, 0.3], scale=[0.3, 0.15, 0.15], sh_dc=rgb_to_dc([0.5, 0.2, 0.5])),
                    _g(mu=[0, 0.4, 0.3], scale=[0.05] * 3),
                    _g(mu=[0.4, 0.4, 0.3], scale=[0.005] * 3),
                    _g(mu=[0, 0, -10], scale=[0.3] * 3)], extent=1.0)
    stats = adc.DensifyStats(grad_accum=np.array([1e-2, 0.0, 1e-2, 1e-2]), denom=np.ones(4))
    run_step("blobs", coarse, cams, gts, stats, AdpSplitConfig(v_views=3), 1)
    # (b) criterion-6 style desk steps (tests/test_acceptance.py:225-265)
    for seed in range(12):
        gt, cams, gts = synth_scene(seed, k=8, cam_count=6, image_size=24)
        scene = init_from_gt(gt, seed)
        n = len(scene.gaussians)
        stats = adc.DensifyStats(grad_accum=np.full(n, 1e-2), denom=np.ones(n))
        run_step(f"desk{seed}", scene, cams, gts, stats, desk_config(v_views=4), seed)
    # (c) paper-default config, larger scenes, mixed gradients, erosion r=2..3
    for seed in range(4):
        gt, cams, gts = synth_scene(100 + seed, k=60, cam_count=5, image_size=48)
        scene = init_from_gt(gt, seed, inflate=3.0)
        n = len(scene.gaussians)
        rng = np.random.default_rng(seed)
        ga = np.where(rng.uniform(size=n) < 0.7, 1e-2, 1e-5)
        den = np.where(rng.uniform(size=n) < 0.1, 0.0, 1.0)
        stats = adc.DensifyStats(grad_accum=ga, denom=den)
        cfg = AdpSplitConfig(v_views=4, r_erode=2 + seed % 2, m_min=3, n_max=4 + seed,
                             tau_s=0.01 if seed < 2 else 0.05)
        run_step(f"paper{seed}", scene, cams, gts, stats, cfg, 7 + seed)


# ------------------------------------------------------- next rows of SURVEY 8(f)
def gen_next_rows():
    # vanilla_densify on the step inputs (n_children 2 and 3; ref/adc.py:248-280)
    specs = []
    for tag in ("blobs", "desk0", "desk3", "paper1", "paper2"):
        for n_children in (2, 3):
            sc = Scene([Gaussian3D(mu=store[f"step__{tag}__in__mu"][i], scale=store[f"step__{tag}__in__scale"][i],
                                   rot=store[f"step__{tag}__in__rot"][i],
                                   opacity=float(store[f"step__{tag}__in__opacity"][i]),
                                   sh_dc=store[f"step__{tag}__in__sh_dc"][i])
                        for i in range(len(store[f"step__{tag}__in__mu"]))],
                       extent=float(store[f"step__{tag}__in__extent"]))
            stats = adc.DensifyStats(grad_accum=store[f"step__{tag}__grad_accum"].copy(),
                                     denom=store[f"step__{tag}__denom"].copy())
            cfg = AdpSplitConfig(**meta["step"][tag]["cfg"])
            seed = 1000 + n_children
            rng = np.random.default_rng(seed)
            new_scene, rep = adc.vanilla_densify(sc, stats, cfg, n_children, rng)
            key = f"vanilla__{tag}__{n_children}"
            put_scene(f"{key}__out", new_scene)
            put(f"{key}__index_map", rep.index_map)
            specs.append(dict(tag=tag, n_children=n_children, seed=seed, report=report_dict(rep),
                              rng_state=json.loads(json.dumps(rng.bit_generator.state))))
    meta["vanilla"] = specs
    # accumulate_stats (ref/adc.py:73-79) with the reference's fp64 GradOutput
    rng = np.random.default_rng(77)
    acc = []
    for c, n in enumerate((1, 7, 1000, 4099)):
        ga = rng.uniform(0, 1e-2, n)
        den = rng.integers(0, 5, n).astype(np.float64)
        vg = rng.normal(0, 1e-3, (n, 2)) * np.exp(rng.normal(0, 3, (n, 1)))
        vis = rng.uniform(size=n) < 0.6
        stats = adc.DensifyStats(grad_accum=ga.copy(), denom=den.copy())
        for rep_ in range(3):      # three views in a row
            z = np.zeros((n, 3))
            adc.accumulate_stats(stats, GradOutput(dmu=z, dscale=z, drot=np.zeros((n, 4)), dopacity=np.zeros(n),
                                                   dsh_dc=z, viewspace_grad=vg * (rep_ + 1), visible=vis))
        for k, v in dict(ga=ga, den=den, vg=vg, vis=vis, ga_out=stats.grad_accum, den_out=stats.denom).items():
            put(f"accum__{c}__{k}", v)
        acc.append(n)
    meta["accum"] = acc
    # _prune (ref/harness.py:320-340) on trainer state built from a scene
    pr = []
    for c, (n, thr) in enumerate(((50, harness.PRUNE_OPACITY), (400, 0.05), (30, 0.5), (20, 0.5), (20, 1e-4))):
        rng = np.random.default_rng(500 + c)
        op = rng.uniform(1e-4, 0.2, n) if thr < 0.5 else rng.uniform(0.3, 0.7, n)
        if c == 3:
            op = np.full(n, 0.9)            # nobody pruned: state returned unchanged
        if c == 4:
            op = np.full(n, 5e-5)           # everybody below: unchanged too
        gs = [Gaussian3D(mu=rng.normal(size=3), scale=np.exp(rng.normal(size=3) - 3), rot=rand_quat(rng),
                         opacity=float(op[i]), sh_dc=rng.normal(size=3)) for i in range(n)]
        params = harness._Params(Scene(gaussians=gs, extent=1.0))
        if c == 1:                          # logits right at the threshold's logit
            params.logit_op[:40] = np.log(thr / (1 - thr)) + rng.integers(-3, 4, 40) * 1e-16
        opt = harness._Adam(params)
        for g in params.groups():
            opt.m[g] = rng.normal(size=opt.m[g].shape)
            opt.v[g] = rng.uniform(size=opt.v[g].shape)
        stats = adc.DensifyStats(grad_accum=np.arange(n, dtype=np.float64), denom=rng.uniform(size=n))
        new_p, new_opt, new_stats = harness._prune(params, opt, stats, thr)
        put(f"prune__{c}__logit", params.logit_op)
        put(f"prune__{c}__keep_index", new_stats.grad_accum.astype(np.int64))
        put(f"prune__{c}__m_mu_in", opt.m["mu"])
        put(f"prune__{c}__m_mu_out", new_opt.m["mu"])
        put(f"prune__{c}__denom_out", new_stats.denom)
        pr.append(dict(n=n, threshold=thr, pruned=new_p is not params))
    meta["prune"] = pr


def main():
    gen_render()
    gen_maps()
    gen_partition()
    gen_child()
    gen_merge()
    gen_merge_large()
    gen_steps()
    gen_next_rows()
    store["meta_json"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT, **store)
    print(f"wrote {OUT}: {len(store)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
