"""Pin the CPU oracle against golden vectors produced by the reference itself.

Every comparison here is against outputs of /root/reference/pkg/src/adpsplit
captured by tests/golden/make_golden.py.  Integer outputs must match exactly;
fp64 outputs must match bit for bit where the oracle follows the reference's
operation order (it does everywhere except the support-window render, which
is proven exact by construction and checked here too).
"""

import numpy as np
import pytest

import golden_io
from oracle import adpsplit_oracle as O

DATA, META = golden_io.load()


@pytest.mark.parametrize("c", range(12))
def test_render_matches_reference(c):
    g, _ = golden_io.scene(DATA, f"render__{c}__scene")
    cam = golden_io.cams(DATA, f"render__{c}__cam")[0]
    img, dom = O.render(g, cam)
    np.testing.assert_array_equal(dom, DATA[f"render__{c}__dominant"])
    np.testing.assert_array_equal(img, DATA[f"render__{c}__image"])


@pytest.mark.parametrize("c", range(24))
def test_maps_match_reference(c):
    cfg = META["maps"][c]
    m = O.compute_maps(DATA[f"maps__{c}__rendered"], DATA[f"maps__{c}__gt"], cfg)
    np.testing.assert_array_equal(m.e, DATA[f"maps__{c}__e"])
    np.testing.assert_array_equal(m.m, DATA[f"maps__{c}__m"])
    np.testing.assert_array_equal(m.b, DATA[f"maps__{c}__b"])


@pytest.mark.parametrize("c", range(40))
def test_partition_and_region_stats_match_reference(c):
    spec = META["part"][c]
    dom = DATA[f"part__{c}__dom"]
    is_cand = np.zeros(max(int(dom.max()), max(spec["cands"])) + 1, dtype=bool)
    is_cand[spec["cands"]] = True
    maps = O.Maps(e=None, m=DATA[f"part__{c}__m"], b=DATA[f"part__{c}__b"])
    regs = O.partition(maps, dom, is_cand, spec["m_min"], view=c)
    rows = np.array([[r.candidate, r.band, r.area, r.minpix] for r in regs],
                    dtype=np.int64).reshape(-1, 4)
    np.testing.assert_array_equal(rows, DATA[f"part__{c}__rows"])
    pix = np.concatenate([r.pixels for r in regs]) if regs else np.zeros((0, 2), np.int64)
    np.testing.assert_array_equal(pix, DATA[f"part__{c}__pixels"])
    gt = DATA[f"part__{c}__gt"]
    for k, r in enumerate(regs):
        O.region_stats(r, gt)
        np.testing.assert_array_equal(r.centroid, DATA[f"part__{c}__centroid"][k])
        np.testing.assert_array_equal(r.e1, DATA[f"part__{c}__e1"][k])
        np.testing.assert_array_equal([r.sigma1, r.sigma2], DATA[f"part__{c}__sigma"][k])
        np.testing.assert_array_equal(r.gt_rgb, DATA[f"part__{c}__gt_rgb"][k])


def test_child_init_matches_reference():
    rows = DATA["child__rows"]
    n_ok = 0
    for row in rows:
        mu, scale, rot, o = row[0:3], row[3:6], row[6:10], row[10]
        cam = O.Cam.from_row(row[11:29])
        reg = O.Region(candidate=0, view=0, band=0, area=7, minpix=0, pixels=None,
                       centroid=row[29:31], e1=row[31:33], e2=row[33:35], sigma1=row[35],
                       sigma2=row[36], gt_rgb=row[37:40])
        t_ref, ok = row[40], bool(row[41])
        g = O.Gaussians(mu[None], scale[None], rot[None], [o], np.zeros((1, 3)))
        orig, d, _ = O.pixel_ray(cam, *reg.centroid)
        assert O.optimal_t(mu, O.covariance(rot, scale), orig, d, 1e-9) == t_ref
        ch = O.init_child(g, 0, reg, cam, 1e-9)
        assert (ch is not None) == ok
        if ok:
            n_ok += 1
            np.testing.assert_array_equal(ch.mu, row[42:45])
            np.testing.assert_array_equal(ch.rot.ravel(), row[45:54])
            np.testing.assert_array_equal(ch.scale, row[54:57])
    assert n_ok > 150


@pytest.mark.parametrize("c", range(150))
def test_merge_and_cap_match_reference(c):
    spec = META["merge"][c]
    props = [O.Proposal(mu=m, rot=r, scale=s, opacity=0.6, rgb=rgb, parent=0, view=0, area=9)
             for m, r, s, rgb in zip(DATA[f"merge__{c}__mu"], DATA[f"merge__{c}__rot"],
                                     DATA[f"merge__{c}__scale"], DATA[f"merge__{c}__rgb"])]
    groups = O.merge_groups(props, spec["gamma_d"], spec["gamma_c"])
    assert [g.members for g in groups] == spec["members"]
    for k, g in enumerate(groups):
        np.testing.assert_array_equal(g.mu, DATA[f"merge__{c}__g_mu"][k])
        np.testing.assert_array_equal(g.cov, DATA[f"merge__{c}__g_cov"][k])
        np.testing.assert_array_equal(g.rgb, DATA[f"merge__{c}__g_rgb"][k])
        assert g.extent == DATA[f"merge__{c}__g_ext"][k]
    capped = O.cap_children(groups, spec["n_max"])
    assert [groups.index(g) for g in capped] == DATA[f"merge__{c}__cap_order"].tolist()


STEP_TAGS = sorted(META["step"])


def run_oracle_step(tag, use_ref_renders):
    g, extent = golden_io.scene(DATA, f"step__{tag}__in")
    cams = golden_io.cams(DATA, f"step__{tag}__cams")
    gts = DATA[f"step__{tag}__gt"]
    m = META["step"][tag]
    renders = None
    if use_ref_renders:
        renders = {v: (DATA[f"step__{tag}__img{v}"], DATA[f"step__{tag}__dom{v}"])
                   for v in m["report"]["sampled_views"]}
    return O.adpsplit_step(g, extent, cams, gts, DATA[f"step__{tag}__grad_accum"],
                           DATA[f"step__{tag}__denom"], golden_io.Cfg(m["cfg"]),
                           np.random.default_rng(m["seed"]), renders=renders)


def assert_step_matches(res, tag):
    rep = META["step"][tag]["report"]
    assert res.count_after == rep["count_after"]
    assert res.sampled_views == rep["sampled_views"]
    assert res.merge_edges == rep["merge_edges"]
    assert res.clones == rep["clones"]
    assert res.reset_indices == rep["reset_indices"]
    got = [dict(index=r.index, regions_per_view=r.regions_per_view, proposals=r.proposals,
                merged=r.merged, children_inserted=r.children_inserted, fallback=r.fallback,
                reset=r.reset) for r in res.candidates]
    assert got == rep["candidates"]
    np.testing.assert_array_equal(res.index_map, DATA[f"step__{tag}__index_map"])
    out, _ = golden_io.scene(DATA, f"step__{tag}__out")
    for f in ("mu", "scale", "rot", "opacity", "sh_dc"):
        np.testing.assert_array_equal(getattr(res.gaussians, f), getattr(out, f), err_msg=f)


@pytest.mark.parametrize("tag", STEP_TAGS)
def test_step_matches_reference_end_to_end(tag):
    res = run_oracle_step(tag, use_ref_renders=False)
    assert_step_matches(res, tag)


@pytest.mark.parametrize("tag", STEP_TAGS)
def test_step_stage_isolated_replay(tag):
    res = run_oracle_step(tag, use_ref_renders=True)
    assert_step_matches(res, tag)


def test_partition_reference_semantics_handcrafted():
    """Known answers of tests/test_error_partition.py:120-163 (area 9 blob, diagonals)."""
    cand = np.array([True])
    m = np.zeros((8, 8), dtype=bool)
    m[2:5, 2:5] = True
    regs = O.partition(O.Maps(None, m, np.zeros((8, 8), np.int64)), np.zeros((8, 8), np.int64),
                       cand, 5)
    assert len(regs) == 1 and regs[0].area == 9
    m = np.zeros((8, 8), dtype=bool)
    for i in range(5):
        m[i, i] = True
    regs = O.partition(O.Maps(None, m, np.zeros((8, 8), np.int64)), np.zeros((8, 8), np.int64),
                       cand, 5)
    assert len(regs) == 1 and regs[0].area == 5


def test_band_edges_known_answer():
    """tests/test_error_partition.py:98-102: tau=0.1, L=3 -> edges 0.4 / 0.7."""
    e = np.array([[0.1, 0.11, 0.39, 0.4, 0.69, 0.7, 0.99, 1.0]])
    assert O.band_map(e, 0.1, 3).tolist() == [[0, 0, 0, 1, 1, 2, 2, 2]]


def test_region_stats_horizontal_line():
    """tests/test_error_partition.py:217-226: centroid (3,3), sigma1=sqrt2, sigma2 floored."""
    gt = np.zeros((8, 8, 3))
    gt[3, 3] = [0.2, 0.4, 0.6]
    reg = O.Region(0, 0, 0, 5, 0, np.array([(x, 3) for x in range(1, 6)]))
    O.region_stats(reg, gt)
    assert np.allclose(reg.centroid, [3.0, 3.0])
    assert reg.sigma1 == pytest.approx(np.sqrt(2.0)) and reg.sigma2 == 0.5
    assert np.allclose(reg.gt_rgb, [0.2, 0.4, 0.6])


# ------------------------------------------------ next rows pinned
def _vanilla_inputs(spec):
    tag = spec["tag"]
    g, extent = golden_io.scene(DATA, f"step__{tag}__in")
    cfg = golden_io.Cfg(META["step"][tag]["cfg"])
    return g, extent, DATA[f"step__{tag}__grad_accum"], DATA[f"step__{tag}__denom"], cfg


@pytest.mark.parametrize("c", range(10))
def test_vanilla_densify_matches_reference(c):
    spec = META["vanilla"][c]
    g, extent, ga, den, cfg = _vanilla_inputs(spec)
    rng = np.random.default_rng(spec["seed"])
    res = O.vanilla_densify(g, extent, ga, den, cfg, spec["n_children"], rng)
    key = f"vanilla__{spec['tag']}__{spec['n_children']}"
    np.testing.assert_array_equal(res.index_map, DATA[f"{key}__index_map"])
    for f in ("mu", "scale", "rot", "opacity", "sh_dc"):
        np.testing.assert_array_equal(getattr(res.gaussians, f), DATA[f"{key}__out__{f}"], err_msg=f)
    want = spec["report"]
    assert res.clones == want["clones"]
    assert [(r.index, r.children_inserted) for r in res.candidates] == \
        [(r["index"], r["children_inserted"]) for r in want["candidates"]]
    st = rng.bit_generator.state
    assert st["state"]["state"] == spec["rng_state"]["state"]["state"]


@pytest.mark.parametrize("tag", sorted(META["step"]))
def test_remap_stats_matches_reference(tag):
    rep = META["step"][tag]["report"]
    ga, den = O.remap_stats(DATA[f"step__{tag}__grad_accum"], DATA[f"step__{tag}__denom"],
                            DATA[f"step__{tag}__index_map"], rep["reset_indices"], rep["clones"])
    np.testing.assert_array_equal(ga, DATA[f"remap__{tag}__grad_accum"])
    np.testing.assert_array_equal(den, DATA[f"remap__{tag}__denom"])


@pytest.mark.parametrize("c", range(4))
def test_accumulate_stats_matches_reference(c):
    ga, den = DATA[f"accum__{c}__ga"].copy(), DATA[f"accum__{c}__den"].copy()
    vg, vis = DATA[f"accum__{c}__vg"], DATA[f"accum__{c}__vis"]
    for k in range(3):
        O.accumulate_stats(ga, den, vg * (k + 1), vis)
    np.testing.assert_array_equal(ga, DATA[f"accum__{c}__ga_out"])
    np.testing.assert_array_equal(den, DATA[f"accum__{c}__den_out"])


@pytest.mark.parametrize("c", range(5))
def test_prune_keep_matches_reference(c):
    spec = META["prune"][c]
    keep = O.prune_keep(DATA[f"prune__{c}__logit"], spec["threshold"])
    if not spec["pruned"]:
        assert keep is None
        return
    np.testing.assert_array_equal(keep, DATA[f"prune__{c}__keep_index"])
    np.testing.assert_array_equal(DATA[f"prune__{c}__m_mu_in"][keep], DATA[f"prune__{c}__m_mu_out"])


@pytest.mark.parametrize("c", range(10))
def test_large_merge_matches_reference(c):
    """30-300 proposals: the oracle's prefiltered union-find vs the reference's all-pairs loop."""
    spec = META["merge_large"][c]
    props = [O.Proposal(mu=m, rot=r, scale=s, opacity=0.6, rgb=rgb, parent=0, view=0, area=9)
             for m, r, s, rgb in zip(DATA[f"mergeL__{c}__mu"], DATA[f"mergeL__{c}__rot"],
                                     DATA[f"mergeL__{c}__scale"], DATA[f"mergeL__{c}__rgb"])]
    groups = O.merge_groups(props, spec["gamma_d"], spec["gamma_c"])
    assert [g.members for g in groups] == spec["members"]
    for k, g in enumerate(groups):
        np.testing.assert_array_equal(g.mu, DATA[f"mergeL__{c}__g_mu"][k])
        np.testing.assert_array_equal(g.cov, DATA[f"mergeL__{c}__g_cov"][k])
