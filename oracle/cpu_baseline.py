"""Timed CPU run of the oracle port on a bounded sample -- BASELINE INFRASTRUCTURE.

Used only by bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm.
It runs the oracle's restatement of ``adpsplit_step`` (ref/adc.py:143-245)
on k of the V sampled views, timing each stage:

  per view      compute_maps, partition, region_stats   (ref/error_partition.py)
                ever-dominant flags                      (ref/adc.py:177-180)
  per proposal  init_child                               (ref/child_init.py)
  per parent    merge_groups, cap_children, group->Gaussian, parent copy
  once          select, compaction / index_map

The full-step CPU time is extrapolated linearly in V from the per-view and
per-proposal/per-parent work of the sample (merge cost grows faster than
linearly with proposals, so this UNDER-estimates the CPU time).  Fallback
children of candidates that are merely unseen in the k-view sample are
timed but excluded from the extrapolation.  With ``workers > 1`` the per-view
stages fan out over processes (fork), one view per worker.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import adpsplit_oracle as O

_G = {}


def _view_work(v):
    """maps + partition + region_stats + init_child for one view (worker)."""
    s = _G
    t0 = time.perf_counter()
    img, dom = s["renders"][v]
    maps = O.compute_maps(img, s["gts"][v], s["cfg"])
    regs = O.partition(maps, dom, s["is_cand"], int(O.cfg_get(s["cfg"], "m_min")), view=v)
    for r in regs:
        O.region_stats(r, s["gts"][v])
    t1 = time.perf_counter()
    d = np.asarray(dom).ravel()
    dominant = np.unique(d[(d >= 0) & (d < len(s["is_cand"]))])
    t2 = time.perf_counter()
    props = []
    for r in regs:
        ch = O.init_child(s["g"], r.candidate, r, s["cams"][v], O.cfg_get(s["cfg"], "eps"))
        props.append(ch)
    t3 = time.perf_counter()
    return v, [r.candidate for r in regs], props, dominant, (t1 - t0, t2 - t1, t3 - t2)


def _merge_work(chunk):
    """merge_groups + cap_children + group->Gaussian for a chunk of parents (worker)."""
    s = _G
    t0 = time.perf_counter()
    n_max = int(O.cfg_get(s["cfg"], "n_max"))
    gd, gc = O.cfg_get(s["cfg"], "gamma_d"), O.cfg_get(s["cfg"], "gamma_c")
    n_children = 0
    for i in chunk:
        props = s["by_cand"][i]
        groups = O.cap_children(O.merge_groups(props, gd, gc), n_max)
        for gr in groups:
            O.group_to_params(gr, float(s["g"].opacity[i]))
        n_children += len(groups)
    return time.perf_counter() - t0, n_children


def time_sample(g: O.Gaussians, extent: float, cams: list, view_ids: list, renders: dict, gts: dict,
                grad_accum, denom, cfg, n_views_total: int, workers: int = 1, rng=None,
                cand_frac: float = 1.0) -> dict:
    """Time the oracle port on ``view_ids``; merges run on every 1/cand_frac-th
    parent with proposals (extrapolated x 1/cand_frac), fanned out over
    ``workers`` processes like the per-view stages."""
    rng = rng or np.random.default_rng(0)
    T = dict(select=0.0, maps_partition_stats=0.0, dominance=0.0, init_child=0.0, merge_emit=0.0,
             fallback=0.0, compaction=0.0)
    wall0 = time.perf_counter()
    t = time.perf_counter()
    split_set, clone_set = O.select(grad_accum, denom, g.scale, O.cfg_get(cfg, "tau_g"),
                                    O.cfg_get(cfg, "tau_s") * extent)
    is_cand = np.zeros(len(g), dtype=bool)
    is_cand[split_set] = True
    T["select"] = time.perf_counter() - t
    _G.update(g=g, cams=cams, renders=renders, gts=gts, cfg=cfg, is_cand=is_cand)
    if workers > 1:
        with mp.get_context("fork").Pool(min(workers, len(view_ids))) as pool:
            outs = pool.map(_view_work, view_ids)
    else:
        outs = [_view_work(v) for v in view_ids]
    per_view_wall = time.perf_counter() - t - T["select"]
    by_cand = {}
    dom_any = np.zeros(len(g), dtype=bool)
    n_regions = 0
    for v, cands, props, dominant, (a, b, c) in sorted(outs, key=lambda o: o[0]):
        T["maps_partition_stats"] += a
        T["dominance"] += b
        T["init_child"] += c
        dom_any[dominant] = True
        n_regions += len(cands)
        for cand, p in zip(cands, props):
            by_cand.setdefault(cand, []).append(p)
    removed = np.zeros(len(g), dtype=bool)
    n_ins = 0
    n_props = 0
    merge_list = []
    for i in (int(k) for k in split_set):
        props = [p for p in by_cand.get(i, []) if p is not None]
        by_cand[i] = props
        n_props += len(props)
        if not dom_any[i]:
            t = time.perf_counter()
            O.vanilla_children(g, i, 2, O.cfg_get(cfg, "eta"), rng)
            removed[i] = True
            n_ins += 2
            T["fallback"] += time.perf_counter() - t
        elif props:
            merge_list.append(i)
            removed[i] = True
    stride = max(1, int(round(1.0 / cand_frac)))
    sampled = merge_list[::stride]
    _G["by_cand"] = by_cand
    t = time.perf_counter()
    if workers > 1 and len(sampled) > 1:
        chunks = [sampled[w::workers] for w in range(workers)]
        with mp.get_context("fork").Pool(workers) as pool:
            res = pool.map(_merge_work, chunks)
        merge_wall = time.perf_counter() - t
        T["merge_emit"] = sum(r[0] for r in res)
        n_ins += sum(r[1] for r in res) + len(sampled)
    else:
        dt, nc = _merge_work(sampled)
        merge_wall = time.perf_counter() - t
        T["merge_emit"] = dt
        n_ins += nc + len(sampled)
    t = time.perf_counter()
    keep = np.flatnonzero(~removed)
    _ = O.Gaussians.concat([g.take(keep), g.take(clone_set)])
    _ = np.concatenate([keep, np.full(n_ins + len(clone_set), -1)])
    T["compaction"] = time.perf_counter() - t
    wall = time.perf_counter() - wall0
    k = len(view_ids)
    scale = n_views_total / k
    if workers > 1:
        # per-view stages ran concurrently: charge their wall time, not the sum
        view_part = per_view_wall
    else:
        view_part = T["maps_partition_stats"] + T["dominance"] + T["init_child"]
    merge_part = (merge_wall if workers > 1 else T["merge_emit"]) * (len(merge_list) / max(len(sampled), 1))
    est = T["select"] + T["compaction"] + scale * (view_part + merge_part)
    return dict(stages_s=T, sample_wall_s=wall, extrapolated_step_s=est, n_split=int(len(split_set)),
                n_clone=int(len(clone_set)), n_regions=n_regions, n_proposals=n_props, views=k,
                views_total=n_views_total, workers=workers, cpu_count=os.cpu_count(),
                parents_merged=len(sampled), parents_with_proposals=len(merge_list))
