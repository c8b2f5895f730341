#!/usr/bin/env python
"""AdpSplit densify-step benchmark (BASELINE.json metric) on B200.

One step = one AdpSplit densification step (stats + split + compaction,
ref/adc.py:165-244) over the attribution (image, dominant map) of the V
sampled views -- the stage boundary of BASELINE.md's "densify-step ms"
(B_step = 28 V H W + 72 N + 64 N_out bytes).  The
attribution render that produces the boundary is compute-bound and is
reported separately under "render" (ms/view, splat-px/s), and the full step
including it under "full_step".

  value     parents/s (|split set| / step time), inputs resident in HBM
  e2e       the same step through the public API from pinned HOST buffers
            (image, gt, dominant, params, stats copied in; grown params and
            index_map copied out) inside the timed region
  roofline  the dominant kernel, minmax_kernel: the one pass over the step's
            attribution inputs (28 B/px = image fp32x3 + gt
            fp32x3 + dominant int32) / its CUDA-event time, vs MEASURED_PEAKS;
            traffic = its ncu dram bytes (it also writes the 2.125 B/px
            16-bit raw-error cache and candidate bits).  "tile_pass" reports the
            bit-plane pass (tile_words_kernel, HBM: 2.125 B/px read) and the
            warp CCL (tile_bits_kernel, latency-bound) that follow.
  cpu_baseline  the oracle port on a bounded view sample (rank 0, N=1)

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config configN]
Multi-GPU: one rank per GPU; launched by torchrun, or bench.py re-executes
itself under torch.distributed.run when --gpus N > 1 and WORLD_SIZE is unset
(it exits with an error line when fewer than N GPUs are visible).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "AdpSplit densify-step ms & parents/s at 1M Gaussians; stat-accum GB/s vs HBM"
UNIT = "parents/s"
BYTES_PER_PX = 28      # image fp32x3 + gt fp32x3 + dominant int32 (the step's attribution inputs)
WORDS_BYTES_PER_PX = 2 + 0.125 + 0.5   # bit-plane pass: 16-bit raw cache + candidate bits read, 4 bit planes written
MINMAX_TRAFFIC_PER_PX = 28 + 2 + 0.125   # minmax pass: inputs read once, 16-bit raw cache + candidate bits written
BYTES_PER_G_IN = 72    # params 56 B + grad_accum/denom 2 x f64
BYTES_PER_G_OUT = 64   # params 56 B + index_map int64


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic(config):
    """dram bytes (read + write) of one minmax_kernel launch from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(config, {}).get("minmax_kernel_dram_bytes")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, period_ms=20):
        self.rows = []
        self.proc = None
        self.index = index
        self.period_ms = period_ms
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def window(self, t0, t1):
        self.t0, self.t1 = t0, t1

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = [r for t, r in self.rows if self.t0 is None or (self.t0 - 0.05 <= t <= self.t1 + 0.05)]
        scope = "timed_region"
        if len(rows) < 3:
            rows = [r for _, r in self.rows]
            scope = "whole_run"
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            parts = [p.strip() for p in r.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(smax)), "reasons": sorted(reasons),
                "samples": len(sm), "scope": scope}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def make_cfg(wl, v_views):
    from paper_2605_06876_b200.types import AdpSplitConfig
    return AdpSplitConfig(v_views=v_views, n_max=wl.n_max)


# ---------------------------------------------------------------------------
# CPU side (oracle port): cpu_baseline leg and --impl reference arm
# ---------------------------------------------------------------------------

def cpu_sample(wl, ini, cams, stats, view_ids, workers, renders, gts, cand_frac=1.0):
    from oracle import adpsplit_oracle as O
    from oracle.cpu_baseline import time_sample

    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    cam_objs = [O.Cam.from_row(r) for r in cams]
    cfg = make_cfg(wl, len(cams))
    return time_sample(g, ini.extent, cam_objs, view_ids, renders, gts, stats[0], stats[1], cfg,
                       n_views_total=len(cams), workers=workers, cand_frac=cand_frac)


def _workload_stats(wl, seed):
    """Candidates of a weighted workload need the rendered weights: on the box's GPU
    when there is one (the same numbers as the GPU arm), else the uniform draw."""
    if wl.stats_mode == "uniform":
        return wl.build(seed=seed), None
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError(f"{wl.name}: the weighted workload needs a GPU to render its statistics")
    from paper_2605_06876_b200 import operator as op
    plan = op.Plan("cuda:0")
    d = wl.build_device(plan, seed=seed)
    out = (d["ini"], d["cams"], d["stats"], d["gt"])
    renders = {v: (d["img"][v].double().cpu().numpy(), d["dom"][v].long().cpu().numpy())
               for v in range(min(len(d["cams"]), 64))}
    gts = {v: d["gt_img"][v].double().cpu().numpy() for v in renders}
    del d, plan
    torch.cuda.empty_cache()
    return out, (renders, gts)


def run_reference(args, wl):
    """--impl reference: the oracle port on the box's host cores (rank 0 only).

    Each step is a bounded sample of the config's step: all per-view stages on
    k of the V sampled views (fanned out over worker processes), the merges of
    the sampled parents, select and compaction; its measured wall time is
    ms_per_step, and value = |split set| / (the sample extrapolated linearly in
    V to the full step), a lower bound on the CPU time since the merge grows
    faster than linearly in V."""
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return
    (ini, cams, stats, gt_scene), attr = _workload_stats(wl, args.seed)
    cores = host_cores()
    k = max(1, min(cores, args.ref_views, len(cams)))
    views = list(range(k))
    if attr is not None:
        renders = {v: attr[0][v] for v in views}
        gts = {v: attr[1][v] for v in views}
    else:
        import multiprocessing as mp

        from oracle import adpsplit_oracle as O
        from oracle import c_render
        c_render.build()
        g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
        gt_g = O.Gaussians(gt_scene.mu, gt_scene.scale, gt_scene.rot, gt_scene.opacity, gt_scene.sh_dc)
        _PREP.update(g=g, gt=gt_g, cams=cams)
        with mp.get_context("fork").Pool(min(k, cores)) as pool:
            outs = pool.map(_prep_view, views)
        renders = {v: (img, dom) for v, img, dom, _ in outs}
        gts = {v: gt for v, _, _, gt in outs}
    walls, ests = [], []
    info = None
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        info = cpu_sample(wl, ini, cams, stats, views, workers=min(k, cores), renders=renders, gts=gts,
                          cand_frac=args.ref_cand_frac)
        if it >= args.warmup:
            walls.append(time.perf_counter() - t0)
            ests.append(info["extrapolated_step_s"])
    t_full = float(np.mean(ests))
    value = info["n_split"] / t_full
    workers = min(k, cores)
    sample = (f"oracle port (numpy): {k} of {len(cams)} views per step on {workers} worker processes "
              f"({workers} of {cores} host cores), merge/cap/emit on {info['parents_merged']} of "
              f"{info['parents_with_proposals']} parents with proposals; measured sample wall "
              f"{np.mean(walls):.2f} s/step (= ms_per_step), extrapolated linearly to all parents and "
              f"V={len(cams)}: {t_full:.2f} s per full step (value = |S| / that; a lower bound on CPU time, "
              f"merges grow faster than linearly in V); {info['n_regions']} regions, "
              f"{info['n_proposals']} proposals in the sample")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": float(np.mean(walls)) * 1e3,
            "extrapolated_ms_per_full_step": t_full * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(wl, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "host_cores": cores, "kind": "port",
                             "sample": sample, "stages_s": info["stages_s"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


_PREP = {}


def _prep_view(v):
    from oracle import c_render
    img, dom = c_render.render(_PREP["g"], _PREP["cams"][v])
    gt, _ = c_render.render(_PREP["gt"], _PREP["cams"][v])
    return v, img, dom, gt


def config_dict(wl, args, extra=None):
    d = {"workload": f"{wl.name}: slab-shaped synthetic {wl.n_gt // 2:,}-Gaussian init "
                     f"({wl.n_gt:,}-Gaussian GT), {wl.n_views} views {wl.width}x{wl.height}, full densify step",
         "n_gaussians": wl.n_gt // 2 + 1, "views": wl.n_views, "width": wl.width, "height": wl.height,
         "v_views": wl.n_views, "n_max": wl.n_max, "cfg": "paper defaults (ref/scene.py:151-163)",
         "rho": wl.rho, "stats": wl.stats_mode, "p_split": wl.p_split, "p_clone": wl.p_clone,
         "l2": "inputs larger than L2 (image+gt+dominant = 28 B/px x V x H x W)"}
    if extra:
        d.update(extra)
    return d


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def time_accumulate(dev, n, peak, launches=10):
    """accumulate_stats (ref/adc.py:73-79) on n Gaussians, one launch per view with
    fp32 viewspace gradients (a GPU rasterizer's): 41 B per Gaussian per view
    (vg 8 + visible 1 + grad_accum/denom read+write 32).  L2 is flushed before
    every launch; each launch is timed with events on the launching stream."""
    import torch

    from paper_2605_06876_b200 import operator as op
    gen = torch.Generator(device=dev).manual_seed(0)
    ga = torch.zeros(n, dtype=torch.float64, device=dev)
    den = torch.zeros(n, dtype=torch.float64, device=dev)
    vg = torch.randn(n, 2, device=dev, generator=gen)
    vis = torch.rand(n, device=dev, generator=gen) < 0.7
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(launches)]
    op.accumulate_stats_(ga, den, vg, vis)
    for e0, e1 in evs:
        flush.zero_()
        e0.record()
        op.accumulate_stats_(ga, den, vg, vis)
        e1.record()
    torch.cuda.synchronize(dev)
    ms = float(np.mean([e0.elapsed_time(e1) for e0, e1 in evs]))
    gbs = 41.0 * n / (ms * 1e-3) / 1e9
    return {"GB/s": gbs, "frac": gbs / peak, "ms_per_launch": ms, "n": n, "bytes_per_gaussian": 41,
            "note": "one launch per view, fp32 viewspace grads, L2 flushed before each launch"}


def time_accumulate_sharded(dev, n, n_views, world, rank, peak, max_over_ranks):
    """The sharded stat feed (sharded.accumulate_stats_sharded_): each rank
    accumulates its block of the n_views training views (fp32 viewspace
    gradients, one kernel per view) and one all_reduce(SUM) of the [2,n] fp64
    partials combines them.  Timed with events, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2605_06876_b200 import sharded as SH
    gen = torch.Generator(device=dev).manual_seed(rank)
    ga = torch.zeros(n, dtype=torch.float64, device=dev)
    den = torch.zeros(n, dtype=torch.float64, device=dev)
    vg = torch.randn(n, 2, device=dev, generator=gen)
    vis = torch.rand(n, device=dev, generator=gen) < 0.7
    lo, hi = SH.view_block(n_views, world, rank)
    views = [(vg, vis)] * (hi - lo)
    SH.accumulate_stats_sharded_(ga, den, views)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0.record()
    for _ in range(reps):
        SH.accumulate_stats_sharded_(ga, den, views)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = max_over_ranks(e0.elapsed_time(e1) / reps)
    gbs = 41.0 * n * n_views / (ms * 1e-3) / 1e9
    return {"ms_per_feed": ms, "views": n_views, "n": n, "GB/s": gbs, "frac_of_world_peak": gbs / (peak * world),
            "allreduce_bytes": 16 * n,
            "note": "per rank its block of views, one kernel per view, one all_reduce(SUM) of the [2,n] fp64 partials"}


def parity_on_sample(op, plan, wl, d, vs, cfg_k):
    """The GPU step and the oracle step on the same k sampled views (stage-isolated:
    the same GPU attribution into both); every integer output compared, near-
    threshold candidates reported (tests/parity.py)."""
    import torch
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import parity as PA
    from oracle import adpsplit_oracle as O
    ini, cams = d["ini"], d["cams"]
    ga, den = d["stats"]
    cams_k = cams[vs]
    rng_seed = 0
    # the k cameras are the step's camera list and v_views = k: both sides sample all
    # of them with the same Generator call (ref/adc.py:161), then draw the same normals
    gres = op.densify_step(d["g"], ini.extent, cams_k, d["gt_img"][vs[0]:vs[-1] + 1],
                           torch.as_tensor(ga, device=plan.device), torch.as_tensor(den, device=plan.device), cfg_k,
                           np.random.default_rng(rng_seed),
                           renders=(d["img"][vs[0]:vs[-1] + 1], d["dom"][vs[0]:vs[-1] + 1]), plan=plan)
    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    cam_objs = [O.Cam.from_row(r) for r in cams_k]
    renders = {k: (d["img"][v].double().cpu().numpy(), d["dom"][v].long().cpu().numpy()) for k, v in enumerate(vs)}
    gts = {k: d["gt_img"][v].double().cpu().numpy() for k, v in enumerate(vs)}
    t0 = time.perf_counter()
    ores = O.adpsplit_step(g, ini.extent, cam_objs, gts, ga, den, cfg_k, np.random.default_rng(rng_seed),
                           renders=renders)
    np.testing.assert_array_equal(PA.gpu_regions(plan), PA.oracle_regions(ores, list(range(len(vs)))))
    flagged = PA.flag_candidates(ores, g, cam_objs, cfg_k)
    st = PA.compare_step(gres, ores, flagged, g)
    return {"views": [int(v) for v in vs], "candidates": st["candidates"], "mismatched": st["mismatched"],
            "flagged": st["flagged"], "regions": int(gres.counts["n_regions"]),
            "rows_compared": st["rows_compared"], "max_rel_cov": st["max_rel_cov"],
            "max_rel_mu": st["max_rel_mu"], "oracle_s": time.perf_counter() - t0,
            "checked": "regions, cases, regions_per_view, proposals, N_i, merge_edges, clones, resets, "
                       "index_map, child_parent, insert offsets exact; child params within tolerance"}


def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    from paper_2605_06876_b200 import operator as op

    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    # ADPS_BENCH_BACKEND=gloo: a functional check of the multi-rank path with host
    # collectives (e.g. ranks sharing one GPU); numbers come from NCCL, one GPU per rank
    backend = os.environ.get("ADPS_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    if world > 1:
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    dev = torch.device("cuda", local if world > 1 else 0)

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    torch.cuda.set_device(dev)
    clocks = ClockSampler(index=dev.index)
    clocks.start()
    plan = op.Plan(dev)

    # ---- workload (seeded numpy scenes; GT images, attribution and statistics rendered on the device)
    t0 = time.time()
    d = wl.build_device(plan, seed=args.seed + (rank if args.replicas else 0))
    ini, cams, stats = d["ini"], d["cams"], d["stats"]
    g, gt_img = d["g"], d["gt_img"]
    ga = torch.as_tensor(stats[0], device=dev)
    den = torch.as_tensor(stats[1], device=dev)
    cfg = make_cfg(wl, len(cams))
    view_ids = list(range(len(cams)))       # v_views = all views of the config
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    # ---- attribution render of the sampled views (reported separately)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    img, dom = d["img"], d["dom"]
    torch.cuda.synchronize()
    ev0.record()
    img, dom = plan.render(g, cams[view_ids], out=(img, dom))
    ev1.record()
    torch.cuda.synchronize()
    render_ms = ev0.elapsed_time(ev1)

    sharded = world > 1 and not args.replicas
    if sharded:
        from paper_2605_06876_b200 import sharded as SH
        lo, hi = SH.view_block(len(view_ids), world, rank)

        def step_fn(gg, gt_, ga_, den_, rng, renders):
            return SH.densify_step_sharded(gg, ini.extent, cams, gt_, ga_, den_, cfg, rng, renders=renders,
                                           plan=plan, view_ids=view_ids, want_report=True, local_views=True)
        # each rank holds (and, e2e, copies in) only its own block of views
        img_l, dom_l, gt_l = img[lo:hi], dom[lo:hi], gt_img[lo:hi]
    else:
        def step_fn(gg, gt_, ga_, den_, rng, renders):
            return op.densify_step(gg, ini.extent, cams, gt_, ga_, den_, cfg, rng, renders=renders, plan=plan,
                                   view_ids=view_ids, want_report=True, one_sync=not args.two_call)
        img_l, dom_l, gt_l = img, dom, gt_img

    def step(rng=None):
        # the caller's Generator is an input of the step (ref/adc.py:154-161);
        # the timed loop hands in identically seeded ones made beforehand
        return step_fn(g, gt_l, ga, den, rng if rng is not None else np.random.default_rng((args.seed, 0)),
                       (img_l, dom_l))

    for _ in range(max(args.warmup, 1)):
        res = step()
    # ---- timed region: value
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    k0, l0 = plan.launch_count()
    tw0 = time.time()
    rngs = [np.random.default_rng((args.seed, 0)) for _ in range(args.steps)]
    ev0.record()
    for i in range(args.steps):
        res = step(rngs[i])
    ev1.record()
    torch.cuda.synchronize()
    tw1 = time.time()
    if world > 1:
        dist.barrier()
    clocks.window(tw0, tw1)
    k1, l1 = plan.launch_count()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        ms = max_over_ranks(ms)
    counts = res.counts
    n_split = counts["n_split"]
    pp = res.report_arrays["cand_proposals"].cpu().numpy()
    props_stats = {"max": int(pp.max()) if len(pp) else 0, "p99": float(np.percentile(pp, 99)) if len(pp) else 0,
                   "mean": float(pp.mean()) if len(pp) else 0, "over_96": int((pp > 96).sum()),
                   "total": int(pp.sum())}
    ns = max(n_split, 1)
    shares = {"split_candidates": n_split, "clone_candidates": counts["n_clone"],
              "adaptive": (n_split - counts["n_fallback"] - counts["n_reset"]) / ns,
              "fallback": counts["n_fallback"] / ns, "reset": counts["n_reset"] / ns}

    # ---- per-stage breakdown with CUDA events on the launching stream (each rank: its own views)
    stages = {}
    plan.set_timing(True)
    stage_acc = {}
    n_t = max(3, min(args.steps, 10))
    for _ in range(n_t):
        step()
        for k_, v_ in plan.stage_ms().items():
            stage_acc[k_] = stage_acc.get(k_, 0.0) + v_
    plan.set_timing(False)
    stages = {k_: v_ / n_t for k_, v_ in stage_acc.items()}

    V, H, W = len(view_ids), wl.height, wl.width
    px = V * H * W
    px_local = (hi - lo) * H * W if sharded else px   # the input pass of this rank
    peak, peak_kind = load_peaks()
    tile_ms = stages.get("tile_ccl", float("nan"))
    mm_ms = stages.get("minmax", float("nan"))
    # stat-accum: 28 B/px over the attribution stages (maps, partition, stats)
    attr_ms = sum(stages.get(k_, 0) for k_ in ("minmax", "thresholds", "tile_ccl", "border_merge"))
    achieved = BYTES_PER_PX * px_local / (mm_ms * 1e-3) / 1e9 if stages.get("minmax") else None
    traffic = load_traffic(wl.name)
    b_step = BYTES_PER_PX * px + BYTES_PER_G_IN * g.n + BYTES_PER_G_OUT * counts["n_out"]
    acc = time_accumulate(dev, g.n, peak) if rank == 0 else None
    acc_sh = None
    if world > 1:   # the sharded stat feed: views over ranks, one all_reduce
        try:
            acc_sh = time_accumulate_sharded(dev, g.n, len(view_ids), world, rank, peak, max_over_ranks)
        except Exception as exc:   # reported, never fatal for the bench line
            acc_sh = {"error": repr(exc)[:200]}

    # ---- K1-epilogue variant (reported separately): the render's
    #      epilogue runs select and the input pass, the step starts from the
    #      6 B/px boundary (16-bit raw cache + dominant map); 1 GPU
    fused = None
    if world == 1 and not args.no_fused:
        gt_v = gt_img   # all views sampled (contiguous): the step's own gt tensor
        img_f = torch.empty_like(img)
        dom_f = torch.empty_like(dom)

        def fused_render():
            return plan.render_fused(g, ini.extent, ga, den, cfg, cams[view_ids], gt_v, out=(img_f, dom_f))

        def fused_step():
            return op.densify_step(g, ini.extent, cams, gt_l, ga, den, cfg, np.random.default_rng((args.seed, 0)),
                                   renders=(img_f, dom_f), plan=plan, view_ids=view_ids, want_report=True,
                                   one_sync=not args.two_call)

        for _ in range(2):
            fused_render()
            rf = fused_step()
        assert rf.counts["n_out"] == counts["n_out"] and rf.counts["n_regions"] == counts["n_regions"]
        n_f = max(3, min(args.steps, 10))
        r_ms, s_ms = [], []
        for _ in range(n_f):
            e_a, e_b, e_c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e_a.record()
            fused_render()
            e_b.record()
            fused_step()
            e_c.record()
            torch.cuda.synchronize()
            r_ms.append(e_a.elapsed_time(e_b))
            s_ms.append(e_b.elapsed_time(e_c))
        fr, fs = float(np.mean(r_ms)), float(np.mean(s_ms))
        b8 = 6 * px + BYTES_PER_G_IN * g.n + BYTES_PER_G_OUT * counts["n_out"]
        fused = {"render_ms": fr, "render_ms_plain": render_ms, "step_ms": fs,
                 "parents_per_s": n_split / (fs * 1e-3), "full_step_ms": fr + fs,
                 "full_step_parents_per_s": n_split / ((fr + fs) * 1e-3),
                 "step_bytes": int(b8), "step_roofline_frac": b8 / (fs * 1e-3) / 1e9 / peak,
                 "note": "render epilogue = select + input pass (raw L1 fp64, per-view min/max, candidate bits, "
                         "ever-dominant flags); step from the 6 B/px boundary (16-bit raw cache + dominant map); "
                         "identical results (tests/test_gpu_rows.py)"}

    # ---- e2e: same step through the API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        host = {k_: t_.cpu().pin_memory() for k_, t_ in
                dict(mu=g.mu, scale=g.scale, rot=g.rot, opacity=g.opacity, sh_dc=g.sh_dc, ga=ga, den=den,
                     img=img_l, gt=gt_l, dom=dom_l).items()}
        h2d = sum(t_.numel() * t_.element_size() for t_ in host.values())
        n_out = counts["n_out"]
        out_h = {k_: torch.empty((n_out,) + tuple(s_), dtype=torch.float32).pin_memory()
                 for k_, s_ in dict(mu=(3,), scale=(3,), rot=(4,), opacity=(), sh_dc=(3,)).items()}
        im_h = torch.empty(n_out, dtype=torch.int64).pin_memory()
        d2h = sum(t_.numel() * t_.element_size() for t_ in out_h.values()) + im_h.numel() * 8

        def e2e_step(rng=None):
            dd = {k_: t_.to(dev, non_blocking=True) for k_, t_ in host.items()}
            gg = op.GaussianTensors(dd["mu"], dd["scale"], dd["rot"], dd["opacity"], dd["sh_dc"])
            r = step_fn(gg, dd["gt"], dd["ga"], dd["den"],
                        rng if rng is not None else np.random.default_rng((args.seed, 0)), (dd["img"], dd["dom"]))
            for k_ in out_h:
                out_h[k_].copy_(getattr(r.gaussians, k_), non_blocking=True)
            im_h.copy_(r.index_map, non_blocking=True)
            return r

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        n_e = max(2, min(args.steps, 5))
        rngs_e = [np.random.default_rng((args.seed, 0)) for _ in range(n_e)]
        ev0.record()
        for i in range(n_e):
            e2e_step(rngs_e[i])
        ev1.record()
        torch.cuda.synchronize()
        serial_ms = ev0.elapsed_time(ev1) / n_e

        # the same steps as a serving loop would run them: step i+1's inputs
        # copied in (copy stream, second device buffer) while step i computes,
        # and step i's results copied out (a D2H stream; PCIe is full duplex)
        # while step i+1's inputs come in.  Every step still moves all of its
        # inputs in and its results out inside the timed region.
        cur_s = torch.cuda.current_stream()
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        slots = [{k_: torch.empty_like(t_, device=dev) for k_, t_ in host.items()} for _ in range(2)]
        done = [None, None]   # compute finished with the slot (its buffers may be overwritten)

        def copy_in(slot):
            with torch.cuda.stream(s_in):
                if done[slot] is not None:
                    s_in.wait_event(done[slot])
                for k_, t_ in host.items():
                    slots[slot][k_].copy_(t_, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s_in)
            return ev

        def pipelined(n, rngs):
            ready = copy_in(0)
            for i in range(n):
                slot = i & 1
                nxt = copy_in(slot ^ 1) if i + 1 < n else None   # queued before this step's host waits
                cur_s.wait_event(ready)
                dd = slots[slot]
                gg = op.GaussianTensors(dd["mu"], dd["scale"], dd["rot"], dd["opacity"], dd["sh_dc"])
                r = step_fn(gg, dd["gt"], dd["ga"], dd["den"], rngs[i], (dd["img"], dd["dom"]))
                fin = torch.cuda.Event()
                fin.record(cur_s)
                done[slot] = fin
                with torch.cuda.stream(s_out):
                    s_out.wait_event(fin)
                    for k_ in out_h:
                        src = getattr(r.gaussians, k_)
                        out_h[k_].copy_(src, non_blocking=True)
                        src.record_stream(s_out)   # its memory is not reused before the copy-out ran
                    im_h.copy_(r.index_map, non_blocking=True)
                    r.index_map.record_stream(s_out)
                ready = nxt
            cur_s.wait_stream(s_out)

        n_p = max(4, min(args.steps, 8))
        pipelined(n_p, [np.random.default_rng((args.seed, 0)) for _ in range(n_p)])   # warm the allocator
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        rngs_p = [np.random.default_rng((args.seed, 0)) for _ in range(n_p)]
        ev0.record()
        pipelined(n_p, rngs_p)
        ev1.record()
        torch.cuda.synchronize()
        e2e_ms = ev0.elapsed_time(ev1) / n_p
        del slots
        if world > 1:
            e2e_ms = max_over_ranks(e2e_ms)
            serial_ms = max_over_ranks(serial_ms)
        e2e = {"value": n_split / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": n_p, "serial_ms_per_step": serial_ms,
               "note": ("per rank: params + stats + its own block of views in, grown params + index_map out"
                        if world > 1 else "params + stats + all views in, grown params + index_map out") +
                       "; steps pipelined: step i+1's copy-in and step i's copy-out overlap step i's compute "
                       "(serial_ms_per_step: one step at a time)"}
        del host

    # ---- full step incl. the attribution render
    full_ms = render_ms + ms
    clocks.stop()
    clk = clocks.summary()

    # ---- CPU baseline + parity on the same sample (rank 0, N = 1)
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        k = max(1, args.cpu_views)
        vs = view_ids[:k]
        renders = {v: (img[v].double().cpu().numpy(), dom[v].long().cpu().numpy()) for v in vs}
        gts = {v: gt_img[v].double().cpu().numpy() for v in vs}
        info = cpu_sample(wl, ini, cams, stats, vs, workers=1, renders=renders, gts=gts,
                          cand_frac=args.cpu_cand_frac)
        cpu = {"value": info["n_split"] / info["extrapolated_step_s"], "unit": UNIT, "cores": 1,
               "host_cores": host_cores(), "kind": "port",
               "sample": (f"oracle port (numpy, 1 of {host_cores()} host cores) on {k} of {V} views of the "
                          f"same step inputs, merge/cap/emit on {info['parents_merged']} of "
                          f"{info['parents_with_proposals']} parents with proposals; per-view + per-parent "
                          f"stages timed and extrapolated linearly to all parents and V={V} "
                          f"(sample wall {info['sample_wall_s']:.1f} s)"),
               "step_s_extrapolated": info["extrapolated_step_s"], "stages_s": info["stages_s"]}
        if not args.no_parity:
            parity = parity_on_sample(op, plan, wl, d, vs, make_cfg(wl, k))

    if rank == 0:
        extra = {"dc_gt": d["dc_gt"], "dc_init": d["dc_init"], "shares": shares,
                 "parallelism": (f"replicas x{world}" if args.replicas else
                                 f"views and parents sharded over {world} ranks") if world > 1 else "single GPU"}
        line = {
            "metric": METRIC, "value": n_split * world / (ms * 1e-3) if args.replicas else n_split / (ms * 1e-3),
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak" if args.replicas else "strong", "vs_baseline": None,
            "dtype": "f64+i64 (decisions), fp32 (params)", "data": "synthetic",
            "config": config_dict(wl, args, extra),
            "densify_step_ms": ms,
            "stat_accum": {"GB/s": BYTES_PER_PX * px_local / (attr_ms * 1e-3) / 1e9 if attr_ms else None,
                           "frac": None, "ms": attr_ms},
            "accumulate_stats": acc,
            "accumulate_stats_sharded": acc_sh,
            "step_roofline": {"bytes": int(b_step), "GB/s": b_step / (ms * 1e-3) / 1e9,
                              "frac": b_step / (ms * 1e-3) / 1e9 / peak},
            "roofline": {"bound": "hbm", "kernel": "minmax2_kernel (input pass: raw L1 error, per-view min/max, "
                                                    "ever-dominant flags, candidate bits, 16-bit raw cache)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "algorithmic_bytes_per_launch": BYTES_PER_PX * px_local, "ms_per_launch": mm_ms,
                         "note": "achieved counts the 28 B/px inputs only; traffic = ncu dram read+write of one "
                                 "launch (incl. the 2.125 B/px caches it writes), profiles/"},
            "tile_pass": {"ms": tile_ms, "kernels": "tile_words_kernel (HBM) + tile_bits_kernel (latency-bound CCL)",
                          "words_bytes_per_launch": WORDS_BYTES_PER_PX * px},
            "stages_ms": stages,
            "render": {"ms_per_view": render_ms / V, "ms_total": render_ms, "views": V,
                       "splat_px_per_s": d["dc_init"] * px / (render_ms * 1e-3),
                       "note": "attribution render (compute-bound), not part of value; splat-px = (pixel, splat) "
                               "pairs with alpha >= 1/255 (measured depth complexity x pixels)"},
            "full_step": {"ms": full_ms, "parents_per_s": n_split / (full_ms * 1e-3)},
            "fused_epilogue": fused,
            "counts": counts,
            "proposals_per_parent": props_stats,
            "e2e": e2e,
            "gpu_launches": int((k1 - k0) / args.steps),
            "library_sort_calls_per_step": (l1 - l0) / args.steps,
            "clocks": clk,
            "cpu_baseline": cpu,
            "parity": parity,
            "setup_s": setup_s,
        }
        if line["stat_accum"]["GB/s"]:
            line["stat_accum"]["frac"] = line["stat_accum"]["GB/s"] / peak
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _free_port():
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        return s_.getsockname()[1]


def _spawn_ranks(args):
    """--gpus N without torchrun: re-exec under torch.distributed.run, one rank per GPU."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but only {have} GPU(s) visible"}),
              flush=True)
        raise SystemExit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="config3")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-views", type=int, default=2)
    ap.add_argument("--ref-views", type=int, default=8)
    ap.add_argument("--ref-cand-frac", type=float, default=1.0)
    ap.add_argument("--cpu-cand-frac", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity check on the cpu sample")
    ap.add_argument("--no-fused", action="store_true", help="skip the K1-epilogue (fused render) variant")
    ap.add_argument("--two-call", action="store_true",
                    help="phase 1 end and phase 2 as two calls (the emit after the host read the counts)")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas (weak scaling) instead of the view-sharded step")
    args = ap.parse_args()
    from paper_2605_06876_b200.synth import CONFIGS
    wl = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, wl)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _spawn_ranks(args)
    run_ours(args, wl)


if __name__ == "__main__":
    main()
