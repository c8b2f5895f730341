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
            traffic = its ncu dram bytes (it also writes the 4.125 B/px
            fp32 raw-error cache and candidate bits).  "tile_pass" reports the
            bit-plane pass (tile_words_kernel, HBM: 4.125 B/px read) and the
            warp CCL (tile_bits_kernel, latency-bound) that follow.
  cpu_baseline  the oracle port on a bounded view sample (rank 0, N=1)

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: launched by torchrun, one rank per GPU.
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
WORDS_BYTES_PER_PX = 4 + 0.125 + 0.5   # bit-plane pass: fp32 raw cache + candidate bits read, 4 bit planes written
MINMAX_TRAFFIC_PER_PX = 28 + 4 + 0.125   # minmax pass: inputs read once, fp32 raw cache + candidate bits written
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


def make_cfg(wl, v_views):
    from paper_2605_06876_b200.types import AdpSplitConfig
    return AdpSplitConfig(v_views=v_views, n_max=wl.n_max)


# ---------------------------------------------------------------------------
# CPU side (oracle port): cpu_baseline leg and --impl reference arm
# ---------------------------------------------------------------------------

def cpu_sample(wl, ini, cams, stats, gt_scene, view_ids, workers, renders=None, gts=None, cand_frac=1.0):
    from oracle import adpsplit_oracle as O
    from oracle import c_render
    from oracle.cpu_baseline import time_sample

    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    cam_objs = [O.Cam.from_row(r) for r in cams]
    if renders is None:
        gt_g = O.Gaussians(gt_scene.mu, gt_scene.scale, gt_scene.rot, gt_scene.opacity, gt_scene.sh_dc)
        renders, gts = {}, {}
        for v in view_ids:
            renders[v] = c_render.render(g, cams[v])
            gts[v] = c_render.render(gt_g, cams[v])[0]
    cfg = make_cfg(wl, len(cams))
    return time_sample(g, ini.extent, cam_objs, view_ids, renders, gts, stats[0], stats[1], cfg,
                       n_views_total=len(cams), workers=workers, cand_frac=cand_frac)


def run_reference(args, wl):
    """--impl reference: the oracle port on the box's host cores (rank 0 only)."""
    world, rank, _ = dist_env()
    if world > 1 and rank != 0:
        return
    import multiprocessing as mp

    from oracle import c_render
    from oracle import adpsplit_oracle as O

    c_render.build()
    ini, cams, stats, gt_scene = wl.build()
    cores = os.cpu_count() or 1
    k = max(1, min(cores, args.ref_views))
    # inputs for all k views (untimed preparation), rendered by the C oracle in parallel
    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    gt_g = O.Gaussians(gt_scene.mu, gt_scene.scale, gt_scene.rot, gt_scene.opacity, gt_scene.sh_dc)
    _PREP.update(g=g, gt=gt_g, cams=cams)
    views = list(range(k))
    with mp.get_context("fork").Pool(min(k, cores)) as pool:
        outs = pool.map(_prep_view, views)
    renders = {v: (img, dom) for v, img, dom, _ in outs}
    gts = {v: gt for v, _, _, gt in outs}
    times = []
    info = None
    for it in range(args.warmup + args.steps):
        info = cpu_sample(wl, ini, cams, stats, gt_scene, views, workers=min(k, cores), renders=renders, gts=gts,
                          cand_frac=args.ref_cand_frac)
        if it >= args.warmup:
            times.append(info["extrapolated_step_s"])
    t = float(np.mean(times))
    value = info["n_split"] / t
    sample = (f"oracle port: {k} of {len(cams)} views per step ({min(k, cores)} worker processes), "
              f"per-view stages timed on all parents, merge/cap/emit on every "
              f"{int(round(1 / args.ref_cand_frac))}th parent with proposals "
              f"({info['parents_merged']} of {info['parents_with_proposals']}), extrapolated linearly "
              f"to all parents and to V={len(cams)}; {info['n_regions']} regions, "
              f"{info['n_proposals']} proposals in the sample")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(wl, args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(k, cores), "kind": "port",
                             "sample": sample, "stages_s": info["stages_s"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


_PREP = {}


def _prep_view(v):
    from oracle import c_render
    img, dom = c_render.render(_PREP["g"], _PREP["cams"][v])
    gt, _ = c_render.render(_PREP["gt"], _PREP["cams"][v])
    return v, img, dom, gt


def config_dict(wl, args):
    return {"workload": f"{wl.name}: bonsai-shaped synthetic {wl.n_gt // 2:,}-Gaussian init "
                        f"({wl.n_gt:,}-Gaussian GT), {wl.n_views} views {wl.width}x{wl.height}, full densify step",
            "n_gaussians": wl.n_gt // 2 + 1, "views": wl.n_views, "width": wl.width, "height": wl.height,
            "v_views": wl.n_views, "n_max": wl.n_max, "cfg": "paper defaults (ref/scene.py:151-163)",
            "l2": "inputs larger than L2 (image+gt+dominant = 28 B/px x V x H x W)"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    from paper_2605_06876_b200 import operator as op

    world, rank, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    clocks = ClockSampler(index=dev.index)
    clocks.start()
    plan = op.Plan(dev)

    # ---- workload (seeded numpy), GT images rendered by the operator's own render
    t0 = time.time()
    ini, cams, stats, gt_scene = wl.build(seed=args.seed + (rank if args.replicas else 0))
    g = op.GaussianTensors.from_numpy(*ini.arrays(), device=dev)
    gt_g = op.GaussianTensors.from_numpy(*gt_scene.arrays(), device=dev)
    gt_img, _ = plan.render(gt_g, cams)
    del gt_g
    ga = torch.as_tensor(stats[0], device=dev)
    den = torch.as_tensor(stats[1], device=dev)
    cfg = make_cfg(wl, len(cams))
    view_ids = list(range(len(cams)))       # v_views = all views of the config
    torch.cuda.synchronize()
    setup_s = time.time() - t0

    # ---- attribution render of the sampled views (reported separately)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    img, dom = plan.render(g, cams[view_ids])
    torch.cuda.synchronize()
    ev0.record()
    img, dom = plan.render(g, cams[view_ids], out=(img, dom))
    ev1.record()
    torch.cuda.synchronize()
    render_ms = ev0.elapsed_time(ev1)

    sharded = world > 1 and not args.replicas
    if sharded:
        from paper_2605_06876_b200 import sharded as SH
        step_fn = SH.densify_step_sharded   # views sharded over ranks, records gathered
    else:
        step_fn = op.densify_step

    def step():
        rng = np.random.default_rng((args.seed, 0))
        return step_fn(g, ini.extent, cams, gt_img, ga, den, cfg, rng, renders=(img, dom),
                       plan=plan, view_ids=view_ids, want_report=True)

    for _ in range(max(args.warmup, 1)):
        res = step()
    # ---- timed region: value
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    k0, l0 = plan.launch_count()
    tw0 = time.time()
    ev0.record()
    for _ in range(args.steps):
        res = step()
    ev1.record()
    torch.cuda.synchronize()
    tw1 = time.time()
    if world > 1:
        dist.barrier()
    clocks.window(tw0, tw1)
    k1, l1 = plan.launch_count()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    counts = res.counts
    n_split = counts["n_split"]
    pp = res.report_arrays["cand_proposals"].cpu().numpy()
    props_stats = {"max": int(pp.max()) if len(pp) else 0, "p99": float(np.percentile(pp, 99)) if len(pp) else 0,
                   "mean": float(pp.mean()) if len(pp) else 0, "over_96": int((pp > 96).sum()),
                   "total": int(pp.sum())}

    # ---- per-stage breakdown with CUDA events on the launching stream
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
    peak, peak_kind = load_peaks()
    tile_ms = stages.get("tile_ccl", float("nan"))
    mm_ms = stages.get("minmax", float("nan"))
    # stat-accum: 28 B/px over the attribution stages (maps, partition, stats)
    attr_ms = sum(stages.get(k_, 0) for k_ in ("minmax", "thresholds", "tile_ccl", "border_merge"))
    achieved = BYTES_PER_PX * px / (mm_ms * 1e-3) / 1e9
    traffic = load_traffic(wl.name)
    b_step = BYTES_PER_PX * px + BYTES_PER_G_IN * g.n + BYTES_PER_G_OUT * counts["n_out"]

    # ---- e2e: same step through the API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        host = {k_: t_.cpu().pin_memory() for k_, t_ in
                dict(mu=g.mu, scale=g.scale, rot=g.rot, opacity=g.opacity, sh_dc=g.sh_dc, ga=ga, den=den,
                     img=img, gt=gt_img, dom=dom).items()}
        h2d = sum(t_.numel() * t_.element_size() for t_ in host.values())
        n_out = counts["n_out"]
        out_h = {k_: torch.empty((n_out,) + tuple(s), dtype=torch.float32).pin_memory()
                 for k_, s in dict(mu=(3,), scale=(3,), rot=(4,), opacity=(), sh_dc=(3,)).items()}
        im_h = torch.empty(n_out, dtype=torch.int64).pin_memory()
        d2h = sum(t_.numel() * t_.element_size() for t_ in out_h.values()) + im_h.numel() * 8

        def e2e_step():
            d = {k_: t_.to(dev, non_blocking=True) for k_, t_ in host.items()}
            gg = op.GaussianTensors(d["mu"], d["scale"], d["rot"], d["opacity"], d["sh_dc"])
            r = step_fn(gg, ini.extent, cams, d["gt"], d["ga"], d["den"], cfg,
                        np.random.default_rng((args.seed, 0)), renders=(d["img"], d["dom"]), plan=plan,
                        view_ids=view_ids, want_report=True)
            for k_ in out_h:
                out_h[k_].copy_(getattr(r.gaussians, k_), non_blocking=True)
            im_h.copy_(r.index_map, non_blocking=True)
            return r

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        n_e = max(2, min(args.steps, 5))
        ev0.record()
        for _ in range(n_e):
            e2e_step()
        ev1.record()
        torch.cuda.synchronize()
        e2e_ms = ev0.elapsed_time(ev1) / n_e
        e2e = {"value": n_split / (e2e_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}
        del host

    # ---- full step incl. the attribution render
    full_ms = render_ms + ms
    clocks.stop()
    clk = clocks.summary()

    # ---- CPU baseline (rank 0, N = 1): oracle port on GPU-produced inputs of k views
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        k = max(1, args.cpu_views)
        vs = view_ids[:k]
        renders = {v: (img[v].double().cpu().numpy(), dom[v].long().cpu().numpy()) for v in vs}
        gts = {v: gt_img[v].double().cpu().numpy() for v in vs}
        info = cpu_sample(wl, ini, cams, stats, gt_scene, vs, workers=1, renders=renders, gts=gts,
                          cand_frac=args.cpu_cand_frac)
        cpu = {"value": info["n_split"] / info["extrapolated_step_s"], "unit": UNIT, "cores": 1, "kind": "port",
               "sample": (f"oracle port (numpy, 1 thread) on {k} of {V} views of the same step inputs, "
                          f"merge/cap/emit on {info['parents_merged']} of {info['parents_with_proposals']} "
                          f"parents with proposals; per-view + per-parent stages timed and extrapolated "
                          f"linearly to all parents and V={V} "
                          f"(sample wall {info['sample_wall_s']:.1f} s; host has {os.cpu_count()} cores)"),
               "step_s_extrapolated": info["extrapolated_step_s"], "stages_s": info["stages_s"]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": n_split * world / (ms * 1e-3) if args.replicas else n_split / (ms * 1e-3),
            "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak" if args.replicas else "strong", "vs_baseline": None,
            "dtype": "f64+i64 (decisions), fp32 (params)", "data": "synthetic", "config": config_dict(wl, args),
            "densify_step_ms": ms,
            "stat_accum": {"GB/s": BYTES_PER_PX * px / (attr_ms * 1e-3) / 1e9, "frac": None, "ms": attr_ms},
            "step_roofline": {"bytes": int(b_step), "GB/s": b_step / (ms * 1e-3) / 1e9,
                              "frac": b_step / (ms * 1e-3) / 1e9 / peak},
            "roofline": {"bound": "hbm", "kernel": "minmax_kernel (input pass: raw L1 error, per-view min/max, "
                                                    "ever-dominant flags, candidate bits, fp32 raw cache)",
                         "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": BYTES_PER_PX * px, "ms_per_launch": mm_ms,
                         "note": "achieved counts the 28 B/px inputs only; traffic = ncu dram read+write of one "
                                 "launch (incl. the 4.125 B/px cache it writes), profiles/"},
            "tile_pass": {"ms": tile_ms, "kernels": "tile_words_kernel (HBM) + tile_bits_kernel (latency-bound CCL)",
                          "words_bytes_per_launch": WORDS_BYTES_PER_PX * px},
            "stages_ms": stages,
            "render": {"ms_per_view": render_ms / V, "ms_total": render_ms, "views": V,
                       "note": "attribution render (compute-bound), not part of value"},
            "full_step": {"ms": full_ms, "parents_per_s": n_split / (full_ms * 1e-3)},
            "counts": counts,
            "proposals_per_parent": props_stats,
            "e2e": e2e,
            "gpu_launches": int((k1 - k0) / args.steps),
            "library_sort_calls_per_step": (l1 - l0) / args.steps,
            "clocks": clk,
            "cpu_baseline": cpu,
            "setup_s": setup_s,
        }
        line["stat_accum"]["frac"] = line["stat_accum"]["GB/s"] / peak
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


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
    ap.add_argument("--ref-cand-frac", type=float, default=0.125)
    ap.add_argument("--cpu-cand-frac", type=float, default=0.5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N>1: independent replicas (weak scaling) instead of the view-sharded step")
    args = ap.parse_args()
    from paper_2605_06876_b200.synth import CONFIGS
    wl = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
