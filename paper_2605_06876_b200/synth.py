"""Seeded synthetic workloads of the BASELINE configs (numpy; host-side).

Distribution follows the reference's synthetic harness
(ref/harness.py:99-210: flat slab of Gaussians, ring of cameras at
elevation 0.9 rad, 50 % subset init with inflated scales plus one dim cover
Gaussian) with one change the survey calls for:
splat size shrinks as 1/sqrt(k) so the mean depth complexity stays fixed
as the Gaussian count grows to millions (the reference's fixed sizes leave
almost every Gaussian occluded at scale).  A log-normal size spread keeps a
realistic share of Gaussians above the split-scale gate tau_s*extent.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SH_C0 = 0.28209479177387814


@dataclass
class SynthScene:
    mu: np.ndarray
    scale: np.ndarray
    rot: np.ndarray
    opacity: np.ndarray
    sh_dc: np.ndarray
    extent: float

    @property
    def n(self):
        return len(self.mu)

    def arrays(self):
        return self.mu, self.scale, self.rot, self.opacity, self.sh_dc


def _look_at(eye, target, world_up):
    """ref/harness.py:99-107: columns right, down, forward."""
    fwd = target - eye
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(-np.asarray(world_up, dtype=np.float64), fwd)
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    return np.stack([right, down, fwd], axis=1)


def ring_cameras(n_cams: int, width: int, height: int, extent: float = 1.0, elev: float = 0.9) -> np.ndarray:
    """Camera ring of ref/harness.py:140-166 for a W x H image -> [C,18] rows."""
    dist = 2.6 * extent
    f = 0.55 * min(width, height) * dist / extent
    rows = []
    for i in range(n_cams):
        ang = 2 * np.pi * i / n_cams
        eye = dist * np.array([np.cos(ang) * np.cos(elev), np.sin(ang) * np.cos(elev), np.sin(elev)])
        r = _look_at(eye, np.zeros(3), (0.0, 0.0, 1.0))
        rows.append(np.concatenate([r.ravel(), eye, [f, f, (width - 1) / 2.0, (height - 1) / 2.0,
                                                    width, height]]))
    return np.array(rows)


def gt_scene(k: int, seed: int, size_factor: float = 1.0, spread: float = 0.0,
             large_frac: float = 0.0, large_range=(0.005, 0.01)) -> SynthScene:
    """GT scene like ref/harness.py:110-138.

    Base size U(.04,.10) x size_factor x lognormal(spread); a fraction
    ``large_frac`` instead gets base U(large_range) (world units, before the
    init inflation) so that a realistic share clears the split gate.
    """
    rng = np.random.default_rng(seed)
    mu = np.stack([rng.uniform(-0.75, 0.75, k), rng.uniform(-0.75, 0.75, k), rng.uniform(-0.12, 0.12, k)], 1)
    base = rng.uniform(0.04, 0.10, k) * size_factor
    if spread > 0:
        base = base * np.exp(rng.normal(0.0, spread, k))
    aniso = rng.uniform(0.4, 1.0, (k, 3))
    if large_frac > 0:
        large = rng.uniform(size=k) < large_frac
        base = np.where(large, rng.uniform(large_range[0], large_range[1], k) / aniso.max(axis=1), base)
    q = rng.standard_normal((k, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    opacity = rng.uniform(0.65, 0.95, k)
    sh_dc = (rng.uniform(0.15, 0.85, (k, 3)) - 0.5) / SH_C0
    scale = base[:, None] * aniso
    radii = np.linalg.norm(mu, axis=1) + scale.max(axis=1)
    extent = max(1.0, float(radii.max()))
    return SynthScene(mu, scale, q, opacity, sh_dc, extent)


def init_scene(gt: SynthScene, seed: int, fraction: float = 0.5, inflate: float = 2.0,
               cover: bool = True) -> SynthScene:
    """Perturbed inflated subset plus a cover Gaussian (ref/harness.py:172-210)."""
    rng = np.random.default_rng((seed, 0xC0FFEE))
    k = gt.n
    n = max(1, int(round(fraction * k)))
    chosen = np.sort(rng.choice(k, size=n, replace=False))
    mu = gt.mu[chosen] + rng.normal(0.0, 0.01 * gt.extent, (n, 3))
    parts = [mu, gt.scale[chosen] * inflate, gt.rot[chosen], gt.opacity[chosen], gt.sh_dc[chosen]]
    if cover:
        parts = [np.concatenate([parts[0], np.zeros((1, 3))]),
                 np.concatenate([parts[1], np.full((1, 3), 0.6 * gt.extent)]),
                 np.concatenate([parts[2], [[1.0, 0.0, 0.0, 0.0]]]),
                 np.concatenate([parts[3], [0.3]]),
                 np.concatenate([parts[4], np.zeros((1, 3))])]
    return SynthScene(*parts, extent=gt.extent)


def synth_stats(scale: np.ndarray, extent: float, tau_g: float, tau_s: float, p_split: float,
                p_clone: float, seed: int):
    """DensifyStats (denom = 1) whose select() yields ~p_split*N split and ~p_clone*N
    clone candidates (ref/adc.py:82-89): g = tau_g*exp(|z|) for the chosen
    Gaussians, tau_g*exp(-|z|-1e-3) for the rest."""
    rng = np.random.default_rng((seed, 0x57A75))
    n = len(scale)
    large = scale.max(axis=1) > tau_s * extent
    high = np.zeros(n, dtype=bool)
    li, si = np.flatnonzero(large), np.flatnonzero(~large)
    high[rng.choice(li, size=min(len(li), int(round(p_split * n))), replace=False)] = True
    high[rng.choice(si, size=min(len(si), int(round(p_clone * n))), replace=False)] = True
    z = np.abs(rng.standard_normal(n))
    ga = np.where(high, tau_g * np.exp(z), tau_g * np.exp(-z - 1e-3))
    return ga, np.ones(n)


def synth_stats_weighted(scale: np.ndarray, extent: float, tau_g: float, tau_s: float, p_split: float,
                         p_clone: float, weight: np.ndarray, floor: float, seed: int):
    """DensifyStats whose candidates follow the Gaussians' rendered contribution.

    In training, ``accumulate_stats`` credits a Gaussian only in views where it
    is visible (ref/adc.py:73-79) and its view-space gradient scales with its
    blending weight T*alpha over the pixels it covers, so high-gradient
    Gaussians are the ones the renders actually use.  Candidates are drawn
    without replacement (Efraimidis-Spirakis keys) with probability
    proportional to weight + floor * mean(weight) among the large (split) and
    the small (clone) Gaussians; ``floor`` keeps stale, occluded Gaussians in
    play.  g = tau_g*exp(|z|) for the drawn ones, tau_g*exp(-|z|-1e-3) else."""
    rng = np.random.default_rng((seed, 0x57A75))
    n = len(scale)
    w = np.asarray(weight, dtype=np.float64)
    large = scale.max(axis=1) > tau_s * extent
    high = np.zeros(n, dtype=bool)
    for sel, p in ((large, p_split), (~large, p_clone)):
        idx = np.flatnonzero(sel)
        k = min(len(idx), int(round(p * n)))
        if k == 0:
            continue
        wi = w[idx] + floor * max(float(w[idx].mean()), 1e-30)
        keys = np.log(rng.uniform(size=len(idx))) / wi
        high[idx[np.argpartition(-keys, k - 1)[:k]]] = True
    z = np.abs(rng.standard_normal(n))
    ga = np.where(high, tau_g * np.exp(z), tau_g * np.exp(-z - 1e-3))
    return ga, np.ones(n)


def rho_of(size_factor: float, k_gt: int) -> float:
    """SURVEY.md 8(d)'s density parameter: base = U(.04,.10) * sqrt(32 rho / k_gt)."""
    return size_factor ** 2 * k_gt / 32.0


def round_f32(s: SynthScene) -> SynthScene:
    """Round parameters to fp32 (what the device stores), renormalising quaternions in fp32."""
    q = s.rot.astype(np.float32)
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    return SynthScene(s.mu.astype(np.float32).astype(np.float64),
                      s.scale.astype(np.float32).astype(np.float64),
                      q.astype(np.float32).astype(np.float64),
                      s.opacity.astype(np.float32).astype(np.float64),
                      s.sh_dc.astype(np.float32).astype(np.float64), s.extent)


def _quat_rot(q):
    q = q / np.linalg.norm(q, axis=1, keepdims=True)
    w, x, y, z = q.T
    return np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                     2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                     2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], axis=1).reshape(-1, 3, 3)


def depth_complexity(s: SynthScene, cam_row, alpha_min=1.0 / 255) -> float:
    """Mean number of splats with alpha >= alpha_min per pixel of one view.

    Exact per-splat footprint of the reference's render (ref/raster.py:66-93):
    alpha = min(.99, o) exp(-q/2) >= alpha_min inside the conic ellipse
    q <= 2 ln(min(o,.99)/alpha_min) of the projected covariance
    J W Sigma W^T J^T + 0.3 I, whose area is pi * 2 ln(.) * sqrt(det).  Summed
    over the splats in front of the camera whose centre projects into the
    image, divided by W*H (border clipping ignored)."""
    r = cam_row[0:9].reshape(3, 3)
    c = cam_row[9:12]
    fx, fy, px, py, w, h = cam_row[12], cam_row[13], cam_row[14], cam_row[15], cam_row[16], cam_row[17]
    p = (s.mu - c) @ r
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    ok = z > 1e-8
    mx, my = fx * x / np.where(ok, z, 1) + px, fy * y / np.where(ok, z, 1) + py
    ok &= (mx >= 0) & (mx <= w - 1) & (my >= 0) & (my <= h - 1)
    R = _quat_rot(s.rot[ok])
    S = np.einsum("nij,nj,nkj->nik", R, s.scale[ok] ** 2, R)
    zz = z[ok]
    J = np.zeros((len(zz), 2, 3))
    J[:, 0, 0] = fx / zz
    J[:, 0, 2] = -fx * x[ok] / zz ** 2
    J[:, 1, 1] = fy / zz
    J[:, 1, 2] = -fy * y[ok] / zz ** 2
    T = J @ r.T
    cov = T @ S @ np.transpose(T, (0, 2, 1)) + 0.3 * np.eye(2)
    det = cov[:, 0, 0] * cov[:, 1, 1] - cov[:, 0, 1] ** 2
    o = np.minimum(s.opacity[ok], 0.99)
    area = np.pi * 2.0 * np.log(np.maximum(o / alpha_min, 1.0)) * np.sqrt(det)
    return float(area.sum() / (w * h))


@dataclass
class Workload:
    name: str
    n_gt: int
    n_views: int
    width: int
    height: int
    p_split: float
    p_clone: float
    size_factor: float
    large_frac: float = 0.06
    large_range: tuple = (0.005, 0.01)
    spread: float = 0.3
    inflate: float = 2.0
    n_max: int = 19
    seed: int = 0
    # "uniform": candidates drawn uniformly among the large / small Gaussians;
    # "weighted": by rendered blending weight; "dominance": by dominated pixels
    stats_mode: str = "uniform"
    weight_floor: float = 0.05

    @property
    def rho(self) -> float:
        return rho_of(self.size_factor, self.n_gt)

    def build(self, seed=None, weight=None):
        """-> (init SynthScene rounded to fp32, camera rows, (grad_accum, denom), gt SynthScene).

        A "weighted" workload needs ``weight`` (the init scene's summed blending
        weights over its views, Plan.render_stats; see build_device)."""
        seed = self.seed if seed is None else seed
        gt = gt_scene(self.n_gt, seed, self.size_factor, self.spread, self.large_frac, self.large_range)
        ini = round_f32(init_scene(gt, seed, inflate=self.inflate))
        cams = ring_cameras(self.n_views, self.width, self.height, gt.extent)
        if self.stats_mode in ("weighted", "dominance") and weight is not None:
            stats = synth_stats_weighted(ini.scale, ini.extent, 2e-4, 0.01, self.p_split, self.p_clone, weight,
                                         self.weight_floor, seed)
        elif self.stats_mode in ("weighted", "dominance"):
            raise ValueError(f"{self.name}: weighted stats need the rendered weights (build_device)")
        else:
            stats = synth_stats(ini.scale, ini.extent, 2e-4, 0.01, self.p_split, self.p_clone, seed)
        return ini, cams, stats, round_f32(gt)

    def build_device(self, plan, seed=None):
        """Everything a step needs, on the plan's device: the init and GT scenes,
        the GT images (rendered), the init attribution of all views (rendered,
        with each Gaussian's blending weight for the weighted stats) and the
        measured depth complexities.  Returns a dict."""
        import torch

        from .operator import GaussianTensors
        seed = self.seed if seed is None else seed
        gt = gt_scene(self.n_gt, seed, self.size_factor, self.spread, self.large_frac, self.large_range)
        ini = round_f32(init_scene(gt, seed, inflate=self.inflate))
        gt = round_f32(gt)
        cams = ring_cameras(self.n_views, self.width, self.height, gt.extent)
        dev = plan.device
        g = GaussianTensors.from_numpy(*ini.arrays(), device=dev)
        gt_g = GaussianTensors.from_numpy(*gt.arrays(), device=dev)
        # statistics renders (no early termination) are separate from the
        # attribution the step consumes, which is the plain render
        _, _, _, dc_gt = plan.render_stats(gt_g, cams)
        gt_img, _ = plan.render(gt_g, cams)
        del gt_g
        _, _, weight, dc_init = plan.render_stats(g, cams)
        img, dom = plan.render(g, cams)
        dom_px = torch.zeros(g.n, dtype=torch.int64, device=dev)
        for v in range(len(cams)):
            dv = dom[v].reshape(-1)
            dom_px += torch.bincount(dv[dv >= 0].long(), minlength=g.n)
        if self.stats_mode in ("weighted", "dominance"):
            w = (weight if self.stats_mode == "weighted" else dom_px).double().cpu().numpy()
            stats = synth_stats_weighted(ini.scale, ini.extent, 2e-4, 0.01, self.p_split, self.p_clone,
                                         w, self.weight_floor, seed)
        else:
            stats = synth_stats(ini.scale, ini.extent, 2e-4, 0.01, self.p_split, self.p_clone, seed)
        torch.cuda.synchronize(dev)
        return dict(ini=ini, gt=gt, cams=cams, stats=stats, g=g, gt_img=gt_img, img=img, dom=dom,
                    weight=weight, dom_px=dom_px, dc_gt=dc_gt, dc_init=dc_init)


# BASELINE.json configs.  Sizes scale as 1/sqrt(k) around the
# 2.4M-GT scene of config 3 (base = U(.04,.10) * 0.01 * sqrt(2.4M/k): rho = 7.5
# in the survey's sqrt(32 rho / k_gt) form, the small Gaussians at the 0.3 px^2
# footprint floor).  The survey's depth complexity of 16-32 cannot be reached at
# these densities: the split candidates must exceed tau_s * extent (a >= 4.8 px
# standard deviation at config 3) and alone cover ~30 splats per pixel of the
# init render; measured values are reported with every bench line.
#
# DensifyStats: p_S of the Gaussians become split candidates, drawn by their
# dominated pixels (the Gaussians the views actually show; "dominance"), with a
# floor so occluded large Gaussians still appear.  On the reference's slab only
# ~12 % of the Gaussians above the split gate are front-most anywhere, so p_S =
# 1 % keeps the fallback (never-dominant) share under one half; config3_p5 is
# the survey's p_S = 5 % (88 % fallbacks) and config3_dc100 round 1's workload
# (rho = 30, uniform draw, 90 % fallbacks).
def _sf(k):
    return float(np.sqrt(2_400_000 / k))


def _wl(name, k, v, w, h, p_split=0.01, size=0.01, mode="dominance", floor=0.01, **kw):
    return Workload(name, k, v, w, h, p_split, 0.02, size * _sf(k),
                    large_range=(0.005 * _sf(k), 0.01 * _sf(k)), stats_mode=mode, weight_floor=floor, **kw)


CONFIGS = {
    "config1": _wl("config1", 10_000, 1, 256, 256),
    "config2": _wl("config2", 200_000, 16, 800, 800),
    "config3": _wl("config3", 2_400_000, 64, 1237, 822),
    "config4": _wl("config4", 6_000_000, 128, 1297, 840, n_max=9),
    "config5": _wl("config5", 16_000_000, 256, 1297, 840, p_split=0.25, large_frac=0.3, inflate=4.0),
    "config3_p5": _wl("config3_p5", 2_400_000, 64, 1237, 822, p_split=0.05),
    "config3_dc100": _wl("config3_dc100", 2_400_000, 64, 1237, 822, p_split=0.05, size=0.02, mode="uniform"),
}
