"""The AdpSplit split operator on B200: host orchestration over the C ABI.

Two entry layers:

* tensor API -- ``densify_step`` / ``render_views`` on SoA fp32 CUDA tensors;
  the benchmark and any GPU trainer call this.
* reference API -- ``adpsplit_step(scene, cameras, gt_images, stats, cfg, rng)``
  and ``render(scene, cam, background)`` with the reference's object types,
  argument meaning, ordering and exceptions (ref/adc.py:143-245,
  ref/raster.py:136-157), so it drops in where the reference is called
  (ref/harness.py:400-404, ref/cli.py:119).

Everything numeric runs in libadps.so; this module only moves buffers,
draws from the caller's numpy Generator in the reference's order and builds
the report.  There is no CPU fallback: without CUDA or without the library
every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi
from .types import CandidateRecord, Gaussian3D, SplitReport

F32 = torch.float32
F64 = torch.float64


def _require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2605_06876_b200 needs a CUDA device (B200); no CPU fallback exists")
    d = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if d.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {d}")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def _ptr(t):
    return C.c_void_p(0 if t is None else t.data_ptr())


# ----------------------------------------------------------------------------
# SoA Gaussians
# ----------------------------------------------------------------------------

@dataclass
class GaussianTensors:
    """N Gaussians as contiguous fp32 CUDA tensors (56 B each at SH degree 0)."""

    mu: torch.Tensor          # [N,3]
    scale: torch.Tensor       # [N,3]
    rot: torch.Tensor         # [N,4] (w,x,y,z)
    opacity: torch.Tensor     # [N]
    sh_dc: torch.Tensor       # [N,3]
    sh_rest: torch.Tensor = None   # [N,K,3] or None

    def __post_init__(self):
        for name in ("mu", "scale", "rot", "opacity", "sh_dc", "sh_rest"):
            t = getattr(self, name)
            if t is not None:
                if t.dtype != F32:
                    raise TypeError(f"{name} must be float32")
                setattr(self, name, t.contiguous())

    @property
    def n(self) -> int:
        return int(self.mu.shape[0])

    @property
    def sh_k(self) -> int:
        return 0 if self.sh_rest is None else int(self.sh_rest.shape[1])

    @property
    def device(self):
        return self.mu.device

    def abi(self) -> _abi.Gaussians:
        return _abi.Gaussians(self.mu.data_ptr(), self.scale.data_ptr(), self.rot.data_ptr(),
                              self.opacity.data_ptr(), self.sh_dc.data_ptr(),
                              self.sh_rest.data_ptr() if self.sh_k else None, self.sh_k)

    @staticmethod
    def empty(n: int, sh_k: int, device) -> "GaussianTensors":
        return GaussianTensors(torch.empty(n, 3, dtype=F32, device=device),
                               torch.empty(n, 3, dtype=F32, device=device),
                               torch.empty(n, 4, dtype=F32, device=device),
                               torch.empty(n, dtype=F32, device=device),
                               torch.empty(n, 3, dtype=F32, device=device),
                               torch.empty(n, sh_k, 3, dtype=F32, device=device) if sh_k else None)

    def head(self, n: int) -> "GaussianTensors":
        """The first n rows (views of the same storage; contiguous, fp32 by construction)."""
        t = object.__new__(GaussianTensors)
        t.mu, t.scale, t.rot, t.opacity, t.sh_dc = self.mu[:n], self.scale[:n], self.rot[:n], self.opacity[:n], \
            self.sh_dc[:n]
        t.sh_rest = self.sh_rest[:n] if self.sh_rest is not None else None
        return t

    @staticmethod
    def from_numpy(mu, scale, rot, opacity, sh_dc, sh_rest=None, device=None) -> "GaussianTensors":
        d = _require_cuda(device)

        def t(a, shape):
            return torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(shape)),
                                   device=d)

        n = len(mu)
        rest = None
        if sh_rest is not None and np.asarray(sh_rest).size:
            rest = t(sh_rest, (n, -1, 3))
        return GaussianTensors(t(mu, (n, 3)), t(scale, (n, 3)), t(rot, (n, 4)), t(opacity, (n,)),
                               t(sh_dc, (n, 3)), rest)

    def numpy(self) -> dict:
        out = {k: getattr(self, k).detach().cpu().numpy() for k in ("mu", "scale", "rot", "opacity", "sh_dc")}
        out["sh_rest"] = (self.sh_rest.cpu().numpy() if self.sh_k
                          else np.zeros((self.n, 0, 3), dtype=np.float32))
        return out


def camera_rows(cameras) -> np.ndarray:
    """Cameras -> [C,18] float64 rows in save_cameras order (ref/scene.py:339-347)."""
    if isinstance(cameras, np.ndarray):
        rows = np.asarray(cameras, dtype=np.float64)
        if rows.ndim != 2 or rows.shape[1] != 18:
            raise ValueError("camera rows must be [C,18]")
        return np.ascontiguousarray(rows)
    return np.ascontiguousarray(np.array(
        [np.concatenate([np.asarray(c.r_c2w, dtype=np.float64).ravel(),
                         np.asarray(c.center, dtype=np.float64),
                         [c.f_x, c.f_y, c.p_x, c.p_y, c.width, c.height]]) for c in cameras],
        dtype=np.float64).reshape(-1, 18))


def config_struct(cfg) -> _abi.Config:
    def get(name):
        return cfg[name] if isinstance(cfg, dict) else getattr(cfg, name)

    return _abi.Config(float(get("tau_l1")), int(get("r_erode")), int(get("m_min")), int(get("l_bands")),
                       int(get("n_max")), int(get("v_views")), 0, float(get("gamma_d")),
                       float(get("gamma_c")), float(get("tau_g")), float(get("tau_s")),
                       float(get("eta")), float(get("eps")))


# ----------------------------------------------------------------------------
# Plan
# ----------------------------------------------------------------------------

class Plan:
    """Owns one native plan (all scratch) on one device; reuse across steps."""

    def __init__(self, device=None):
        self.device = _require_cuda(device)
        self._dev_index = self.device.index if self.device.index is not None else torch.cuda.current_device()
        self.lib = _abi.load()
        self._h = C.c_void_p()
        with torch.cuda.device(self.device):
            _abi.check(self.lib.adps_plan_create(C.byref(self._h), self.device.index, 0, 0, 0, 0))
        self.timing = False

    def close(self):
        if self._h:
            self.lib.adps_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        # the raw cudaStream_t of torch's current stream on this device (what
        # torch.cuda.current_stream(dev).cuda_stream returns, without the wrapper)
        return C.c_void_p(torch._C._cuda_getCurrentRawStream(self._dev_index))

    def check_guards(self):
        """(bytes, buffers) written past the end of a plan buffer since allocation (debug; syncs)."""
        nb, nbuf = C.c_int64(), C.c_int32()
        _abi.check(self.lib.adps_check_guards(self._h, C.byref(nb), C.byref(nbuf)))
        return int(nb.value), int(nbuf.value)

    def set_timing(self, on: bool):
        self.timing = bool(on)
        _abi.check(self.lib.adps_set_timing(self._h, int(on)))

    def stage_ms(self) -> dict:
        """Per-stage device times (ms) of the last phase 1 + phase 2 (timing mode)."""
        ms = (C.c_double * 32)()
        names = (C.c_char_p * 32)()
        n = C.c_int32()
        _abi.check(self.lib.adps_get_timing(self._h, ms, 32, C.byref(n), names))
        out = {}
        for i in range(n.value):
            k = names[i].decode()
            out[k] = out.get(k, 0.0) + float(ms[i])
        return out

    def launch_count(self):
        """(own kernels, library sort calls) launched by this plan so far."""
        k, lib = C.c_int64(), C.c_int64()
        _abi.check(self.lib.adps_get_launch_count(self._h, C.byref(k), C.byref(lib)))
        return int(k.value), int(lib.value)

    def set_large_threshold(self, p: int):
        """Parents with more than p proposals take the grid-wide merge path (default 32)."""
        _abi.check(self.lib.adps_set_param(self._h, _abi.PARAM_LARGE_THRESHOLD, int(p)))

    def set_tile_path(self, path: int):
        """0: warp-per-tile CCL (+ block CCL for deferred tiles), 1: block CCL only."""
        _abi.check(self.lib.adps_set_param(self._h, _abi.PARAM_TILE_PATH, int(path)))

    def set_raw_cache(self, on: bool):
        """Minmax pass caches the fp64 raw L1 error for the warp CCL (default on)."""
        _abi.check(self.lib.adps_set_param(self._h, _abi.PARAM_RAW_CACHE, int(bool(on))))

    def set_render_binning(self, fast: bool):
        """Render depth order: 32-bit keys + fix-up, no per-view sync (default), or the 64-bit sort."""
        _abi.check(self.lib.adps_set_param(self._h, _abi.PARAM_RENDER_BINNING, int(bool(fast))))

    def set_param(self, key: int, value: int):
        _abi.check(self.lib.adps_set_param(self._h, int(key), int(value)))

    def get_param(self, key: int) -> int:
        v = C.c_int64()
        _abi.check(self.lib.adps_get_param(self._h, int(key), C.byref(v)))
        return int(v.value)

    def deferred_tiles(self) -> int:
        """Tiles the warp CCL of the last phase 1 handed to the block CCL."""
        return self.get_param(_abi.PARAM_DEFERRED_TILES)

    def normals_pcg64(self, bitgen_state: dict, n: int, out: torch.Tensor = None, sync=True):
        """numpy Generator(PCG64).standard_normal(n) on the device, bit-identical.

        bitgen_state: ``rng.bit_generator.state``.  Returns (out, consumed,
        status) when sync, else (out, None, None) with consumed/status
        readable via normals_result() after the next phase1_end; sync=2
        leaves the launch to that phase1_end (adps.h)."""
        st = bitgen_state["state"]
        m64 = (1 << 64) - 1
        state = (C.c_uint64 * 2)(st["state"] & m64, st["state"] >> 64)
        inc = (C.c_uint64 * 2)(st["inc"] & m64, st["inc"] >> 64)
        if out is None:
            out = torch.empty(max(n, 0), dtype=F64, device=self.device)
        consumed, status = C.c_int64(), C.c_int32()
        _abi.check(self.lib.adps_normals_pcg64(self._h, self._stream(), state, inc, int(n), _ptr(out) if n else None,
                                               int(sync), C.byref(consumed), C.byref(status)))
        if sync is True or sync == 1:
            return out, int(consumed.value), int(status.value)
        return out, None, None

    def normals_result(self):
        """(consumed, status) of the last normals_pcg64 after the plan synchronised."""
        return self.get_param(_abi.PARAM_NORMALS_CONSUMED), self.get_param(_abi.PARAM_NORMALS_STATUS)

    def set_debug_records(self, on: bool):
        _abi.check(self.lib.adps_set_debug_records(self._h, int(on)))

    def set_debug_maps(self, m: torch.Tensor = None, b: torch.Tensor = None):
        _abi.check(self.lib.adps_set_debug_maps(self._h, _ptr(m), _ptr(b)))

    # -- render (ref/raster.py:136-157)
    def render(self, g: GaussianTensors, cams: np.ndarray, bg=(0.0, 0.0, 0.0), out=None):
        cams = camera_rows(cams)
        v = len(cams)
        w, h = int(cams[0, 16]), int(cams[0, 17])
        if out is None:
            image = torch.empty(v, h, w, 3, dtype=F32, device=self.device)
            dom = torch.empty(v, h, w, dtype=torch.int32, device=self.device)
        else:
            image, dom = out
        bgv = (C.c_float * 3)(*[float(x) for x in bg])
        ga = g.abi()
        _abi.check(self.lib.adps_render(self._h, self._stream(), C.byref(ga), g.n,
                                        cams.ctypes.data_as(C.c_void_p), v, bgv, _ptr(image), _ptr(dom)))
        return image, dom

    def render_fused(self, g: GaussianTensors, extent, grad_accum, denom, cfg, cams_v, gt_v, bg=(0.0, 0.0, 0.0),
                     out=None):
        """Attribution render of the sampled views with the step's input pass
        fused into its epilogue (adps_render_fused): returns (image, dominant);
        the next phase1_begin on the same tensors starts from the raw cache."""
        cams_v = camera_rows(cams_v)
        v = len(cams_v)
        w, h = int(cams_v[0, 16]), int(cams_v[0, 17])
        if out is None:
            image = torch.empty(v, h, w, 3, dtype=F32, device=self.device)
            dom = torch.empty(v, h, w, dtype=torch.int32, device=self.device)
        else:
            image, dom = out
        self._check_inputs(grad_accum, denom, image, gt_v, dom)
        bgv = (C.c_float * 3)(*[float(x) for x in bg])
        ga = g.abi()
        cs = config_struct(cfg)
        _abi.check(self.lib.adps_render_fused(self._h, self._stream(), C.byref(ga), g.n, float(extent),
                                              _ptr(grad_accum), _ptr(denom), C.byref(cs),
                                              cams_v.ctypes.data_as(C.c_void_p), v, bgv, _ptr(gt_v), _ptr(image),
                                              _ptr(dom)))
        return image, dom

    def render_stats(self, g: GaussianTensors, cams: np.ndarray, bg=(0.0, 0.0, 0.0)):
        """(image, dominant, weight [n] fp32, depth complexity): the render plus each
        Gaussian's summed blending weight T*alpha and the mean number of splats with
        alpha >= 1/255 per pixel (workload statistics for the benchmark)."""
        cams = camera_rows(cams)
        v = len(cams)
        w, h = int(cams[0, 16]), int(cams[0, 17])
        image = torch.empty(v, h, w, 3, dtype=F32, device=self.device)
        dom = torch.empty(v, h, w, dtype=torch.int32, device=self.device)
        weight = torch.zeros(max(g.n, 1), dtype=F32, device=self.device)
        bgv = (C.c_float * 3)(*[float(x) for x in bg])
        ga = g.abi()
        contrib = C.c_uint64()
        _abi.check(self.lib.adps_render_stats(self._h, self._stream(), C.byref(ga), g.n,
                                              cams.ctypes.data_as(C.c_void_p), v, bgv, _ptr(image), _ptr(dom),
                                              _ptr(weight), C.byref(contrib)))
        return image, dom, weight[:g.n], contrib.value / float(v * h * w)

    # -- phase 1 / 2 (ref/adc.py:165-244)
    @staticmethod
    def _check_inputs(grad_accum, denom, image, gt, dom):
        """The C ABI takes raw pointers: reject tensors of the wrong type/layout loudly."""
        for name, t, dt in (("grad_accum", grad_accum, F64), ("denom", denom, F64), ("image", image, F32),
                            ("gt", gt, F32), ("dominant", dom, torch.int32)):
            if t.dtype != dt:
                raise ValueError(f"{name} must be {dt}, got {t.dtype}")
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous CUDA tensor")

    def phase1(self, g, extent, grad_accum, denom, cfg, cams_v, image, gt, dom) -> dict:
        cams_v = camera_rows(cams_v)
        self._check_inputs(grad_accum, denom, image, gt, dom)
        counts = _abi.Counts()
        cs = config_struct(cfg)
        ga = g.abi()
        self._g_keep = (g, grad_accum, denom, image, gt, dom)
        st = self.lib.adps_step_phase1(self._h, self._stream(), C.byref(ga), g.n, float(extent),
                                       _ptr(grad_accum), _ptr(denom), C.byref(cs),
                                       cams_v.ctypes.data_as(C.c_void_p), len(cams_v), _ptr(image),
                                       _ptr(gt), _ptr(dom), C.byref(counts))
        _abi.check(st)
        return counts.as_dict()

    def phase1_begin(self, g, extent, grad_accum, denom, cfg, cams_v, image, gt, dom) -> dict:
        """select + ever-dominant flags; returns n_split/n_clone/n_fallback after one sync."""
        cams_v = camera_rows(cams_v)
        self._check_inputs(grad_accum, denom, image, gt, dom)
        counts = _abi.Counts()
        cs = config_struct(cfg)
        ga = g.abi()
        self._g_keep = (g, grad_accum, denom, image, gt, dom)
        _abi.check(self.lib.adps_step_phase1_begin(self._h, self._stream(), C.byref(ga), g.n, float(extent),
                                                   _ptr(grad_accum), _ptr(denom), C.byref(cs),
                                                   cams_v.ctypes.data_as(C.c_void_p), len(cams_v), _ptr(image),
                                                   _ptr(gt), _ptr(dom), C.byref(counts)))
        return counts.as_dict()

    def phase1_end(self) -> dict:
        """The rest of phase 1 (maps ... offsets); releases the GIL while the GPU works."""
        counts = _abi.Counts()
        _abi.check(self.lib.adps_step_phase1_end(self._h, self._stream(), C.byref(counts)))
        return counts.as_dict()

    def capacity(self) -> tuple:
        """(out_cap, app_cap): row bounds of the step begun by phase1_begin."""
        oc, ac = C.c_int64(), C.c_int64()
        _abi.check(self.lib.adps_step_capacity(self._h, C.byref(oc), C.byref(ac)))
        return int(oc.value), int(ac.value)

    def phase1_end_emit(self, g, normals, out: GaussianTensors, index_map: torch.Tensor,
                        child_parent: torch.Tensor, insert_offset: torch.Tensor, report: torch.Tensor = None) -> dict:
        """phase1_end + phase2 with one synchronisation (adps_step_phase1_end_emit):
        out/index_map hold capacity()[0] rows, child_parent capacity()[1]; report
        (optional) int32 [4 n_split + n_split V + n_clone] gets the report arrays."""
        counts = _abi.Counts()
        ga = g.abi()
        oa = _abi.GaussiansOut(out.mu.data_ptr(), out.scale.data_ptr(), out.rot.data_ptr(),
                               out.opacity.data_ptr(), out.sh_dc.data_ptr(),
                               out.sh_rest.data_ptr() if out.sh_k else None, out.sh_k)
        _abi.check(self.lib.adps_step_phase1_end_emit(
            self._h, self._stream(), C.byref(ga), _ptr(normals), C.byref(oa), _ptr(index_map),
            _ptr(child_parent) if child_parent.numel() else None,
            _ptr(insert_offset) if insert_offset.numel() else None,
            out.n, child_parent.numel(), _ptr(report) if report is not None and report.numel() else None,
            C.byref(counts)))
        return counts.as_dict()

    # -- view-sharded phase 1 (multi-GPU; see sharded.py and include/adps.h)
    def set_view_sharding(self, offset: int, stride: int, n_views_global: int):
        _abi.check(self.lib.adps_set_view_sharding(self._h, int(offset), int(stride), int(n_views_global)))

    def buffer(self, which: int):
        """(device pointer, count, element bytes) of a plan-owned buffer."""
        ptr, cnt, eb = C.c_void_p(), C.c_int64(), C.c_int64()
        _abi.check(self.lib.adps_get_buffer(self._h, int(which), C.byref(ptr), C.byref(cnt), C.byref(eb)))
        return ptr.value, int(cnt.value), int(eb.value)

    def _buffer_copy(self, which: int) -> torch.Tensor:
        ptr, cnt, eb = self.buffer(which)
        out = torch.empty(cnt * eb, dtype=torch.uint8, device=self.device)
        if cnt:
            _copy_device(out, ptr, cnt * eb, self.device)
        return out

    def dom_flags(self) -> torch.Tensor:
        """Copy of the ever-dominant flags of the last phase1_begin (uint8 [n])."""
        return self._buffer_copy(_abi.BUF_DOM_FLAG)

    def set_dom_flags(self, flags: torch.Tensor):
        ptr, cnt, eb = self.buffer(_abi.BUF_DOM_FLAG)
        if flags.numel() != cnt * eb or flags.dtype != torch.uint8:
            raise ValueError("dom flags must be uint8 [n]")
        if cnt:
            global _cudart
            if _cudart is None:
                from cuda.bindings import runtime as _rt
                _cudart = _rt
            stream = torch.cuda.current_stream(self.device).cuda_stream
            err, = _cudart.cudaMemcpyAsync(ptr, flags.contiguous().data_ptr(), cnt,
                                           _cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice, stream)
            if int(err) != 0:
                raise RuntimeError(f"cudaMemcpyAsync failed: {err}")

    def phase1_refresh(self) -> dict:
        """Fallback count from the (externally reduced) ever-dominant flags."""
        counts = _abi.Counts()
        _abi.check(self.lib.adps_step_phase1_refresh(self._h, self._stream(), C.byref(counts)))
        return counts.as_dict()

    def phase1_local(self) -> int:
        n = C.c_int64()
        _abi.check(self.lib.adps_step_phase1_local(self._h, self._stream(), C.byref(n)))
        return int(n.value)

    def export_records(self) -> dict:
        """This rank's region records, proposals and valid flags as uint8 tensors."""
        return {"regions": self._buffer_copy(_abi.BUF_REGIONS), "proposals": self._buffer_copy(_abi.BUF_PROPOSALS),
                "valid": self._buffer_copy(_abi.BUF_VALID)}

    def record_sizes(self):
        return self.buffer(_abi.BUF_REGIONS)[2], self.buffer(_abi.BUF_PROPOSALS)[2]

    def phase1_import(self, regions: torch.Tensor, proposals: torch.Tensor, valid: torch.Tensor):
        n = valid.numel()
        self._import_keep = (regions, proposals, valid)
        _abi.check(self.lib.adps_step_phase1_import(self._h, self._stream(), _ptr(regions) if n else None,
                                                    _ptr(proposals) if n else None, _ptr(valid) if n else None, n))

    def phase1_merge(self) -> dict:
        """Merge + cap (+ offsets unless parent-sharded: then only this rank's
        candidates, and counts holds its merge_edges / n_children)."""
        counts = _abi.Counts()
        _abi.check(self.lib.adps_step_phase1_merge(self._h, self._stream(), C.byref(counts)))
        return counts.as_dict()

    def set_parent_sharding(self, rank: int, world: int):
        _abi.check(self.lib.adps_set_parent_sharding(self._h, int(rank), int(world)))

    def shard(self):
        """(k_lo, k_hi, p_lo, p_hi) of this rank's parent range after a parent-sharded merge."""
        v = [C.c_int64() for _ in range(4)]
        _abi.check(self.lib.adps_get_shard(self._h, *[C.byref(x) for x in v]))
        return tuple(int(x.value) for x in v)

    def export_shard(self, merge_edges: int, n_children: int) -> torch.Tensor:
        """This rank's merge results as one byte blob: header (k_lo, k_hi, p_lo, p_hi,
        merge_edges, n_children) int64, cand_merged and cand_ins [k_lo, k_hi) int32,
        children rows [p_lo, p_hi) (14 fp32 each)."""
        k_lo, k_hi, p_lo, p_hi = self.shard()
        head = torch.tensor([k_lo, k_hi, p_lo, p_hi, merge_edges, n_children], dtype=torch.int64,
                            device=self.device).view(torch.uint8)
        parts = [head]
        for which, lo, hi in ((_abi.BUF_CAND_MERGED, k_lo, k_hi), (_abi.BUF_CAND_INS, k_lo, k_hi),
                              (_abi.BUF_CHILDREN, p_lo, p_hi)):
            ptr, _, eb = self.buffer(which)
            t = torch.empty((hi - lo) * eb, dtype=torch.uint8, device=self.device)
            if hi > lo:
                _copy_device(t, ptr + lo * eb, (hi - lo) * eb, self.device)
            parts.append(t)
        return torch.cat(parts)

    def import_shards(self, blobs) -> tuple:
        """Write every other rank's merge results into this plan; returns the summed
        (merge_edges, n_children)."""
        own = self.shard()
        me = nc = 0
        for b in blobs:
            head = b[:48].clone().view(torch.int64).tolist()
            k_lo, k_hi, p_lo, p_hi, e, c = head
            me += e
            nc += c
            if (k_lo, k_hi, p_lo, p_hi) == own:
                continue
            off = 48
            for which, lo, hi in ((_abi.BUF_CAND_MERGED, k_lo, k_hi), (_abi.BUF_CAND_INS, k_lo, k_hi),
                                  (_abi.BUF_CHILDREN, p_lo, p_hi)):
                ptr, _, eb = self.buffer(which)
                nb = (hi - lo) * eb
                if nb:
                    src = b[off:off + nb].contiguous()
                    _copy_to_ptr(ptr + lo * eb, src, self.device)
                off += nb
        return me, nc

    def phase1_finish(self, merge_edges: int, n_children: int) -> dict:
        counts = _abi.Counts()
        _abi.check(self.lib.adps_step_phase1_finish(self._h, self._stream(), int(merge_edges), int(n_children),
                                                    C.byref(counts)))
        return counts.as_dict()

    def vanilla_phase1(self, g, extent, grad_accum, denom, cfg, n_children: int) -> dict:
        """select + every split candidate -> n_children vanilla children (ref/adc.py:248-280)."""
        counts = _abi.Counts()
        cs = config_struct(cfg)
        ga = g.abi()
        self._g_keep = (g, grad_accum, denom)
        _abi.check(self.lib.adps_vanilla_phase1(self._h, self._stream(), C.byref(ga), g.n, float(extent),
                                                _ptr(grad_accum), _ptr(denom), C.byref(cs), int(n_children),
                                                C.byref(counts)))
        return counts.as_dict()

    def reset_flags(self, include_clones: bool) -> torch.Tensor:
        """uint8 [n_before]: the last step's reset candidates (and clone sources)."""
        n = self._g_keep[0].n
        flags = torch.empty(max(n, 1), dtype=torch.uint8, device=self.device)
        _abi.check(self.lib.adps_reset_flags(self._h, self._stream(), _ptr(flags), int(bool(include_clones))))
        return flags[:n]

    def phase2(self, g, normals, out: GaussianTensors, index_map: torch.Tensor, child_parent: torch.Tensor = None,
               insert_offset: torch.Tensor = None):
        ga = g.abi()
        oa = _abi.GaussiansOut(out.mu.data_ptr(), out.scale.data_ptr(), out.rot.data_ptr(),
                               out.opacity.data_ptr(), out.sh_dc.data_ptr(),
                               out.sh_rest.data_ptr() if out.sh_k else None, out.sh_k)
        _abi.check(self.lib.adps_step_phase2(self._h, self._stream(), C.byref(ga), _ptr(normals),
                                             C.byref(oa), _ptr(index_map),
                                             _ptr(child_parent) if child_parent is not None and child_parent.numel()
                                             else None,
                                             _ptr(insert_offset) if insert_offset is not None and insert_offset.numel()
                                             else None))

    def prune_index(self, threshold: float, opacity: torch.Tensor = None, logit_op: torch.Tensor = None):
        """(index_map [n_keep] int64, n_keep, n_near) of ref/harness.py:320-340's keep test."""
        src = opacity if opacity is not None else logit_op
        if src is None:
            raise ValueError("need opacity (fp32) or logit_op (fp64)")
        want = F32 if opacity is not None else F64
        if src.dtype != want or not src.is_cuda or src.dim() != 1:
            raise ValueError(f"{'opacity' if opacity is not None else 'logit_op'} must be a 1-D {want} CUDA tensor")
        src = src.contiguous()
        n = src.numel()
        im = torch.empty(max(n, 1), dtype=torch.int64, device=self.device)
        nk, nn = C.c_int64(), C.c_int64()
        _abi.check(self.lib.adps_prune_index(self._h, self._stream(), _ptr(src) if opacity is not None else None,
                                             _ptr(src) if opacity is None else None, n, float(threshold),
                                             _ptr(im), C.byref(nk), C.byref(nn)))
        return im[:nk.value], int(nk.value), int(nn.value)

    def report_arrays(self, n_split: int, n_clone: int) -> dict:
        r = _abi.Report()
        _abi.check(self.lib.adps_get_report(self._h, C.byref(r)))
        v = int(r.n_views)
        # one buffer, one native call for the six copies
        buf = torch.empty(4 * n_split + n_split * v + n_clone, dtype=torch.int32, device=self.device)
        _abi.check(self.lib.adps_copy_report(self._h, self._stream(), _ptr(buf), int(n_split), int(n_clone)))
        return _report_views(buf, n_split, n_clone, v)

    def regions(self) -> dict:
        """Region records of the last phase 1, in reference order (diagnostic)."""
        rec, order, valid, stats, child = (C.c_void_p() for _ in range(5))
        n = C.c_int64()
        _abi.check(self.lib.adps_get_regions(self._h, C.byref(rec), C.byref(order), C.byref(valid),
                                             C.byref(stats), C.byref(child), C.byref(n)))
        n = n.value
        raw = torch.empty(n * 16, dtype=torch.int32, device=self.device)
        ordt = torch.empty(n, dtype=torch.int32, device=self.device)
        val = torch.empty(n, dtype=torch.uint8, device=self.device)
        if n:
            _copy_device(raw, rec.value, n * 64, self.device)
            _copy_device(ordt, order.value, n * 4, self.device)
            _copy_device(val, valid.value, n, self.device)
        raw = raw.view(n, 16)
        o = ordt.long()
        out = dict(view_pos=raw[:, 0][o], candidate=raw[:, 1][o], band=raw[:, 2][o], minpix=raw[:, 3][o],
                   moments=raw[:, 4:].contiguous().view(torch.int64).view(n, 6)[o], valid=val[o])
        if stats.value and n:
            st = torch.empty(n, 10, dtype=F64, device=self.device)
            ch = torch.empty(n, 16, dtype=F64, device=self.device)
            _copy_device(st, stats.value, n * 80, self.device)
            _copy_device(ch, child.value, n * 128, self.device)
            out["stats"] = st[o]
            out["child"] = ch[o]
        return out


_cudart = None


def _copy_to_ptr(dst_ptr: int, src: torch.Tensor, device):
    """Device-to-device copy into a raw pointer owned by the plan."""
    global _cudart
    if _cudart is None:
        from cuda.bindings import runtime as _rt
        _cudart = _rt
    stream = torch.cuda.current_stream(device).cuda_stream
    err, = _cudart.cudaMemcpyAsync(dst_ptr, src.data_ptr(), src.numel() * src.element_size(),
                                   _cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice, stream)
    if int(err) != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed: {err}")


def _copy_device(dst: torch.Tensor, src_ptr: int, nbytes: int, device):
    """Device-to-device copy from a raw pointer owned by the plan."""
    global _cudart
    if _cudart is None:
        from cuda.bindings import runtime as _rt  # cuda-python
        _cudart = _rt
    stream = torch.cuda.current_stream(device).cuda_stream
    err, = _cudart.cudaMemcpyAsync(dst.data_ptr(), src_ptr, nbytes,
                                   _cudart.cudaMemcpyKind.cudaMemcpyDeviceToDevice, stream)
    if int(err) != 0:
        raise RuntimeError(f"cudaMemcpyAsync failed: {err}")


_plans: dict = {}


def default_plan(device=None) -> Plan:
    d = _require_cuda(device)
    if d.index not in _plans:
        _plans[d.index] = Plan(d)
    return _plans[d.index]


# ----------------------------------------------------------------------------
# tensor API
# ----------------------------------------------------------------------------

def sample_views(n_cams: int, v_views: int, rng) -> list:
    """sorted(rng.choice(#cams, V, replace=False)), ref/adc.py:154-161."""
    if v_views > n_cams:
        raise ValueError(f"v_views={v_views} exceeds available cameras ({n_cams})")
    return [int(v) for v in sorted(rng.choice(n_cams, size=v_views, replace=False))]


def _gather_views(x, view_ids, device):
    """Stack per-view images of the sampled views on the device (no copy if contiguous)."""
    if isinstance(x, torch.Tensor):
        if x.device != device:
            x = x.to(device)
        if view_ids == list(range(view_ids[0], view_ids[0] + len(view_ids))):
            return x[view_ids[0]:view_ids[0] + len(view_ids)].to(F32).contiguous()
        return x.index_select(0, torch.as_tensor(view_ids, device=device)).to(F32).contiguous()
    return torch.stack([torch.as_tensor(np.asarray(x[v], dtype=np.float32), device=device)
                        for v in view_ids]).contiguous()


@dataclass
class StepResult:
    gaussians: GaussianTensors
    index_map: torch.Tensor
    counts: dict
    view_ids: list
    _report: object = None         # the report arrays, or (buffer, n_split, n_clone, V) split on first use
    normals: torch.Tensor = None   # the 6F fallback normals (device)
    child_parent: torch.Tensor = None    # int32 [n_out - n_keep]: old index of every appended row
    insert_offset: torch.Tensor = None   # int64 [n_split]: output row of candidate k's first insert
    stage_ms: dict = field(default_factory=dict)

    @property
    def report_arrays(self) -> dict:
        """The SplitReport arrays on the device (views of one buffer)."""
        if isinstance(self._report, tuple):
            self._report = _report_views(*self._report)
        return self._report

    @report_arrays.setter
    def report_arrays(self, value):
        self._report = value

    def report(self) -> SplitReport:
        """Host SplitReport (ref/adc.py:60-70) built from the device arrays."""
        ra = {k: v.cpu().numpy() for k, v in self.report_arrays.items()}
        rep = SplitReport(count_before=self.counts["n_before"], count_after=self.counts["n_out"])
        rep.sampled_views = list(self.view_ids)
        rep.merge_edges = self.counts["merge_edges"]
        rep.clones = [int(i) for i in ra["clone_index"]]
        for k, i in enumerate(ra["cand_index"]):
            case = int(ra["cand_case"][k])
            rpv = ra["regions_per_view"]
            rec = CandidateRecord(index=int(i),
                                  regions_per_view=[int(x) for x in rpv[k]] if rpv.ndim == 2 and k < len(rpv) else [],
                                  proposals=int(ra["cand_proposals"][k]))
            if case == _abi.CASE_FALLBACK:
                rec.fallback = True
            elif case == _abi.CASE_RESET:
                rec.reset = True
                rep.reset_indices.append(int(i))
            else:
                rec.merged = int(ra["cand_merged"][k])
                rec.children_inserted = rec.merged
            rep.candidates.append(rec)
        rep.index_map = self.index_map.cpu().numpy().astype(np.int64)
        return rep


class FallbackNormals:
    """The 6F normals of the fallback children (ref/adc.py:97).

    The caller's Generator draws 3 normals per fallback child in ascending
    parent order; the stream is chunk-invariant, so the 6F values are one
    slice of rng.standard_normal.  A PCG64 Generator's slice is produced on
    the device, bit-identical (adps_normals_pcg64), and the host Generator is
    advanced past it once phase 1 has synchronised; any other bit generator is
    drawn on a host thread while the GPU finishes phase 1 (the C calls
    release the GIL).  Start it after phase1_begin, call join() after the
    phase-1 end, then result().
    """

    def __init__(self, plan: Plan, rng, nf: int, children: int = 2):
        self.plan, self.rng, self.nf = plan, rng, int(nf)
        self.count = 3 * int(children) * self.nf
        self.gpu = self.nf > 0 and isinstance(rng.bit_generator, np.random.PCG64)
        self.normals, self._drawn, self._th = None, {}, None
        if self.gpu:
            # launched by phase1_end at its first host wait (sync=2): the ~80 us
            # of launch calls then overlap the attribution instead of idling the GPU
            self.normals, _, _ = plan.normals_pcg64(rng.bit_generator.state, self.count, sync=2)
        elif self.nf > 0:
            def _draw():
                self._drawn["z"] = rng.standard_normal(self.count)

            self._th = threading.Thread(target=_draw)
            self._th.start()

    def join(self):
        if self._th is not None:
            self._th.join()
            self._th = None

    def result(self):
        """Device tensor of the normals (None when there are no fallbacks)."""
        self.join()
        if self.gpu:
            consumed, status = self.plan.normals_result()
            if status == 0:
                self.rng.bit_generator.advance(consumed)
            else:   # a wedge test too close to call against the host libm: draw on the host
                self.normals = torch.from_numpy(self.rng.standard_normal(self.count)).to(self.plan.device)
            self.gpu = False
        elif self.nf > 0 and self.normals is None:
            self.normals = torch.from_numpy(self._drawn["z"]).to(self.plan.device)
        return self.normals


def _report_views(buf: torch.Tensor, n_split: int, n_clone: int, v: int) -> dict:
    """The SplitReport arrays as views of adps_copy_report's buffer."""
    parts = torch.split(buf, [n_split] * 4 + [n_split * v, n_clone])
    return dict(cand_index=parts[0], cand_case=parts[1], cand_proposals=parts[2], cand_merged=parts[3],
                regions_per_view=parts[4].view(-1, max(v, 1)), clone_index=parts[5])


def _step_outputs(n_out: int, sh_k: int, n_app: int, n_split: int, dev, out: GaussianTensors = None):
    """(GaussianTensors, index_map int64, child_parent int32, insert_offset int64) for phase 2.
    (Separate allocations: the caching allocator serves these sizes from its
    pools faster than one large carved buffer, measured at config 3.)"""
    if out is None:
        out = GaussianTensors.empty(n_out, sh_k, dev)
    return (out, torch.empty(n_out, dtype=torch.int64, device=dev), torch.empty(n_app, dtype=torch.int32, device=dev),
            torch.empty(n_split, dtype=torch.int64, device=dev))


def densify_step(g: GaussianTensors, extent: float, cameras, gt, grad_accum: torch.Tensor,
                 denom: torch.Tensor, cfg, rng, *, renders=None, plan: Plan = None,
                 view_ids=None, want_report: bool = True, out: GaussianTensors = None,
                 fused: bool = False, one_sync: bool = True) -> StepResult:
    """One AdpSplit densify step on device tensors (ref/adc.py:143-245).

    cameras: all C cameras ([C,18] rows or Camera objects).  gt: [C,H,W,3]
    fp32 tensor (or a per-camera sequence).  renders: optional (image,
    dominant) of the sampled views (the stage boundary the reference tests
    reach by monkeypatching ``adc.render``); rendered on the GPU otherwise --
    with ``fused`` by the render whose epilogue also runs the step's input
    pass (adps_render_fused; same results).  one_sync: when the fallback
    normals are drawn on the device (PCG64) and no ``out`` is given, phase 1's
    end and the emit are one call with one synchronisation
    (adps_step_phase1_end_emit); the outputs are then row-prefix views of
    arrays sized by the step's bounds.  Same results either way.
    """
    plan = plan or default_plan(g.device)
    cams = camera_rows(cameras)
    if view_ids is None:
        view_ids = sample_views(len(cams), int(cfg["v_views"] if isinstance(cfg, dict) else cfg.v_views), rng)
    cams_v = cams[view_ids]
    dev = plan.device
    gt_v = _gather_views(gt, view_ids, dev)
    grad_accum = grad_accum.to(dev, F64).contiguous()
    denom = denom.to(dev, F64).contiguous()
    if renders is None and fused:
        image, dom = plan.render_fused(g, extent, grad_accum, denom, cfg, cams_v, gt_v)
    elif renders is None:
        image, dom = plan.render(g, cams_v)
    else:
        image, dom = renders
        image = image.to(dev, F32).contiguous()
        dom = dom.to(dev, torch.int32).contiguous()
    counts = plan.phase1_begin(g, extent, grad_accum, denom, cfg, cams_v, image, gt_v, dom)
    nf = counts["n_fallback"]
    draw = FallbackNormals(plan, rng, nf)
    if one_sync and out is None and (nf == 0 or draw.gpu):
        # normals on the device: the emit goes out with phase 1's end, into
        # arrays sized by the step's row bounds, before the host reads a count
        out_cap, app_cap = plan.capacity()
        out_full, im_full, cp_full, insert_offset = _step_outputs(out_cap, g.sh_k, app_cap, counts["n_split"], dev)
        ns, ncl, nv = counts["n_split"], counts["n_clone"], len(view_ids)
        rep_buf = torch.empty(4 * ns + ns * nv + ncl, dtype=torch.int32, device=dev) if want_report else None
        dev_normals = draw.normals
        counts = plan.phase1_end_emit(g, dev_normals, out_full, im_full, cp_full, insert_offset, rep_buf)
        if counts["n_fallback"] != nf:
            raise RuntimeError("fallback count changed between phase-1 halves")
        normals = draw.result()
        n_out = counts["n_out"]
        out, index_map = out_full.head(n_out), im_full[:n_out]
        child_parent = cp_full[:n_out - counts["n_keep"]]
        if normals is not dev_normals:
            # the device normals failed their wedge test: emit again with the host's
            plan.phase2(g, normals, out, index_map, child_parent, insert_offset)
    else:
        rep_buf = None
        try:
            counts = plan.phase1_end()
        finally:
            draw.join()
        if counts["n_fallback"] != nf:
            raise RuntimeError("fallback count changed between phase-1 halves")
        normals = draw.result()
        n_out = counts["n_out"]
        out, index_map, child_parent, insert_offset = _step_outputs(n_out, g.sh_k, n_out - counts["n_keep"],
                                                                    counts["n_split"], dev, out)
        plan.phase2(g, normals, out, index_map, child_parent, insert_offset)
    res = StepResult(gaussians=out, index_map=index_map, counts=counts, view_ids=list(view_ids),
                     normals=normals, child_parent=child_parent, insert_offset=insert_offset)
    if want_report:
        res.report_arrays = ((rep_buf, ns, ncl, nv) if rep_buf is not None
                             else plan.report_arrays(counts["n_split"], counts["n_clone"]))
    if plan.timing:
        res.stage_ms = plan.stage_ms()
    return res


def vanilla_densify_step(g: GaussianTensors, extent: float, grad_accum: torch.Tensor, denom: torch.Tensor, cfg,
                         n_children: int, rng, *, plan: Plan = None, want_report: bool = True) -> StepResult:
    """The binary ADC baseline on the device (ref/adc.py:248-280): every split
    candidate becomes n_children vanilla_split children, clones appended."""
    plan = plan or default_plan(g.device)
    dev = plan.device
    counts = plan.vanilla_phase1(g, extent, grad_accum.to(dev, F64).contiguous(), denom.to(dev, F64).contiguous(),
                                 cfg, n_children)
    nf, count = counts["n_split"], 3 * int(n_children) * counts["n_split"]
    normals = None
    if nf > 0 and isinstance(rng.bit_generator, np.random.PCG64):
        normals, consumed, status = plan.normals_pcg64(rng.bit_generator.state, count, sync=True)
        if status == 0:
            rng.bit_generator.advance(consumed)
        else:   # a wedge test too close to call against the host libm
            normals = torch.from_numpy(rng.standard_normal(count)).to(dev)
    elif nf > 0:
        normals = torch.from_numpy(rng.standard_normal(count)).to(dev)
    out = GaussianTensors.empty(counts["n_out"], g.sh_k, dev)
    index_map = torch.empty(counts["n_out"], dtype=torch.int64, device=dev)
    child_parent = torch.empty(counts["n_out"] - counts["n_keep"], dtype=torch.int32, device=dev)
    insert_offset = torch.empty(counts["n_split"], dtype=torch.int64, device=dev)
    plan.phase2(g, normals, out, index_map, child_parent, insert_offset)
    res = StepResult(gaussians=out, index_map=index_map, counts=counts, view_ids=[], normals=normals,
                     child_parent=child_parent, insert_offset=insert_offset)
    if want_report:
        res.report_arrays = plan.report_arrays(counts["n_split"], counts["n_clone"])
    return res


def remap_rows(index_map: torch.Tensor, values: torch.Tensor, zero_old: torch.Tensor = None) -> torch.Tensor:
    """out[new] = values[index_map[new]] for carried rows not flagged in zero_old,
    zeros for new rows (ref/adc.py:283-296, ref/harness.py:285-295), on the device."""
    lib = _abi.load()
    n_out = index_map.numel()
    v = values.contiguous()
    out = torch.empty((n_out,) + tuple(v.shape[1:]), dtype=v.dtype, device=v.device)
    row_bytes = v.element_size() * (v[0].numel() if v.dim() > 1 and v.shape[0] else
                                    int(np.prod(v.shape[1:], dtype=np.int64)))
    stream = torch.cuda.current_stream(v.device).cuda_stream
    _abi.check(lib.adps_remap_rows(C.c_void_p(stream), _ptr(index_map.contiguous()), n_out,
                                   _ptr(zero_old) if zero_old is not None else None, _ptr(v), row_bytes,
                                   _ptr(out)))
    return out


def remap_stats(plan: Plan, res: StepResult, grad_accum: torch.Tensor, denom: torch.Tensor):
    """remap_stats (ref/adc.py:283-296) after densify_step / vanilla_densify_step:
    carried Gaussians keep their accumulators unless reset or cloned; new ones start at 0."""
    flags = plan.reset_flags(include_clones=True)
    return (remap_rows(res.index_map, grad_accum.to(F64), flags), remap_rows(res.index_map, denom.to(F64), flags))


def render_views(g: GaussianTensors, cameras, bg=(0.0, 0.0, 0.0), plan: Plan = None):
    plan = plan or default_plan(g.device)
    return plan.render(g, camera_rows(cameras), bg)


def accumulate_stats_(grad_accum: torch.Tensor, denom: torch.Tensor, viewspace_grad: torch.Tensor,
                      visible: torch.Tensor):
    """In-place DensifyStats feed on device (ref/adc.py:73-79):
    grad_accum[visible] += |viewspace_grad|_2, denom[visible] += 1.

    viewspace_grad is the [N,2] d loss / d projected mean (GradOutput,
    ref/raster.py:49-58) in fp64 (the reference's precision, bit-identical
    norms) or fp32 (a GPU rasterizer's); visible is a [N] bool/uint8 mask.
    grad_accum/denom are updated in place and must be contiguous fp64 CUDA
    tensors on the gradient's device."""
    lib = _abi.load()
    if grad_accum.dtype != F64 or denom.dtype != F64:
        raise TypeError("stats must be float64")
    n = len(grad_accum)
    if len(denom) != n or len(visible) != n or len(viewspace_grad) != n:
        raise ValueError("stats dimensions do not match gradient output")
    if viewspace_grad.dim() != 2 or viewspace_grad.shape[1] != 2:
        raise ValueError(f"viewspace_grad must be [N,2], got {tuple(viewspace_grad.shape)}")
    if viewspace_grad.dtype not in (F32, F64):
        raise TypeError("viewspace_grad must be float32 or float64")
    for name, t in (("grad_accum", grad_accum), ("denom", denom), ("viewspace_grad", viewspace_grad),
                    ("visible", visible)):
        if not t.is_cuda or t.device != grad_accum.device:
            raise ValueError(f"{name} must be on {grad_accum.device}")
    for name, t in (("grad_accum", grad_accum), ("denom", denom)):
        if t.dim() != 1 or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous 1-D tensor (updated in place)")
    vg = viewspace_grad.contiguous()
    vis = visible.to(torch.uint8).contiguous()
    stream = C.c_void_p(torch.cuda.current_stream(grad_accum.device).cuda_stream)
    fn = lib.adps_accumulate_stats_f64 if vg.dtype == F64 else lib.adps_accumulate_stats
    _abi.check(fn(stream, _ptr(grad_accum), _ptr(denom), _ptr(vg), _ptr(vis), n))


def prune(g: GaussianTensors, threshold: float, *, rows=(), logit_op: torch.Tensor = None, plan: Plan = None):
    """Opacity prune on the device (ref/harness.py:320-340, ``_prune``).

    keep = opacity >= threshold (the fp32 opacity, or sigmoid(logit_op) when
    the trainer keeps fp64 logits, ref/harness.py:217-218); like the
    reference, nothing is pruned when every or no Gaussian survives.  ``rows``
    are per-Gaussian tensors carried over for the survivors (optimizer
    moments, DensifyStats, logits), gathered by adps_remap_rows.
    Returns (GaussianTensors, [rows...], index_map [n_keep] int64 or None, n_near)."""
    plan = plan or default_plan(g.device)
    im, nk, near = plan.prune_index(threshold, opacity=None if logit_op is not None else g.opacity,
                                    logit_op=logit_op)
    if nk == 0 or nk == g.n:
        return g, list(rows), None, near
    gather = [remap_rows(im, getattr(g, f)) for f in ("mu", "scale", "rot", "opacity", "sh_dc")]
    rest = remap_rows(im, g.sh_rest) if g.sh_k else None
    return GaussianTensors(*gather, rest), [remap_rows(im, r) for r in rows], im, near


# ----------------------------------------------------------------------------
# reference API (object types)
# ----------------------------------------------------------------------------

def _scene_arrays(gaussians):
    n = len(gaussians)
    k = max((len(x.sh_rest) for x in gaussians), default=0)
    rest = np.zeros((n, k, 3))
    for i, x in enumerate(gaussians):
        for j, c in enumerate(x.sh_rest):
            rest[i, j] = c
    return (np.array([x.mu for x in gaussians], dtype=np.float64).reshape(n, 3),
            np.array([x.scale for x in gaussians], dtype=np.float64).reshape(n, 3),
            np.array([x.rot for x in gaussians], dtype=np.float64).reshape(n, 4),
            np.array([x.opacity for x in gaussians], dtype=np.float64).reshape(n),
            np.array([x.sh_dc for x in gaussians], dtype=np.float64).reshape(n, 3), rest)


def _clamp_opacity(o):
    return min(max(o, 1e-6), 1.0 - 1e-6)


def adpsplit_step(scene, cameras, gt_images, stats, cfg, rng, *, plan: Plan = None, renders=None):
    """Drop-in for ``adpsplit.adc.adpsplit_step`` (ref/adc.py:143-245).

    Mutates ``scene.gaussians`` (survivors are the same objects, in the old
    order, followed by the inserted Gaussians) and returns (scene, SplitReport).
    Parameters are processed in fp32 on the GPU; inserted parent copies,
    clones and the exact-copy fields of fallback children are taken from
    the original objects so the opacity bookkeeping holds to fp64.
    """
    if cfg.v_views > len(cameras):
        raise ValueError(f"v_views={cfg.v_views} exceeds available cameras ({len(cameras)})")
    dev = _require_cuda()
    plan = plan or default_plan(dev)
    gs = list(scene.gaussians)
    mu, scale, rot, op, dc, rest = _scene_arrays(gs)
    g = GaussianTensors.from_numpy(mu, scale, rot, op, dc, rest if rest.shape[1] else None, dev)
    view_ids = sample_views(len(cameras), cfg.v_views, rng)
    rnd = None
    if renders is not None:
        rnd = renders(view_ids) if callable(renders) else renders
    res = densify_step(g, scene.extent, cameras, gt_images,
                       torch.as_tensor(np.asarray(stats.grad_accum, dtype=np.float64), device=dev),
                       torch.as_tensor(np.asarray(stats.denom, dtype=np.float64), device=dev),
                       cfg, rng, renders=rnd, plan=plan, view_ids=view_ids)
    rep = res.report()
    outg = res.gaussians.numpy()
    make = type(gs[0]) if gs else Gaussian3D
    new = [gs[int(i)] for i in rep.index_map[rep.index_map >= 0]]
    pos = len(new)
    for rec in rep.candidates:
        p = gs[rec.index]
        if rec.fallback:
            for _ in range(2):
                new.append(make(mu=outg["mu"][pos].astype(np.float64), scale=p.scale / (cfg.eta * 2),
                                rot=p.rot, opacity=p.opacity, sh_dc=p.sh_dc, sh_rest=p.sh_rest))
                pos += 1
        elif not rec.reset:
            for _ in range(rec.children_inserted):
                q = outg["rot"][pos].astype(np.float64)
                new.append(make(mu=outg["mu"][pos].astype(np.float64),
                                scale=outg["scale"][pos].astype(np.float64), rot=q / np.linalg.norm(q),
                                opacity=_clamp_opacity(float(p.opacity)),
                                sh_dc=outg["sh_dc"][pos].astype(np.float64), sh_rest=()))
                pos += 1
            new.append(make(mu=p.mu, scale=p.scale, rot=p.rot,
                            opacity=_clamp_opacity(p.opacity / (rec.children_inserted + 1)),
                            sh_dc=p.sh_dc, sh_rest=p.sh_rest))
            pos += 1
    for i in rep.clones:
        p = gs[i]
        new.append(make(mu=p.mu, scale=p.scale, rot=p.rot, opacity=p.opacity, sh_dc=p.sh_dc,
                        sh_rest=p.sh_rest))
        pos += 1
    if pos != rep.count_after:
        raise RuntimeError(f"population mismatch: built {pos}, device reported {rep.count_after}")
    scene.gaussians = new
    return scene, rep


def vanilla_densify(scene, stats, cfg, n_children: int, rng, *, plan: Plan = None):
    """Drop-in for ``adpsplit.adc.vanilla_densify`` (ref/adc.py:248-280): the
    binary ADC baseline, computed on the GPU; mutates ``scene.gaussians``
    (survivors are the same objects) and returns (scene, SplitReport)."""
    dev = _require_cuda()
    plan = plan or default_plan(dev)
    gs = list(scene.gaussians)
    mu, scale, rot, op, dc, rest = _scene_arrays(gs)
    g = GaussianTensors.from_numpy(mu, scale, rot, op, dc, rest if rest.shape[1] else None, dev)
    res = vanilla_densify_step(g, scene.extent, torch.as_tensor(np.asarray(stats.grad_accum, dtype=np.float64),
                                                                device=dev),
                               torch.as_tensor(np.asarray(stats.denom, dtype=np.float64), device=dev), cfg,
                               n_children, rng, plan=plan)
    rep = res.report()
    for rec in rep.candidates:
        rec.children_inserted = int(n_children)
    outg = res.gaussians.numpy()
    make = type(gs[0]) if gs else Gaussian3D
    new = [gs[int(i)] for i in rep.index_map[rep.index_map >= 0]]
    pos = len(new)
    for rec in rep.candidates:
        p = gs[rec.index]
        for _ in range(n_children):
            new.append(make(mu=outg["mu"][pos].astype(np.float64), scale=p.scale / (cfg.eta * n_children),
                            rot=p.rot, opacity=p.opacity, sh_dc=p.sh_dc, sh_rest=p.sh_rest))
            pos += 1
    for i in rep.clones:
        p = gs[i]
        new.append(make(mu=p.mu, scale=p.scale, rot=p.rot, opacity=p.opacity, sh_dc=p.sh_dc, sh_rest=p.sh_rest))
        pos += 1
    if pos != rep.count_after:
        raise RuntimeError(f"population mismatch: built {pos}, device reported {rep.count_after}")
    scene.gaussians = new
    return scene, rep


def remap_stats_ref(stats, report):
    """Drop-in for ``adpsplit.adc.remap_stats`` (ref/adc.py:283-296) on the GPU:
    carried Gaussians keep their accumulators unless reset or cloned."""
    dev = _require_cuda()
    n_old = len(np.asarray(stats.grad_accum))
    flags = np.zeros(max(n_old, 1), np.uint8)
    flags[[int(i) for i in report.reset_indices] + [int(i) for i in report.clones]] = 1
    im = torch.as_tensor(np.asarray(report.index_map, dtype=np.int64), device=dev)
    fl = torch.as_tensor(flags, device=dev)
    ga = remap_rows(im, torch.as_tensor(np.asarray(stats.grad_accum, dtype=np.float64), device=dev), fl)
    de = remap_rows(im, torch.as_tensor(np.asarray(stats.denom, dtype=np.float64), device=dev), fl)
    return type(stats)(grad_accum=ga.cpu().numpy(), denom=de.cpu().numpy())


@dataclass
class RenderOutput:
    image: np.ndarray
    dominant_map: np.ndarray
    background: np.ndarray


def render(scene, cam, background) -> RenderOutput:
    """Drop-in for ``adpsplit.raster.render`` (ref/raster.py:136-157), fp32 on the GPU."""
    dev = _require_cuda()
    bg = np.asarray(background, dtype=np.float64)
    mu, scale, rot, op, dc, rest = _scene_arrays(list(scene.gaussians))
    g = GaussianTensors.from_numpy(mu, scale, rot, op, dc, rest if rest.shape[1] else None, dev)
    img, dom = render_views(g, camera_rows([cam]), bg)
    return RenderOutput(image=img[0].double().cpu().numpy(), dominant_map=dom[0].long().cpu().numpy(),
                        background=bg)
