"""Multi-GPU AdpSplit densify step: one process per GPU over torch.distributed.

SURVEY.md 8(e), following the path's own data dependencies:

  Phase A (view-sharded).  Rank r owns a contiguous block of the sampled-view
  positions, [r*V/g, (r+1)*V/g) (g = world size), so its attribution inputs
  (image, dominant, gt) are zero-copy slices of the [V,H,W,...] arrays.  It runs select, the per-view error maps,
  partition, region statistics and child initialisation for its views only
  (ref/adc.py:165-196) -- every per-view stage is independent across views.
  The ever-dominant flags (ref/adc.py:177-180, an OR over all sampled views)
  are combined with ONE all_reduce(MAX) of an N-byte vector, after which the
  global fallback count is known and the fallback normals can be drawn.

  Exchange.  Region records (64 B, global view positions), their proposals
  (152 B) and valid flags are packed into one byte blob per rank and
  all-gathered (one size all_gather + one padded data all_gather, one host
  read of the sizes); each rank hands the concatenation to its plan.
  Records are merged in their (candidate, view, band, first pixel) key order,
  which is the reference's order (ref/adc.py:190-195), so the concatenation
  order is irrelevant and every rank sees identical inputs.

  Phase B (parent-sharded).  The split candidates are cut into contiguous
  ranges balanced by their gate work (sum of P_k^2 + 1, shard_parents); each
  rank gates, groups and caps only its range (ref/cross_view_merge.py), then
  the per-parent results (children per parent, inserted counts) and the
  children rows are all-gathered, and the offsets and compaction run on every
  rank over identical inputs -- every rank ends with the identical grown
  arrays (what the next data-parallel training step needs).

  Stat feed.  accumulate_stats_sharded_ shards the per-view accumulation of
  the training's DensifyStats (ref/adc.py:73-79) over views and sums the
  per-rank partials with one all_reduce(SUM) of a [2,N] fp64 buffer.

The orchestration is written against a small executor interface so that the
same code drives the CUDA plan (GpuExecutor) and, in the CPU tests, a
stand-in executor built on the oracle (tests/test_sharded.py, gloo, world 2).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import operator as op


def view_block(n_views: int, world: int, rank: int) -> tuple:
    """[lo, hi) of the sampled-view positions owned by `rank` (contiguous blocks)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * n_views // world, (rank + 1) * n_views // world


def shard_views(n_views: int, world: int, rank: int) -> list:
    """Positions (into the sorted sampled view ids) owned by `rank`: one contiguous block."""
    lo, hi = view_block(n_views, world, rank)
    return list(range(lo, hi))


def shard_parents(p_counts, world: int, rank: int) -> tuple:
    """[lo, hi) of the split candidates `rank` merges: candidate k goes to rank
    floor(W_<k * world / W), W_<k the exclusive prefix of w = P_k^2 + 1 (the
    host statement of the device rule in merge.cu shard_range_kernel)."""
    w = [int(p) * int(p) + 1 for p in p_counts]
    total = sum(w)
    lo, hi, excl = len(w), 0, 0
    for k, wk in enumerate(w):
        owner = min(world - 1, excl * world // total) if total else 0
        if owner == rank:
            lo, hi = min(lo, k), max(hi, k + 1)
        excl += wk
    return (lo, hi) if hi > lo else (0, 0)


def _comm_device(t: torch.Tensor, group=None) -> torch.device:
    """Where a collective on `t` runs: gloo takes host tensors, NCCL device tensors."""
    return torch.device("cpu") if dist.get_backend(group) == "gloo" else t.device


def all_reduce_max_(t: torch.Tensor, group=None) -> torch.Tensor:
    cd = _comm_device(t, group)
    if cd == t.device:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return t
    h = t.to(cd)
    dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
    t.copy_(h)
    return t


def all_reduce_sum_(t: torch.Tensor, group=None) -> torch.Tensor:
    cd = _comm_device(t, group)
    if cd == t.device:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return t
    h = t.to(cd)
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    t.copy_(h)
    return t


def accumulate_stats_sharded_(grad_accum: torch.Tensor, denom: torch.Tensor, views, group=None,
                              accumulate=None) -> None:
    """The stat feed of data-parallel training (ref/adc.py:73-79 per view),
    sharded over training views: each rank accumulates the gradient outputs of
    ITS views -- ``views`` is a sequence of (viewspace_grad [N,2], visible [N])
    -- into zeroed per-Gaussian partial sums with the CUDA kernel
    (``operator.accumulate_stats_``), the partials of all ranks are summed
    with ONE all_reduce(SUM) of a packed [2,N] fp64 buffer (NCCL over NVLink
    on a GPU box), and every rank adds the identical totals to its
    grad_accum / denom.  The counts in ``denom`` are exact; ``grad_accum``
    differs from one process's view-by-view sum only in the fp64 rounding of
    the summation order (the reference has no multi-process form)."""
    n = grad_accum.numel()
    part = torch.zeros(2, n, dtype=torch.float64, device=grad_accum.device)
    acc = accumulate or op.accumulate_stats_
    for vg, vis in views:
        acc(part[0], part[1], vg, vis)
    all_reduce_sum_(part.view(-1), group)
    grad_accum.add_(part[0])
    denom.add_(part[1])


def all_gather_bytes(t: torch.Tensor, group=None) -> list:
    """all_gather of 1-D uint8 tensors of different lengths: one all_gather of the
    sizes (one host read), one all_gather_into_tensor of the blobs padded to the
    largest.  Returns the per-rank blobs on t's device."""
    world = dist.get_world_size(group)
    cd = _comm_device(t, group)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=cd)
    sizes_t = torch.empty(world, dtype=torch.int64, device=cd)
    dist.all_gather_into_tensor(sizes_t, n, group=group)
    sizes = sizes_t.tolist()
    m = max(sizes) if sizes else 0
    if m == 0:
        return [t.new_empty(0) for _ in range(world)]
    pad = torch.zeros(m, dtype=torch.uint8, device=cd)
    pad[:t.numel()] = t.to(cd)
    out = torch.empty(world * m, dtype=torch.uint8, device=cd)
    dist.all_gather_into_tensor(out, pad, group=group)
    out = out.to(t.device)
    return [out[r * m:r * m + k] for r, k in enumerate(sizes)]


def _pack(parts: dict) -> torch.Tensor:
    """{name: uint8 tensor} -> one blob: int64 lengths header, then the parts in key order."""
    keys = sorted(parts)
    dev = parts[keys[0]].device
    head = torch.tensor([parts[k].numel() for k in keys], dtype=torch.int64).view(torch.uint8).to(dev)
    return torch.cat([head] + [parts[k].reshape(-1) for k in keys])


def _unpack(blob: torch.Tensor, keys) -> dict:
    keys = sorted(keys)
    h = 8 * len(keys)
    lens = blob[:h].cpu().clone().view(torch.int64).tolist() if blob.numel() else [0] * len(keys)
    out, off = {}, h
    for k, ln in zip(keys, lens):
        out[k] = blob[off:off + ln]
        off += ln
    return out


def run_sharded(ex, n_views: int, group=None):
    """The sharded step over an executor; returns the executor's emit() result.

    Executor interface (all tensors on the collective backend's device):
      begin(positions) -> counts       select + ever-dominant flags of the local views
      dom_flags() / set_dom_flags(t)   uint8 [N]
      refresh() -> n_fallback          fallback count from the reduced flags
      start_normals(n_fallback)        start drawing the 6F fallback normals
      local() -> {name: uint8 tensor}  local region records / proposals / valid flags
      import_(dict of per-rank lists)  the gathered records
      merge() -> counts                merge + cap of this rank's parents (all, if not parent-sharded)
      export_shard() -> uint8 tensor   this rank's per-parent results (parent-sharded executors)
      import_shards(list of blobs)     every rank's results; finishes phase 1 (offsets)
      emit() -> result                 the grown Gaussians (identical on every rank)
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world > n_views:
        raise ValueError(f"{world} ranks but only {n_views} sampled views to shard")
    ex.begin(shard_views(n_views, world, rank))
    flags = ex.dom_flags()
    all_reduce_max_(flags, group)
    ex.set_dom_flags(flags)
    ex.start_normals(ex.refresh())
    recs = ex.local()
    blobs = all_gather_bytes(_pack(recs), group)
    per_rank = [_unpack(b, recs.keys()) for b in blobs]
    ex.import_({k: [p[k] for p in per_rank] for k in recs})
    ex.merge()
    if getattr(ex, "parent_sharded", False):
        ex.import_shards(all_gather_bytes(ex.export_shard(), group))
    return ex.emit()


def run_lockstep(executors: list, n_views: int):
    """run_sharded for a list of executors (rank = list position) in ONE process,
    with the two collectives done in place (OR of the flags, concatenation of
    the records).  Same stage sequence as run_sharded; used to check the
    sharded C-ABI flow on a single GPU."""
    world = len(executors)
    if world > n_views:
        raise ValueError(f"{world} ranks but only {n_views} sampled views to shard")
    for r, ex in enumerate(executors):
        ex.begin(shard_views(n_views, world, r))
    flags = [ex.dom_flags() for ex in executors]
    red = flags[0].clone()
    for f in flags[1:]:
        red = torch.maximum(red, f.to(red.device))
    for ex in executors:
        ex.set_dom_flags(red.to(flags[0].device))
        ex.start_normals(ex.refresh())
    recs = [ex.local() for ex in executors]
    gathered = {k: [r[k] for r in recs] for k in recs[0]}
    for ex in executors:
        ex.import_(gathered)
    for ex in executors:
        ex.merge()
    if getattr(executors[0], "parent_sharded", False):
        blobs = [ex.export_shard() for ex in executors]
        for ex in executors:
            ex.import_shards(blobs)
    return [ex.emit() for ex in executors]


class GpuExecutor:
    """The executor interface over one rank's CUDA plan."""

    def __init__(self, g: op.GaussianTensors, extent: float, cameras, gt, grad_accum, denom, cfg, rng, *,
                 renders=None, plan: op.Plan = None, view_ids=None, want_report: bool = True,
                 world: int = 1, rank: int = 0, parent_shard: bool = True, local_views: bool = False):
        self.plan = plan or op.default_plan(g.device)
        self.g, self.extent, self.cfg, self.rng = g, extent, cfg, rng
        self.cams = op.camera_rows(cameras)
        v_views = int(cfg["v_views"] if isinstance(cfg, dict) else cfg.v_views)
        self.view_ids = list(view_ids) if view_ids is not None else op.sample_views(len(self.cams), v_views, rng)
        self.gt, self.renders = gt, renders
        self.ga = grad_accum.to(self.plan.device, op.F64).contiguous()
        self.den = denom.to(self.plan.device, op.F64).contiguous()
        self.want_report, self.world, self.rank = want_report, world, rank
        self.parent_sharded = bool(parent_shard) and world > 1
        self.local_views = bool(local_views)   # renders / gt hold only this rank's view block
        self.counts = None
        self.normals = None

    def begin(self, positions):
        P, dev = self.plan, self.plan.device
        self.positions = list(positions)
        vids = [self.view_ids[p] for p in self.positions]
        cams_v = self.cams[vids]
        lo, hi = self.positions[0], self.positions[-1] + 1
        if self.positions != list(range(lo, hi)):
            raise ValueError("view shards must be contiguous blocks of sampled-view positions")
        if self.renders is None:
            image, dom = P.render(self.g, cams_v)
        elif self.local_views:
            image = self.renders[0].to(dev, op.F32).contiguous()
            dom = self.renders[1].to(dev, torch.int32).contiguous()
        else:   # zero-copy slices of the [V,...] attribution of all sampled views
            image = self.renders[0].to(dev, op.F32)[lo:hi].contiguous()
            dom = self.renders[1].to(dev, torch.int32)[lo:hi].contiguous()
        if self.local_views:
            gt_v = self.gt.to(dev, op.F32).contiguous()
            if image.shape[0] != hi - lo or gt_v.shape[0] != hi - lo:
                raise ValueError(f"local_views: expected the {hi - lo} views of this rank's block")
        else:
            gt_v = op._gather_views(self.gt, vids, dev)
        self._keep = (image, dom, gt_v)
        P.set_view_sharding(lo, 1, len(self.view_ids))
        P.set_parent_sharding(self.rank, self.world) if self.parent_sharded else P.set_parent_sharding(0, 1)
        self.counts = P.phase1_begin(self.g, self.extent, self.ga, self.den, self.cfg, cams_v, image, gt_v, dom)
        return self.counts

    def dom_flags(self):
        return self.plan.dom_flags()

    def set_dom_flags(self, t):
        self.plan.set_dom_flags(t)

    def refresh(self):
        self.counts["n_fallback"] = self.plan.phase1_refresh()["n_fallback"]
        return self.counts["n_fallback"]

    def start_normals(self, nf):
        self._draw = op.FallbackNormals(self.plan, self.rng, nf)

    def local(self):
        self.plan.phase1_local()
        return self.plan.export_records()

    def import_(self, gathered):
        cat = {k: torch.cat(v) if v else torch.empty(0, dtype=torch.uint8, device=self.plan.device)
               for k, v in gathered.items()}
        self.plan.phase1_import(cat["regions"], cat["proposals"], cat["valid"])

    def merge(self):
        try:
            part = self.plan.phase1_merge()
            if self.parent_sharded:
                self._part = part
            else:
                self.counts = part
        finally:
            if not self.parent_sharded:
                self._unshard()
        return part

    def _unshard(self):
        self._draw.join()
        self.plan.set_view_sharding(0, 1, 0)
        self.plan.set_parent_sharding(0, 1)

    def export_shard(self):
        return self.plan.export_shard(self._part["merge_edges"], self._part["n_children"])

    def import_shards(self, blobs):
        try:
            me, nc = self.plan.import_shards(blobs)
            self.counts = self.plan.phase1_finish(me, nc)
        finally:
            self._unshard()

    def emit(self):
        normals = self._draw.result()
        counts, dev = self.counts, self.plan.device
        out = op.GaussianTensors.empty(counts["n_out"], self.g.sh_k, dev)
        index_map = torch.empty(counts["n_out"], dtype=torch.int64, device=dev)
        child_parent = torch.empty(counts["n_out"] - counts["n_keep"], dtype=torch.int32, device=dev)
        insert_offset = torch.empty(counts["n_split"], dtype=torch.int64, device=dev)
        self.plan.phase2(self.g, normals, out, index_map, child_parent, insert_offset)
        res = op.StepResult(gaussians=out, index_map=index_map, counts=counts, view_ids=list(self.view_ids),
                            normals=normals, child_parent=child_parent, insert_offset=insert_offset)
        if self.want_report:
            res.report_arrays = self.plan.report_arrays(counts["n_split"], counts["n_clone"])
        return res


def densify_step_sharded(g: op.GaussianTensors, extent: float, cameras, gt, grad_accum, denom, cfg, rng, *,
                         renders=None, plan: op.Plan = None, view_ids=None, want_report: bool = True,
                         group=None, local_views: bool = False) -> op.StepResult:
    """op.densify_step over all ranks of `group` (one GPU each); identical result on every rank.

    Every rank passes the same arguments (same Generator state, same sampled
    views; `renders`, if given, are the attribution of ALL sampled views, of
    which each rank reads only its own block).  With ``local_views`` the
    renders and gt hold only this rank's block of sampled views
    (view_block(V, world, rank)), so a rank never stages the others' pixels.
    With world size 1 this is op.densify_step.
    """
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return op.densify_step(g, extent, cameras, gt, grad_accum, denom, cfg, rng, renders=renders, plan=plan,
                               view_ids=view_ids, want_report=want_report)
    ex = GpuExecutor(g, extent, cameras, gt, grad_accum, denom, cfg, rng, renders=renders, plan=plan,
                     view_ids=view_ids, want_report=want_report, world=dist.get_world_size(group),
                     rank=dist.get_rank(group), local_views=local_views)
    return run_sharded(ex, len(ex.view_ids), group)


__all__ = ["view_block", "shard_views", "all_reduce_max_", "all_reduce_sum_", "accumulate_stats_sharded_",
           "all_gather_bytes", "run_sharded", "run_lockstep", "GpuExecutor", "densify_step_sharded"]
