"""Sharded densify step (paper_2605_06876_b200/sharded.py) on CPU: gloo, world size 2 and 3.

The orchestration -- view sharding, the all_reduce(MAX) of the ever-dominant
flags, the variable-length all_gather of the region records -- runs for real
over gloo with a stand-in executor built on the oracle's phases
(O.view_regions / O.ever_dominant / O.step_finish), and every rank's result
must equal the single-process oracle step bit for bit.  The CUDA executor
drives the same run_sharded over the plan's C ABI (tests/test_gpu_parity.py
checks that flow on one GPU with run_lockstep).
"""
import os
import pickle
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import golden_io  # noqa: E402
import parity as PA  # noqa: E402
from oracle import adpsplit_oracle as O  # noqa: E402
from paper_2605_06876_b200 import sharded as SH  # noqa: E402

TAGS = ["blobs", "desk0", "desk3", "paper1"]


def _inputs(tag):
    data, meta = golden_io.load()
    g, extent = golden_io.scene(data, f"step__{tag}__in")
    g = PA.oracle_gaussians_f32(g)
    cams = golden_io.cams(data, f"step__{tag}__cams")
    gts = PA.f32(data[f"step__{tag}__gt"])
    m = meta["step"][tag]
    return (g, extent, cams, gts, data[f"step__{tag}__grad_accum"], data[f"step__{tag}__denom"],
            golden_io.Cfg(m["cfg"]), m["seed"])


class OracleExecutor:
    """run_sharded's executor interface over the oracle's per-phase functions.

    Parent-sharded like the CUDA executor: after the merge each rank exports
    the per-candidate results of ITS range (shard_parents) and the final
    population is assembled from all ranks' exports."""

    parent_sharded = True

    def __init__(self, g, extent, cams, gts, ga, den, cfg, rng, renders):
        self.g, self.extent, self.cams, self.gts, self.cfg, self.rng = g, extent, cams, gts, cfg, rng
        self.ga, self.den, self.renders = ga, den, renders
        self.view_ids = O.sample_views(len(cams), int(O.cfg_get(cfg, "v_views")), rng)

    def begin(self, positions):
        n = len(self.g)
        self.split, self.clone = O.select(self.ga, self.den, self.g.scale, O.cfg_get(self.cfg, "tau_g"),
                                          O.cfg_get(self.cfg, "tau_s") * self.extent)
        is_cand = np.zeros(n, dtype=bool)
        is_cand[self.split] = True
        local = [self.view_ids[p] for p in positions]
        self.flags = O.ever_dominant([self.renders[v][1] for v in local], n).astype(np.uint8)
        self.regions = {v: O.view_regions(self.renders[v], self.gts[v], is_cand, self.cfg, v) for v in local}

    def dom_flags(self):
        return torch.from_numpy(self.flags.copy())

    def set_dom_flags(self, t):
        self.dom_any = t.numpy().astype(bool)

    def refresh(self):
        return int((~self.dom_any[np.asarray(self.split, dtype=np.int64)]).sum())

    def start_normals(self, nf):
        self.nf = nf   # the oracle draws them inline, in ascending parent order

    def local(self):
        return {"regions": torch.frombuffer(bytearray(pickle.dumps(self.regions)), dtype=torch.uint8)}

    def import_(self, gathered):
        self.all_regions = {}
        for t in gathered["regions"]:
            self.all_regions.update(pickle.loads(t.numpy().tobytes()))

    def merge(self):
        assert sorted(self.all_regions) == self.view_ids
        self.full = O.step_finish(self.g, self.cams, self.view_ids, self.all_regions, self.dom_any, self.split,
                                  self.clone, self.cfg, self.rng)
        self.k_lo, self.k_hi = SH.shard_parents([c.proposals for c in self.full.candidates],
                                                dist.get_world_size(), dist.get_rank())

    @staticmethod
    def _rows(c):
        return 2 if c.fallback else (0 if c.reset else c.children_inserted + 1)

    def export_shard(self):
        f = self.full
        n_keep = int((f.index_map >= 0).sum())
        start = n_keep + sum(self._rows(c) for c in f.candidates[:self.k_lo])
        stop = start + sum(self._rows(c) for c in f.candidates[self.k_lo:self.k_hi])
        rows = f.gaussians.take(np.arange(start, stop))
        edges = sum(len(gr.members) - 1 for c in f.candidates[self.k_lo:self.k_hi]
                    for gr in f.all_groups.get(c.index, []))
        return torch.frombuffer(bytearray(pickle.dumps(
            (self.k_lo, self.k_hi, f.candidates[self.k_lo:self.k_hi], rows, edges))), dtype=torch.uint8)

    def import_shards(self, blobs):
        parts = sorted((pickle.loads(b.numpy().tobytes()) for b in blobs if b.numel()), key=lambda t: t[0])
        f = self.full
        cands, rows, edges, nxt = [], [], 0, 0
        for k_lo, k_hi, cs, r, e in parts:
            if k_hi <= k_lo:
                continue
            assert k_lo == nxt, "candidate ranges must tile the split set"
            cands += cs
            rows.append(r)
            edges += e
            nxt = k_hi
        assert nxt == len(f.candidates)
        keep = np.flatnonzero(f.index_map >= 0)
        clones = [self.g.take([i]) for i in f.clones]
        res = O.StepResult(gaussians=O.Gaussians.concat([self.g.take(f.index_map[keep])] + rows + clones),
                           count_before=f.count_before, count_after=0, index_map=f.index_map, candidates=cands,
                           clones=f.clones, reset_indices=f.reset_indices, sampled_views=f.sampled_views,
                           merge_edges=edges)
        res.count_after = len(res.gaussians)
        self.assembled = res

    def emit(self):
        return self.assembled


def _digest(res):
    gs = res.gaussians
    return {"mu": gs.mu, "scale": gs.scale, "rot": gs.rot, "opacity": gs.opacity, "sh_dc": gs.sh_dc,
            "index_map": res.index_map, "clones": np.array(res.clones), "reset": np.array(res.reset_indices),
            "merge_edges": np.array([res.merge_edges]),
            "cands": np.array([[c.index, c.proposals, c.merged, c.children_inserted, int(c.fallback), int(c.reset)]
                               + list(c.regions_per_view) for c in res.candidates])}


def _renders(g, cams):
    return {v: O.render(g, cams[v]) for v in range(len(cams))}


def _worker(rank, world, port, tag, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g, extent, cams, gts, ga, den, cfg, seed = _inputs(tag)
        renders = _renders(g, cams)
        ex = OracleExecutor(g, extent, cams, gts, ga, den, cfg, np.random.default_rng(seed), renders)
        res = SH.run_sharded(ex, len(ex.view_ids))
        with open(os.path.join(out_dir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump((_digest(res), ex.rng.bit_generator.state), f)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_parents_partition():
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 1000):
        p = rng.integers(0, 50, n)
        if n:
            p[rng.integers(0, n)] = 3000   # one heavy parent
        for world in (1, 2, 3, 8):
            ranges = [SH.shard_parents(p, world, r) for r in range(world)]
            nonempty = [r for r in ranges if r[1] > r[0]]
            assert sum(hi - lo for lo, hi in nonempty) == n
            assert all(a[1] == b[0] for a, b in zip(nonempty, nonempty[1:]))


def test_shard_views_partition():
    for V in (1, 5, 64):
        for world in range(1, min(V, 8) + 1):
            parts = [SH.shard_views(V, world, r) for r in range(world)]
            assert sorted(sum(parts, [])) == list(range(V))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        SH.shard_views(4, 2, 2)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("tag", TAGS)
def test_sharded_step_matches_single_process(tmp_path, tag, world):
    g, extent, cams, gts, ga, den, cfg, seed = _inputs(tag)
    if world > int(O.cfg_get(cfg, "v_views")):
        pytest.skip("fewer sampled views than ranks")
    mp.spawn(_worker, args=(world, _free_port(), tag, str(tmp_path)), nprocs=world, join=True)
    rng = np.random.default_rng(seed)
    want = _digest(O.adpsplit_step(g, extent, cams, gts, ga, den, cfg, rng, renders=_renders(g, cams)))
    for r in range(world):
        with open(tmp_path / f"r{r}.pkl", "rb") as f:
            got, state = pickle.load(f)
        for k in want:
            np.testing.assert_array_equal(got[k], want[k], err_msg=f"rank {r}: {k}")
        assert state == rng.bit_generator.state   # the Generator advanced exactly as one process would


def test_all_gather_bytes_ragged(tmp_path):
    mp.spawn(_gather_worker, args=(3, _free_port(), str(tmp_path)), nprocs=3, join=True)
    for r in range(3):
        with open(tmp_path / f"g{r}.pkl", "rb") as f:
            got = pickle.load(f)
        assert got == [list(range(k * 5)) for k in range(3)]


def _gather_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = torch.arange(rank * 5, dtype=torch.uint8)
        parts = SH.all_gather_bytes(t)
        with open(os.path.join(out_dir, f"g{rank}.pkl"), "wb") as f:
            pickle.dump([p.tolist() for p in parts], f)
    finally:
        dist.destroy_process_group()


# ------------------------------------------------ the CUDA executor across processes
def _gpu_worker(rank, world, port, out_dir):
    """One rank of densify_step_sharded on cuda:0 (the test box has one GPU):
    the collectives run over gloo on host copies, the plan's kernels never wait
    on another rank's."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_06876_b200 import operator as op
        g, extent, cams, gts, ga, den, cfg, seed, img, dom = _gpu_inputs()
        plan = op.Plan("cuda:0")
        rng = np.random.default_rng(seed)
        res = SH.densify_step_sharded(PA.to_tensors(g), extent, cams, torch.as_tensor(gts, dtype=torch.float32,
                                                                                      device="cuda:0"),
                                      torch.as_tensor(ga, device="cuda:0"), torch.as_tensor(den, device="cuda:0"),
                                      cfg, rng, renders=(img.cuda(), dom.cuda()), plan=plan,
                                      view_ids=list(range(len(cams))))
        with open(os.path.join(out_dir, f"gpu{rank}.pkl"), "wb") as f:
            pickle.dump((_gpu_digest(res), rng.bit_generator.state), f)
    finally:
        dist.destroy_process_group()


def _gpu_inputs():
    from paper_2605_06876_b200 import synth as S
    from paper_2605_06876_b200.types import AdpSplitConfig
    wl = S.Workload("sharded", 20_000, 6, 160, 112, 0.05, 0.02, 0.02 * np.sqrt(2_400_000 / 20_000),
                    large_range=(0.005 * np.sqrt(120), 0.01 * np.sqrt(120)), seed=3)
    ini, cams, (ga, den), gt = wl.build()
    g = O.Gaussians(ini.mu, ini.scale, ini.rot, ini.opacity, ini.sh_dc)
    gt_g = O.Gaussians(gt.mu, gt.scale, gt.rot, gt.opacity, gt.sh_dc)
    from paper_2605_06876_b200 import operator as op
    plan = op.Plan("cuda:0")
    gts, _ = plan.render(PA.to_tensors(gt_g), cams)
    img, dom = plan.render(PA.to_tensors(g), cams)
    return (g, ini.extent, cams, gts.cpu().numpy(), ga, den, AdpSplitConfig(v_views=len(cams), n_max=wl.n_max), 11,
            img.cpu(), dom.cpu())


def _gpu_digest(res):
    out = dict(res.gaussians.numpy())
    out.update(index_map=res.index_map.cpu().numpy(), child_parent=res.child_parent.cpu().numpy(),
               insert_offset=res.insert_offset.cpu().numpy(),
               counts=np.array([v for k, v in sorted(res.counts.items()) if k != "n_partials"]))
    out.update({k: v.cpu().numpy() for k, v in res.report_arrays.items()})
    return out


@pytest.mark.gpu
def test_sharded_two_processes_one_gpu(tmp_path):
    """densify_step_sharded with the CUDA executor in 2 real processes (gloo
    collectives) equals the single-process densify_step bit for bit."""
    from paper_2605_06876_b200 import operator as op
    g, extent, cams, gts, ga, den, cfg, seed, img, dom = _gpu_inputs()
    rng = np.random.default_rng(seed)
    single = op.densify_step(PA.to_tensors(g), extent, cams, torch.as_tensor(gts, dtype=torch.float32,
                                                                            device="cuda:0"),
                             torch.as_tensor(ga, device="cuda:0"), torch.as_tensor(den, device="cuda:0"), cfg, rng,
                             renders=(img.cuda(), dom.cuda()), plan=op.Plan("cuda:0"),
                             view_ids=list(range(len(cams))))
    want = _gpu_digest(single)
    assert single.counts["n_regions"] > 0
    mp.spawn(_gpu_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        with open(tmp_path / f"gpu{r}.pkl", "rb") as f:
            got, state = pickle.load(f)
        for k in want:
            np.testing.assert_array_equal(got[k], want[k], err_msg=f"rank {r}: {k}")
        assert state == rng.bit_generator.state


# ------------------------------------------------ sharded stat feed (ref/adc.py:73-79)
def _acc_views(n, n_views, seed):
    rng = np.random.default_rng(seed)
    return [(rng.normal(size=(n, 2)), rng.uniform(size=n) < 0.6) for _ in range(n_views)]


def _torch_acc(ga, den, vg, vis):
    """The oracle's accumulate_stats on torch CPU tensors (stand-in for the kernel)."""
    g = ga.numpy()
    d = den.numpy()
    O.accumulate_stats(g, d, np.asarray(vg), np.asarray(vis))


def _stats_worker(rank, world, port, out_dir, n, n_views):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        views = _acc_views(n, n_views, 5)
        lo, hi = SH.view_block(n_views, world, rank)
        ga = torch.full((n,), 0.25, dtype=torch.float64)
        den = torch.full((n,), 2.0, dtype=torch.float64)
        SH.accumulate_stats_sharded_(ga, den, views[lo:hi], accumulate=_torch_acc)
        with open(os.path.join(out_dir, f"s{rank}.pkl"), "wb") as f:
            pickle.dump((ga.numpy(), den.numpy()), f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_accumulate_stats_sharded_over_views(tmp_path, world):
    """Each rank accumulates its block of views, one all_reduce(SUM) combines
    them: every rank holds the same stats, denom exact, grad_accum equal to
    the one-process view-by-view oracle within fp64 summation-order rounding."""
    n, n_views = 2000, 7
    views = _acc_views(n, n_views, 5)
    ga = np.full(n, 0.25)
    den = np.full(n, 2.0)
    for vg, vis in views:
        O.accumulate_stats(ga, den, vg, vis)
    mp.spawn(_stats_worker, args=(world, _free_port(), str(tmp_path), n, n_views), nprocs=world, join=True)
    got = []
    for r in range(world):
        with open(tmp_path / f"s{r}.pkl", "rb") as f:
            got.append(pickle.load(f))
    for g_, d_ in got:
        np.testing.assert_array_equal(g_, got[0][0])
        np.testing.assert_array_equal(d_, got[0][1])
        np.testing.assert_array_equal(d_, den)
        np.testing.assert_allclose(g_, ga, rtol=1e-13, atol=0)


def _stats_gpu_worker(rank, world, port, out_dir, n, n_views):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        views = [(torch.as_tensor(vg, device="cuda:0"), torch.as_tensor(vis, device="cuda:0"))
                 for vg, vis in _acc_views(n, n_views, 9)]
        lo, hi = SH.view_block(n_views, world, rank)
        ga = torch.full((n,), 0.25, dtype=torch.float64, device="cuda:0")
        den = torch.full((n,), 2.0, dtype=torch.float64, device="cuda:0")
        SH.accumulate_stats_sharded_(ga, den, views[lo:hi])   # the CUDA kernel per view
        with open(os.path.join(out_dir, f"sg{rank}.pkl"), "wb") as f:
            pickle.dump((ga.cpu().numpy(), den.cpu().numpy()), f)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_accumulate_stats_sharded_two_processes_one_gpu(tmp_path):
    """The sharded stat feed with the CUDA kernel in 2 real processes: ranks
    identical, denom exact, grad_accum within summation-order rounding of the
    one-process kernel sum (itself bit-exact to the reference per view)."""
    from paper_2605_06876_b200 import operator as op
    n, n_views = 50_001, 6
    ga = torch.full((n,), 0.25, dtype=torch.float64, device="cuda:0")
    den = torch.full((n,), 2.0, dtype=torch.float64, device="cuda:0")
    for vg, vis in _acc_views(n, n_views, 9):
        op.accumulate_stats_(ga, den, torch.as_tensor(vg, device="cuda:0"), torch.as_tensor(vis, device="cuda:0"))
    mp.spawn(_stats_gpu_worker, args=(2, _free_port(), str(tmp_path), n, n_views), nprocs=2, join=True)
    got = []
    for r in range(2):
        with open(tmp_path / f"sg{r}.pkl", "rb") as f:
            got.append(pickle.load(f))
    for g_, d_ in got:
        np.testing.assert_array_equal(g_, got[0][0])
        np.testing.assert_array_equal(d_, den.cpu().numpy())
        np.testing.assert_allclose(g_, ga.cpu().numpy(), rtol=1e-13, atol=0)
