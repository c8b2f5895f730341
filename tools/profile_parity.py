"""cProfile of the bench's parity leg (oracle step on k views) on the GPU box (dev tool)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_06876_b200 import operator as op  # noqa: E402
from paper_2605_06876_b200 import synth as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config3"
wl = S.CONFIGS[name]
plan = op.Plan("cuda:0")
d = wl.build_device(plan)
t = time.time()
pr = cProfile.Profile()
pr.enable()
res = bench.parity_on_sample(op, plan, wl, d, [0, 1], bench.make_cfg(wl, 2))
pr.disable()
print("parity", res, "wall", time.time() - t, "cpu_count", os.cpu_count(), flush=True)
pstats.Stats(pr).sort_stats("cumtime").print_stats(35)
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
