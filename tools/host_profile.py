"""cProfile of the host path of training iterations at config A (launch /
host bound): where the per-iteration host time goes.
    python tools/host_profile.py [iters]"""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
from bench_configs import iteration, make  # noqa: E402

import paper_2503_01199_b200 as sb  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 200
scene, state, views, targets = make(10_000, (128, 128), 1, scaled=False)
lrs = sb.LearningRates().at(0.0, position_scale=3.2)
for _ in range(5):
    iteration(scene, state, views[0], targets[0], lrs)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
for _ in range(iters):
    iteration(scene, state, views[0], targets[0], lrs)
torch.cuda.synchronize()
pr.disable()
print(f"{(time.perf_counter() - t0) / iters * 1e3:.3f} ms/iter (profiled)")
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
