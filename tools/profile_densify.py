"""Phase timings of one densification event at config C (3M Gaussians, 1080p).

    python tools/profile_densify.py
Each phase is bracketed by a device synchronisation (host wall clock), so
the numbers add up to the event's cost including allocator growth.
"""
from __future__ import annotations

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200 import densify as D  # noqa: E402
from bench_configs import make, iteration  # noqa: E402


def main():
    n0 = 3_000_000
    scene, state, views, targets = make(n0, (1920, 1080), 100)
    lrs = sb.LearningRates().at(0.0, position_scale=3.2)
    for vi in range(20):
        iteration(scene, state, views[vi], targets[vi % len(targets)], lrs)
    dcfg = sb.DensifyConfig(start_epoch=1, densify_interval_epochs=1, budget=int(1.05 * n0))
    out = {}
    for rnd in range(2):
        ph = {}
        torch.cuda.synchronize()

        def tick(name, t0):
            torch.cuda.synchronize()
            t = time.perf_counter()
            ph[name] = (t - t0) * 1e3
            return t

        t = time.perf_counter()
        stats = sb.DensifyStats.from_scene(scene)
        scores = D.variance_score(stats)
        t = tick("score", t)
        thr = dcfg.resolve_split_threshold(scene)
        t = tick("threshold", t)
        clone_idx, split_idx = D.select_and_grow(scene, scores, dcfg.budget, thr)
        t = tick("select", t)
        D.apply_growth(scene, clone_idx, split_idx)
        t = tick("grow", t)
        D.prune(scene, dcfg.prune_opacity)
        t = tick("prune", t)
        sb.DensifyStats.from_scene(scene).reset()
        t = tick("reset", t)
        sb.morton_sort(scene)
        t = tick("morton_sort", t)
        iteration(scene, state, views[0], targets[0], lrs)
        t = tick("first_iteration_after", t)
        iteration(scene, state, views[1], targets[1], lrs)
        t = tick("second_iteration_after", t)
        ph["n"] = scene.n
        ph["n_clone"] = int(clone_idx.numel())
        out[f"event{rnd}"] = ph
        dcfg.budget = int(1.10 * n0)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
