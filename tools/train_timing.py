"""Wall-clock time per view of the reference-facing train() loop at config B
(1M Gaussians, 1920x1080, synthetic), deterministic and fast backward, next
to the bench's device-timed iteration: what a user of train() sees.
    python tools/train_timing.py [views] [epochs]"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_configs import make  # noqa: E402

import paper_2503_01199_b200 as sb  # noqa: E402

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 20
epochs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
scene0, _, views, targets = make(1_000_000, (1920, 1080), nv)
pairs = [(views[i], targets[i % len(targets)]) for i in range(nv)]
for det in (True, False):
    scene = scene0.copy() if hasattr(scene0, "copy") else scene0
    cfg = sb.TrainConfig(epochs=1, deterministic=det, densify=sb.DensifyConfig(budget=0))
    sb.train(cfg, scene, pairs)            # warm-up epoch
    torch.cuda.synchronize()
    cfg = sb.TrainConfig(epochs=epochs, deterministic=det, densify=sb.DensifyConfig(budget=0))
    t = time.perf_counter()
    sb.train(cfg, scene, pairs)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(json.dumps({"deterministic": det, "views": nv, "epochs": epochs,
                      "ms_per_view": 1e3 * dt / (nv * epochs), "views_per_s": nv * epochs / dt}))
