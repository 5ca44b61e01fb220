"""Minimal driver for ncu captures: config B scene, Morton sort, then
`--iters` full training iterations (forward, loss, backward, Adam).

Per iteration the onesweep kernels launch in this order:
  hist_kernel: depth sort, tile sort       (2 per iteration, +1 for the Morton sort)
  pass_kernel: 4 depth passes, 2 tile passes (6 per iteration, +8 for the Morton sort)
so e.g. the tile-sort passes of iteration i are pass_kernel launches
8 + 6 i + 4 and 8 + 6 i + 5.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--res", default="1920x1080")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--deterministic", action="store_true")
a = ap.parse_args()
W, H = (int(v) for v in a.res.split("x"))
arr = scaled_scene_arrays(a.n, 7, (W, H))
scene = sb.SceneSoA(*[arr[k] for k in ("position", "log_scale", "rotation", "color", "opacity_logit")], device="cuda")
state = sb.AdamState(scene)
sb.DensifyStats.zeros(scene.n).attach(scene)
sb.morton_sort(scene)
cam = camera_ring(SyntheticSceneSpec(n_gaussians=a.n, n_views=1, view_resolution=(W, H), seed=7))[0]
target = torch.rand(H, W, 3, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
lrs = sb.LearningRates().at(0.0, 3.2)
for _ in range(a.iters):
    out, ctx = sb.forward(scene, cam, sb.RasterConfig(deterministic=a.deterministic))
    loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
    res = sb.backward(scene, ctx, dI)
    sb.adam_step(scene, res.grads, state, res.cluster_mask, lrs)
torch.cuda.synchronize()
print("P", ctx.n_pairs, "Nc", ctx.n_compact)
