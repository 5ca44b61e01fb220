"""Deterministic backward at 4K (config E scene, 64,800 tiles): two det runs
bit-identical, det vs fast within float-atomic noise."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_configs import make  # noqa: E402

import paper_2503_01199_b200 as sb  # noqa: E402

scene, _, views, targets = make(6_000_000, (3840, 2160), 1)
res = {}
for name, det in (("det1", True), ("det2", True), ("fast", False)):
    cfg = sb.RasterConfig(deterministic=det)
    out, ctx = sb.forward(scene, views[0], cfg)
    _, dI = sb.loss_and_grad(out.color, targets[0], 0.2, return_tensor=True)
    r = sb.backward(scene, ctx, dI, sb.DensifyStats.zeros(scene.n, scene.device))
    res[name] = (r.grads.packed.clone(), r.stats.S.clone(), r.stats.C.clone())
    print(name, "P", ctx.n_pairs, "tiles", ctx.camera.tiles)
same = [torch.equal(a, b) for a, b in zip(res["det1"], res["det2"])]
g1, g2 = res["det1"][0], res["fast"][0]
rel = ((g1 - g2).abs().max() / g2.abs().max()).item()
print(f"det runs bit-identical (grads, S, C): {same}; det vs fast max rel diff {rel:.3e}; "
      f"C equal {torch.equal(res['det1'][2], res['fast'][2])}")
