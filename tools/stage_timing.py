"""Per-stage device timing of one training iteration at a BASELINE config.

    python tools/stage_timing.py [--n 1000000] [--res 1920x1080] [--iters 10]

Times each public call with CUDA events on the current stream (after warm-up)
and prints one JSON object.  Diagnostic only; bench.py is the contract.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--res", default="1920x1080")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--deterministic", action="store_true", help="RasterConfig(deterministic=True)")
    a = ap.parse_args()
    W, H = (int(v) for v in a.res.split("x"))
    arr = scaled_scene_arrays(a.n, 7, (W, H))
    scene = sb.SceneSoA(*[arr[k] for k in ("position", "log_scale", "rotation", "color", "opacity_logit")],
                        device="cuda")
    state = sb.AdamState(scene)
    sb.DensifyStats.zeros(scene.n).attach(scene)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    sb.morton_sort(scene)
    e1.record()
    torch.cuda.synchronize()
    t_sort = e0.elapsed_time(e1)
    cam = camera_ring(SyntheticSceneSpec(n_gaussians=a.n, n_views=1, view_resolution=(W, H), seed=7))[0]
    target = torch.rand(H, W, 3, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    lrs = sb.LearningRates().at(0.0, 3.2)
    rcfg = sb.RasterConfig(deterministic=a.deterministic)
    rows = []
    for it in range(a.iters + 3):
        es = [ev() for _ in range(5)]
        es[0].record()
        out, ctx = sb.forward(scene, cam, rcfg)
        es[1].record()
        loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
        es[2].record()
        res = sb.backward(scene, ctx, dI)
        es[3].record()
        sb.adam_step(scene, res.grads, state, res.cluster_mask, lrs)
        es[4].record()
        torch.cuda.synchronize()
        if it >= 3:
            rows.append([es[i].elapsed_time(es[i + 1]) for i in range(4)])
    r = np.median(np.array(rows), axis=0)
    print(json.dumps({"deterministic": a.deterministic, "n": a.n, "res": [W, H], "P": ctx.n_pairs, "n_compact": ctx.n_compact,
                      "morton_sort_ms": t_sort, "forward_ms": r[0], "loss_ms": r[1], "backward_ms": r[2],
                      "adam_ms": r[3], "iter_ms": float(r.sum())}))


if __name__ == "__main__":
    main()
