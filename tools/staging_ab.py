"""A/B of the raster kernels' record staging (register prefetch vs TMA bulk
copies into a double-buffered slab) at a BASELINE config, same process, same
scene, interleaved rounds; CUDA events around each raster call.

    python tools/staging_ab.py [--n 1000000] [--res 1920x1080] [--rounds 5] [--iters 10]

Prints one JSON line per staging mode (median ms of sb_raster_fwd /
sb_raster_bwd) and checks that the modes produce the same image and the same
gradients (to float-atomic order).  Diagnostic; bench.py is the contract.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200 import _lib  # noqa: E402
from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays  # noqa: E402

MODES = ("reg", "tma", "tma32")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--res", default="1920x1080")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--modes", default=",".join(MODES))
    a = ap.parse_args()
    modes = a.modes.split(",")
    W, H = (int(v) for v in a.res.split("x"))
    arr = scaled_scene_arrays(a.n, 7, (W, H))
    scene = sb.SceneSoA(*[arr[k] for k in ("position", "log_scale", "rotation", "color", "opacity_logit")],
                        device="cuda")
    sb.morton_sort(scene)
    cam = camera_ring(SyntheticSceneSpec(n_gaussians=a.n, n_views=1, view_resolution=(W, H), seed=7))[0]
    target = torch.rand(H, W, 3, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    times = {m: {"sb_raster_fwd": [], "sb_raster_bwd": []} for m in modes}
    outs = {}
    for rnd in range(a.rounds):
        for m in modes:
            os.environ["SB_RASTER_STAGING"] = m
            for it in range(a.iters + 2):
                _lib.enable_call_timing(it >= 2)
                out, ctx = sb.forward(scene, cam)
                loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
                res = sb.backward(scene, ctx, dI, sb.DensifyStats.zeros(scene.n))
                torch.cuda.synchronize()
                if it >= 2:
                    t = _lib.call_timings()
                    for k in times[m]:
                        times[m][k] += t.get(k, [])
            _lib.enable_call_timing(False)
            if rnd == 0:
                outs[m] = (out.color.clone(), out.frag_count.clone(), res.grads.packed.clone())
    ref = outs[modes[0]]
    for m in modes:
        c, f, g = outs[m]
        same_img = bool(torch.equal(c, ref[0]) and torch.equal(f, ref[1]))
        gd = float(((g - ref[2]).abs() / ref[2].abs().clamp_min(1e-3 * ref[2].abs().max())).max())
        row = {"mode": m, "P": ctx.n_pairs, "fwd_ms": float(np.median(times[m]["sb_raster_fwd"])),
               "bwd_ms": float(np.median(times[m]["sb_raster_bwd"])), "image_identical": same_img,
               "grad_floored_rel_vs_" + modes[0]: gd}
        print(json.dumps(row))


if __name__ == "__main__":
    main()
