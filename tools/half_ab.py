"""Blending-state precision A/B at a BASELINE config: the fp32 forward, the
fp16 (reference half path, forward.py:194-230) and bf16 forwards, each 16-bit
one as the scalar kernel and the pixel-pair packed (half2 / bfloat162)
kernel.  CUDA events around sb_raster_fwd, median over interleaved rounds;
the packed kernels must reproduce the scalar ones bit for bit.

    python tools/half_ab.py [--n 1000000] [--res 1920x1080] [--rounds 5] [--iters 10]
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

MODES = (("fp32", False, None), ("fp16_scalar", True, "1"), ("fp16_packed", True, "0"),
         ("bf16_scalar", "bf16", "1"), ("bf16_packed", "bf16", "0"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--res", default="1920x1080")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    W, H = (int(v) for v in a.res.split("x"))
    arr = scaled_scene_arrays(a.n, 7, (W, H))
    scene = sb.SceneSoA(*[arr[k] for k in ("position", "log_scale", "rotation", "color", "opacity_logit")],
                        device="cuda")
    sb.morton_sort(scene)
    cam = camera_ring(SyntheticSceneSpec(n_gaussians=a.n, n_views=1, view_resolution=(W, H), seed=7))[0]
    times = {m[0]: [] for m in MODES}
    outs = {}
    for rnd in range(a.rounds):
        for name, half, scalar in MODES:
            if scalar is not None:
                os.environ["SB_HALF_SCALAR"] = scalar
            for it in range(a.iters + 2):
                _lib.enable_call_timing(it >= 2)
                out, ctx = sb.forward(scene, cam, half=half)
                torch.cuda.synchronize()
                if it >= 2:
                    times[name] += _lib.call_timings().get("sb_raster_fwd", [])
            _lib.enable_call_timing(False)
            if rnd == 0:
                outs[name] = (out.color.clone(), out.transmittance.clone(), out.frag_count.clone())
    os.environ.pop("SB_HALF_SCALAR", None)
    ref = outs["fp32"][0].double()
    for name, half, scalar in MODES:
        c = outs[name][0].double()
        mse = float(((c - ref) ** 2).mean())
        row = {"mode": name, "P": ctx.n_pairs, "raster_fwd_ms": float(np.median(times[name])),
               "psnr_vs_fp32_db": 99.0 if mse == 0 else float(10 * np.log10(1 / mse))}
        if name.endswith("packed"):
            sc = outs[name.replace("packed", "scalar")]
            row["bit_identical_to_scalar"] = all(torch.equal(x, y) for x, y in zip(outs[name], sc))
        print(json.dumps(row))


if __name__ == "__main__":
    main()
