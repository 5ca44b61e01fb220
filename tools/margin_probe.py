"""Parity margin of the backward on every fixture over repeated runs (the
backward's atomics make the low bits run-dependent): the largest
conditioned_rel_excess / floored_rel per channel group.   python tools/margin_probe.py [runs]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_01199_b200 as sb  # noqa: E402
from tests import goldens as G  # noqa: E402

CH = ((0, 3), (3, 6), (6, 10), (10, 13), (13, 14))
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 10
for fname, prefix in G.CASES:
    d = G.load(fname)
    sc = G.scene(d, prefix)
    scene = sb.SceneSoA(*[sc[k] for k in G.CH], device="cuda")
    cam = G.camera(d, prefix)
    cfg = sb.RasterConfig(background=tuple(float(b) for b in d[f"{prefix}cfg_bg"]),
                          use_culling=bool(d[f"{prefix}cfg_cull"]),
                          conic_reduce="tree" if int(d[f"{prefix}cfg_tree"]) else "exp_aligned")
    g32 = d[f"{prefix}grads"].astype(np.float64)
    g64 = d.get(f"{prefix}grads64")
    worst = np.zeros(len(CH))
    for _ in range(runs):
        out, ctx = sb.forward(scene, cam, cfg)
        res = sb.backward(scene, ctx, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n))
        g = res.grads.packed[:, :14].double().cpu().numpy()
        for q, (lo, hi) in enumerate(CH):
            v = (G.floored_rel(g[:, lo:hi], g32[:, lo:hi]) / 1e-2 if g64 is None else
                 G.conditioned_rel_excess(g[:, lo:hi], g32[:, lo:hi], g64[:, lo:hi].astype(np.float64), 1e-2))
            worst[q] = max(worst[q], v)
    print(f"{fname}:{prefix or 'A'} worst (<= 1 passes): " + " ".join(f"{w:.3f}" for w in worst))
