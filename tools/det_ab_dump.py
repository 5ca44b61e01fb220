"""A/B of the deterministic backward between two library builds: dump the
grads and S/M/C of two det-mode views at config B and a small scene.
    SB_LIB_VARIANT=... python tools/det_ab_dump.py OUT.npz"""
import sys, numpy as np, torch
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import paper_2503_01199_b200 as sb
from bench_configs import make
out = {}
for name, n, res in (("B", 1_000_000, (1920, 1080)), ("small", 20_000, (320, 240))):
    scene, state, views, targets = make(n, res, 2, scaled=(n > 100000))
    cfg = sb.RasterConfig(deterministic=True)
    for v in range(2):
        o, ctx = sb.forward(scene, views[v], cfg)
        _, dI = sb.loss_and_grad(o.color, targets[v], 0.2, return_tensor=True)
        r = sb.backward(scene, ctx, dI)
        torch.cuda.synchronize()
        out[f"{name}{v}_grads"] = r.grads.packed.cpu().numpy()
        out[f"{name}{v}_S"] = r.stats.S.cpu().numpy()
        out[f"{name}{v}_M"] = r.stats.M.cpu().numpy()
        out[f"{name}{v}_C"] = r.stats.C.cpu().numpy()
np.savez(sys.argv[1], **out)
print("saved", sys.argv[1])
