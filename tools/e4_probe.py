import sys, os, dataclasses
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from tests import goldens as G
from tests.test_gpu_parity import _scene, _cfg, CH_SLICES
import paper_2503_01199_b200 as sb
d = G.load("golden_edge.npz"); prefix = "e4_"
scene, cam, cfg = _scene(d, prefix), G.camera(d, prefix), _cfg(d, prefix)
g64 = d[f"{prefix}grads64"].astype(np.float64); g32 = d[f"{prefix}grads"].astype(np.float64)
def errs(c):
    out, ctx = sb.forward(scene, cam, c)
    res = sb.backward(scene, ctx, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n))
    g = res.grads.packed[:, :14].double().cpu().numpy()
    r = []
    for lo, hi in CH_SLICES:
        den = np.maximum(np.abs(g64[:, lo:hi]), 1e-3 * np.abs(g64[:, lo:hi]).max())
        err = np.abs(g[:, lo:hi] - g64[:, lo:hi]) / den
        ref_err = np.abs(g32[:, lo:hi] - g64[:, lo:hi]) / den
        exc = ref_err.max(axis=1) > 0.5e-2
        r.append(err[~exc].max(initial=0.0))
    return r
fast = np.array([errs(cfg) for _ in range(40)])
print("fast max per slice", fast.max(0)); print("fast median", np.median(fast, 0))
print("det", errs(dataclasses.replace(cfg, deterministic=True)))

# fast (atomic order) vs the fixed-order backward, floored relative over all channels
def grads(c):
    out, ctx = sb.forward(scene, cam, c)
    return sb.backward(scene, ctx, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n)).grads.packed.double().cpu().numpy()
det = grads(dataclasses.replace(cfg, deterministic=True))
rel = []
for _ in range(40):
    f = grads(cfg)
    den = np.maximum(np.abs(det), 1e-3 * np.abs(det).max(axis=0, keepdims=True))
    rel.append(float((np.abs(f - det) / np.maximum(den, 1e-30)).max()))
print("fast vs det floored rel: median %.2e max %.2e" % (np.median(rel), max(rel)))
