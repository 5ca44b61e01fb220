"""Host-side time of each sb_* call and of the forward's device-to-host read
inside a config B training step (diagnostic for launch gaps).

    python tools/host_timing.py
"""
import collections
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200 import _lib  # noqa: E402
from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays  # noqa: E402

arr = scaled_scene_arrays(1_000_000, 7, (1920, 1080))
scene = sb.SceneSoA(*[arr[k] for k in ("position", "log_scale", "rotation", "color", "opacity_logit")], device="cuda")
state = sb.AdamState(scene)
sb.DensifyStats.zeros(scene.n).attach(scene)
sb.morton_sort(scene)
cam = camera_ring(SyntheticSceneSpec(n_gaussians=scene.n, n_views=1, view_resolution=(1920, 1080), seed=7))[0]
target = torch.rand(1080, 1920, 3, device="cuda")
lrs = sb.LearningRates().at(0.0, 3.2)

acc = collections.defaultdict(list)
orig = _lib.call


def timed_call(name, *args):
    t0 = time.perf_counter()
    r = orig(name, *args)
    acc[name].append(time.perf_counter() - t0)
    return r


_lib.call = timed_call
orig_tolist = torch.Tensor.tolist


def step():
    out, ctx = sb.forward(scene, cam)
    loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
    res = sb.backward(scene, ctx, dI)
    sb.adam_step(scene, res.grads, state, res.cluster_mask, lrs)


for _ in range(5):
    step()
torch.cuda.synchronize()
acc.clear()
phases = collections.defaultdict(list)
for _ in range(20):
    t0 = time.perf_counter()
    out, ctx = sb.forward(scene, cam)
    t1 = time.perf_counter()
    loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
    t2 = time.perf_counter()
    res = sb.backward(scene, ctx, dI)
    t3 = time.perf_counter()
    sb.adam_step(scene, res.grads, state, res.cluster_mask, lrs)
    t4 = time.perf_counter()
    phases["forward"].append(t1 - t0)
    phases["loss"].append(t2 - t1)
    phases["backward"].append(t3 - t2)
    phases["adam"].append(t4 - t3)
torch.cuda.synchronize()
for k, v in phases.items():
    print(f"host {k:10s} {1e6 * sum(v) / len(v):8.1f} us")
for k, v in acc.items():
    print(f"call {k:28s} {1e6 * sum(v) / len(v):8.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
t0 = time.perf_counter()
for _ in range(20):
    step()
e1.record()
torch.cuda.synchronize()
print(f"step: device {e0.elapsed_time(e1) / 20 * 1e3:.1f} us, host {(time.perf_counter() - t0) / 20 * 1e6:.1f} us")
