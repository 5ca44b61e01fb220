"""Device timeline of config B training steps (torch.profiler / CUPTI):
every kernel, memset and memcpy with its start and duration, and the idle
gaps between them.  Diagnostic only.   python tools/timeline.py"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays  # noqa: E402

arr = scaled_scene_arrays(1_000_000, 7, (1920, 1080))
scene = sb.SceneSoA(*[arr[k] for k in ("position", "log_scale", "rotation", "color", "opacity_logit")], device="cuda")
state = sb.AdamState(scene)
sb.DensifyStats.zeros(scene.n).attach(scene)
sb.morton_sort(scene)
cam = camera_ring(SyntheticSceneSpec(n_gaussians=scene.n, n_views=1, view_resolution=(1920, 1080), seed=7))[0]
target = torch.rand(1080, 1920, 3, device="cuda")
lrs = sb.LearningRates().at(0.0, 3.2)


def step():
    out, ctx = sb.forward(scene, cam)
    loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
    res = sb.backward(scene, ctx, dI)
    sb.adam_step(scene, res.grads, state, res.cluster_mask, lrs)


for _ in range(5):
    step()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
# last step only: from the last projection kernel on
starts = [i for i, e in enumerate(ev) if "project_cull" in e.name]
period = ev[starts[-1]].time_range.start - ev[starts[-2]].time_range.start
ev = ev[starts[-2]:starts[-1]]
prev_end = None
idle = 0.0
# with programmatic dependent launch a kernel's CTAs may start before its
# predecessor ends (negative gap); "own" is the time it adds after that end
print("    gap       own      span")
for e in ev:
    s, d = e.time_range.start, e.time_range.elapsed_us()
    gap = 0.0 if prev_end is None else s - prev_end
    idle += max(gap, 0.0)
    own = d if prev_end is None else s + d - max(s, prev_end)
    print(f"gap {gap:7.1f}  {own:8.1f}  {d:8.1f} us  {e.name[:90]}")
    prev_end = max(s + d, prev_end or 0.0)
print(f"total idle between operations: {idle:.1f} us")
print(f"step period (projection to projection): {period:.1f} us")
