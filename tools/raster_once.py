"""Config-B forward + loss + backward, a few times: the target process for
ncu captures of the raster kernels (`ncu -k regex:raster ... python
tools/raster_once.py`).  SB_RASTER_STAGING selects the staging variant."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays  # noqa: E402

n = int(os.environ.get("SB_N", "1000000"))
W, H = 1920, 1080
arr = scaled_scene_arrays(n, 7, (W, H))
scene = sb.SceneSoA(*[arr[k] for k in ("position", "log_scale", "rotation", "color", "opacity_logit")], device="cuda")
sb.morton_sort(scene)
cam = camera_ring(SyntheticSceneSpec(n_gaussians=n, n_views=1, view_resolution=(W, H), seed=7))[0]
target = torch.rand(H, W, 3, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
for _ in range(int(os.environ.get("SB_ITERS", "3"))):
    out, ctx = sb.forward(scene, cam)
    loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
    res = sb.backward(scene, ctx, dI)
torch.cuda.synchronize()
