"""paper_2503_01199_b200: a B200-native (sm_100a) implementation of the LiteGS
3D Gaussian Splatting training hot path, drop-in for the reference package's
Python API (pkg/src/tinysplat/__init__.py:8-25).

Morton sort, cluster-cull-compact, projection, tile binning and per-tile
depth sort, the warp-per-tile rasterizer (forward + backward with warp
reductions), the opacity-gradient statistics and the cluster-sparse Adam
step run as hand-written CUDA kernels in libsplat_b200.so, called through
its C-ABI (include/splat_b200.h).  There is no CPU fallback.
"""
from .backward import BackwardResult, DensifyStats, SceneGrads, backward
from .camera import CameraView, Frustum, build_frustum, look_at
from .ccc import (ClusterIndex, build_clusters, cluster_visibility, compact_arrays, cull_clusters, morton_encode,
                  morton_sort, scatter_grads)
from .checkpoint import adam_state_from, checkpoint, load_checkpoint, load_ply, save_checkpoint, save_ply
from .densify import DensifyConfig, densify_step, opacity_decay, prune, variance_score
from .errors import ShapeMismatchError, StaleSceneError, TrainingDiverged, ValidationError
from .forward import (RasterConfig, RenderContext, RenderOutput, TileWorkload, blend_tile, forward, half_path_blend,
                      render)
from .projection import ProjectedScene, compose_cov3d, project_scene, quat_to_rotmat
from .metrics import loss_and_grad, psnr, ssim
from .optim import AdamState, LearningRates, adam_step
from .reduction import exp_aligned_reduce, lane_group_reduce
from .scene import SceneSoA, activate
from .train import TrainConfig, TrainResult, multiview_step, train

__all__ = [
    "BackwardResult", "DensifyStats", "SceneGrads", "backward",
    "CameraView", "Frustum", "build_frustum", "look_at", "morton_sort", "morton_encode", "ClusterIndex",
    "build_clusters", "cull_clusters", "cluster_visibility", "compact_arrays", "scatter_grads",
    "adam_state_from", "checkpoint", "load_checkpoint", "load_ply", "save_checkpoint", "save_ply",
    "DensifyConfig", "densify_step", "opacity_decay", "prune", "variance_score",
    "ShapeMismatchError", "StaleSceneError", "TrainingDiverged", "ValidationError",
    "RasterConfig", "RenderContext", "RenderOutput", "TileWorkload", "blend_tile", "half_path_blend", "forward",
    "render", "ProjectedScene", "project_scene", "compose_cov3d", "quat_to_rotmat", "activate",
    "loss_and_grad", "psnr", "ssim", "AdamState", "LearningRates", "adam_step",
    "exp_aligned_reduce", "lane_group_reduce", "SceneSoA", "TrainConfig", "TrainResult", "multiview_step", "train",
]

__version__ = "0.1.0"
