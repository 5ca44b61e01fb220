"""Seeded synthetic inputs (input generator for benches and parity tests).

Reproduces the reference's generator draw-for-draw with numpy's PCG64
(pkg/src/tinysplat/synthetic.py:22-90: random_scene, camera_ring) so the
device path and the CPU oracle see identical float32-representable
parameters, and adds the N-scaled scenes of SURVEY.md 8(d) (configs B-E:
log_scale -= ln((N/512)^(1/3)), then every channel re-rounded through fp32).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .camera import CameraView, look_at

CHANNELS = ("position", "log_scale", "rotation", "color", "opacity_logit")


@dataclass
class SyntheticSceneSpec:
    n_gaussians: int = 512
    scene_extent: float = 1.0
    n_views: int = 8
    view_resolution: tuple = (128, 128)
    seed: int = 0
    target_kind: str = "random_gaussians"

    def __post_init__(self):
        if self.n_views < 1:
            raise ValueError("need n_views >= 1")
        if min(self.view_resolution) < 16:
            raise ValueError("resolution must be at least 16x16")


def _f32(d: dict) -> dict:
    return {k: np.asarray(v, np.float64).astype(np.float32).astype(np.float64) for k, v in d.items()}


def random_scene_arrays(spec: SyntheticSceneSpec) -> dict:
    """Raw channels as float64 arrays holding float32 values."""
    rng = np.random.default_rng(spec.seed)
    n, ext = spec.n_gaussians, spec.scene_extent
    d = {}
    d["position"] = rng.uniform(-ext, ext, size=(n, 3))
    d["log_scale"] = np.log(rng.uniform(0.04, 0.16, size=(n, 3)) * ext)
    d["rotation"] = rng.normal(size=(n, 4))
    d["color"] = rng.uniform(-1.5, 1.5, size=(n, 3))
    d["opacity_logit"] = rng.uniform(-0.5, 2.0, size=n)
    return _f32(d)


def scaled_scene_arrays(n: int, seed: int = 7, resolution=(1920, 1080)) -> dict:
    """footprints shrunk by (N/512)^(1/3)."""
    d = random_scene_arrays(SyntheticSceneSpec(n_gaussians=n, n_views=1, view_resolution=resolution, seed=seed))
    d["log_scale"] = d["log_scale"] - np.log((n / 512.0) ** (1.0 / 3.0))
    return _f32(d)


def random_scene(spec: SyntheticSceneSpec, device=None):
    from .scene import SceneSoA
    d = random_scene_arrays(spec)
    return SceneSoA(*[d[k] for k in CHANNELS], device=device)


def camera_ring(spec: SyntheticSceneSpec, center=(0.0, 0.0, 0.0)) -> list:
    """Views evenly spaced on a ring of radius 3.2 * extent, raised 0.35 of
    the radius, aimed at `center` (synthetic.py:73-90)."""
    W, H = spec.view_resolution
    f = 1.1 * max(W, H)
    rad = 3.2 * spec.scene_extent
    views = []
    for k in range(spec.n_views):
        ang = 2.0 * np.pi * k / spec.n_views
        eye = np.array(center) + rad * np.array([np.sin(ang), 0.35, np.cos(ang)])
        views.append(CameraView(world_to_camera=look_at(eye, center), focal=(f, f),
                                principal_point=((W - 1) / 2.0, (H - 1) / 2.0), resolution=(W, H),
                                near=0.05 * spec.scene_extent, far=20.0 * spec.scene_extent))
    return views
