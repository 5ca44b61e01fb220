"""project_scene: the reference's projection API on the device.

Reference: pkg/src/tinysplat/projection.py:24-190 (Frustum, build_frustum,
ProjectedScene, project_scene) and scene.py:46-73 (quat_to_rotmat,
compose_cov3d).  The raster fields -- xy, depth, conic, radius, colour,
opacity, valid, in_image -- come from the fused projection kernel
(sb_project_cull_compact with culling off, so the compact records are every
Gaussian in order), bit-exact with the reference's float32 path.  The chain
fields the reference also returns (t_cam, M, cov_screen, cov_world, scale,
unit_quat) are formed on first access in float64 torch ops from the same
parameters (the device backward recomputes them inside its chain kernel; they
are not on the hot path).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .camera import CameraView, Frustum, build_frustum  # noqa: F401 (re-exported: projection.py:24-65)
from .scene import SceneSoA

LOW_PASS_DEFAULT = 0.3
EXTENT_SIGMA = 3.0


def quat_to_rotmat(q: torch.Tensor) -> torch.Tensor:
    """scene.py:46-59: unit quaternions (..., 4) wxyz -> (..., 3, 3)."""
    w, x, y, z = q.unbind(-1)
    return torch.stack([
        torch.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        torch.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        torch.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def compose_cov3d(scale, rotation) -> torch.Tensor:
    """scene.py:62-73: R diag(scale^2) R^T, symmetrised, float64; (3,) + (4,)
    or batched (N, 3) + (N, 4)."""
    s = torch.as_tensor(scale, dtype=torch.float64)
    q = torch.as_tensor(rotation, dtype=torch.float64, device=s.device)
    R = quat_to_rotmat(q)
    RD = R * (s * s)[..., None, :]
    cov = RD @ R.transpose(-1, -2)
    return 0.5 * (cov + cov.transpose(-1, -2))


@dataclass
class ProjectedScene:
    """projection.py:68-90, device tensors (N rows)."""
    xy: torch.Tensor           # (N, 2) float32
    depth: torch.Tensor        # (N,)
    conic: torch.Tensor        # (N, 3)
    radius: torch.Tensor       # (N,)
    color: torch.Tensor        # (N, 3)
    opacity: torch.Tensor      # (N,)
    valid: torch.Tensor        # (N,) bool
    in_image: torch.Tensor     # (N,) bool
    n_degenerate: int = 0
    _scene: SceneSoA | None = field(default=None, repr=False)
    _camera: CameraView | None = field(default=None, repr=False)
    _low_pass: float = LOW_PASS_DEFAULT
    _chain: dict | None = field(default=None, repr=False)

    def _chain_fields(self) -> dict:
        if self._chain is None:
            sc, cam = self._scene, self._camera
            dev = sc.device
            pos = sc.position.double()
            scale = torch.exp(sc.log_scale.double())
            quat = sc.rotation.double()
            quat = quat / torch.linalg.vector_norm(quat, dim=-1, keepdim=True)
            R = torch.as_tensor(cam.rotation, dtype=torch.float64, device=dev)
            tr = torch.as_tensor(cam.translation, dtype=torch.float64, device=dev)
            t = pos @ R.T + tr
            tz = t[:, 2]
            tz_safe = torch.where((tz > cam.near) & (tz < cam.far), tz, torch.ones_like(tz))
            fx, fy = (float(v) for v in cam.focal)
            J = torch.zeros((sc.n, 2, 3), dtype=torch.float64, device=dev)
            J[:, 0, 0] = fx / tz_safe
            J[:, 1, 1] = fy / tz_safe
            J[:, 0, 2] = -fx * t[:, 0] / tz_safe ** 2
            J[:, 1, 2] = -fy * t[:, 1] / tz_safe ** 2
            M = J @ R
            cov_world = compose_cov3d(scale, quat)
            S = M @ cov_world @ M.transpose(1, 2)
            cov_screen = torch.stack([S[:, 0, 0] + self._low_pass, S[:, 0, 1], S[:, 1, 1] + self._low_pass], 1)
            self._chain = dict(t_cam=t, M=M, cov_screen=cov_screen, cov_world=cov_world, scale=scale, unit_quat=quat)
        return self._chain

    t_cam = property(lambda s: s._chain_fields()["t_cam"])
    M = property(lambda s: s._chain_fields()["M"])
    cov_screen = property(lambda s: s._chain_fields()["cov_screen"])
    cov_world = property(lambda s: s._chain_fields()["cov_world"])
    scale = property(lambda s: s._chain_fields()["scale"])
    unit_quat = property(lambda s: s._chain_fields()["unit_quat"])


def _dtype_ok(dtype) -> bool:
    return dtype in (np.float32, "float32", torch.float32) or np.dtype(dtype) == np.float32


def project_scene(scene: SceneSoA, camera, dtype=np.float32, low_pass: float = LOW_PASS_DEFAULT) -> ProjectedScene:
    """projection.py:130-190: project every primitive on the device.

    The device path projects in float32 (the reference's RasterConfig
    default, bit-exact); the reference's float64 numeric mode exists only in
    the CPU oracle, so dtype=float64 raises ValueError (note: the reference's
    project_scene itself defaults to float64)."""
    if not _dtype_ok(dtype):
        raise ValueError("the B200 path projects in float32 (dtype=np.float32); float64 exists only in the "
                         "CPU oracle")
    from .forward import REC_FLOATS, RasterConfig
    _lib.require_cuda(scene.data)
    camera = CameraView.from_any(camera)
    dev = scene.device
    n = scene.n
    K = (n + 127) // 128
    cam_s = camera.struct()
    cfg_s = RasterConfig(use_culling=False, low_pass=low_pass).struct()
    recs = torch.empty((max(n, 1), REC_FLOATS), dtype=torch.float32, device=dev)
    cmap = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    coff = torch.empty(max(K, 1), dtype=torch.int32, device=dev)
    cvis = torch.empty(max(K, 1), dtype=torch.uint8, device=dev)
    counters = torch.zeros(8, dtype=torch.int32, device=dev)
    lib = _lib.load()
    ws = _lib.workspace("project", lib.sb_project_workspace_bytes(n), dev)
    _lib.call("sb_project_cull_compact", _lib.ptr(scene.data), n, C.byref(cam_s), C.byref(cfg_s), _lib.ptr(recs),
              _lib.ptr(cmap), _lib.ptr(coff), _lib.ptr(cvis), _lib.ptr(counters), None, None, None, None,
              _lib.ptr(ws), ws.numel(), C.c_void_p(_lib.stream_ptr(dev)))
    r = recs[:n]
    flags = r[:, 11].contiguous().view(torch.int32)
    return ProjectedScene(
        xy=r[:, 0:2], depth=r[:, 9], conic=torch.stack([r[:, 2], r[:, 3], r[:, 4]], 1), radius=r[:, 10],
        color=r[:, 6:9], opacity=r[:, 5], valid=(flags & 1) != 0, in_image=(flags & 2) != 0,
        n_degenerate=int(counters[2]), _scene=scene, _camera=camera, _low_pass=float(low_pass))
