"""Pinhole camera contract (host side, float64) and its C-ABI struct.

Same fields and conventions as the reference CameraView
(pkg/src/tinysplat/camera.py:14-51): x right, y down, z forward; pixel =
focal * xy / z + principal_point with integer pixel centres.  The frustum
planes (projection.py:38-65) are computed here once per view with the same
float64 expressions and shipped to the device inside `sb_camera`.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import SbCamera


@dataclass
class CameraView:
    world_to_camera: np.ndarray  # (4, 4) rigid transform
    focal: np.ndarray            # (fx, fy) pixels
    principal_point: np.ndarray  # (cx, cy) pixels
    resolution: tuple            # (width, height)
    near: float
    far: float

    def __post_init__(self):
        self.world_to_camera = np.asarray(self.world_to_camera, dtype=np.float64).reshape(4, 4)
        self.focal = np.asarray(self.focal, dtype=np.float64).reshape(2)
        self.principal_point = np.asarray(self.principal_point, dtype=np.float64).reshape(2)
        self.resolution = (int(self.resolution[0]), int(self.resolution[1]))
        self.near, self.far = float(self.near), float(self.far)
        if not (0.0 < self.near < self.far):
            raise ValueError(f"need 0 < near < far, got near={self.near} far={self.far}")
        R = self.rotation
        if not np.allclose(R @ R.T, np.eye(3), atol=1e-6):
            raise ValueError("world_to_camera rotation block is not orthonormal")

    @classmethod
    def from_any(cls, cam) -> "CameraView":
        """Accept the reference's CameraView (or any duck-typed equivalent)."""
        if isinstance(cam, cls):
            return cam
        return cls(cam.world_to_camera, cam.focal, cam.principal_point, cam.resolution, cam.near, cam.far)

    @property
    def rotation(self):
        return self.world_to_camera[:3, :3]

    @property
    def translation(self):
        return self.world_to_camera[:3, 3]

    @property
    def center(self):
        return -self.rotation.T @ self.translation

    @property
    def tiles(self):
        W, H = self.resolution
        return (W + 15) // 16, (H + 7) // 8

    def frustum_planes(self) -> np.ndarray:
        return frustum_planes(self)

    def struct(self) -> SbCamera:
        """The C-ABI struct, rebuilt only when a field changed (the frustum
        planes cost ~50 us of numpy per build; callers pass the struct by
        reference and the library copies it at launch)."""
        key = (self.world_to_camera.tobytes(), self.focal.tobytes(), self.principal_point.tobytes(),
               self.resolution, self.near, self.far)
        cached = self.__dict__.get("_struct_cache")
        if cached is not None and cached[0] == key:
            return cached[1]
        s = self._build_struct()
        self.__dict__["_struct_cache"] = (key, s)
        return s

    def _build_struct(self) -> SbCamera:
        s = SbCamera()
        s.w2c[:] = [float(v) for v in self.world_to_camera.reshape(16)]
        s.fx, s.fy = float(self.focal[0]), float(self.focal[1])
        s.cx, s.cy = float(self.principal_point[0]), float(self.principal_point[1])
        s.near_plane, s.far_plane = self.near, self.far
        s.planes[:] = [float(v) for v in frustum_planes(self).reshape(24)]
        s.width, s.height = self.resolution
        return s


@dataclass
class Frustum:
    """projection.py:24-35: six inward-facing unit planes (n, d), a point x
    is inside iff n.x + d >= 0 for all six."""
    planes: np.ndarray  # (6, 4) float64

    def signed_distances(self, points) -> np.ndarray:
        points = np.atleast_2d(np.asarray(points, dtype=np.float64))
        return points @ self.planes[:, :3].T + self.planes[:, 3]

    def contains(self, points) -> np.ndarray:
        return np.all(self.signed_distances(points) >= 0.0, axis=-1)


def build_frustum(camera) -> Frustum:
    """projection.py:38-65: (6, 4) inward unit planes n.x + d >= 0: near,
    far, left (u >= 0), right (u <= W-1), top (v >= 0), bottom (v <= H-1)."""
    return Frustum(frustum_planes(camera))


def frustum_planes(camera) -> np.ndarray:
    """The planes of build_frustum as a (6, 4) float64 array (same float64
    expressions and order as the reference)."""
    R = np.asarray(camera.world_to_camera, dtype=np.float64)[:3, :3]
    t = np.asarray(camera.world_to_camera, dtype=np.float64)[:3, 3]
    centre = -R.T @ t
    fx, fy = (float(v) for v in camera.focal)
    cx, cy = (float(v) for v in camera.principal_point)
    W, H = camera.resolution
    normals_cam = (
        (np.array([0.0, 0.0, 1.0]), -camera.near),
        (np.array([0.0, 0.0, -1.0]), camera.far),
        (np.array([fx, 0.0, cx]), 0.0),
        (np.array([-fx, 0.0, (W - 1) - cx]), 0.0),
        (np.array([0.0, fy, cy]), 0.0),
        (np.array([0.0, -fy, (H - 1) - cy]), 0.0),
    )
    planes = np.empty((6, 4))
    for i, (n_cam, offset) in enumerate(normals_cam):
        n_world = R.T @ n_cam
        d = offset - n_world @ centre
        norm = np.linalg.norm(n_world)
        planes[i, :3] = n_world / norm
        planes[i, 3] = d / norm
    return planes


def look_at(eye, target, up=(0.0, 1.0, 0.0)) -> np.ndarray:
    """World-to-camera rigid transform for a camera at `eye` aimed at `target`
    (camera.py:54-72 conventions)."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(np.asarray(up, dtype=np.float64), fwd)
    nr = np.linalg.norm(right)
    if nr < 1e-9:
        alt = np.array([1.0, 0.0, 0.0]) if abs(fwd[0]) < 0.9 else np.array([0.0, 0.0, 1.0])
        right = np.cross(alt, fwd)
        nr = np.linalg.norm(right)
    right = right / nr
    down = np.cross(fwd, right)
    R = np.stack([right, down, fwd])
    m = np.eye(4)
    m[:3, :3] = R
    m[:3, 3] = -R @ eye
    return m
