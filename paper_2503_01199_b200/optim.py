"""Cluster-sparse Adam on the device.

Reference: pkg/src/tinysplat/optim.py:20-98.  Moments are (N, 16) float32
rows aligned with the parameter rows and registered as scene extras (so
Morton re-sorts and densification carry them); per-primitive step counters
are int32.  sb_adam_sparse computes in float32 on the float32 state (beta1
0.9, beta2 0.999, eps 1e-15, per-row bias corrections 1 - beta^t formed as
-expm1(t ln beta) in float32, <= 1.9e-7 relative for t <= 2e6).  The
reference keeps float64 state and arithmetic; against it the parameters
agree to ~2e-6 relative after a few steps (tests/test_gpu_parity.py
test_adam_vs_reference), i.e. well inside one step of size ~lr.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from .scene import RAW_CHANNELS, SceneSoA

BETA1 = 0.9
BETA2 = 0.999
EPS = 1e-15
CLUSTER_SIZE = 128


@dataclass
class LearningRates:
    position: float = 1.6e-4
    position_final: float = 1.6e-6
    log_scale: float = 5e-3
    rotation: float = 1e-3
    color: float = 2.5e-3
    opacity_logit: float = 5e-2

    def at(self, progress: float, position_scale: float = 1.0) -> dict:
        """Per-channel rates at training progress in [0, 1] (optim.py:34-44)."""
        p = min(max(progress, 0.0), 1.0)
        pos = self.position * (self.position_final / self.position) ** p
        return {"position": pos * position_scale, "log_scale": self.log_scale, "rotation": self.rotation,
                "color": self.color, "opacity_logit": self.opacity_logit}


class AdamState:
    """m / v as (N, 16) float32 extras, step as (N,) int32 extra."""

    def __init__(self, scene: SceneSoA):
        dev = scene.device
        scene.register_extra("adam_m", torch.zeros((scene.n, 16), dtype=torch.float32, device=dev))
        scene.register_extra("adam_v", torch.zeros((scene.n, 16), dtype=torch.float32, device=dev))
        scene.register_extra("adam_step", torch.zeros(scene.n, dtype=torch.int32, device=dev))
        self.scene = scene

    @property
    def m_rows(self):
        return self.scene.extras["adam_m"]

    @property
    def v_rows(self):
        return self.scene.extras["adam_v"]

    @property
    def step(self):
        return self.scene.extras["adam_step"]

    def m(self, name):
        from .scene import CHANNEL_COLS
        a, b = CHANNEL_COLS[name]
        return self.m_rows[:, a] if b - a == 1 else self.m_rows[:, a:b]

    def v(self, name):
        from .scene import CHANNEL_COLS
        a, b = CHANNEL_COLS[name]
        return self.v_rows[:, a] if b - a == 1 else self.v_rows[:, a:b]


def adam_step(scene: SceneSoA, grads, state: AdamState, cluster_mask, lrs: dict,
              cluster_size: int = CLUSTER_SIZE, rows: tuple | None = None):
    """One sparse Adam update confined to true-masked clusters (optim.py:69-98).

    rows=(r0, r1) (r0 a multiple of 128) updates only scene rows [r0, r1):
    `grads` and `cluster_mask` then hold just those rows / their clusters (a
    ZeRO-1 shard, parallel.ViewParallel(zero1=True))."""
    n = scene.n
    if n == 0:
        return
    if cluster_size != CLUSTER_SIZE:
        raise ValueError("the device optimiser uses 128-primitive clusters")
    r0, r1 = (0, n) if rows is None else (int(rows[0]), int(rows[1]))
    if r0 % CLUSTER_SIZE or not (0 <= r0 <= r1 <= n):
        raise ValueError(f"row range {rows} must be cluster-aligned within [0, {n}]")
    m = r1 - r0
    if m == 0:
        return
    from .backward import SceneGrads
    if not isinstance(grads, SceneGrads):
        grads = SceneGrads.from_dict(grads.as_dict() if hasattr(grads, "as_dict") else grads, m, scene.device)
    from .errors import ShapeMismatchError
    packed = grads.packed
    if tuple(packed.shape) != (m, 16) or packed.dtype != torch.float32 or packed.device != scene.data.device:
        raise ShapeMismatchError(f"gradient rows {tuple(packed.shape)} {packed.dtype} on {packed.device} "
                                 f"!= ({m}, 16) float32 on {scene.data.device}")
    packed = packed.contiguous()
    mask = torch.as_tensor(cluster_mask, device=scene.device)
    k = (m + CLUSTER_SIZE - 1) // CLUSTER_SIZE
    if mask.numel() != k:
        raise ShapeMismatchError(f"cluster mask length {mask.numel()} != {k} clusters")
    mask = (mask.view(torch.uint8) if mask.dtype == torch.bool else (mask != 0).to(torch.uint8)).contiguous()
    for name, t in (("m", state.m_rows), ("v", state.v_rows), ("step", state.step)):
        if t.shape[0] != n or t.device != scene.data.device:
            raise ShapeMismatchError(f"Adam {name} has {t.shape[0]} rows on {t.device} != {n} on {scene.data.device}")
    lr = (C.c_double * 5)(*[float(lrs[k]) for k in RAW_CHANNELS])
    _lib.call("sb_adam_sparse", _lib.ptr(scene.data[r0:r1]), _lib.ptr(packed), _lib.ptr(state.m_rows[r0:r1]),
              _lib.ptr(state.v_rows[r0:r1]), _lib.ptr(state.step[r0:r1]), _lib.ptr(mask), m, lr,
              C.c_void_p(_lib.stream_ptr(scene.device)))
