"""Gaussian parameter tensors on the device (the SceneSoA contract).

Reference: pkg/src/tinysplat/scene.py:146-260.  Same raw channels, shapes
and restructuring semantics (single writer; permute / keep / append move
every raw channel and every registered extra together and bump
`generation` exactly once), stored B200-first:

* one float32 (N, 16) row per Gaussian — position 3 | log_scale 3 |
  rotation 4 (w x y z) | color 3 | opacity_logit 1 | pad 2 — so every kernel
  reads a Gaussian with four coalesced 128-bit loads; the channel attributes
  are views into that buffer;
* extras (Adam moments, densification statistics, ...) are device tensors
  with a leading N dimension, permuted by the same sb_permute_rows launch.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .errors import ShapeMismatchError, ValidationError

RAW_CHANNELS = ("position", "log_scale", "rotation", "color", "opacity_logit")
CHANNEL_WIDTHS = {"position": 3, "log_scale": 3, "rotation": 4, "color": 3, "opacity_logit": 1}
CHANNEL_COLS = {"position": (0, 3), "log_scale": (3, 6), "rotation": (6, 10), "color": (10, 13),
                "opacity_logit": (13, 14)}
ROW = 16


def _sigmoid64(x: torch.Tensor) -> torch.Tensor:
    """scene.py:31-38: 1 / (1 + exp(-x)) for x >= 0, exp(x) / (1 + exp(x))
    otherwise -- both are exp(-|x|) and one division (float64)."""
    e = torch.exp(-x.abs())
    return torch.where(x >= 0, 1.0 / (1.0 + e), e / (1.0 + e))


def activate(position, log_scale, rotation, color, opacity_logit):
    """scene.py:103-126: raw channels -> activated (position, scale, unit
    quaternion, color, opacity) in float64 (torch, on the inputs' device).
    Raises ValidationError naming the channel / index for non-finite values
    or zero-norm quaternions."""
    arrays = {}
    for name, v in (("position", position), ("log_scale", log_scale), ("rotation", rotation), ("color", color),
                    ("opacity_logit", opacity_logit)):
        t = v if torch.is_tensor(v) else torch.as_tensor(np.asarray(v, dtype=np.float64))
        t = t.to(torch.float64)
        bad = ~torch.isfinite(t)
        if bool(bad.any()):
            raise ValidationError(name, int(torch.nonzero(bad.reshape(t.shape[0], -1).any(1))[0, 0])
                                  if t.dim() else 0, "non-finite value")
        arrays[name] = t
    qn = torch.linalg.vector_norm(arrays["rotation"], dim=-1)
    if bool((qn == 0).any()):
        raise ValidationError("rotation", int(torch.nonzero(qn == 0).reshape(-1)[0]), "zero-norm quaternion")
    return (arrays["position"], torch.exp(arrays["log_scale"]), arrays["rotation"] / qn[..., None],
            _sigmoid64(arrays["color"]), _sigmoid64(arrays["opacity_logit"]))


def pack_rows(position, log_scale, rotation, color, opacity_logit, device=None) -> torch.Tensor:
    """Raw channels (numpy or torch, any float dtype) -> (N, 16) float32 rows."""
    chans = {"position": position, "log_scale": log_scale, "rotation": rotation, "color": color,
             "opacity_logit": opacity_logit}
    ts = {}
    for k, v in chans.items():
        if not torch.is_tensor(v):
            a = np.asarray(v)
            v = a if a.flags.writeable else a.copy()   # read-only inputs (e.g. npz views)
        t = torch.as_tensor(v)
        ts[k] = t.to(torch.float32).reshape(-1, CHANNEL_WIDTHS[k])
    n = ts["position"].shape[0]
    for k, t in ts.items():
        if t.shape[0] != n:
            raise ShapeMismatchError(f"channel '{k}' has {t.shape[0]} rows, position has {n}")
    dev = device if device is not None else (ts["position"].device if ts["position"].is_cuda else "cuda")
    out = torch.zeros((n, ROW), dtype=torch.float32, device=dev)
    for k, (a, b) in CHANNEL_COLS.items():
        out[:, a:b] = ts[k].to(dev)
    return out


class SceneSoA:
    """Device-resident scene; see module docstring."""

    def __init__(self, position, log_scale, rotation, color, opacity_logit, device=None):
        self.data = pack_rows(position, log_scale, rotation, color, opacity_logit, device)
        self.extras: dict[str, torch.Tensor] = {}
        self.generation = 0

    # ---- construction ------------------------------------------------------
    @classmethod
    def from_rows(cls, rows: torch.Tensor) -> "SceneSoA":
        obj = cls.__new__(cls)
        if rows.dim() != 2 or rows.shape[1] != ROW or rows.dtype != torch.float32:
            raise ShapeMismatchError("rows must be (N, 16) float32")
        obj.data = rows.contiguous()
        obj.extras = {}
        obj.generation = 0
        return obj

    @classmethod
    def from_reference(cls, scene, device=None) -> "SceneSoA":
        """From a reference tinysplat.SceneSoA (float64 numpy) or a dict."""
        get = (lambda k: scene[k]) if isinstance(scene, dict) else (lambda k: getattr(scene, k))
        return cls(*[get(k) for k in RAW_CHANNELS], device=device)

    @classmethod
    def empty(cls, device=None) -> "SceneSoA":
        z = np.zeros((0, 3))
        return cls(z, z, np.zeros((0, 4)), z, np.zeros(0), device=device)

    def to_numpy(self) -> dict:
        h = self.data.detach().cpu().numpy().astype(np.float64)
        return {k: (h[:, a:b] if b - a > 1 else h[:, a]).copy() for k, (a, b) in CHANNEL_COLS.items()}

    # ---- channels ------------------------------------------------------------
    def __len__(self):
        return self.data.shape[0]

    @property
    def n(self) -> int:
        return self.data.shape[0]

    @property
    def device(self):
        return self.data.device

    def _col(self, name):
        a, b = CHANNEL_COLS[name]
        return self.data[:, a] if b - a == 1 else self.data[:, a:b]

    position = property(lambda s: s._col("position"))
    log_scale = property(lambda s: s._col("log_scale"))
    rotation = property(lambda s: s._col("rotation"))
    color = property(lambda s: s._col("color"))
    opacity_logit = property(lambda s: s._col("opacity_logit"))

    def raw_channels(self):
        return {k: self._col(k) for k in RAW_CHANNELS}

    def register_extra(self, name: str, array: torch.Tensor):
        if array.shape[0] != self.n:
            raise ShapeMismatchError(f"extra '{name}' has length {array.shape[0]}, scene has {self.n}")
        self.extras[name] = array

    def validate(self):
        """scene.py:96-127 checks on the device; raises ValidationError."""
        for name in RAW_CHANNELS:
            bad = ~torch.isfinite(self._col(name))
            if bad.any():
                idx = int(torch.nonzero(bad.reshape(self.n, -1).any(1))[0, 0])
                raise ValidationError(name, idx, "non-finite value")
        qn = torch.linalg.vector_norm(self.rotation, dim=-1)
        if (qn == 0).any():
            raise ValidationError("rotation", int(torch.nonzero(qn == 0)[0, 0]), "zero-norm quaternion")

    # activated views (host convenience; the kernels activate on the fly)
    def scales(self):
        return torch.exp(self.log_scale.double())

    def unit_rotations(self):
        q = self.rotation.double()
        return q / torch.linalg.vector_norm(q, dim=-1, keepdim=True)

    def colors(self):
        return torch.sigmoid(self.color.double())

    def opacities(self):
        return torch.sigmoid(self.opacity_logit.double())

    # ---- restructuring -------------------------------------------------------
    def permute(self, perm, trusted: bool = False):
        """Gather every row (params + extras) by `perm` with sb_permute_rows."""
        perm_t = torch.as_tensor(perm, device=self.device)
        if perm_t.shape != (self.n,):
            raise ShapeMismatchError(f"permutation length {tuple(perm_t.shape)} != {self.n}")
        if perm_t.dtype.is_floating_point or perm_t.dtype == torch.bool:
            raise ValueError(f"permutation must be integer, not {perm_t.dtype}")
        if self.n and not trusted:
            # the gather kernel reads rows perm[i]: out-of-range indices would
            # read outside the arrays (the reference raises IndexError)
            lo, hi = int(perm_t.min()), int(perm_t.max())
            if lo < 0 or hi >= self.n:
                raise IndexError(f"permutation index out of range [0, {self.n}): min {lo}, max {hi}")
        perm_u = perm_t.to(torch.int32).contiguous()
        arrays = [("__data__", self.data)] + list(self.extras.items())
        outs = []
        for start in range(0, len(arrays), 16):
            chunk = arrays[start:start + 16]
            src, dst, rb = [], [], []
            for name, a in chunk:
                a = a.contiguous()
                o = torch.empty_like(a)
                src.append(a.data_ptr()); dst.append(o.data_ptr())
                rb.append(a.element_size() * (a.numel() // max(a.shape[0], 1)))
                outs.append((name, o))
            k = len(chunk)
            _lib.call("sb_permute_rows", _lib.ptr(perm_u), self.n, k, (C.c_void_p * k)(*src),
                      (C.c_void_p * k)(*dst), (C.c_int32 * k)(*rb), C.c_void_p(_lib.stream_ptr(self.device)))
        for name, o in outs:
            if name == "__data__":
                self.data = o
            else:
                self.extras[name] = o
        self.generation += 1

    def keep(self, mask):
        mask_t = torch.as_tensor(mask, device=self.device, dtype=torch.bool)
        if mask_t.shape != (self.n,):
            raise ShapeMismatchError(f"mask length {tuple(mask_t.shape)} != {self.n}")
        self.data = self.data[mask_t].contiguous()
        for k in list(self.extras):
            self.extras[k] = self.extras[k][mask_t].contiguous()
        self.generation += 1

    def append_raw(self, position, log_scale, rotation, color, opacity_logit):
        """Append primitives; extras grow with zero rows (scene.py:226-242)."""
        rows = pack_rows(position, log_scale, rotation, color, opacity_logit, self.device)
        k = rows.shape[0]
        self.data = torch.cat([self.data, rows]).contiguous()
        for name in list(self.extras):
            a = self.extras[name]
            self.extras[name] = torch.cat([a, torch.zeros((k,) + tuple(a.shape[1:]), dtype=a.dtype,
                                                          device=a.device)]).contiguous()
        self.generation += 1

    def copy(self) -> "SceneSoA":
        out = SceneSoA.from_rows(self.data.clone())
        out.extras = {k: v.clone() for k, v in self.extras.items()}
        out.generation = self.generation
        return out

    def bounds(self):
        if self.n == 0:
            z = torch.zeros(3, dtype=torch.float64, device=self.device)
            return z, z.clone()
        p = self.position
        return p.amin(0).double(), p.amax(0).double()
