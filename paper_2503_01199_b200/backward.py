"""Backward: raster replay + warp reductions + projection chain, on device.

Reference API: pkg/src/tinysplat/backward.py:37-92 (SceneGrads,
DensifyStats, BackwardResult) and 205-279 (backward).  Two launches:

  sb_raster_bwd            backward.py:112-267: back-to-front tile replay,
                           per-fragment dL/dalpha, scanline fold, one warp
                           reduction per channel, one atomic per (primitive,
                           tile, channel), S/M/C opacity-gradient statistics
  sb_chain_projection_bwd  backward.py:272-278: float64 chain to the raw
                           channels + scatter_grads + stats accumulation
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from .errors import ShapeMismatchError, StaleSceneError
from .ccc import CLUSTER_SIZE
from .forward import SGRAD_BYTES, RenderContext, _sgrad_clean, _stream_key
from .scene import CHANNEL_COLS, RAW_CHANNELS, SceneSoA

GRAD_CHANNELS = RAW_CHANNELS


class SceneGrads:
    """Per-channel gradient views over one (N, 16) float32 buffer (the
    optimiser consumes the packed rows directly)."""

    def __init__(self, packed: torch.Tensor):
        self.packed = packed

    def _col(self, name):
        a, b = CHANNEL_COLS[name]
        return self.packed[:, a] if b - a == 1 else self.packed[:, a:b]

    position = property(lambda s: s._col("position"))
    log_scale = property(lambda s: s._col("log_scale"))
    rotation = property(lambda s: s._col("rotation"))
    color = property(lambda s: s._col("color"))
    opacity_logit = property(lambda s: s._col("opacity_logit"))

    def as_dict(self):
        return {k: self._col(k) for k in GRAD_CHANNELS}

    @classmethod
    def zeros(cls, n, device="cuda"):
        return cls(torch.zeros((n, 16), dtype=torch.float32, device=device))

    @classmethod
    def from_dict(cls, d, n, device="cuda"):
        out = cls.zeros(n, device)
        for k, (a, b) in CHANNEL_COLS.items():
            out.packed[:, a:b] = torch.as_tensor(d[k], device=device).to(torch.float32).reshape(n, b - a)
        return out


@dataclass
class DensifyStats:
    """backward.py:59-86: S = sum f^2, M = sum f (float64), C = contributing
    fragment count (int32 on the device), per primitive."""
    S: torch.Tensor
    M: torch.Tensor
    C: torch.Tensor

    @classmethod
    def zeros(cls, n, device="cuda"):
        return cls(S=torch.zeros(n, dtype=torch.float64, device=device),
                   M=torch.zeros(n, dtype=torch.float64, device=device),
                   C=torch.zeros(n, dtype=torch.int32, device=device))

    def reset(self):
        self.S.zero_()
        self.M.zero_()
        self.C.zero_()

    def attach(self, scene: SceneSoA):
        scene.register_extra("densify_S", self.S)
        scene.register_extra("densify_M", self.M)
        scene.register_extra("densify_C", self.C)

    @classmethod
    def from_scene(cls, scene: SceneSoA):
        return cls(S=scene.extras["densify_S"], M=scene.extras["densify_M"], C=scene.extras["densify_C"])


def check_stats(stats: DensifyStats, n: int, device):
    """The chain kernel accumulates into S / M (float64) and C (int32) in
    place: wrong dtypes, lengths or devices would be misread or overrun, so
    they raise (the reference raises on mismatched lengths in np.add.at)."""
    dev = torch.device(device)
    for name, t, dt in (("S", stats.S, torch.float64), ("M", stats.M, torch.float64), ("C", stats.C, torch.int32)):
        if not torch.is_tensor(t) or t.device != dev:
            raise ValueError(f"DensifyStats.{name} must be a tensor on {dev}")
        if t.dtype != dt:
            raise ValueError(f"DensifyStats.{name} must be {dt} on the device, not {t.dtype}")
        if tuple(t.shape) != (n,):
            raise ShapeMismatchError(f"DensifyStats.{name} shape {tuple(t.shape)} != {(n,)}")
        if not t.is_contiguous():
            raise ValueError(f"DensifyStats.{name} must be contiguous (accumulated in place)")


@dataclass
class BackwardResult:
    grads: SceneGrads
    stats: DensifyStats
    cluster_mask: torch.Tensor   # (K,) bool: clusters eligible for the optimiser


def backward(scene: SceneSoA, ctx: RenderContext, dL_dI, stats: DensifyStats | None = None,
             trace=None, grads_out: torch.Tensor | None = None, accumulate: bool = False,
             chain_after: torch.cuda.Event | None = None, chain_chunks=None) -> BackwardResult:
    """backward.py:205-279.  dL_dI is (H, W, 3) (any float dtype / device;
    cast to float32 on the scene's device).  grads_out: optional preallocated
    float32 rows (>= N, 16), e.g. padded for a reduce-scatter; the gradient
    rows are its first N rows.  chain_chunks(chain, grads): runs the
    projection chain itself as chain(r0, r1) over cluster-aligned row ranges
    (ViewParallel.overlapped_step interleaves them with the gradient
    all-reduce).  chain_after: the projection chain (which
    writes grads_out and the statistics) waits for this event -- views on
    two streams serialise only their chains.  accumulate=True (needs grads_out) ADDS this
    view's rows into grads_out (rows of culled clusters untouched): a
    multi-view step sums its views in place (sb_chain_projection_bwd_accumulate)."""
    if trace is not None:
        raise ValueError("per-fragment traces are a CPU-oracle debug feature")
    if ctx.generation != scene.generation:
        raise StaleSceneError(
            f"render context generation {ctx.generation} != scene generation {scene.generation}")
    W, H = ctx.camera.resolution
    dI = torch.as_tensor(dL_dI)
    if tuple(dI.shape) != (H, W, 3):
        raise ShapeMismatchError(f"dL_dI shape {tuple(dI.shape)} != {(H, W, 3)}")
    dev = scene.device
    dI = dI.to(device=dev, dtype=torch.float32).contiguous()
    if stats is None:
        stats = DensifyStats.from_scene(scene) if "densify_S" in scene.extras else DensifyStats.zeros(scene.n, dev)
    n = scene.n
    check_stats(stats, n, dev)
    cam_s = ctx.camera.struct()
    cfg_s = ctx.config.struct()
    stream = C.c_void_p(_lib.stream_ptr(dev))
    nc = max(ctx.n_compact, 1)
    T_final, last = ctx.transmittance, ctx.last
    if ctx.half:
        # the reference's backward replays in float32 regardless of the
        # forward's blending precision: recover float32 T_final / last
        T_final = torch.empty_like(ctx.transmittance)
        last = torch.empty_like(ctx.last)
        scratch = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
        frags = torch.empty_like(ctx.last)
        ws_f = _lib.workspace("raster_fwd", _lib.load().sb_raster_workspace_bytes(), dev)
        _lib.call("sb_raster_fwd", _lib.ptr(ctx.recs), _lib.ptr(ctx.rows), _lib.ptr(ctx.tile_buffer),
                  _lib.ptr(ctx.tile_prims),
                  C.byref(cam_s), C.byref(cfg_s), _lib.ptr(scratch), _lib.ptr(T_final), _lib.ptr(frags),
                  _lib.ptr(last), _lib.ptr(ws_f), ws_f.numel(), stream)
    sgrad = _lib.workspace("sgrad", nc * SGRAD_BYTES, dev)
    # rows already zeroed by this context's forward (project kernel), unless
    # another forward or backward has used the workspace since
    prezeroed = ctx.token != 0 and _sgrad_clean.get(_stream_key(dev)) == ctx.token
    _sgrad_clean.pop(_stream_key(dev), None)
    det = int(bool(ctx.config.deterministic))
    ws_r = _lib.workspace("raster_bwd",
                          _lib.load().sb_raster_bwd_workspace_bytes(det, ctx.n_pairs, ctx.n_compact), dev)
    _lib.call("sb_raster_bwd", _lib.ptr(ctx.recs), _lib.ptr(ctx.rows), _lib.ptr(ctx.tile_buffer),
              _lib.ptr(ctx.tile_prims),
              C.byref(cam_s), C.byref(cfg_s), _lib.ptr(dI), _lib.ptr(T_final), _lib.ptr(last),
              _lib.ptr(sgrad), 0 if prezeroed else ctx.n_compact, ctx.n_pairs, ctx.n_compact, _lib.ptr(ws_r),
              ws_r.numel(), stream)
    if accumulate and grads_out is None:
        raise ValueError("accumulate=True needs grads_out (the running sum)")
    if grads_out is None:
        grads = torch.empty((n, 16), dtype=torch.float32, device=dev)
    else:
        if (grads_out.dtype != torch.float32 or grads_out.dim() != 2 or grads_out.shape[1] != 16
                or grads_out.shape[0] < n or not grads_out.is_contiguous() or grads_out.device != scene.data.device):
            raise ShapeMismatchError(f"grads_out {tuple(grads_out.shape)} {grads_out.dtype} must be contiguous "
                                     f"float32 (>= {n}, 16) on {scene.data.device}")
        grads = grads_out[:n]
    if chain_after is not None:
        torch.cuda.current_stream(dev).wait_event(chain_after)
    name = "sb_chain_projection_bwd_accumulate" if accumulate else "sb_chain_projection_bwd"

    def chain(r0: int, r1: int):
        """The chain on scene rows [r0, r1) (r0 cluster-aligned): row-offset
        views of the parameters, cluster offsets, gradients and statistics."""
        m = r1 - r0
        if m <= 0:
            return
        f4, f8, i4 = 16 * 4, 8, 4
        _lib.call(name, C.c_void_p(scene.data.data_ptr() + r0 * f4), m, C.byref(cam_s), C.byref(cfg_s),
                  C.c_void_p(ctx.cluster_offset.data_ptr() + (r0 // CLUSTER_SIZE) * i4), _lib.ptr(ctx.recs),
                  _lib.ptr(sgrad), C.c_void_p(grads.data_ptr() + r0 * f4),
                  C.c_void_p(stats.S.data_ptr() + r0 * f8), C.c_void_p(stats.M.data_ptr() + r0 * f8),
                  C.c_void_p(stats.C.data_ptr() + r0 * i4), stream)

    if chain_chunks is None:
        chain(0, n)
    else:
        # the caller's schedule: chain_chunks(chain, grads) runs the chain
        # over row ranges, e.g. interleaved with gradient exchanges
        chain_chunks(chain, grads)
    return BackwardResult(grads=SceneGrads(grads), stats=stats, cluster_mask=ctx.cluster_vis.view(torch.bool))
