"""Forward render: project -> cluster cull -> compact -> bin -> per-tile
depth sort -> warp-per-tile raster, all on the device.

Reference API: pkg/src/tinysplat/forward.py:56-94 (RasterConfig,
RenderOutput, RenderContext) and 258-308 (forward, render).  The call chain
per view is four calls through the C-ABI (include/splat_b200.h):

  sb_project_cull_compact  projection.py:130-190 + ccc.py:112-194
  sb_bin_prepare           tiles.py:75-91 exact hits counted per tile ->
                           tile offsets (-> P)
  sb_bin_finish            tiles.py:94-106: scatter (depth, slot) keys into
                           tile ranges, per-tile sort in shared memory
  sb_raster_fwd            forward.py:161-191 blend + 240-255 assembly
"""
from __future__ import annotations

import ctypes as C
import itertools
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .camera import CameraView
from .scene import SceneSoA

TILE_W, TILE_H, LANES, PIXELS_PER_LANE = 16, 8, 32, 4
CLUSTER_SIZE = 128
REC_FLOATS = 12  # 48-byte compact record
ROW_FLOATS = 16  # 64-byte raster row
TMA_STAGING = ("tma", "tma32", "g4")


@dataclass
class RasterConfig:
    """forward.py:56-71 fields.  The device path computes in float32 (the
    reference default); float64 is the CPU oracle's numeric mode only."""
    dtype: str = "float32"
    kernel: str = "scanline"
    alpha_min: float = 1.0 / 255.0
    alpha_max: float = 0.99
    t_stop: float = 1e-4
    background: tuple = (0.0, 0.0, 0.0)
    low_pass: float = 0.3
    use_culling: bool = True
    conic_reduce: str = "exp_aligned"   # backward: "exp_aligned" | "tree"
    # backward without float atomics: per-(primitive, tile) rows reduced per
    # primitive in tile order, bit-reproducible (the
    # reference's "deterministic" mode).  train() turns it on
    # with TrainConfig(deterministic=True), the reference's default.
    deterministic: bool = False

    def struct(self, half=False) -> _lib.SbRasterCfg:
        if self.dtype != "float32":
            raise ValueError("the B200 path rasterizes in float32 (dtype='float32'); "
                             "float64 exists only in the CPU oracle")
        if self.kernel != "scanline":
            raise ValueError("only the scanline kernel is implemented on the device")
        if self.conic_reduce not in ("exp_aligned", "tree"):
            raise ValueError(f"unknown conic_reduce {self.conic_reduce!r}")
        s = _lib.SbRasterCfg()
        s.alpha_min, s.alpha_max, s.t_stop = self.alpha_min, self.alpha_max, self.t_stop
        s.background[:] = [float(b) for b in self.background]
        s.low_pass = self.low_pass
        s.use_culling = int(bool(self.use_culling))
        s.conic_reduce = 0 if self.conic_reduce == "exp_aligned" else 1
        s.half_state = _half_mode(half)
        s.deterministic = int(bool(self.deterministic))
        return s


@dataclass
class RenderOutput:
    color: torch.Tensor          # (H, W, 3) float32
    transmittance: torch.Tensor  # (H, W) float32
    frag_count: torch.Tensor     # (H, W) int32


@dataclass
class TileWorkload:
    """tiles.py:30-35, materialised on demand from the device lists."""
    tile_x: int
    tile_y: int
    origin: tuple
    primitives: np.ndarray


@dataclass
class RenderContext:
    """forward.py:80-94: what the backward replays, pinned to a generation.
    Device buffers stay resident; host views are built lazily."""
    generation: int
    camera: CameraView
    config: RasterConfig
    n_total: int
    n_clusters: int
    n_compact: int
    n_pairs: int
    visible_clusters: int
    culled_clusters: int
    recs: torch.Tensor            # (N, 12) float32 compact records (first n_compact rows)
    rows: torch.Tensor | None     # (N, 16) float32 raster rows (TMA staging only; sb_raster_row_bytes)
    compact_map_full: torch.Tensor  # (N,) int32
    cluster_offset: torch.Tensor  # (K,) int32
    cluster_vis: torch.Tensor     # (K,) uint8
    tile_offsets: torch.Tensor    # (T + 1,) int32
    tile_prims: torch.Tensor      # (P,) int32 compact slots, per-tile depth order
    transmittance: torch.Tensor   # (H, W)
    last: torch.Tensor            # (H, W) int32
    n_degenerate: int = 0
    half: bool | str = False      # produced by a 16-bit blending-state path
    token: int = 0                # owner token of the pre-zeroed sgrad workspace (0: none)
    tile_buffer: torch.Tensor | None = field(default=None, repr=False)   # offsets + raster schedule (2T + 1)
    cluster_cull: torch.Tensor | None = field(default=None, repr=False)  # (K,) uint8 pure frustum test
    cluster_aabb: torch.Tensor | None = field(default=None, repr=False)  # (K, 6) float64 min xyz, max xyz
    _tiles: list | None = field(default=None, repr=False)

    @property
    def compact_map(self) -> torch.Tensor:
        return self.compact_map_full[: self.n_compact]

    @property
    def tiles(self) -> list:
        """Non-empty tiles in tile-id order (the reference's ctx.tiles)."""
        if self._tiles is None:
            offs = self.tile_offsets.cpu().numpy()
            prims = self.tile_prims.cpu().numpy()
            tx_n = self.camera.tiles[0]
            out = []
            for t in np.flatnonzero(np.diff(offs) > 0):
                ty, tx = divmod(int(t), tx_n)
                out.append(TileWorkload(tile_x=tx, tile_y=ty, origin=(tx * TILE_W, ty * TILE_H),
                                        primitives=prims[offs[t]:offs[t + 1]].astype(np.int64)))
            self._tiles = out
        return self._tiles

    @property
    def projected(self) -> dict:
        """Compact projected arrays decoded from the device records."""
        r = self.recs[: self.n_compact]
        flags = r[:, 11].contiguous().view(torch.int32)
        return {
            "xy": r[:, 0:2], "conic": torch.stack([r[:, 2], r[:, 3], r[:, 4]], 1), "opacity": r[:, 5],
            "color": r[:, 6:9], "depth": r[:, 9], "radius": r[:, 10],
            "valid": (flags & 1) != 0, "in_image": (flags & 2) != 0,
        }


# (device, W, H) -> (pair, super-tile entry) capacities of the binning buffers
_bin_capacity: dict = {}
_pinned: dict = {}
# The backward's screen-gradient workspace ("sgrad", 64 B per compact slot)
# is zeroed by the forward's project kernel; _sgrad_clean[device] names the
# one context whose backward may use it without zeroing again.
SGRAD_BYTES = 64
_sgrad_clean: dict = {}
_ctx_tokens = itertools.count(1)


def _stream_key(dev):
    """(device, current stream): per-stream host state (counter mirror,
    clean screen-gradient workspace)."""
    return _lib.raw_stream(dev)


def _pinned_counters(dev):
    """Pinned host mirror of the counters and its device address (one per
    device and stream; the forward reads it before returning, so it is never
    in flight twice).  The bin scan kernel writes it directly when the
    buffer is mapped (address not None); otherwise it is filled by a copy."""
    key = _stream_key(dev)
    if key not in _pinned:
        host = torch.zeros(8, dtype=torch.int32, pin_memory=True)
        addr = C.c_void_p()
        rc = _lib.load().sb_host_mapped_pointer(C.c_void_p(host.data_ptr()), C.byref(addr))
        _pinned[key] = (host, addr if rc == 0 and addr.value else None)
    return _pinned[key]


def _half_mode(half) -> int:
    """half=False: float32 state; True / "fp16": the reference's binary16
    path (forward.py:194-230); "bf16": a bfloat16 variant."""
    if half is False or half is None:
        return 0
    if half is True or half == "fp16":
        return 1
    if half == "bf16":
        return 2
    raise ValueError(f"half must be False, True, 'fp16' or 'bf16', not {half!r}")


def _launch_forward(scene: SceneSoA, camera: CameraView, config: RasterConfig, half, zero_sgrad=True):
    _lib.require_cuda(scene.data)
    dev = scene.device
    n = scene.n
    W, H = camera.resolution
    tx_n, ty_n = camera.tiles
    ntiles = tx_n * ty_n
    K = (n + CLUSTER_SIZE - 1) // CLUSTER_SIZE
    cam_s = camera.struct()
    cfg_s = config.struct(half)
    stream = C.c_void_p(_lib.stream_ptr(dev))

    recs = torch.empty((max(n, 1), REC_FLOATS), dtype=torch.float32, device=dev)
    # 64-byte raster rows, consumed only by the TMA-staged raster variants
    # (SB_RASTER_STAGING=tma|tma32|g4; the default register staging reads
    # the 48-byte records): not written otherwise
    rows = (torch.empty((max(n, 1), ROW_FLOATS), dtype=torch.float32, device=dev)
            if os.environ.get("SB_RASTER_STAGING", "reg") in TMA_STAGING else None)
    cmap = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    coff = torch.empty(max(K, 1), dtype=torch.int32, device=dev)
    cvis = torch.empty(max(K, 1), dtype=torch.uint8, device=dev)   # written for every cluster
    ccull = torch.empty(max(K, 1), dtype=torch.uint8, device=dev)  # pure frustum test (cull_clusters)
    caabb = torch.empty((max(K, 1), 6), dtype=torch.float64, device=dev)   # build_clusters AABBs
    counters = torch.empty(8, dtype=torch.int32, device=dev)   # vis, N_c, ndeg, 0 (project); P, E (bin)
    lib = _lib.load()
    # offsets (T + 1) followed by the heavy-first raster schedule (T)
    tile_buf = torch.empty(2 * ntiles + 1, dtype=torch.int32, device=dev)
    tile_offsets = tile_buf[: ntiles + 1]
    ws = _lib.workspace("project", lib.sb_project_workspace_bytes(n), dev)
    sgrad = _lib.workspace("sgrad", max(n, 1) * SGRAD_BYTES, dev) if zero_sgrad else None
    _sgrad_clean.pop(_stream_key(dev), None)
    _lib.call("sb_project_cull_compact", _lib.ptr(scene.data), n, C.byref(cam_s), C.byref(cfg_s), _lib.ptr(recs),
              _lib.ptr(cmap), _lib.ptr(coff), _lib.ptr(cvis), _lib.ptr(counters),
              _lib.ptr(sgrad) if sgrad is not None else None, _lib.ptr(rows), _lib.ptr(caabb), _lib.ptr(ccull),
              _lib.ptr(ws), ws.numel(), stream)
    # one zero-initialised state per tile grid (its count arrays stay zeroed)
    state = _lib.workspace(f"bin_state_{tx_n}x{ty_n}", lib.sb_bin_state_workspace_bytes(n, ntiles), dev)
    host, mirror = _pinned_counters(dev)
    _lib.call("sb_bin_prepare", _lib.ptr(recs), _lib.ptr(counters), n, C.byref(cam_s), _lib.ptr(tile_buf),
              _lib.ptr(counters[4:]), mirror, _lib.ptr(state), state.numel(), stream)
    # Binning part 2 is launched before the host knows P and E, with the
    # capacities of earlier views of this resolution; the one device-to-host
    # read below then overlaps it, and it is re-launched only if they were
    # exceeded (its kernels write nothing in that case).
    key = (str(dev), W, H)
    p_cap, e_cap = _bin_capacity.get(key, (0, 0))

    def finish(p_cap, e_cap):
        prims = torch.empty(max(p_cap, 1), dtype=torch.int32, device=dev)
        ws_f = _lib.workspace("bin_finish", lib.sb_bin_finish_workspace_bytes(e_cap, ntiles), dev)
        _lib.call("sb_bin_finish", _lib.ptr(recs), _lib.ptr(counters), n, C.byref(cam_s), p_cap, e_cap,
                  _lib.ptr(tile_offsets), _lib.ptr(state), _lib.ptr(prims), _lib.ptr(ws_f), ws_f.numel(), stream)
        return prims

    if mirror is None:
        host.copy_(counters, non_blocking=True)       # queued before part 2
    ready = torch.cuda.Event()
    ready.record()
    prims = finish(p_cap, e_cap) if p_cap else None
    ready.synchronize()                                # the one device-to-host read
    vis, nc, ndeg, _, P, E = (int(v) for v in host[:6].tolist())
    if P > p_cap or E > e_cap:
        p_cap, e_cap = P + P // 4 + 1024, E + E // 4 + 1024
        _bin_capacity[key] = (p_cap, e_cap)
        prims = finish(p_cap, e_cap)
    if prims is None:
        prims = torch.empty(1, dtype=torch.int32, device=dev)
    color = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    T = torch.empty((H, W), dtype=torch.float32, device=dev)
    frags = torch.empty((H, W), dtype=torch.int32, device=dev)
    last = torch.empty((H, W), dtype=torch.int32, device=dev)
    ws_r = _lib.workspace("raster_fwd", _lib.load().sb_raster_workspace_bytes(), dev)
    _lib.call("sb_raster_fwd", _lib.ptr(recs), _lib.ptr(rows), _lib.ptr(tile_buf), _lib.ptr(prims), C.byref(cam_s),
              C.byref(cfg_s), _lib.ptr(color), _lib.ptr(T), _lib.ptr(frags), _lib.ptr(last), _lib.ptr(ws_r),
              ws_r.numel(), stream)
    out = RenderOutput(color=color, transmittance=T, frag_count=frags)
    ctx = RenderContext(generation=scene.generation, camera=camera, config=config, n_total=n, n_clusters=K,
                        n_compact=nc, n_pairs=P, visible_clusters=vis, culled_clusters=K - vis, recs=recs, rows=rows,
                        compact_map_full=cmap, cluster_offset=coff[:K], cluster_vis=cvis[:K],
                        tile_offsets=tile_offsets, tile_prims=prims[:P], transmittance=T, last=last,
                        tile_buffer=tile_buf, cluster_cull=ccull[:K], cluster_aabb=caabb[:K],
                        n_degenerate=ndeg, half=half)
    if sgrad is not None:
        ctx.token = next(_ctx_tokens)
        _sgrad_clean[_stream_key(dev)] = ctx.token
    return out, ctx


def forward(scene: SceneSoA, camera, config: RasterConfig | None = None, counter=None, half=False):
    """Render `scene` from `camera`; returns (RenderOutput, RenderContext).

    forward.py:258-304.  half=True (or "fp16") renders with fp16 blending
    state (forward.py:194-230), half="bf16" with bfloat16 state; the backward
    then replays in float32 as the reference does.  `counter` (the reference's CPU op tally) is not
    applicable on the device and must be None; use ncu counters instead."""
    if counter is not None:
        raise ValueError("OpCounter instrumentation is CPU-only; profile the device path with ncu")
    config = config or RasterConfig()
    camera = CameraView.from_any(camera)
    return _launch_forward(scene, camera, config, half)


def render(scene: SceneSoA, camera, config: RasterConfig | None = None) -> RenderOutput:
    """forward.py:307-308 (no backward follows: the sgrad rows are left alone)."""
    return _launch_forward(scene, CameraView.from_any(camera), config or RasterConfig(), False,
                           zero_sgrad=False)[0]


# ---- single-tile blending (forward.py:161-230) -------------------------------
def _lane_pixels(origin, resolution):
    """forward.py:117-127: lane l -> pixel x0 + l % 16, rows y0 + 4 (l // 16) + i."""
    x0, y0 = origin
    W, H = resolution
    lane = np.arange(LANES)
    px = x0 + lane % TILE_W
    py = y0 + 4 * (lane // TILE_W)[:, None] + np.arange(PIXELS_PER_LANE)[None, :]
    valid = (px[:, None] < W) & (py < H)
    return px, py, valid


def _records_from_projected(projected) -> torch.Tensor:
    """Pack projected arrays (ProjectedScene or a ctx.projected dict) into
    the device's 48-byte compact records."""
    get = (lambda k: projected[k]) if isinstance(projected, dict) else (lambda k: getattr(projected, k))
    xy = torch.as_tensor(get("xy"))
    dev = xy.device if xy.is_cuda else torch.device("cuda")
    f = lambda k: torch.as_tensor(get(k), device=dev).to(torch.float32)  # noqa: E731
    xy, conic, color = f("xy").reshape(-1, 2), f("conic").reshape(-1, 3), f("color").reshape(-1, 3)
    n = xy.shape[0]
    flags = (torch.as_tensor(get("valid"), device=dev).to(torch.int32)
             | (torch.as_tensor(get("in_image"), device=dev).to(torch.int32) << 1))
    recs = torch.empty((max(n, 1), REC_FLOATS), dtype=torch.float32, device=dev)
    recs[:n, 0:2] = xy
    recs[:n, 2:5] = conic
    recs[:n, 5] = f("opacity").reshape(-1)
    recs[:n, 6:9] = color
    recs[:n, 9] = f("depth").reshape(-1)
    recs[:n, 10] = f("radius").reshape(-1)
    recs[:n, 11] = flags.view(torch.float32)
    return recs


def _blend_one_tile(tile, projected, config, resolution, half):
    config = config or RasterConfig()
    W, H = int(resolution[0]), int(resolution[1])
    tx_n, ty_n = (W + TILE_W - 1) // TILE_W, (H + TILE_H - 1) // TILE_H
    ntiles = tx_n * ty_n
    t = int(tile.tile_y) * tx_n + int(tile.tile_x)
    recs = _records_from_projected(projected)
    dev = recs.device
    prims = torch.as_tensor(np.asarray(tile.primitives), device=dev).to(torch.int32).reshape(-1)
    P = prims.numel()
    offs = torch.zeros(2 * ntiles + 1, dtype=torch.int32, device=dev)
    offs[t + 1:ntiles + 1] = P
    sched = torch.arange(ntiles, dtype=torch.int32, device=dev)
    sched[0], sched[t] = t, 0                  # the one non-empty tile first
    offs[ntiles + 1:] = sched
    color = torch.empty((H, W, 3), dtype=torch.float32, device=dev)
    T = torch.empty((H, W), dtype=torch.float32, device=dev)
    frags = torch.empty((H, W), dtype=torch.int32, device=dev)
    last = torch.empty((H, W), dtype=torch.int32, device=dev)
    cam = CameraView(np.eye(4), (1.0, 1.0), (0.0, 0.0), (W, H), 0.05, 20.0)
    cam_s, cfg_s = cam.struct(), config.struct(half)
    ws = _lib.workspace("raster_fwd", _lib.load().sb_raster_workspace_bytes(), dev)
    _lib.call("sb_raster_fwd", _lib.ptr(recs), None, _lib.ptr(offs), _lib.ptr(prims if P else offs), C.byref(cam_s),
              C.byref(cfg_s), _lib.ptr(color), _lib.ptr(T), _lib.ptr(frags), _lib.ptr(last), _lib.ptr(ws),
              ws.numel(), C.c_void_p(_lib.stream_ptr(dev)))
    px, py, valid = _lane_pixels(tile.origin, (W, H))
    bg = torch.tensor(config.background, dtype=torch.float32, device=dev)
    rgb = bg.expand(LANES, PIXELS_PER_LANE, 3).clone()
    Tl = torch.ones((LANES, PIXELS_PER_LANE), dtype=torch.float32, device=dev)
    fl = torch.zeros((LANES, PIXELS_PER_LANE), dtype=torch.int32, device=dev)
    li, ii = np.nonzero(valid)
    if li.size:
        ys = torch.as_tensor(py[li, ii], device=dev)
        xs = torch.as_tensor(px[li], device=dev)
        lt, it = torch.as_tensor(li, device=dev), torch.as_tensor(ii, device=dev)
        rgb[lt, it] = color[ys, xs]
        Tl[lt, it] = T[ys, xs]
        fl[lt, it] = frags[ys, xs]
    return rgb, Tl, fl, torch.as_tensor(valid, device=dev)


def blend_tile(tile: TileWorkload, projected, config: RasterConfig | None = None, resolution=None, counter=None):
    """forward.py:161-191: composite ONE tile with the device's warp kernel;
    returns (rgb (32, 4, 3), T (32, 4), frags (32, 4), valid (32, 4)) in lane
    layout (lane l -> column l % 16, rows 4 (l // 16) + i).  `projected` holds
    the arrays `tile.primitives` indexes (ProjectedScene or ctx.projected)."""
    if counter is not None:
        raise ValueError("OpCounter instrumentation is CPU-only; profile the device path with ncu")
    if resolution is None:
        raise ValueError("resolution is required")
    return _blend_one_tile(tile, projected, config, resolution, False)


def half_path_blend(tile: TileWorkload, projected, config: RasterConfig | None = None, resolution=None):
    """forward.py:194-230: the same with binary16 blending state (rgb / T
    returned in float32, as the reference upcasts them)."""
    if resolution is None:
        raise ValueError("resolution is required")
    return _blend_one_tile(tile, projected, config, resolution, True)
