"""Tile binning host API (reference: pkg/src/tinysplat/tiles.py).

The forward bins its compact records inside `forward` (sb_bin_prepare +
sb_bin_finish).  `bin_tiles` exposes the same two device calls for caller
arrays, with the reference's signature: it packs (xy, depth, radius, mask)
into compact records and returns the per-tile (depth, index)-ordered lists,
exactly np.lexsort((prim, depth, tile_id)) restricted to each tile
(tiles.py:94-106).

  tile_grid      tiles.py:38-41
  bin_tiles      tiles.py:50-107  -> list of TileWorkload (non-empty tiles)
  bin_tiles_device                -> (tile_offsets (T + 1), prims (P)) device
                                     tensors, no host materialisation
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from .camera import CameraView
from .forward import REC_FLOATS, TileWorkload

TILE_W, TILE_H = 16, 8
_REC_X, _REC_Y, _REC_DEPTH, _REC_RADIUS, _REC_FLAGS = 0, 1, 9, 10, 11
_IN_IMAGE = 2   # record flag bit 1: generates fragments (forward.py:279)


def tile_grid(resolution):
    """tiles.py:38-41: (tiles_x, tiles_y) of 16 x 8 tiles."""
    W, H = resolution
    return (W + TILE_W - 1) // TILE_W, (H + TILE_H - 1) // TILE_H


def _grid_camera(resolution) -> CameraView:
    # the binning reads only the resolution (and the tile grid it implies)
    return CameraView(np.eye(4), (1.0, 1.0), (0.0, 0.0), resolution, 0.01, 100.0)


def bin_tiles_device(xy, depth, radius, mask, resolution, device=None):
    """Device binning of caller arrays over the compact primitive buffer.
    Returns (tile_offsets int32 (T + 1), prims int32 (P)) on the device.
    Masked depths must be positive (the pipeline's depths exceed the near
    plane): the kernels order depths by their float32 bit patterns."""
    if device is None:
        device = xy.device if torch.is_tensor(xy) and xy.is_cuda else torch.device("cuda")
    xy = torch.as_tensor(xy, device=device).to(torch.float32).reshape(-1, 2)
    n = xy.shape[0]
    depth = torch.as_tensor(depth, device=device).to(torch.float32).reshape(n)
    radius = torch.as_tensor(radius, device=device).to(torch.float32).reshape(n)
    mask = torch.as_tensor(mask, device=device).to(torch.bool).reshape(n)
    _lib.require_cuda(xy)
    if bool((mask & ~(depth > 0)).any()):
        raise ValueError("masked primitives need positive depths")
    W, H = resolution
    tx_n, ty_n = tile_grid(resolution)
    ntiles = tx_n * ty_n
    cam_s = _grid_camera(resolution).struct()
    lib = _lib.load()
    stream = C.c_void_p(_lib.stream_ptr(device))
    recs = torch.zeros((max(n, 1), REC_FLOATS), dtype=torch.float32, device=device)
    recs[:n, _REC_X] = xy[:, 0]
    recs[:n, _REC_Y] = xy[:, 1]
    recs[:n, _REC_DEPTH] = depth
    recs[:n, _REC_RADIUS] = radius
    recs.view(torch.int32)[:n, _REC_FLAGS] = torch.where(mask, _IN_IMAGE, 0).to(torch.int32)
    counters = torch.zeros(8, dtype=torch.int32, device=device)
    counters[1] = n                                  # N_c: every row is a compact record
    tile_buf = torch.empty(2 * ntiles + 1, dtype=torch.int32, device=device)
    state = _lib.workspace(f"bin_state_{tx_n}x{ty_n}", lib.sb_bin_state_workspace_bytes(n, ntiles), device)
    _lib.call("sb_bin_prepare", _lib.ptr(recs), _lib.ptr(counters), n, C.byref(cam_s), _lib.ptr(tile_buf),
              _lib.ptr(counters[4:]), None, _lib.ptr(state), state.numel(), stream)
    P, E = (int(v) for v in counters[4:6].tolist())
    prims = torch.empty(max(P, 1), dtype=torch.int32, device=device)
    ws = _lib.workspace("bin_finish", lib.sb_bin_finish_workspace_bytes(E, ntiles), device)
    _lib.call("sb_bin_finish", _lib.ptr(recs), _lib.ptr(counters), n, C.byref(cam_s), P, E,
              _lib.ptr(tile_buf), _lib.ptr(state), _lib.ptr(prims), _lib.ptr(ws), ws.numel(), stream)
    return tile_buf[: ntiles + 1], prims[:P]


def bin_tiles(xy, depth, radius, mask, resolution):
    """tiles.py:50-107: TileWorkload per non-empty tile, tile-id order, each
    with its primitives (indices into the given arrays) in depth order."""
    offsets, prims = bin_tiles_device(xy, depth, radius, mask, resolution)
    tx_n, _ = tile_grid(resolution)
    offs = offsets.cpu().numpy().astype(np.int64)
    pr = prims.cpu().numpy().astype(np.int64)
    tiles = []
    for t in np.flatnonzero(np.diff(offs)):
        tyi, txi = divmod(int(t), tx_n)
        tiles.append(TileWorkload(tile_x=txi, tile_y=tyi, origin=(txi * TILE_W, tyi * TILE_H),
                                  primitives=pr[offs[t]:offs[t + 1]]))
    return tiles
