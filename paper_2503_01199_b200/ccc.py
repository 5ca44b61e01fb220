"""Cluster-Cull-Compact host API: Morton keys / sort on the device.

Reference: pkg/src/tinysplat/ccc.py.  Culling and compaction run fused
inside the forward (sb_project_cull_compact); this module exposes the Morton
re-sort (ccc.py:59-90) and the reference's cluster-index API as separate
device calls:

  build_clusters      -> sb_build_clusters (float64 AABB per 128-row block)
  cull_clusters       -> sb_cull_clusters (p-vertex frustum test)
  cluster_visibility  -> sb_cull_clusters with the in_image widening
  compact_arrays      -> device gather of the visible clusters' rows

  morton_encode  -> sb_morton_encode (caller positions and bounds, float64
                    quantise + bit interleave); morton_encode_scene ->
                    sb_morton_keys (the scene's own bounds on the device)
  morton_sort    -> sb_morton_keys + sb_radix_sort_pairs_u64 (63-bit keys,
                    8 stable LSD passes) + sb_permute_rows over the parameter
                    rows and every registered extra
"""
from __future__ import annotations

import ctypes as C

import torch

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeMismatchError, ValidationError
from .scene import SceneSoA

CLUSTER_SIZE = 128
MORTON_BITS = 21


def cluster_count(n: int, cluster_size: int = CLUSTER_SIZE) -> int:
    return (n + cluster_size - 1) // cluster_size


def _keys(rows: torch.Tensor, n: int):
    dev = rows.device
    stream = C.c_void_p(_lib.stream_ptr(dev))
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    vals = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    lohi = torch.empty(6, dtype=torch.float64, device=dev)
    bad = torch.empty(1, dtype=torch.int32, device=dev)
    ws = _lib.workspace("morton", _lib.load().sb_morton_keys_workspace_bytes(n), dev)
    _lib.call("sb_morton_keys", _lib.ptr(rows), n, _lib.ptr(keys), _lib.ptr(vals), _lib.ptr(lohi), _lib.ptr(bad),
              _lib.ptr(ws), ws.numel(), stream)
    return keys, vals, lohi, bad


def morton_encode(positions, bounds_min, bounds_max, device=None) -> torch.Tensor:
    """ccc.py:59-66 on the device (sb_morton_encode): 63-bit Z-order keys of
    (N, 3) positions, quantised in float64 within the given bounds.  Keys are
    uint64 values carried in an int64 tensor (view as uint64 on the host).
    Raises ValidationError on a non-finite position, as quantize does."""
    if device is None:
        device = positions.device if torch.is_tensor(positions) and positions.is_cuda else torch.device("cuda")
    pos = torch.as_tensor(positions, dtype=torch.float64, device=device).reshape(-1, 3).contiguous()
    _lib.require_cuda(pos)
    n = pos.shape[0]
    lohi = torch.cat([torch.as_tensor(bounds_min, dtype=torch.float64).reshape(3),
                      torch.as_tensor(bounds_max, dtype=torch.float64).reshape(3)]).to(device)
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=device)
    bad = torch.empty(1, dtype=torch.int32, device=device)
    _lib.call("sb_morton_encode", _lib.ptr(pos), n, _lib.ptr(lohi), _lib.ptr(keys), _lib.ptr(bad),
              C.c_void_p(_lib.stream_ptr(device)))
    b = int(bad.item())
    if b < n:
        raise ValidationError("position", b, "non-finite position")
    return keys[:n]


def morton_encode_scene(scene: SceneSoA):
    """(keys uint64-as-int64, lo, hi) for the scene's own bounds."""
    _lib.require_cuda(scene.data)
    keys, _, lohi, bad = _keys(scene.data, scene.n)
    b = int(bad.item())
    if b < scene.n:
        raise ValidationError("position", b, "non-finite position")
    return keys[: scene.n], lohi[:3], lohi[3:]


def morton_sort(scene: SceneSoA) -> torch.Tensor:
    """Stable in-place sort of the scene and all extras by Morton key
    (ccc.py:79-90).  Returns the applied permutation (int64); bumps
    generation even when the order was already sorted."""
    n = scene.n
    if n == 0:
        scene.generation += 1
        return torch.zeros(0, dtype=torch.int64, device=scene.device)
    _lib.require_cuda(scene.data)
    dev = scene.device
    keys, vals, _, bad = _keys(scene.data, n)
    keys_alt = torch.empty_like(keys)
    vals_alt = torch.empty_like(vals)
    ws = _lib.workspace("sort", _lib.load().sb_sort_workspace_bytes(n), dev)
    flip = C.c_int(0)
    _lib.call("sb_radix_sort_pairs_u64", _lib.ptr(keys), _lib.ptr(vals), _lib.ptr(keys_alt), _lib.ptr(vals_alt), n,
              63, C.byref(flip), _lib.ptr(ws), ws.numel(), C.c_void_p(_lib.stream_ptr(dev)))
    b = int(bad.item())
    if b < n:
        raise ValidationError("position", b, "non-finite position")
    perm = (vals_alt if flip.value else vals)[:n]
    scene.permute(perm, trusted=True)   # a device sort's output: a permutation of [0, n)
    return perm.to(torch.int64)


def sort_pairs(keys: torch.Tensor, vals: torch.Tensor, bits: int = 64):
    """Stable (key, value) sort with the hand-written LSD radix sort; keys are
    uint64 carried in int64 tensors (unsigned order)."""
    n = keys.numel()
    dev = keys.device
    k = keys.contiguous().clone()
    v = vals.to(torch.int32).contiguous().clone()
    ka, va = torch.empty_like(k), torch.empty_like(v)
    ws = _lib.workspace("sort", _lib.load().sb_sort_workspace_bytes(n), dev)
    flip = C.c_int(0)
    _lib.call("sb_radix_sort_pairs_u64", _lib.ptr(k), _lib.ptr(v), _lib.ptr(ka), _lib.ptr(va), n, bits,
              C.byref(flip), _lib.ptr(ws), ws.numel(), C.c_void_p(_lib.stream_ptr(dev)))
    return (ka, va) if flip.value else (k, v)


def scatter_grads(compact_grads: torch.Tensor, compact_map: torch.Tensor, n: int,
                  cluster_size: int = CLUSTER_SIZE):
    """ccc.py:197-216 for a (N_c, ...) tensor: full-length rows (zeros
    elsewhere) and the per-cluster update mask."""
    out = torch.zeros((n,) + tuple(compact_grads.shape[1:]), dtype=compact_grads.dtype,
                      device=compact_grads.device)
    idx = compact_map.long()
    out[idx] = compact_grads
    mask = torch.zeros(cluster_count(n, cluster_size), dtype=torch.bool, device=compact_grads.device)
    if idx.numel():
        mask[idx // cluster_size] = True
    return out, mask


# ---- cluster index (ccc.py:97-194) ------------------------------------------
@dataclass
class ClusterIndex:
    """ccc.py:97-109: per-cluster float64 AABBs (device tensors)."""
    cluster_size: int
    aabb_min: torch.Tensor   # (K, 3) float64
    aabb_max: torch.Tensor   # (K, 3) float64
    n: int

    @property
    def n_clusters(self) -> int:
        return int(self.aabb_min.shape[0])

    def member_slice(self, k: int) -> slice:
        return slice(k * self.cluster_size, min((k + 1) * self.cluster_size, self.n))


def build_clusters(scene: SceneSoA, cluster_size: int = CLUSTER_SIZE) -> ClusterIndex:
    """ccc.py:112-131: AABBs of p -+ 3 max(exp(log_scale)) over consecutive
    blocks of the (Morton-sorted) scene, on the device (sb_build_clusters)."""
    _lib.require_cuda(scene.data)
    n = scene.n
    k = cluster_count(n, cluster_size)
    aabb = torch.empty((max(k, 1), 6), dtype=torch.float64, device=scene.device)
    if n:
        _lib.call("sb_build_clusters", _lib.ptr(scene.data), n, int(cluster_size), _lib.ptr(aabb),
                  C.c_void_p(_lib.stream_ptr(scene.device)))
    return ClusterIndex(cluster_size=int(cluster_size), aabb_min=aabb[:k, :3], aabb_max=aabb[:k, 3:], n=n)


def _planes(frustum) -> C.Array:
    planes = np.asarray(getattr(frustum, "planes", frustum), dtype=np.float64).reshape(-1)
    if planes.size != 24:
        raise ShapeMismatchError(f"frustum planes must be (6, 4), got {planes.size} values")
    return (C.c_double * 24)(*[float(v) for v in planes])


def _cull(index: ClusterIndex, frustum, in_image=None):
    k = index.n_clusters
    dev = index.aabb_min.device
    aabb = torch.cat([index.aabb_min, index.aabb_max], dim=1).to(torch.float64).contiguous()
    out = torch.zeros(max(k, 1), dtype=torch.uint8, device=dev)
    ii = None
    if in_image is not None:
        ii = torch.as_tensor(in_image, device=dev)
        if ii.numel() != index.n:
            raise ShapeMismatchError(f"in_image length {ii.numel()} != {index.n}")
        ii = ii.to(torch.uint8).contiguous()
    if k:
        _lib.call("sb_cull_clusters", _lib.ptr(aabb), k, index.cluster_size, index.n, _planes(frustum), _lib.ptr(ii),
                  None if ii is not None else _lib.ptr(out), _lib.ptr(out) if ii is not None else None,
                  C.c_void_p(_lib.stream_ptr(dev)))
    return out[:k].bool()


def cull_clusters(index: ClusterIndex, frustum) -> torch.Tensor:
    """ccc.py:134-146: (K,) bool -- a cluster survives unless its AABB lies
    entirely behind some frustum plane (p-vertex test, the reference's einsum
    order)."""
    return _cull(index, frustum)


def cluster_visibility(index: ClusterIndex, frustum, in_image) -> torch.Tensor:
    """ccc.py:149-164: cull_clusters widened by any member with in_image
    (culling is then exactly invisible in the render)."""
    return _cull(index, frustum, in_image)


def compact_arrays(struct_or_dict, cluster_mask, cluster_size: int, n: int):
    """ccc.py:171-194: the visible clusters' rows of every length-n array
    (dict values or ndarray / tensor attributes), gathered on the device;
    returns (compacted, compact_map int64)."""
    mask = torch.as_tensor(cluster_mask)
    dev = mask.device if mask.is_cuda else torch.device("cuda")
    mask = mask.to(dev).bool()
    k = mask.numel()
    starts = torch.arange(k, device=dev, dtype=torch.int64) * cluster_size
    ends = torch.clamp(starts + cluster_size, max=n)
    keep = mask & (ends > starts)
    rows = torch.arange(k * cluster_size, device=dev, dtype=torch.int64)
    member = rows < n
    cmap = rows[keep.repeat_interleave(cluster_size) & member]

    def gather(v):
        t = torch.as_tensor(v, device=dev) if not torch.is_tensor(v) else v.to(dev)
        return t.index_select(0, cmap).contiguous()

    if isinstance(struct_or_dict, dict):
        return {kk: gather(v) for kk, v in struct_or_dict.items()}, cmap
    import copy as _copy
    out = _copy.copy(struct_or_dict)
    for name, value in vars(struct_or_dict).items():
        if (isinstance(value, (np.ndarray, torch.Tensor)) and value.ndim >= 1 and len(value) == n):
            setattr(out, name, gather(value))
    return out, cmap
