"""Deterministic 32-lane reductions on real warps.

Reference: pkg/src/tinysplat/reduction.py:21-58, which emulates a warp in
software.  Here they are the device functions the raster backward uses,
exposed for parity tests:

  lane_group_reduce   __shfl_xor butterfly (strides 16..1) — bit-identical to
                      the reference's v[:s] + v[s:2s] tree (fp add commutes)
  exp_aligned_reduce  REDUX.MAX of the binary exponents, rint to 23 fractional
                      bits, exact REDUX.SUM of the integers, rescale
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib

LANES = 32


def _run(values, mode):
    v = torch.as_tensor(values)
    if v.shape[-1] != LANES:
        raise ValueError(f"lane axis must have {LANES} entries, got {v.shape[-1]}")
    lead = tuple(v.shape[:-1])
    dev = v.device if v.is_cuda else torch.device("cuda")
    _lib.require_cuda()
    flat = v.to(device=dev, dtype=torch.float32).reshape(-1, LANES).contiguous()
    g = flat.shape[0]
    out_f = torch.empty(max(g, 1), dtype=torch.float32, device=dev)
    out_d = torch.empty(max(g, 1), dtype=torch.float64, device=dev)
    _lib.call("sb_lane_reduce", _lib.ptr(flat), g, mode, _lib.ptr(out_f), _lib.ptr(out_d),
              C.c_void_p(_lib.stream_ptr(dev)))
    return (out_d if mode == 2 else out_f)[:g].reshape(lead)


def backward_row_reduce(values, exp_aligned: bool = False):
    """The raster backward's in-register row reductions (test hook): must
    equal lane_group_reduce / exp_aligned_reduce bit for bit."""
    return _run(torch.as_tensor(values), 4 if exp_aligned else 3)


def lane_group_reduce(values, axis: int = -1, float64: bool = False):
    v = torch.as_tensor(values)
    v = torch.movedim(v, axis, -1)
    return _run(v, 2 if float64 else 0)


def exp_aligned_reduce(values, axis: int = -1):
    v = torch.as_tensor(values)
    v = torch.movedim(v, axis, -1)
    return _run(v, 1)
