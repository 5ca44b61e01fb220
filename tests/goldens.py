"""Fixture loading helpers for tests/golden/*.npz (made by tools/make_golden.py
from the reference itself)."""
from __future__ import annotations

import json
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CH = ("position", "log_scale", "rotation", "color", "opacity_logit")
_cache = {}


def load(name):
    if name not in _cache:
        path = os.path.join(GOLDEN, name)
        if name.endswith(".json"):
            with open(path) as f:
                _cache[name] = json.load(f)
        else:
            _cache[name] = dict(np.load(path))
    return _cache[name]


def scene(d, prefix=""):
    return {c: d[f"{prefix}{c}"].astype(np.float64) for c in CH}


def camera(d, prefix=""):
    res = d[f"{prefix}res"]
    nf = d[f"{prefix}nearfar"]
    return SimpleNamespace(world_to_camera=d[f"{prefix}w2c"], focal=d[f"{prefix}focal"],
                           principal_point=d[f"{prefix}pp"], resolution=(int(res[0]), int(res[1])),
                           near=float(nf[0]), far=float(nf[1]))


def raster_cfg(d, prefix="", dtype="float32"):
    from oracle.oracle import RasterConfig
    return RasterConfig(dtype=dtype, background=tuple(float(b) for b in d[f"{prefix}cfg_bg"]),
                        use_culling=bool(d[f"{prefix}cfg_cull"]),
                        conic_reduce="tree" if int(d[f"{prefix}cfg_tree"]) else "exp_aligned")


def floored_rel(a, b, floor=1e-3):
    """max |a-b| / max(|b|, floor * max|b|), per SURVEY 8(c) parity rules."""
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    if b.size == 0:
        return 0.0
    den = np.maximum(np.abs(b), floor * max(np.abs(b).max(), 1e-300))
    return float((np.abs(a - b) / den).max())


CASES = [("golden_A.npz", ""), ("golden_edge.npz", "e1_"), ("golden_edge.npz", "e2_"),
         ("golden_edge.npz", "e3_"), ("golden_edge.npz", "e4_")]


def conditioned_rel_excess(got, ref, ref64, base_tol, k=4.0, floor=1e-3):
    """Elementwise parity with an allowance for ill-conditioned entries.

    err = |got - ref| / den with den = max(|ref64|, floor * max|ref64|); the
    allowance is max(base_tol, k * |ref - ref64| / den), i.e. an entry may miss
    base_tol only where the reference's own float32 path is itself that far
    from its float64 path.  Returns max(err / allowance) (<= 1 passes)."""
    got = np.asarray(got, np.float64); ref = np.asarray(ref, np.float64); ref64 = np.asarray(ref64, np.float64)
    if ref.size == 0:
        return 0.0
    den = np.maximum(np.abs(ref64), floor * max(np.abs(ref64).max(), 1e-300))
    allow = np.maximum(base_tol, k * np.abs(ref - ref64) / den)
    return float((np.abs(got - ref) / den / allow).max())
