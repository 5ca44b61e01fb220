"""Generate tests/golden/* by running the REFERENCE (read-only, in-process).

    PYTHONDONTWRITEBYTECODE=1 python tools/make_golden.py [--big]

Only runs in the build container (the reference does not exist on the GPU
box).  Every fixture records the reference's own outputs on seeded inputs:

  golden_A.npz      BASELINE config A: 10K Gaussians, 128x128, seed 7, view 0
                    (projection, Morton keys/perm, AABBs, cull/visibility masks,
                    compact map, tile lists, fp32 forward, fp32 backward, and
                    the fp64 forward/backward numeric oracle)
  golden_edge.npz   edge cases: ragged resolution + background, culling off,
                    tree conic reduction, out-of-frustum / behind-camera
                    primitives, empty scene, reductions, Adam, variance score,
                    Morton edge cases
  golden_big.json   configs B, C, E (N-scaled scenes): SHA-256 of the reference's
                    Morton keys/perm, projection arrays, cluster masks, compact
                    map and tile lists, plus pair counts and (B) a forward-image
                    pixel sample.  (--big; a few minutes)
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")

import tinysplat as ts  # noqa: E402
from tinysplat import ccc  # noqa: E402
from tinysplat.backward import DensifyStats  # noqa: E402
from tinysplat.densify import variance_score  # noqa: E402
from tinysplat.optim import AdamState, adam_step  # noqa: E402
from tinysplat.projection import project_scene  # noqa: E402
from tinysplat.reduction import exp_aligned_reduce, lane_group_reduce  # noqa: E402
from tinysplat.scene import SceneSoA  # noqa: E402
from tinysplat.tiles import bin_tiles  # noqa: E402
from tinysplat.synthetic import SyntheticSceneSpec, camera_ring, random_scene  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
CH = ("position", "log_scale", "rotation", "color", "opacity_logit")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def scaled_scene(n, seed, res, n_views=1):
    """configs B-E shrink log_scale by ln((N/512)^(1/3)) and
    re-round every channel through float32."""
    spec = SyntheticSceneSpec(n_gaussians=n, n_views=n_views, view_resolution=res, seed=seed)
    sc = random_scene(spec)
    sc.log_scale = sc.log_scale - np.log((n / 512.0) ** (1.0 / 3.0))
    sc = SceneSoA(*[getattr(sc, c).astype(np.float32).astype(np.float64) for c in CH])
    return sc, camera_ring(spec)


def cam_arrays(prefix, cam):
    return {
        f"{prefix}w2c": cam.world_to_camera, f"{prefix}focal": cam.focal,
        f"{prefix}pp": cam.principal_point, f"{prefix}res": np.array(cam.resolution),
        f"{prefix}nearfar": np.array([cam.near, cam.far]),
    }


def scene_arrays(prefix, sc):
    return {f"{prefix}{c}": getattr(sc, c).astype(np.float32) for c in CH}


def tiles_flat(tiles, res):
    txn = (res[0] + 15) // 16
    tyn = (res[1] + 7) // 8
    counts = np.zeros(txn * tyn, np.int64)
    prims = []
    for t in tiles:
        counts[t.tile_y * txn + t.tile_x] = len(t.primitives)
        prims.append(t.primitives)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    prims = np.concatenate(prims).astype(np.int64) if prims else np.zeros(0, np.int64)
    return offs, prims


def full_case(prefix, sc, cam, cfg, target_seed, with_f64=True):
    """Projection + CCC + tiles + forward + loss + backward for one view."""
    d = {}
    d.update(scene_arrays(prefix, sc))
    d.update(cam_arrays(prefix, cam))
    d[f"{prefix}cfg_bg"] = np.array(cfg.background, np.float64)
    d[f"{prefix}cfg_cull"] = np.array(int(cfg.use_culling))
    d[f"{prefix}cfg_tree"] = np.array(int(cfg.conic_reduce == "tree"))
    n = sc.n
    pr = project_scene(sc, cam, dtype=np.float32, low_pass=cfg.low_pass)
    for k in ("xy", "depth", "conic", "radius", "color", "opacity"):
        d[f"{prefix}proj_{k}"] = getattr(pr, k)
    d[f"{prefix}proj_valid"] = pr.valid
    d[f"{prefix}proj_in_image"] = pr.in_image
    if n:
        lo, hi = sc.bounds()
        keys = ccc.morton_encode(sc.position, lo, hi)
        d[f"{prefix}morton_keys"] = keys
        d[f"{prefix}morton_perm"] = np.argsort(keys, kind="stable").astype(np.int32)
        idx = ccc.build_clusters(sc)
        fr = ts.build_frustum(cam)
        d[f"{prefix}aabb_min"] = idx.aabb_min
        d[f"{prefix}aabb_max"] = idx.aabb_max
        d[f"{prefix}planes"] = fr.planes
        d[f"{prefix}cull_mask"] = ccc.cull_clusters(idx, fr)
        d[f"{prefix}vis_mask"] = ccc.cluster_visibility(idx, fr, pr.in_image)
    out, ctx = ts.forward(sc, cam, cfg)
    d[f"{prefix}compact_map"] = ctx.compact_map.astype(np.int32)
    offs, prims = tiles_flat(ctx.tiles, cam.resolution)
    d[f"{prefix}tile_offsets"] = offs.astype(np.int32)
    d[f"{prefix}tile_prims"] = prims.astype(np.int32)
    d[f"{prefix}fwd_color"] = out.color
    d[f"{prefix}fwd_T"] = out.transmittance
    d[f"{prefix}fwd_frags"] = out.frag_count
    rng = np.random.default_rng(target_seed)
    target = rng.uniform(0.0, 1.0, out.color.shape)
    loss, dI = ts.loss_and_grad(out.color, target, 0.2)
    d[f"{prefix}target_seed"] = np.array(target_seed)
    d[f"{prefix}loss"] = np.array(loss)
    d[f"{prefix}dL_dI"] = dI.astype(np.float32)   # backward casts to the raster dtype
    stats = DensifyStats.zeros(n)
    res = ts.backward(sc, ctx, dI.astype(np.float32).astype(np.float64), stats)
    d[f"{prefix}grads"] = np.concatenate(
        [getattr(res.grads, c).reshape(n, -1) for c in CH], axis=1).astype(np.float32)
    d[f"{prefix}stat_S"] = stats.S
    d[f"{prefix}stat_M"] = stats.M
    d[f"{prefix}stat_C"] = stats.C.astype(np.int32)
    d[f"{prefix}score"] = variance_score(stats)
    d[f"{prefix}upd_mask"] = res.cluster_mask
    # fp16 blending state (forward.py:194-230)
    outh, _ = ts.forward(sc, cam, cfg, half=True)
    d[f"{prefix}fwdh_color"] = outh.color
    d[f"{prefix}fwdh_T"] = outh.transmittance
    d[f"{prefix}fwdh_frags"] = outh.frag_count
    if with_f64:
        cfg64 = ts.RasterConfig(**{**cfg.__dict__, "dtype": "float64"})
        out64, ctx64 = ts.forward(sc, cam, cfg64)
        d[f"{prefix}fwd64_color"] = out64.color.astype(np.float32)
        d[f"{prefix}fwd64_frags"] = out64.frag_count
        st64 = DensifyStats.zeros(n)
        res64 = ts.backward(sc, ctx64, dI.astype(np.float32).astype(np.float64), st64)
        d[f"{prefix}grads64"] = np.concatenate(
            [getattr(res64.grads, c).reshape(n, -1) for c in CH], axis=1).astype(np.float32)
        d[f"{prefix}stat64_S"] = st64.S
        d[f"{prefix}stat64_M"] = st64.M
        d[f"{prefix}stat64_C"] = st64.C.astype(np.int32)
    return d


def make_A():
    t = time.time()
    spec = SyntheticSceneSpec(n_gaussians=10_000, n_views=1, view_resolution=(128, 128), seed=7)
    sc = random_scene(spec)
    cam = camera_ring(spec)[0]
    d = full_case("", sc, cam, ts.RasterConfig(), target_seed=1234)
    np.savez_compressed(os.path.join(OUT, "golden_A.npz"), **d)
    print(f"golden_A: {time.time() - t:.1f}s")


def make_edge():
    t = time.time()
    d = {}
    # (1) 512-primitive standard scene, ragged 61x45 view, non-zero background
    spec = SyntheticSceneSpec(n_gaussians=512, n_views=8, view_resolution=(61, 45), seed=0)
    sc = random_scene(spec)
    cams = camera_ring(spec)
    cfg = ts.RasterConfig(background=(0.2, 0.5, 0.8))
    d.update(full_case("e1_", sc, cams[3], cfg, target_seed=11))
    # (2) culling off, (3) tree conic reduction
    d.update(full_case("e2_", sc, cams[5], ts.RasterConfig(use_culling=False), target_seed=12, with_f64=False))
    d.update(full_case("e3_", sc, cams[1], ts.RasterConfig(conic_reduce="tree"), target_seed=13,
                       with_f64=False))
    # (4) wide scene: primitives behind the camera, beyond far, off-screen
    spec4 = SyntheticSceneSpec(n_gaussians=3000, n_views=4, view_resolution=(96, 64), seed=3,
                               scene_extent=4.0)
    sc4 = random_scene(spec4)
    spec4c = SyntheticSceneSpec(n_gaussians=3000, n_views=4, view_resolution=(96, 64), seed=3,
                                scene_extent=1.0)
    cam4 = camera_ring(spec4c)[2]
    cam4.far = 4.0
    d.update(full_case("e4_", sc4, cam4, ts.RasterConfig(), target_seed=14))
    # (5) empty scene
    sc5 = SceneSoA.empty()
    out5, _ = ts.forward(sc5, cams[0], ts.RasterConfig(background=(0.1, 0.2, 0.3)))
    d["e5_fwd_color"] = out5.color
    d.update(cam_arrays("e5_", cams[0]))
    # reductions
    rng = np.random.default_rng(5)
    v = rng.normal(size=(4000, 32)).astype(np.float32)
    v[::7] *= np.float32(1e-30)
    v[1::7, :17] = 0
    v[2::7] = 0
    v[3::7] *= rng.uniform(1e-3, 1e3, size=(1, 32)).astype(np.float32)
    v[4::7, 5] = np.float32(1e30)
    d["red_in"] = v
    d["red_tree"] = lane_group_reduce(v, axis=-1)
    d["red_tree64"] = lane_group_reduce(v.astype(np.float64), axis=-1)
    d["red_exp"] = exp_aligned_reduce(v, axis=-1)
    # Adam (dense oracle): 3 steps, varying cluster masks
    n = 700
    rng = np.random.default_rng(9)
    base = SceneSoA(rng.normal(size=(n, 3)), rng.normal(size=(n, 3)) - 2, rng.normal(size=(n, 4)),
                    rng.normal(size=(n, 3)), rng.normal(size=n))
    base = SceneSoA(*[getattr(base, c).astype(np.float32).astype(np.float64) for c in CH])
    d.update({f"adam_in_{c}": getattr(base, c).copy() for c in CH})
    st = AdamState(base)
    lrs = {"position": 1.6e-4 * 3.2, "log_scale": 5e-3, "rotation": 1e-3, "color": 2.5e-3,
           "opacity_logit": 5e-2}
    d["adam_lrs"] = np.array([lrs[c] for c in CH])
    for k in range(3):
        g = {c: (rng.normal(size=getattr(base, c).shape) * (10.0 ** rng.uniform(-6, 0)))
             .astype(np.float32).astype(np.float64) for c in CH}
        mask = rng.uniform(size=(n + 127) // 128) < 0.7
        d[f"adam_g{k}"] = np.concatenate([g[c].reshape(n, -1) for c in CH], axis=1)
        d[f"adam_mask{k}"] = mask
        adam_step(base, g, st, mask, lrs)
    d["adam_out"] = np.concatenate([getattr(base, c).reshape(n, -1) for c in CH], axis=1)
    d["adam_m"] = np.concatenate([st.m(c).reshape(n, -1) for c in CH], axis=1)
    d["adam_v"] = np.concatenate([st.v(c).reshape(n, -1) for c in CH], axis=1)
    d["adam_step"] = st.step.copy()
    # variance score
    S = rng.uniform(0, 2, 5000); M = rng.normal(size=5000); Cn = rng.integers(0, 50, 5000)
    S[:10] = 0; M[:10] = 0
    stats = DensifyStats(S=S, M=M, C=Cn)
    d["var_S"], d["var_M"], d["var_C"] = S, M, Cn
    d["var_score"] = variance_score(stats)
    # Morton edge cases: flat axis, duplicate points, exact bounds
    p = rng.uniform(-1, 1, (3000, 3))
    p[:, 1] = 0.25
    p[100:200] = p[0]
    d["mort_pos"] = p
    lo, hi = p.min(0), p.max(0)
    d["mort_keys"] = ccc.morton_encode(p, lo, hi)
    d["mort_perm"] = np.argsort(d["mort_keys"], kind="stable").astype(np.int32)
    # densification (densify.py:57-187): selection, growth, prune, re-sort
    from tinysplat.densify import DensifyConfig, densify_step, select_and_grow
    rng = np.random.default_rng(21)
    nd = 2000
    spd = SyntheticSceneSpec(n_gaussians=nd, n_views=1, view_resolution=(64, 64), seed=21)
    scd = random_scene(spd)
    scd.opacity_logit[:40] = -8.0          # prune candidates (sigmoid < 0.005)
    scd.log_scale[80:] -= 1.6             # small primitives -> clone; 40:80 stay large -> split
    scd = SceneSoA(*[getattr(scd, c).astype(np.float32).astype(np.float64) for c in CH])
    std = DensifyStats(S=rng.uniform(0, 1, nd), M=rng.normal(0, 0.3, nd), C=rng.integers(0, 30, nd))
    std.S[::17] = 0.0
    std.attach(scd)
    d.update({f"dens_in_{c}": getattr(scd, c).copy() for c in CH})
    d["dens_S"], d["dens_M"], d["dens_C"] = std.S.copy(), std.M.copy(), std.C.copy()
    cfgd = DensifyConfig(start_epoch=1, densify_interval_epochs=1, budget=2600)
    scores = variance_score(std)
    thr = cfgd.resolve_split_threshold(scd)
    ci, si = select_and_grow(scd, scores, cfgd.budget, thr)
    d["dens_clone"], d["dens_split"], d["dens_thr"] = ci, si, np.array(thr)
    row = densify_step(scd, std, cfgd, epoch=1)
    d.update({f"dens_out_{c}": getattr(scd, c).copy() for c in CH})
    d["dens_row"] = np.array([row.n_before, row.n_after, row.n_split, row.n_clone, row.n_pruned])
    np.savez_compressed(os.path.join(OUT, "golden_edge.npz"), **d)
    print(f"golden_edge: {time.time() - t:.1f}s")


def make_big():
    out = {}
    for name, n, res, fwd in (("B", 1_000_000, (1920, 1080), True),
                              ("C", 3_000_000, (1920, 1080), False),
                              ("E", 6_000_000, (3840, 2160), False)):
        t = time.time()
        sc, cams = scaled_scene(n, 7, res)
        cam = cams[0]
        e = {"n": n, "res": list(res),
             "scene_sha": {c: sha(getattr(sc, c).astype(np.float32)) for c in CH}}
        lo, hi = sc.bounds()
        keys = ccc.morton_encode(sc.position, lo, hi)
        perm = np.argsort(keys, kind="stable")
        e["morton_keys_sha"] = sha(keys)
        e["morton_perm_sha"] = sha(perm.astype(np.int64))
        # the hot path runs on the Morton-sorted scene
        sc.permute(perm)
        pr = project_scene(sc, cam, dtype=np.float32)
        for k in ("xy", "depth", "conic", "radius"):
            a = getattr(pr, k).copy()
            a[~pr.valid] = 0
            e[f"proj_{k}_sha_valid"] = sha(a)
        e["proj_valid_sha"] = sha(pr.valid.astype(np.uint8))
        e["proj_in_image_sha"] = sha(pr.in_image.astype(np.uint8))
        idx = ccc.build_clusters(sc)
        fr = ts.build_frustum(cam)
        vis = ccc.cluster_visibility(idx, fr, pr.in_image)
        e["vis_mask_sha"] = sha(vis.astype(np.uint8))
        e["cull_mask_sha"] = sha(ccc.cull_clusters(idx, fr).astype(np.uint8))
        e["visible_clusters"] = int(vis.sum())
        cp, cmap = ccc.compact_arrays(pr, vis, 128, sc.n)
        e["n_compact"] = int(len(cmap))
        e["compact_map_sha"] = sha(cmap.astype(np.int64))
        tiles = bin_tiles(cp.xy, cp.depth, cp.radius, cp.in_image, cam.resolution)
        offs, prims = tiles_flat(tiles, cam.resolution)
        e["P"] = int(len(prims))
        e["nonempty_tiles"] = len(tiles)
        e["tile_offsets_sha"] = sha(offs.astype(np.int64))
        e["tile_prims_sha"] = sha(prims.astype(np.int64))
        print(f"{name}: stages {time.time() - t:.1f}s  P={len(prims)}  Nc={len(cmap)}")
        if fwd:
            t = time.time()
            o, _ = ts.forward(sc, cam)
            rng = np.random.default_rng(77)
            H, W = res[1], res[0]
            pix = rng.choice(H * W, 20000, replace=False)
            e["fwd_sample_pix"] = pix.tolist()
            e["fwd_sample_color"] = o.color.reshape(-1, 3)[pix].astype(float).tolist()
            e["fwd_sample_T"] = o.transmittance.reshape(-1)[pix].astype(float).tolist()
            e["fwd_sample_frags"] = o.frag_count.reshape(-1)[pix].astype(int).tolist()
            e["fwd_color_sum"] = float(o.color.astype(np.float64).sum())
            e["fwd_frags_sum"] = int(o.frag_count.sum())
            print(f"{name}: forward {time.time() - t:.1f}s")
        out[name] = e
    with open(os.path.join(OUT, "golden_big.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    if a.only in ("", "A"):
        make_A()
    if a.only in ("", "edge"):
        make_edge()
    if a.big or a.only == "big":
        make_big()
