"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The fixtures in tests/golden/ were produced by importing the reference
(/root/reference/pkg/src/tinysplat) in the build container
(tools/make_golden.py).  If these pass, the oracle may be trusted as the
checker for the CUDA path on the GPU box, where the reference is absent.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests import goldens as G


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_projection_bit_exact(fname, prefix):
    d = G.load(fname)
    sc, cam = G.scene(d, prefix), G.camera(d, prefix)
    p = O.project(sc, cam, "float32", 0.3)
    valid = d[f"{prefix}proj_valid"]
    assert np.array_equal(p["valid"], valid)
    assert np.array_equal(p["in_image"], d[f"{prefix}proj_in_image"])
    for k in ("xy", "depth", "conic", "radius", "color", "opacity"):
        ref = d[f"{prefix}proj_{k}"]
        got = p[k]
        # entries where valid is False are unspecified (projection.py:108-110)
        assert np.array_equal(got[valid].view(np.uint32), ref[valid].view(np.uint32)), k
    for k in ("color", "opacity"):
        assert np.array_equal(p[k], d[f"{prefix}proj_{k}"]), k


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_morton_and_ccc_bit_exact(fname, prefix):
    d = G.load(fname)
    sc, cam = G.scene(d, prefix), G.camera(d, prefix)
    n = len(sc["position"])
    keys, perm = O.morton_perm(sc["position"])
    assert np.array_equal(keys, d[f"{prefix}morton_keys"])
    assert np.array_equal(perm, d[f"{prefix}morton_perm"])
    amin, amax = O.build_clusters(sc["position"], sc["log_scale"])
    # AABBs go through float64 exp: numpy's SIMD exp and glibc exp may differ by 1 ulp
    np.testing.assert_allclose(amin, d[f"{prefix}aabb_min"], rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(amax, d[f"{prefix}aabb_max"], rtol=1e-15, atol=1e-15)
    planes = d[f"{prefix}planes"]
    W, H = cam.resolution
    mine = O.frustum_planes(cam.world_to_camera, *cam.focal, *cam.principal_point, W, H, cam.near, cam.far)
    assert np.array_equal(mine, planes)
    assert np.array_equal(O.cull_clusters(amin, amax, planes), d[f"{prefix}cull_mask"])
    p = O.project(sc, cam, "float32", 0.3)
    vis = O.cluster_visibility(n, amin, amax, planes, p["in_image"])
    assert np.array_equal(vis, d[f"{prefix}vis_mask"])
    if int(d[f"{prefix}cfg_cull"]):
        assert np.array_equal(O.compact_map(n, vis), d[f"{prefix}compact_map"])


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_forward_backward_vs_reference(fname, prefix):
    d = G.load(fname)
    sc, cam = G.scene(d, prefix), G.camera(d, prefix)
    cfg = G.raster_cfg(d, prefix)
    color, T, frags, ctx = O.forward(sc, cam, cfg)
    assert np.array_equal(ctx.compact_map, d[f"{prefix}compact_map"])
    assert np.array_equal(ctx.tile_offsets, d[f"{prefix}tile_offsets"])
    assert np.array_equal(ctx.prims, d[f"{prefix}tile_prims"])
    # fp32 vs fp32: differences only from np.exp (SIMD, up to ~2.5 ulp) vs expf
    assert np.abs(color - d[f"{prefix}fwd_color"]).max() <= 1e-5
    assert np.abs(T - d[f"{prefix}fwd_T"]).max() <= 1e-5
    assert (frags != d[f"{prefix}fwd_frags"]).sum() <= 2
    # loss gradient restatement is bit-exact
    rng = np.random.default_rng(int(d[f"{prefix}target_seed"]))
    target = rng.uniform(0.0, 1.0, color.shape)
    loss, dI = O.loss_and_grad(d[f"{prefix}fwd_color"], target, 0.2)
    assert loss == float(d[f"{prefix}loss"])
    assert np.array_equal(dI.astype(np.float32), d[f"{prefix}dL_dI"])
    b = O.backward(sc, ctx, d[f"{prefix}dL_dI"])
    g_ref = d[f"{prefix}grads"].astype(np.float64)
    g64 = d.get(f"{prefix}grads64")
    for lo, hi in ((0, 3), (3, 6), (6, 10), (10, 13), (13, 14)):
        if g64 is None:
            assert G.floored_rel(b["grads"][:, lo:hi], g_ref[:, lo:hi]) <= 1e-3
        else:
            assert G.conditioned_rel_excess(b["grads"][:, lo:hi], g_ref[:, lo:hi],
                                            g64[:, lo:hi], 1e-3) <= 1.0
    assert np.array_equal(b["C"], d[f"{prefix}stat_C"])
    assert G.floored_rel(b["S"], d[f"{prefix}stat_S"]) <= 1e-4
    assert G.floored_rel(b["M"], d[f"{prefix}stat_M"]) <= 1e-3
    assert np.array_equal(b["cluster_mask"], d[f"{prefix}upd_mask"])
    sc_o = O.variance_score(b["S"], b["M"], b["C"])
    assert G.floored_rel(sc_o, d[f"{prefix}score"]) <= 1e-2


@pytest.mark.parametrize("fname,prefix", [c for c in G.CASES if c[1] in ("", "e1_", "e4_")])
def test_float64_numeric_oracle(fname, prefix):
    d = G.load(fname)
    sc, cam = G.scene(d, prefix), G.camera(d, prefix)
    cfg = G.raster_cfg(d, prefix, dtype="float64")
    color, T, frags, ctx = O.forward(sc, cam, cfg)
    assert np.abs(color - d[f"{prefix}fwd64_color"]).max() <= 1e-6
    assert np.array_equal(frags, d[f"{prefix}fwd64_frags"])
    b = O.backward(sc, ctx, d[f"{prefix}dL_dI"].astype(np.float64))
    g_ref = d[f"{prefix}grads64"].astype(np.float64)
    for lo, hi in ((0, 3), (3, 6), (6, 10), (10, 13), (13, 14)):
        assert G.floored_rel(b["grads"][:, lo:hi], g_ref[:, lo:hi]) <= 1e-5
    assert np.array_equal(b["C"], d[f"{prefix}stat64_C"])
    assert G.floored_rel(b["S"], d[f"{prefix}stat64_S"]) <= 1e-6
    assert G.floored_rel(b["M"], d[f"{prefix}stat64_M"]) <= 1e-4


def test_empty_scene():
    d = G.load("golden_edge.npz")
    cam = G.camera(d, "e5_")
    sc = {c: np.zeros((0, w)) if w > 1 else np.zeros(0) for c, w in O.WIDTHS.items()}
    color, T, frags, ctx = O.forward(sc, cam, O.RasterConfig(background=(0.1, 0.2, 0.3)))
    assert np.array_equal(color, d["e5_fwd_color"])
    assert (T == 1).all() and (frags == 0).all()


def test_reductions_bit_exact():
    d = G.load("golden_edge.npz")
    v = d["red_in"]
    assert np.array_equal(O.lane_group_reduce(v), d["red_tree"])
    assert np.array_equal(O.lane_group_reduce(v.astype(np.float64)), d["red_tree64"])
    assert np.array_equal(O.exp_aligned_reduce(v), d["red_exp"])


def test_adam_dense_oracle():
    d = G.load("golden_edge.npz")
    n = len(d["adam_in_position"])
    params = np.ascontiguousarray(np.concatenate(
        [d[f"adam_in_{c}"].reshape(n, -1) for c in G.CH], axis=1))
    m = np.zeros_like(params); v = np.zeros_like(params); step = np.zeros(n, np.int64)
    for k in range(3):
        O.adam_step(params, np.ascontiguousarray(d[f"adam_g{k}"]), m, v, step, d[f"adam_mask{k}"],
                    d["adam_lrs"])
    np.testing.assert_allclose(params, d["adam_out"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(m, d["adam_m"], rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(v, d["adam_v"], rtol=1e-13, atol=1e-300)
    assert np.array_equal(step, d["adam_step"])


def test_variance_score_exact():
    d = G.load("golden_edge.npz")
    assert np.array_equal(O.variance_score(d["var_S"], d["var_M"], d["var_C"]), d["var_score"])


def test_morton_edge_cases():
    d = G.load("golden_edge.npz")
    keys, perm = O.morton_perm(d["mort_pos"])
    assert np.array_equal(keys, d["mort_keys"])
    assert np.array_equal(perm, d["mort_perm"])


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_half_path_vs_reference(fname, prefix):
    """forward.py:194-230: fp16 blending state; numpy's float16 ops round
    once per op like the oracle's _Float16 casts (G comes from different
    float32 exp implementations, so allow one binary16 ulp-scale slack)."""
    d = G.load(fname)
    sc, cam = G.scene(d, prefix), G.camera(d, prefix)
    color, T, frags, _ = O.forward(sc, cam, G.raster_cfg(d, prefix), half=True)
    assert np.abs(color - d[f"{prefix}fwdh_color"]).max() <= 2e-3
    assert np.abs(T - d[f"{prefix}fwdh_T"]).max() <= 2e-3
    assert (frags != d[f"{prefix}fwdh_frags"]).sum() <= 0.002 * frags.size + 2
    ref32 = d[f"{prefix}fwd_color"].astype(np.float64)
    mse = ((color.astype(np.float64) - ref32) ** 2).mean()
    assert mse == 0 or 10 * np.log10(1 / mse) >= 58.0
