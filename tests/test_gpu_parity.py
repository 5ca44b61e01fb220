"""Parity of the CUDA path (through the C-ABI) with the reference's own
outputs (tests/golden, made from /root/reference) and with the CPU oracle.

Bars (BASELINE.json north_star):
  bit-exact  Morton keys / sort order, cull masks, compact maps, tile lists,
             projected xy/depth/conic/radius/colour/opacity
  1e-3       rendered image max abs (fp32 accumulation)
  1e-2       per-Gaussian gradients and S/M/variance, floored relative
             |g - g_ref| <= 1e-2 * max(|g_ref|, 1e-3 * max|g_ref|) per channel,
             with an allowance only where the reference's own fp32 path is
             equally far from its fp64 path (ill-conditioned rows)
"""
import hashlib

import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import goldens as G

pytestmark = pytest.mark.gpu

CH_SLICES = ((0, 3), (3, 6), (6, 10), (10, 13), (13, 14))


def _sb():
    import paper_2503_01199_b200 as sb
    return sb


def _scene(d, prefix=""):
    sb = _sb()
    sc = G.scene(d, prefix)
    return sb.SceneSoA(*[sc[k] for k in G.CH], device="cuda")


def _cfg(d, prefix=""):
    sb = _sb()
    return sb.RasterConfig(background=tuple(float(b) for b in d[f"{prefix}cfg_bg"]),
                           use_culling=bool(d[f"{prefix}cfg_cull"]),
                           conic_reduce="tree" if int(d[f"{prefix}cfg_tree"]) else "exp_aligned")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_forward_bit_exact_stages_and_image(fname, prefix):
    sb = _sb()
    d = G.load(fname)
    scene, cam, cfg = _scene(d, prefix), G.camera(d, prefix), _cfg(d, prefix)
    out, ctx = sb.forward(scene, cam, cfg)
    cmap = ctx.compact_map.cpu().numpy()
    assert np.array_equal(cmap, d[f"{prefix}compact_map"])
    assert np.array_equal(ctx.tile_offsets.cpu().numpy(), d[f"{prefix}tile_offsets"])
    assert np.array_equal(ctx.tile_prims.cpu().numpy(), d[f"{prefix}tile_prims"])
    if int(d[f"{prefix}cfg_cull"]) and len(cmap):
        vis = d[f"{prefix}vis_mask"]
        assert np.array_equal(ctx.cluster_vis.cpu().numpy().astype(bool), vis)
    p = {k: v.cpu().numpy() for k, v in ctx.projected.items()}
    valid = d[f"{prefix}proj_valid"][cmap]
    assert np.array_equal(p["valid"], valid)
    assert np.array_equal(p["in_image"], d[f"{prefix}proj_in_image"][cmap])
    for k in ("xy", "depth", "conic", "radius", "color", "opacity"):
        ref = d[f"{prefix}proj_{k}"][cmap]
        assert np.array_equal(p[k][valid].view(np.uint32), ref[valid].view(np.uint32)), k
    color = out.color.cpu().numpy()
    assert np.abs(color - d[f"{prefix}fwd_color"]).max() <= 1e-3
    assert np.abs(out.transmittance.cpu().numpy() - d[f"{prefix}fwd_T"]).max() <= 1e-3
    # frag counts: exact except alpha / T threshold flips
    assert (out.frag_count.cpu().numpy() != d[f"{prefix}fwd_frags"]).sum() <= 2
    if f"{prefix}fwd64_color" in d:
        assert np.abs(color - d[f"{prefix}fwd64_color"]).max() <= 1e-3


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_backward_vs_reference(fname, prefix):
    sb = _sb()
    d = G.load(fname)
    scene, cam, cfg = _scene(d, prefix), G.camera(d, prefix), _cfg(d, prefix)
    n = scene.n
    out, ctx = sb.forward(scene, cam, cfg)
    stats = sb.DensifyStats.zeros(n)
    res = sb.backward(scene, ctx, torch.from_numpy(d[f"{prefix}dL_dI"]), stats)
    g = res.grads.packed[:, :14].double().cpu().numpy()
    g32 = d[f"{prefix}grads"].astype(np.float64)
    g64 = d.get(f"{prefix}grads64")
    for lo, hi in CH_SLICES:
        if g64 is None:
            assert G.floored_rel(g[:, lo:hi], g32[:, lo:hi]) <= 1e-2, (lo, hi)
        else:
            assert G.conditioned_rel_excess(g[:, lo:hi], g32[:, lo:hi], g64[:, lo:hi].astype(np.float64),
                                            1e-2) <= 1.0, (lo, hi)
    C = stats.C.cpu().numpy()
    assert (C != d[f"{prefix}stat_C"]).sum() <= 2
    assert G.floored_rel(stats.S.cpu().numpy(), d[f"{prefix}stat_S"]) <= 1e-2
    assert G.floored_rel(stats.M.cpu().numpy(), d[f"{prefix}stat_M"]) <= 1e-2
    assert np.array_equal(res.cluster_mask.cpu().numpy(), d[f"{prefix}upd_mask"])
    score = sb.variance_score(stats).cpu().numpy()
    assert G.floored_rel(score, d[f"{prefix}score"]) <= 1e-2


@pytest.mark.parametrize("fname,prefix", [c for c in G.CASES if c[1] in ("", "e1_", "e4_")])
def test_backward_vs_float64_oracle(fname, prefix):
    """Against the reference's float64 path: the back-to-front fp32 replay is
    closer to fp64 than the reference's own fp32 path."""
    sb = _sb()
    import dataclasses
    d = G.load(fname)
    scene, cam, cfg = _scene(d, prefix), G.camera(d, prefix), _cfg(d, prefix)
    g64 = d[f"{prefix}grads64"].astype(np.float64)
    g32 = d[f"{prefix}grads"].astype(np.float64)
    # e4's near-plane rows amplify the float-atomic summation order of the
    # fast backward through the chain (log-scale slice: 3.1e-3 median, 9.1e-3
    # max over 40 runs, tools/e4_probe.py): the plain 1e-2 bar is asserted on
    # the deterministic (fixed-order) backward, the fast one gets 2e-2
    for det, bar in (((False, 1e-2),) if prefix != "e4_" else ((True, 1e-2), (False, 2e-2))):
        _check_vs_float64(sb, scene, cam, dataclasses.replace(cfg, deterministic=det), d, prefix, g64, g32, bar)


def _check_vs_float64(sb, scene, cam, cfg, d, prefix, g64, g32, bar):
    out, ctx = sb.forward(scene, cam, cfg)
    res = sb.backward(scene, ctx, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n))
    g = res.grads.packed[:, :14].double().cpu().numpy()
    for lo, hi in CH_SLICES:
        den = np.maximum(np.abs(g64[:, lo:hi]), 1e-3 * np.abs(g64[:, lo:hi]).max())
        err = np.abs(g[:, lo:hi] - g64[:, lo:hi]) / den
        # rows the reference's OWN float32 path misses by more than half the
        # bar: ill-conditioned in float32 (e4: one Gaussian at depth 0.062,
        # 1.24x the near plane, whose rotation gradient the reference's fp32
        # path gets 1.6e-2 wrong).  The device shares the reference's
        # bit-exact fp32 projection, so it inherits that error there; such
        # rows may be no worse than twice the reference's own.
        ref_err = np.abs(g32[:, lo:hi] - g64[:, lo:hi]) / den
        excused = ref_err.max(axis=1) > 0.5e-2
        assert excused.sum() <= (1 if prefix == "e4_" else 0), (lo, hi, np.flatnonzero(excused))
        assert err[~excused].max(initial=0.0) <= bar, (lo, hi, cfg.deterministic)
        assert (err[excused] <= 2 * ref_err[excused] + bar).all(), (lo, hi, cfg.deterministic)


def test_morton_keys_and_sort_bit_exact():
    sb = _sb()
    from paper_2503_01199_b200.ccc import morton_encode_scene
    for fname, prefix in (("golden_A.npz", ""), ("golden_edge.npz", "e4_")):
        d = G.load(fname)
        scene = _scene(d, prefix)
        keys, lo, hi = morton_encode_scene(scene)
        assert np.array_equal(keys.cpu().numpy().view(np.uint64), d[f"{prefix}morton_keys"])
        sc2 = scene.copy()
        perm = sb.morton_sort(sc2)
        assert np.array_equal(perm.cpu().numpy(), d[f"{prefix}morton_perm"])
        assert torch.equal(sc2.data, scene.data[perm])
        assert sc2.generation == scene.generation + 1
    d = G.load("golden_edge.npz")
    pos = d["mort_pos"]
    z = np.zeros((len(pos), 3))
    scene = sb.SceneSoA(pos, z, np.tile([1.0, 0, 0, 0], (len(pos), 1)), z, np.zeros(len(pos)), device="cuda")
    # mort_pos is float64 data not representable in fp32; compare with the
    # oracle on the fp32-rounded positions instead of the fixture
    keys, perm = O.morton_perm(pos.astype(np.float32).astype(np.float64))
    got, _, _ = morton_encode_scene(scene)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), keys)
    assert np.array_equal(sb.morton_sort(scene.copy()).cpu().numpy(), perm)
    # ccc.morton_encode on the float64 positions themselves: the reference's
    # own keys (fixture), bounds as morton_sort takes them (scene.py:256-260)
    from paper_2503_01199_b200.ccc import morton_encode
    k64 = morton_encode(pos, pos.min(axis=0), pos.max(axis=0))
    assert np.array_equal(k64.cpu().numpy().view(np.uint64), d["mort_keys"])
    # explicit bounds narrower than the data: clipped to the grid edges
    lo, hi = np.full(3, -0.25), np.full(3, 0.25)
    kk = morton_encode(torch.from_numpy(pos).cuda(), lo, hi).cpu().numpy().view(np.uint64)
    assert np.array_equal(kk, O.morton_encode(pos, lo, hi))
    with pytest.raises(sb.ValidationError):
        bad = pos.copy()
        bad[3, 1] = np.nan
        morton_encode(bad, lo, hi)


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_bin_tiles_api_vs_reference(fname, prefix):
    """tiles.bin_tiles (tiles.py:50-107) on the reference's own compact
    projected arrays: per-tile lists bit-exact with the reference's."""
    from paper_2503_01199_b200.tiles import bin_tiles, bin_tiles_device
    d = G.load(fname)
    cm = d[f"{prefix}compact_map"].astype(np.int64)
    xy, depth = d[f"{prefix}proj_xy"][cm], d[f"{prefix}proj_depth"][cm]
    radius, mask = d[f"{prefix}proj_radius"][cm], d[f"{prefix}proj_in_image"][cm]
    res = tuple(int(v) for v in d[f"{prefix}res"])
    offs, prims = bin_tiles_device(xy, depth, radius, mask, res)
    assert np.array_equal(offs.cpu().numpy().astype(np.int64), d[f"{prefix}tile_offsets"])
    assert np.array_equal(prims.cpu().numpy().astype(np.int64), d[f"{prefix}tile_prims"])
    tiles = bin_tiles(xy, depth, radius, mask, res)
    ref_offs = d[f"{prefix}tile_offsets"]
    assert len(tiles) == int((np.diff(ref_offs) > 0).sum())
    for tw in tiles[:50]:
        t = tw.tile_y * ((res[0] + 15) // 16) + tw.tile_x
        assert np.array_equal(tw.primitives, d[f"{prefix}tile_prims"][ref_offs[t]:ref_offs[t + 1]])
        assert tw.origin == (16 * tw.tile_x, 8 * tw.tile_y)
    assert bin_tiles(xy, depth, radius, np.zeros_like(mask), res) == []


def test_radix_sort_random_keys_stable():
    from paper_2503_01199_b200.ccc import sort_pairs
    rng = np.random.default_rng(3)
    for n in (1, 7, 4096, 4097, 100_003):
        k = rng.integers(0, 1 << 20, n, dtype=np.uint64) << np.uint64(30)   # many duplicates
        kt = torch.from_numpy(k.view(np.int64)).cuda()
        vt = torch.arange(n, dtype=torch.int32, device="cuda")
        ks, vs = sort_pairs(kt, vt, bits=64)
        ref = np.argsort(k, kind="stable")
        assert np.array_equal(vs.cpu().numpy(), ref)
        assert np.array_equal(ks.cpu().numpy().view(np.uint64), k[ref])


def test_lane_reductions_bit_exact():
    sb = _sb()
    d = G.load("golden_edge.npz")
    v = torch.from_numpy(d["red_in"]).cuda()
    assert np.array_equal(sb.lane_group_reduce(v).cpu().numpy(), d["red_tree"])
    assert np.array_equal(sb.lane_group_reduce(v, float64=True).cpu().numpy(), d["red_tree64"])
    assert np.array_equal(sb.exp_aligned_reduce(v).cpu().numpy(), d["red_exp"].astype(np.float32))


def test_adam_vs_reference():
    sb = _sb()
    d = G.load("golden_edge.npz")
    n = len(d["adam_in_position"])
    scene = sb.SceneSoA(*[d[f"adam_in_{c}"] for c in G.CH], device="cuda")
    st = sb.AdamState(scene)
    lrs = dict(zip(G.CH, d["adam_lrs"]))
    for k in range(3):
        g = d[f"adam_g{k}"]
        grads = sb.SceneGrads.from_dict({c: g[:, a:b] for c, (a, b) in zip(G.CH, CH_SLICES)}, n)
        sb.adam_step(scene, grads, st, torch.from_numpy(d[f"adam_mask{k}"]), lrs)
    got = scene.data[:, :14].double().cpu().numpy()
    # fp32 state vs the reference's fp64: ~1e-7 relative; Adam steps are ~lr
    np.testing.assert_allclose(got, d["adam_out"], rtol=2e-6, atol=2e-7)
    # moments are float32 state: identical grads in, float64 arithmetic, one
    # rounding per step (cancellation in 0.9 m + 0.1 g needs the floor)
    for lo, hi in CH_SLICES:
        assert G.floored_rel(st.m_rows[:, lo:hi].double().cpu().numpy(), d["adam_m"][:, lo:hi]) <= 1e-5
        assert G.floored_rel(st.v_rows[:, lo:hi].double().cpu().numpy(), d["adam_v"][:, lo:hi]) <= 1e-5
    assert np.array_equal(st.step.cpu().numpy(), d["adam_step"])


def test_variance_score_exact():
    sb = _sb()
    d = G.load("golden_edge.npz")
    stats = sb.DensifyStats(S=torch.from_numpy(d["var_S"]).cuda(), M=torch.from_numpy(d["var_M"]).cuda(),
                            C=torch.from_numpy(d["var_C"].astype(np.int32)).cuda())
    assert np.array_equal(sb.variance_score(stats).cpu().numpy(), d["var_score"])


def test_empty_scene_and_errors():
    sb = _sb()
    d = G.load("golden_edge.npz")
    cam = G.camera(d, "e5_")
    scene = sb.SceneSoA.empty(device="cuda")
    out, ctx = sb.forward(scene, cam, sb.RasterConfig(background=(0.1, 0.2, 0.3)))
    assert np.array_equal(out.color.cpu().numpy(), d["e5_fwd_color"])
    # the counters of an empty scene are reported, not left uninitialised
    assert ctx.n_compact == 0 and ctx.visible_clusters == 0 and ctx.culled_clusters == 0
    assert ctx.n_pairs == 0 and ctx.n_degenerate == 0
    res = sb.backward(scene, ctx, torch.zeros(cam.resolution[1], cam.resolution[0], 3))
    assert res.grads.packed.shape == (0, 16)
    # staleness and shape errors (backward.py:213-218)
    d = G.load("golden_A.npz")
    scene = _scene(d)
    out, ctx = sb.forward(scene, G.camera(d))
    with pytest.raises(sb.ShapeMismatchError):
        sb.backward(scene, ctx, torch.zeros(3, 3, 3))
    sb.morton_sort(scene)
    with pytest.raises(sb.StaleSceneError):
        sb.backward(scene, ctx, torch.zeros(128, 128, 3))


def test_forward_deterministic_and_culling_invisible():
    sb = _sb()
    d = G.load("golden_A.npz")
    scene, cam = _scene(d), G.camera(d)
    a, _ = sb.forward(scene, cam)
    b, _ = sb.forward(scene, cam)
    c, _ = sb.forward(scene, cam, sb.RasterConfig(use_culling=False))
    assert torch.equal(a.color, b.color) and torch.equal(a.frag_count, b.frag_count)
    assert torch.equal(a.color, c.color) and torch.equal(a.frag_count, c.frag_count)


@pytest.mark.parametrize("n,res,seed", [(50_000, (256, 192), 11), (200_000, (640, 360), 5)])
def test_seeded_vs_oracle(n, res, seed):
    """Size-scaled scenes against the oracle run here."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays
    arr = scaled_scene_arrays(n, seed, res)
    cam = camera_ring(SyntheticSceneSpec(n_gaussians=n, n_views=3, view_resolution=res, seed=seed))[2]
    scene = sb.SceneSoA(*[arr[k] for k in G.CH], device="cuda")
    sb.morton_sort(scene)
    arr = {k: v for k, v in zip(G.CH, [None] * 5)}
    h = scene.data.cpu().numpy().astype(np.float64)
    arr = {"position": h[:, 0:3], "log_scale": h[:, 3:6], "rotation": h[:, 6:10], "color": h[:, 10:13],
           "opacity_logit": h[:, 13]}
    out, ctx = sb.forward(scene, cam)
    col, T, frags, octx = O.forward(arr, cam, O.RasterConfig())
    assert np.array_equal(ctx.compact_map.cpu().numpy(), octx.compact_map)
    assert np.array_equal(ctx.tile_offsets.cpu().numpy().astype(np.int64), octx.tile_offsets)
    assert np.array_equal(ctx.tile_prims.cpu().numpy().astype(np.int64), octx.prims)
    assert np.abs(out.color.cpu().numpy() - col).max() <= 1e-3
    assert (out.frag_count.cpu().numpy() != frags).sum() <= 5
    rng = np.random.default_rng(seed)
    _, dI = O.loss_and_grad(col, rng.uniform(0, 1, col.shape), 0.2)
    dI = dI.astype(np.float32)
    res_ = sb.backward(scene, ctx, torch.from_numpy(dI), sb.DensifyStats.zeros(scene.n))
    ob = O.backward(arr, octx, dI)
    g = res_.grads.packed[:, :14].double().cpu().numpy()
    for lo, hi in CH_SLICES:
        assert G.floored_rel(g[:, lo:hi], ob["grads"][:, lo:hi]) <= 1e-2, (lo, hi)
    st = res_.stats
    assert G.floored_rel(st.S.cpu().numpy(), ob["S"]) <= 1e-2
    assert G.floored_rel(st.M.cpu().numpy(), ob["M"]) <= 1e-2
    assert (st.C.cpu().numpy() != ob["C"]).sum() <= 5


@pytest.mark.parametrize("n,res", [(30_000, (64, 64)), (120_000, (64, 48))])
def test_long_tile_lists_vs_oracle(n, res):
    """Unscaled footprints on a tiny view: thousands of primitives per tile,
    so the per-tile sort takes its long-list paths (> 2048 keys, and chunked
    merges beyond 4096).  Tile lists bit-exact with the oracle."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, random_scene_arrays
    spec = SyntheticSceneSpec(n_gaussians=n, n_views=1, view_resolution=res, seed=3)
    arr = random_scene_arrays(spec)
    cam = camera_ring(spec)[0]
    scene = sb.SceneSoA(*[arr[k] for k in G.CH], device="cuda")
    out, ctx = sb.forward(scene, cam)
    col, T, frags, octx = O.forward({k: np.asarray(arr[k], np.float64) for k in G.CH}, cam, O.RasterConfig())
    offs = octx.tile_offsets
    assert np.diff(offs).max() > 4096
    assert np.array_equal(ctx.tile_offsets.cpu().numpy().astype(np.int64), offs)
    assert np.array_equal(ctx.tile_prims.cpu().numpy().astype(np.int64), octx.prims)
    assert np.abs(out.color.cpu().numpy() - col).max() <= 1e-3


def test_long_super_tile_degenerate_depths_vs_oracle():
    """8000 identical Gaussians (one depth) plus one far behind them, all on
    the same super-tiles: the long super-tiles' key-range histogram puts the
    cluster into one bin above the group quantum, so the sort takes its
    chunk-sort + merge fallback.  Tile lists bit-exact with the oracle."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring
    res = (128, 128)
    cam = camera_ring(SyntheticSceneSpec(n_gaussians=8001, n_views=1, view_resolution=res, seed=1))[0]
    n = 8001
    c = np.asarray(cam.center, np.float64)
    far = -2.0 * c / np.linalg.norm(c)          # behind the origin on the same view ray
    arr = {"position": np.zeros((n, 3)), "log_scale": np.full((n, 3), np.log(0.05)),
           "rotation": np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)), "color": np.full((n, 3), 0.25),
           "opacity_logit": np.full(n, -4.0)}
    arr["position"][n // 2] = far
    arr["color"][n // 2] = [1.0, -1.0, 0.5]
    arr = {k: v.astype(np.float32) for k, v in arr.items()}
    scene = sb.SceneSoA(*[arr[k] for k in G.CH], device="cuda")
    out, ctx = sb.forward(scene, cam)
    col, T, frags, octx = O.forward({k: np.asarray(arr[k], np.float64) for k in G.CH}, cam, O.RasterConfig())
    assert np.diff(octx.tile_offsets).max() > 6144
    assert np.array_equal(ctx.tile_offsets.cpu().numpy().astype(np.int64), octx.tile_offsets)
    assert np.array_equal(ctx.tile_prims.cpu().numpy().astype(np.int64), octx.prims)
    assert np.abs(out.color.cpu().numpy() - col).max() <= 1e-3


@pytest.mark.parametrize("name", ["B", "C", "E"])
def test_big_configs_bit_exact_hashes(name):
    """Configs B/C/E at full size: Morton order, projection, cull masks,
    compact map and tile lists hash-identical to the reference's."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays
    gb = G.load("golden_big.json")[name]
    n, res = gb["n"], tuple(gb["res"])
    arr = scaled_scene_arrays(n, 7, res)
    for c in G.CH:
        assert _sha(arr[c].astype(np.float32)) == gb["scene_sha"][c], c
    scene = sb.SceneSoA(*[arr[k] for k in G.CH], device="cuda")
    from paper_2503_01199_b200.ccc import morton_encode_scene
    keys, _, _ = morton_encode_scene(scene)
    assert _sha(keys.cpu().numpy().view(np.uint64)) == gb["morton_keys_sha"]
    perm = sb.morton_sort(scene)
    assert _sha(perm.cpu().numpy()) == gb["morton_perm_sha"]
    cam = camera_ring(SyntheticSceneSpec(n_gaussians=n, n_views=1, view_resolution=res, seed=7))[0]
    out, ctx = sb.forward(scene, cam)
    assert ctx.n_compact == gb["n_compact"] and ctx.visible_clusters == gb["visible_clusters"]
    assert _sha(ctx.cluster_vis.cpu().numpy().astype(np.uint8)) == gb["vis_mask_sha"]
    assert _sha(ctx.compact_map.cpu().numpy().astype(np.int64)) == gb["compact_map_sha"]
    assert ctx.n_pairs == gb["P"]
    assert _sha(ctx.tile_offsets.cpu().numpy().astype(np.int64)) == gb["tile_offsets_sha"]
    assert _sha(ctx.tile_prims.cpu().numpy().astype(np.int64)) == gb["tile_prims_sha"]
    if "fwd_sample_pix" in gb:
        pix = np.array(gb["fwd_sample_pix"])
        col = out.color.reshape(-1, 3).cpu().numpy()[pix]
        assert np.abs(col - np.array(gb["fwd_sample_color"])).max() <= 1e-3
        fr = out.frag_count.reshape(-1).cpu().numpy()[pix]
        assert (fr != np.array(gb["fwd_sample_frags"])).sum() <= 5


def test_backward_row_reductions_bit_exact():
    """The register row reductions the raster backward actually uses."""
    from paper_2503_01199_b200.reduction import backward_row_reduce
    d = G.load("golden_edge.npz")
    v = torch.from_numpy(d["red_in"]).cuda()
    assert np.array_equal(backward_row_reduce(v).cpu().numpy(), d["red_tree"])
    assert np.array_equal(backward_row_reduce(v, exp_aligned=True).cpu().numpy(), d["red_exp"].astype(np.float32))


@pytest.mark.parametrize("W,H", [(1920, 1080), (97, 61), (300, 17), (64, 200), (11, 11)])
def test_fused_loss_sizes_vs_torch(W, H):
    """The fused loss over image sizes that exercise partial strips, partial
    and single row segments and a one-pixel SSIM interior, and the
    benchmarked 1080p frame, against the separable-conv2d restatement
    (metrics.py:118-132) run in float64 on the host: loss within 1e-5
    relative, gradient within 1e-4 of its largest entry; repeat calls
    bit-identical."""
    sb = _sb()
    from paper_2503_01199_b200.metrics import _chw, _ssim_terms
    g = torch.Generator(device="cuda").manual_seed(W * 1000 + H)
    x = torch.rand((H, W, 3), device="cuda", generator=g)
    y = torch.rand((H, W, 3), device="cuda", generator=g)
    loss, grad = sb.loss_and_grad(x, y, 0.2)
    xd, yd = x.double().cpu(), y.double().cpu()
    vals, gs = _ssim_terms(_chw(xd), _chw(yd), True)
    l_ref = 0.8 * (xd - yd).abs().mean().item() + 0.2 * (1.0 - vals.mean().item())
    g_ref = torch.sign(xd - yd) * (0.8 / xd.numel()) - 0.2 * (gs[:, 0].permute(1, 2, 0) / 3)
    assert abs(loss - l_ref) <= 1e-5 * abs(l_ref)
    assert (grad.double().cpu() - g_ref).abs().max().item() <= 1e-4 * g_ref.abs().max().item()
    loss_b, grad_b = sb.loss_and_grad(x, y, 0.2)
    assert loss_b == loss and torch.equal(grad_b, grad)
    # the same kernel's sum of squared errors (train()'s per-view PSNR)
    sse = torch.full((1,), -1.0, dtype=torch.float64, device="cuda")
    sb.loss_and_grad(x, y, 0.2, sse_out=sse)
    ref = ((xd - yd) ** 2).sum().item()
    assert abs(sse.item() - ref) <= 1e-8 * ref   # float32 per-thread partials (4 terms)
    mse = ref / xd.numel()
    assert abs(10 * np.log10(1 / (sse.item() / xd.numel())) - sb.psnr(x, y)) <= 1e-8 * abs(10 * np.log10(1 / mse))


def test_fused_loss_nonfinite_and_wide_range():
    """metrics.py:118-132 in float64: a NaN in the target makes the loss NaN
    and an inf makes it non-finite (the divergence guard, train.py:100);
    0-255-valued float images (far outside [0, 1]) give the float64 loss."""
    sb = _sb()
    from paper_2503_01199_b200.metrics import _chw, _ssim_terms
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.rand((1080, 1920, 3), device="cuda", generator=g)
    y = torch.rand((1080, 1920, 3), device="cuda", generator=g)
    for bad, check in ((float("nan"), np.isnan), (float("inf"), lambda v: not np.isfinite(v))):
        yb = y.clone()
        yb[7, 11, 1] = bad
        loss, grad = sb.loss_and_grad(x, yb, 0.2)
        assert check(loss), (bad, loss)
        loss1, _ = sb.loss_and_grad(x, yb, 0.0)
        assert check(loss1), (bad, loss1)
        l_ok, _ = sb.loss_and_grad(x, y, 0.2)     # the workspace is clean again
        assert np.isfinite(l_ok)
    xs, ys = x * 255.0, y * 255.0
    loss, _ = sb.loss_and_grad(xs, ys, 0.2)
    xd, yd = xs.double().cpu(), ys.double().cpu()
    vals, _ = _ssim_terms(_chw(xd), _chw(yd), False)
    l_ref = 0.8 * (xd - yd).abs().mean().item() + 0.2 * (1.0 - vals.mean().item())
    assert abs(loss - l_ref) <= 1e-5 * abs(l_ref)


def test_train_epoch_psnr_from_loss_kernel():
    """train()'s per-view PSNR comes from the loss kernel's squared-error sum
    (no host sync per view): with zero learning rates the epoch row equals
    metrics.psnr / loss_and_grad of the rendered image (train.py:107-121)."""
    sb = _sb()
    d = G.load("golden_A.npz")
    sc = G.scene(d)
    scene = sb.SceneSoA(*[sc[k] for k in G.CH], device="cuda")
    sb.morton_sort(scene)
    cam = sb.CameraView.from_any(G.camera(d))
    W, H = cam.resolution
    target = np.random.default_rng(4).uniform(0.0, 1.0, (H, W, 3))
    out, _ = sb.forward(scene, cam)
    ref_psnr = sb.psnr(out.color, torch.from_numpy(target).float().cuda())
    ref_loss, _ = sb.loss_and_grad(out.color, torch.from_numpy(target).float().cuda(), 0.2)
    lrs = sb.LearningRates(position=1e-30, position_final=1e-30, log_scale=0.0, rotation=0.0, color=0.0,
                           opacity_logit=0.0)
    r = sb.train(sb.TrainConfig(epochs=1, lrs=lrs), scene, [(cam, target)])
    row = r.metrics[0]
    assert abs(row.psnr - ref_psnr) <= 1e-8 * abs(ref_psnr)
    assert row.loss == ref_loss


def test_train_divergence_guard():
    """test_train.py:96-104: a NaN in the target raises TrainingDiverged in
    epoch 1."""
    sb = _sb()
    d = G.load("golden_A.npz")
    sc = G.scene(d)
    scene = sb.SceneSoA(*[sc[k] for k in G.CH], device="cuda")
    cam = sb.CameraView.from_any(G.camera(d))
    W, H = cam.resolution
    bad = np.zeros((H, W, 3))
    bad[0, 0, 0] = np.nan
    with pytest.raises(sb.TrainingDiverged) as e:
        sb.train(sb.TrainConfig(epochs=1), scene, [(cam, bad)])
    assert e.value.epoch == 1


@pytest.mark.parametrize("fname,prefix", [("golden_A.npz", ""), ("golden_edge.npz", "e1_")])
def test_fused_loss_vs_reference(fname, prefix):
    """metrics.py:118-132: the fused kernel against the reference's float64
    loss / gradient (fixture) and the torch restatement."""
    sb = _sb()
    from paper_2503_01199_b200.metrics import loss_and_grad_torch
    d = G.load(fname)
    col = d[f"{prefix}fwd_color"]
    rng = np.random.default_rng(int(d[f"{prefix}target_seed"]))
    target = rng.uniform(0.0, 1.0, col.shape)
    x = torch.from_numpy(col).cuda()
    y = torch.from_numpy(target).cuda()
    loss, g = sb.loss_and_grad(x, y, 0.2)
    assert abs(loss - float(d[f"{prefix}loss"])) <= 1e-5 * abs(float(d[f"{prefix}loss"]))
    ref = d[f"{prefix}dL_dI"].astype(np.float64)
    assert np.abs(g.cpu().numpy() - ref).max() <= 1e-4 * np.abs(ref).max()
    l2, g2 = loss_and_grad_torch(x, y, 0.2)
    assert abs(loss - l2) <= 1e-5 * abs(l2)
    # uint8 targets (value / 255)
    t8 = (target * 255).round().astype(np.uint8)
    l8, g8 = sb.loss_and_grad(x, torch.from_numpy(t8).cuda(), 0.2)
    l8r, g8r = O.loss_and_grad(col, t8.astype(np.float64) / 255.0, 0.2)
    assert abs(l8 - l8r) <= 1e-5 * abs(l8r)
    assert np.abs(g8.cpu().numpy() - g8r).max() <= 1e-4 * np.abs(g8r).max()
    # loss written straight into mapped pinned host memory (no D2H copy)
    host = torch.full((3,), -1.0, dtype=torch.float64, pin_memory=True)
    lt, g9 = sb.loss_and_grad(x, torch.from_numpy(t8).cuda(), 0.2, return_tensor=True, loss_out=host[1:2])
    torch.cuda.synchronize()
    assert float(host[1]) == l8 and float(lt) == l8 and host[0] == -1.0 and host[2] == -1.0
    assert torch.equal(g9, g8)


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_half_path_vs_reference(fname, prefix):
    """forward.py:194-230 (half=True): fp16 blending state vs the reference's
    own half path, and >= 58 dB against its fp32 image."""
    sb = _sb()
    d = G.load(fname)
    scene, cam, cfg = _scene(d, prefix), G.camera(d, prefix), _cfg(d, prefix)
    out, ctx = sb.forward(scene, cam, cfg, half=True)
    col = out.color.cpu().numpy()
    assert np.abs(col - d[f"{prefix}fwdh_color"]).max() <= 2e-3
    assert np.abs(out.transmittance.cpu().numpy() - d[f"{prefix}fwdh_T"]).max() <= 2e-3
    fr = out.frag_count.cpu().numpy()
    assert (fr != d[f"{prefix}fwdh_frags"]).sum() <= 0.002 * fr.size + 2
    mse = ((col.astype(np.float64) - d[f"{prefix}fwd_color"]) ** 2).mean()
    assert mse == 0 or 10 * np.log10(1 / mse) >= 58.0
    # the backward replays in float32 whatever the forward precision: with
    # the fixed-order reduction the half and fp32 contexts give bit-identical
    # gradients (the float-atomic reduction differs by summation order only)
    import dataclasses
    dcfg = dataclasses.replace(cfg, deterministic=True)
    _, ctx_h = sb.forward(scene, cam, dcfg, half=True)
    res_h = sb.backward(scene, ctx_h, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n))
    _, ctx32 = sb.forward(scene, cam, dcfg)
    res_f = sb.backward(scene, ctx32, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n))
    assert torch.equal(res_h.grads.packed, res_f.grads.packed)


@pytest.mark.parametrize("fname,prefix", G.CASES)
def test_bf16_state_variant(fname, prefix):
    """bfloat16 blending state (unpinned by the
    reference, which only has the fp16 path): PSNR against the fp32 image
    and a float32 backward replay identical to the fp32 forward's."""
    sb = _sb()
    d = G.load(fname)
    scene, cam, cfg = _scene(d, prefix), G.camera(d, prefix), _cfg(d, prefix)
    out, ctx = sb.forward(scene, cam, cfg, half="bf16")
    col = out.color.cpu().numpy().astype(np.float64)
    mse = ((col - d[f"{prefix}fwd_color"]) ** 2).mean()
    db = 99.0 if mse == 0 else 10 * np.log10(1 / mse)
    print(f"bf16 state PSNR vs fp32: {db:.1f} dB")
    assert db >= 42.0   # measured 46.4-51.4 dB on the fixtures
    # the backward replays in float32 from the recovered fp32 T_final / last:
    # with the fixed-order (deterministic) reduction the two are bit-identical
    # (the float-atomic one differs by summation order, which e4's near-plane
    # rows amplify -- tools/e4_probe.py)
    import dataclasses
    dcfg = dataclasses.replace(cfg, deterministic=True)
    _, ctx_b = sb.forward(scene, cam, dcfg, half="bf16")
    res_b = sb.backward(scene, ctx_b, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n))
    _, ctx32 = sb.forward(scene, cam, dcfg)
    res_f = sb.backward(scene, ctx32, torch.from_numpy(d[f"{prefix}dL_dI"]), sb.DensifyStats.zeros(scene.n))
    assert torch.equal(res_b.grads.packed, res_f.grads.packed)
    with pytest.raises(ValueError):
        sb.forward(scene, cam, cfg, half="fp8")


def test_densify_hooks_vs_reference():
    """densify.py:57-187: variance score -> top-k selection (score desc, index
    asc) -> clone / split -> prune -> stats reset -> Morton re-sort."""
    sb = _sb()
    from paper_2503_01199_b200.densify import select_and_grow
    d = G.load("golden_edge.npz")
    scene = sb.SceneSoA(*[d[f"dens_in_{c}"] for c in G.CH], device="cuda")
    stats = sb.DensifyStats(S=torch.from_numpy(d["dens_S"]).cuda(), M=torch.from_numpy(d["dens_M"]).cuda(),
                            C=torch.from_numpy(d["dens_C"].astype(np.int32)).cuda())
    stats.attach(scene)
    cfg = sb.DensifyConfig(start_epoch=1, densify_interval_epochs=1, budget=2600)
    thr = cfg.resolve_split_threshold(scene)
    assert abs(thr - float(d["dens_thr"])) <= 1e-7 * float(d["dens_thr"])
    ci, si = select_and_grow(scene, sb.variance_score(stats), cfg.budget, thr)
    assert np.array_equal(ci.cpu().numpy(), d["dens_clone"])
    assert np.array_equal(si.cpu().numpy(), d["dens_split"])
    assert sb.densify_step(scene, stats, cfg, epoch=0) is None            # off schedule
    row = sb.densify_step(scene, stats, cfg, epoch=1)
    assert [row.n_before, row.n_after, row.n_split, row.n_clone, row.n_pruned] == d["dens_row"].tolist()
    st = sb.DensifyStats.from_scene(scene)     # restructuring replaced the attached arrays
    assert len(st.S) == scene.n and float(st.S.abs().sum()) == 0.0 and int(st.C.abs().sum()) == 0
    # same multiset of primitives (the reference keeps float64, the device
    # float32, so Morton order can differ where a coordinate straddles a cell)
    got = scene.data[:, :14].double().cpu().numpy()
    ref = np.concatenate([d[f"dens_out_{c}"].reshape(len(d["dens_out_position"]), -1) for c in G.CH], axis=1)
    key = lambda a: a[np.lexsort(np.round(a[:, ::-1], 4).T)]  # noqa: E731
    np.testing.assert_allclose(key(got), key(ref), rtol=2e-6, atol=2e-6)


def test_short_training_run_reduces_loss():
    """train.py:61-136 through the device path: loss falls on a small fit."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, random_scene_arrays
    spec = SyntheticSceneSpec(n_gaussians=600, n_views=4, view_resolution=(64, 64), seed=2)
    gt = random_scene_arrays(spec)
    cams = camera_ring(spec)
    gt_scene = sb.SceneSoA(*[gt[k] for k in G.CH], device="cuda")
    views = [(c, sb.render(gt_scene, c).color.clone()) for c in cams]
    init = {k: v.copy() for k, v in gt.items()}
    init["color"] = np.zeros_like(init["color"])
    init["position"] = init["position"] + np.random.default_rng(0).normal(0, 0.02, init["position"].shape)
    scene = sb.SceneSoA(*[init[k] for k in G.CH], device="cuda")
    res = sb.train(sb.TrainConfig(epochs=12, lrs=sb.LearningRates(color=2e-2)), scene, views)
    assert res.metrics[-1].loss < 0.6 * res.metrics[0].loss
    assert res.metrics[-1].psnr > res.metrics[0].psnr


def test_input_validation():
    """Raw device pointers are only handed to the kernels after dtype / shape
    / device checks (the reference raises on the same mismatches)."""
    sb = _sb()
    d = G.load("golden_A.npz")
    scene, cam = _scene(d), G.camera(d)
    n = scene.n
    out, ctx = sb.forward(scene, cam)
    dI = torch.zeros(128, 128, 3)
    bad_stats = [
        sb.DensifyStats(S=torch.zeros(n, dtype=torch.float32, device="cuda"),
                        M=torch.zeros(n, dtype=torch.float64, device="cuda"),
                        C=torch.zeros(n, dtype=torch.int32, device="cuda")),
        sb.DensifyStats(S=torch.zeros(n, dtype=torch.float64, device="cuda"),
                        M=torch.zeros(n, dtype=torch.float64, device="cuda"),
                        C=torch.zeros(n, dtype=torch.int64, device="cuda")),
    ]
    for st in bad_stats:
        with pytest.raises(ValueError):
            sb.backward(scene, ctx, dI, st)
    with pytest.raises(sb.ShapeMismatchError):
        sb.backward(scene, ctx, dI, sb.DensifyStats.zeros(n - 1))
    res = sb.backward(scene, ctx, dI, sb.DensifyStats.zeros(n))
    state = sb.AdamState(scene)
    lrs = sb.LearningRates().at(0.0)
    with pytest.raises(sb.ShapeMismatchError):
        sb.adam_step(scene, res.grads, state, res.cluster_mask[:-1], lrs)
    with pytest.raises(sb.ShapeMismatchError):
        sb.adam_step(scene, sb.SceneGrads(res.grads.packed[:-1]), state, res.cluster_mask, lrs)
    with pytest.raises(ValueError):
        sb.variance_score(sb.DensifyStats(S=torch.zeros(n, device="cuda"), M=torch.zeros(n, device="cuda"),
                                          C=torch.zeros(n, dtype=torch.int32, device="cuda")))
    perm = torch.arange(n, device="cuda")
    perm[3] = n
    with pytest.raises(IndexError):
        scene.copy().permute(perm)
    with pytest.raises(sb.ShapeMismatchError):
        scene.copy().permute(perm[:-1])


def test_second_device_or_noncurrent_stream():
    """Launch facts are per device: a scene on the last visible device renders
    the same image as on device 0 while device 0 stays current."""
    sb = _sb()
    if torch.cuda.device_count() < 2:
        pytest.skip("one visible device")
    d = G.load("golden_A.npz")
    dev = torch.device("cuda", torch.cuda.device_count() - 1)
    sc = G.scene(d)
    a, _ = sb.forward(sb.SceneSoA(*[sc[k] for k in G.CH], device="cuda:0"), G.camera(d))
    b, _ = sb.forward(sb.SceneSoA(*[sc[k] for k in G.CH], device=dev), G.camera(d))
    assert torch.equal(a.color, b.color.to(a.color.device))


def test_single_fragment_primitives_score_zero():
    """Primitives with exactly one contributing fragment get S == M^2, so a
    variance score of exactly 0 (never densified), as in the reference; and
    the candidate set (score > 0) from DEVICE statistics matches the
    reference's own statistics."""
    sb = _sb()
    from paper_2503_01199_b200.densify import select_and_grow
    d = G.load("golden_A.npz")
    scene, cam = _scene(d), G.camera(d)
    out, ctx = sb.forward(scene, cam)
    stats = sb.DensifyStats.zeros(scene.n)
    sb.backward(scene, ctx, torch.from_numpy(d["dL_dI"]), stats)
    C = stats.C.cpu().numpy()
    score = sb.variance_score(stats).cpu().numpy()
    one = C == 1
    assert one.any() and (score[one] == 0).all()
    ref = d["score"]
    assert ((score > 0) != (ref > 0)).sum() <= 2
    # a budget large enough to take every candidate: the same selection
    ci, si = select_and_grow(scene, sb.variance_score(stats), 10 * scene.n, 1e9)
    sel = np.sort(np.concatenate([ci.cpu().numpy(), si.cpu().numpy()]))
    assert np.array_equal(sel, np.flatnonzero(score > 0))


@pytest.mark.parametrize("fname,prefix", [("golden_A.npz", ""), ("golden_edge.npz", "e4_")])
def test_deterministic_backward(fname, prefix):
    """RasterConfig(deterministic=True): no float atomics -- per-(primitive,
    tile) rows summed per primitive in tile order (the reference's np.add.at
    order).  Two runs are bit-identical; parity with the reference holds;
    the fast (atomic) mode agrees to float-summation order."""
    sb = _sb()
    import dataclasses
    d = G.load(fname)
    scene, cam = _scene(d, prefix), G.camera(d, prefix)
    cfg = dataclasses.replace(_cfg(d, prefix), deterministic=True)
    dI = torch.from_numpy(d[f"{prefix}dL_dI"])
    runs = []
    for _ in range(2):
        out, ctx = sb.forward(scene, cam, cfg)
        st = sb.DensifyStats.zeros(scene.n)
        res = sb.backward(scene, ctx, dI, st)
        runs.append((res.grads.packed.clone(), st.S.clone(), st.M.clone(), st.C.clone()))
    for a, b in zip(*runs):
        assert torch.equal(a, b)
    g = runs[0][0][:, :14].double().cpu().numpy()
    g32 = d[f"{prefix}grads"].astype(np.float64)
    g64 = d.get(f"{prefix}grads64")
    for lo, hi in CH_SLICES:
        if g64 is None:
            assert G.floored_rel(g[:, lo:hi], g32[:, lo:hi]) <= 1e-2, (lo, hi)
        else:
            assert G.conditioned_rel_excess(g[:, lo:hi], g32[:, lo:hi], g64[:, lo:hi].astype(np.float64),
                                            1e-2) <= 1.0, (lo, hi)
    assert (runs[0][3].cpu().numpy() != d[f"{prefix}stat_C"]).sum() <= 2
    assert G.floored_rel(runs[0][1].cpu().numpy(), d[f"{prefix}stat_S"]) <= 1e-2
    out, ctx = sb.forward(scene, cam, _cfg(d, prefix))
    fast = sb.backward(scene, ctx, dI, sb.DensifyStats.zeros(scene.n))
    # (float summation order only; e4's near-plane rows amplify it through the chain)
    assert G.floored_rel(fast.grads.packed.double().cpu().numpy(), runs[0][0].double().cpu().numpy()) <= 2e-3
    # the loss is reduced in a fixed order too
    t = torch.rand(cam.resolution[1], cam.resolution[0], 3, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    l1, g1 = sb.loss_and_grad(out.color, t, 0.2)
    l2, g2 = sb.loss_and_grad(out.color, t, 0.2)
    assert l1 == l2 and torch.equal(g1, g2)


def test_deterministic_backward_config_b():
    """The deterministic backward at the benchmarked size (config B: 1M
    Gaussians, 1080p, 16,200 tiles -- several rounds of the tile scan, 13.7M
    tile-list positions): two runs bit-identical in gradients and S / M / C,
    C equal to the fast path's integer counts, gradients within float-atomic
    order noise of the fast path."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays
    n, res = 1_000_000, (1920, 1080)
    arr = scaled_scene_arrays(n, 7, res)
    scene = sb.SceneSoA(*[arr[k] for k in G.CH], device="cuda")
    sb.morton_sort(scene)
    cam = camera_ring(SyntheticSceneSpec(n_gaussians=n, n_views=1, view_resolution=res, seed=7))[0]
    g = torch.Generator(device="cuda").manual_seed(3)
    target = torch.rand((res[1], res[0], 3), device="cuda", generator=g)
    runs = {}
    for name, det in (("d1", True), ("d2", True), ("fast", False)):
        out, ctx = sb.forward(scene, cam, sb.RasterConfig(deterministic=det))
        _, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
        st = sb.DensifyStats.zeros(scene.n, scene.device)
        r = sb.backward(scene, ctx, dI, st)
        runs[name] = (r.grads.packed.clone(), st.S.clone(), st.M.clone(), st.C.clone())
    assert ctx.camera.tiles[0] * ctx.camera.tiles[1] > 8 * 1024
    assert all(torch.equal(a, b) for a, b in zip(runs["d1"], runs["d2"]))
    assert torch.equal(runs["d1"][3], runs["fast"][3])
    gd, gf = runs["d1"][0], runs["fast"][0]
    assert ((gd - gf).abs().max() / gf.abs().max()).item() <= 1e-5


def test_deterministic_training_checkpoints(tmp_path):
    """The reference's acceptance criterion 12 (test_acceptance.py:397-418)
    through the device path: two seeded deterministic train() runs with
    densification give byte-identical checkpoints and CSVs."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, random_scene_arrays
    spec = SyntheticSceneSpec(n_gaussians=300, n_views=3, view_resolution=(48, 48), seed=8)
    gt = random_scene_arrays(spec)
    cams = camera_ring(spec)
    views = [(c, O.forward(gt, c, O.RasterConfig(dtype="float64"))[0]) for c in cams]
    init = random_scene_arrays(SyntheticSceneSpec(n_gaussians=200, n_views=1, view_resolution=(48, 48), seed=44))
    dirs = []
    for run in range(2):
        scene = sb.SceneSoA(*[init[k] for k in G.CH], device="cuda")
        cfg = sb.TrainConfig(epochs=12, lrs=sb.LearningRates(position=3.2e-3, position_final=3.2e-5, log_scale=0.1,
                                                              rotation=0.02, color=0.05, opacity_logit=0.1),
                             seed=9, deterministic=True,
                             densify=sb.DensifyConfig(start_epoch=2, densify_interval_epochs=3, budget=260))
        result = sb.train(cfg, scene, views)
        assert len(result.densify_log) > 0
        dd = tmp_path / f"run{run}"
        sb.checkpoint(result, dd, manifest_text="seed = 9\n")
        dirs.append(dd)
    names = sorted(p.name for p in dirs[0].iterdir())
    assert "scene.ply" in names and "metrics.csv" in names
    for fname in names:
        assert (dirs[0] / fname).read_bytes() == (dirs[1] / fname).read_bytes(), fname


def test_native_densify_surgery_vs_oracle():
    """sb_densify_select / sb_densify_apply (densify.py:66-157 as kernels)
    against the oracle's restatement: the same clone / split lists, the same
    surviving rows in the same order (children to float32 rounding), extras
    moved with their rows and zero for new rows."""
    sb = _sb()
    from paper_2503_01199_b200 import densify as D
    rng = np.random.default_rng(5)
    n = 20000
    rows = np.zeros((n, 16), np.float32)
    rows[:, 0:3] = rng.normal(0, 2, (n, 3))
    rows[:, 3:6] = rng.normal(-2.5, 0.8, (n, 3))
    rows[:, 6:10] = rng.normal(0, 1, (n, 4))
    rows[:, 10:13] = rng.normal(0, 1, (n, 3))
    rows[:, 13] = rng.normal(-2, 2.5, n)
    scores = np.maximum(rng.normal(0, 1, n), 0.0)
    scores[rng.integers(0, n, 300)] = 0.75          # ties broken by index
    extras = {"m": rng.normal(0, 1, (n, 16)).astype(np.float32), "step": rng.integers(0, 9, n).astype(np.int32),
              "S": rng.normal(0, 1, n), "flag8": rng.integers(0, 2, (n, 3)).astype(np.uint8)}
    scene = sb.SceneSoA.from_rows(torch.from_numpy(rows).cuda())
    for k, v in extras.items():
        scene.register_extra(k, torch.from_numpy(v).cuda())
    budget, thr, prune_thr = n + 4000, float(np.exp(-2.0)), 0.01
    ci, si = D.select_and_grow(scene, torch.from_numpy(scores).cuda(), budget, thr)
    oc, os_ = O.select_and_grow(rows, scores, budget, thr)
    assert np.array_equal(ci.cpu().numpy(), oc) and np.array_equal(si.cpu().numpy(), os_)
    assert len(oc) > 100 and len(os_) > 100
    flags, c32, s32 = D._select(scene, torch.from_numpy(scores).cuda(), budget, thr)
    m = D._apply(scene, flags, c32, s32, prune_thr)
    orow, oex = O.apply_growth_and_prune(rows, extras, oc, os_, prune_thr)
    assert m == len(orow) == scene.n
    got = scene.data.cpu().numpy()
    # copies and clones bit-exact; children to float32 rounding of float64 math
    np.testing.assert_allclose(got, orow, rtol=1e-6, atol=1e-6)
    nkeep_orig = int(((1 / (1 + np.exp(-rows[:, 13].astype(np.float64)))) >= prune_thr)[
        np.setdiff1d(np.arange(n), os_)].sum())
    assert np.array_equal(got[:nkeep_orig], orow[:nkeep_orig])
    for k, v in oex.items():
        assert np.array_equal(scene.extras[k].cpu().numpy(), v), k
    # prune alone (no growth) and the growth API without prune
    sc2 = sb.SceneSoA.from_rows(torch.from_numpy(rows).cuda())
    npr = D.prune(sc2, 0.2)
    r2, _ = O.apply_growth_and_prune(rows, {}, [], [], 0.2)
    assert sc2.n == len(r2) and npr == n - len(r2) and np.array_equal(sc2.data.cpu().numpy(), r2)
    sc3 = sb.SceneSoA.from_rows(torch.from_numpy(rows).cuda())
    D.apply_growth(sc3, torch.from_numpy(oc), torch.from_numpy(os_))
    r3, _ = O.apply_growth_and_prune(rows, {}, oc, os_, -np.inf)
    assert sc3.n == len(r3)
    np.testing.assert_allclose(sc3.data.cpu().numpy(), r3, rtol=1e-6, atol=1e-6)


def test_multiview_step_streams_bit_identical():
    """multiview_step on two (and three) streams == on one stream, bit for
    bit (fixed-order backward): per-stream workspaces, the chains serialised
    in view order, masks OR-ed after the join; parameters, moments, step
    counters and statistics after two steps of 5 views."""
    sb = _sb()
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, random_scene_arrays
    spec = SyntheticSceneSpec(n_gaussians=20000, n_views=5, view_resolution=(160, 120), seed=11)
    arrays = random_scene_arrays(spec)
    cams = camera_ring(spec)
    rng = np.random.default_rng(3)
    views = [(c, torch.from_numpy(rng.uniform(0, 1, (120, 160, 3))).float().cuda()) for c in cams]
    raster = sb.RasterConfig(deterministic=True)
    lrs = sb.LearningRates().at(0.0, position_scale=1.0)
    runs = {}
    for k in (1, 2, 3):
        scene = sb.SceneSoA(*[arrays[c] for c in G.CH], device="cuda")
        sb.morton_sort(scene)
        state = sb.AdamState(scene)
        stats = sb.DensifyStats.zeros(scene.n)
        losses = []
        for _ in range(2):
            losses.append(sb.multiview_step(scene, state, views, lrs, raster=raster, stats=stats, streams=k))
        torch.cuda.synchronize()
        runs[k] = (scene.data.clone(), state.m_rows.clone(), state.v_rows.clone(), state.step.clone(),
                   stats.S.clone(), stats.M.clone(), stats.C.clone(), losses)
    for k in (2, 3):
        for x, y in zip(runs[1][:7], runs[k][:7]):
            assert torch.equal(x, y), k
        assert runs[1][7] == runs[k][7]
    assert not torch.equal(runs[1][0], sb.SceneSoA(*[arrays[c] for c in G.CH], device="cuda").data)


def _ref_make_camera(sb, resolution=(32, 32), eye=(0.6, 0.4, -2.5), target=(0, 0, 0), focal=40.0, near=0.1,
                     far=50.0):
    """The reference suite's camera helper (pkg/tests/conftest.py:8-17)."""
    W, H = resolution
    return sb.CameraView(sb.look_at(eye, target), (focal, focal), ((W - 1) / 2.0, (H - 1) / 2.0), resolution, near,
                         far)


def _ref_make_scene(sb, n, rng, extent=0.3, scale_range=(0.08, 0.2), opacity_range=(-0.5, 1.0)):
    """The reference suite's random scene (pkg/tests/conftest.py:20-29)."""
    return sb.SceneSoA(rng.uniform(-extent, extent, (n, 3)), np.log(rng.uniform(*scale_range, (n, 3))),
                       rng.normal(size=(n, 4)), rng.uniform(-1.0, 1.0, (n, 3)), rng.uniform(*opacity_range, n),
                       device="cuda")


def test_criteria_06_07_culling_and_resort_invisible():
    """The reference's acceptance criterion 6 (test_acceptance.py:257-272):
    20 random scene / camera pairs (generated as the reference does), cluster
    culling on vs off give identical colour, transmittance and fragment
    counts; and criterion 7's invariance (test_acceptance.py:296-300): a
    Morton re-sort never changes the render."""
    sb = _sb()
    culled_any = False
    for trial in range(20):
        rng = np.random.default_rng(trial + 400)
        scene = _ref_make_scene(sb, int(rng.integers(100, 400)), rng, extent=2.5)
        sb.morton_sort(scene)
        eye = (float(rng.uniform(-2, 2)), float(rng.uniform(-1, 1)), float(rng.uniform(-5, -2.5)))
        cam = _ref_make_camera(sb, (64, 48), eye=eye, target=tuple(rng.uniform(-0.3, 0.3, 3)))
        on, ctx = sb.forward(scene, cam, sb.RasterConfig(use_culling=True))
        off, _ = sb.forward(scene, cam, sb.RasterConfig(use_culling=False))
        culled_any |= ctx.culled_clusters > 0
        assert torch.equal(on.color, off.color), trial
        assert torch.equal(on.transmittance, off.transmittance), trial
        assert torch.equal(on.frag_count, off.frag_count), trial
    scene = _ref_make_scene(sb, 60, np.random.default_rng(5))
    cam = _ref_make_camera(sb, (48, 48))
    before, _ = sb.forward(scene, cam)
    before = before.color.clone()
    sb.morton_sort(scene)
    after, _ = sb.forward(scene, cam)
    assert torch.equal(before, after.color)


def test_criterion_05_exp_aligned_reduce_device():
    """The reference's acceptance criterion 5 (test_acceptance.py:234-254) on
    the device reduction the backward uses: 10^5 random 32-sets in
    [2^-10, 2^10] within 32 * 2^(e_max - 23) of the exact sum (the device
    rounds the exact integer sum once to float32, inside that bound); an
    all-equal set and one-hot sets exact."""
    sb = _sb()
    rng = np.random.default_rng(13)
    n = 100_000
    v = (2.0 ** rng.uniform(-10, 10, (n, 32)) * rng.choice([-1.0, 1.0], (n, 32))).astype(np.float32)
    got = sb.exp_aligned_reduce(torch.from_numpy(v)).double().cpu().numpy()
    v64 = v.astype(np.float64)
    exact = v64.sum(axis=1)
    e_max = np.floor(np.log2(np.abs(v64).max(axis=1)))
    bound = 32 * 2.0 ** (e_max - 23)
    assert np.all(np.abs(got - exact) <= bound)
    assert float(sb.exp_aligned_reduce(torch.ones(32))) == 32.0
    xs = (rng.normal(size=1000) * 2.0 ** rng.integers(-10, 11, 1000)).astype(np.float32)
    one = np.zeros((1000, 32), np.float32)
    one[np.arange(1000), rng.integers(0, 32, 1000)] = xs
    assert np.array_equal(sb.exp_aligned_reduce(torch.from_numpy(one)).cpu().numpy(), xs)
