"""The reference's cluster-index, projection and tile-blending API mirrors on
the device (ccc.py:97-194, projection.py:24-190,
forward.py:161-230, scene.py:46-126) against the reference's own outputs
(tests/golden) and the CPU oracle."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests import goldens as G

pytestmark = pytest.mark.gpu

FULL_CASES = [c for c in G.CASES]


def _sb():
    import paper_2503_01199_b200 as sb
    return sb


def _scene(d, prefix=""):
    sb = _sb()
    sc = G.scene(d, prefix)
    return sb.SceneSoA(*[sc[k] for k in G.CH], device="cuda")


def _ulps(a, b):
    a = np.ascontiguousarray(a, np.float64).view(np.int64)
    b = np.ascontiguousarray(b, np.float64).view(np.int64)
    return int(np.abs(a - b).max()) if a.size else 0


@pytest.mark.parametrize("fname,prefix", FULL_CASES)
def test_cluster_index_vs_reference(fname, prefix):
    """build_clusters AABBs, the pure cull mask and the widened visibility
    mask -- standalone calls and the forward kernel's optional outputs --
    against the reference's (golden aabb_min / aabb_max / cull_mask /
    vis_mask).  Masks bit-exact; AABBs to the float64 exp's last ulp."""
    sb = _sb()
    d = G.load(fname)
    if f"{prefix}aabb_min" not in d:
        pytest.skip("case without clusters")
    scene, cam = _scene(d, prefix), G.camera(d, prefix)
    idx = sb.build_clusters(scene)
    amin, amax = idx.aabb_min.cpu().numpy(), idx.aabb_max.cpu().numpy()
    ulp = max(_ulps(amin, d[f"{prefix}aabb_min"]), _ulps(amax, d[f"{prefix}aabb_max"]))
    print(f"{prefix or 'A'}: AABB max ulp difference {ulp} over {idx.n_clusters} clusters")
    assert ulp <= 2
    fr = sb.build_frustum(cam)
    assert isinstance(fr, sb.Frustum) and np.array_equal(fr.planes, d[f"{prefix}planes"])
    assert np.array_equal(sb.cull_clusters(idx, fr).cpu().numpy(), d[f"{prefix}cull_mask"])
    pr = sb.project_scene(scene, cam)
    vis = sb.cluster_visibility(idx, fr, pr.in_image).cpu().numpy()
    assert np.array_equal(vis, d[f"{prefix}vis_mask"])
    # the fused forward kernel's own AABB / cull outputs
    out, ctx = sb.forward(scene, cam)
    assert np.array_equal(ctx.cluster_cull.cpu().numpy().astype(bool), d[f"{prefix}cull_mask"])
    caabb = ctx.cluster_aabb.cpu().numpy()
    assert np.array_equal(caabb[:, :3], amin) and np.array_equal(caabb[:, 3:], amax)
    # the same from the reference's own AABBs (cull / visibility exactly)
    ref_idx = sb.ClusterIndex(cluster_size=128, aabb_min=torch.from_numpy(d[f"{prefix}aabb_min"]).cuda(),
                              aabb_max=torch.from_numpy(d[f"{prefix}aabb_max"]).cuda(), n=scene.n)
    assert np.array_equal(sb.cull_clusters(ref_idx, fr.planes).cpu().numpy(), d[f"{prefix}cull_mask"])
    # frustum helpers (projection.py:30-35)
    pts = d[f"{prefix}position"][:50].astype(np.float64)
    assert np.array_equal(fr.contains(pts), np.all(pts @ fr.planes[:, :3].T + fr.planes[:, 3] >= 0, axis=1))


@pytest.mark.parametrize("fname,prefix", FULL_CASES)
def test_project_scene_vs_reference(fname, prefix):
    """project_scene on the device: xy / depth / conic / radius / colour /
    opacity bit-exact on valid rows, valid / in_image exact (golden); the
    chain fields against the oracle's float32 projection."""
    sb = _sb()
    d = G.load(fname)
    scene, cam = _scene(d, prefix), G.camera(d, prefix)
    pr = sb.project_scene(scene, cam)
    valid = d[f"{prefix}proj_valid"]
    assert np.array_equal(pr.valid.cpu().numpy(), valid)
    assert np.array_equal(pr.in_image.cpu().numpy(), d[f"{prefix}proj_in_image"])
    for k in ("xy", "depth", "conic", "radius", "color", "opacity"):
        got = getattr(pr, k).contiguous().cpu().numpy()
        ref = d[f"{prefix}proj_{k}"]
        assert np.array_equal(got[valid].view(np.uint32), ref[valid].view(np.uint32)), k
    if scene.n:
        op = O.project(G.scene(d, prefix), cam)
        for k in ("t_cam", "M", "cov_screen", "cov_world", "scale", "unit_quat"):
            got = getattr(pr, k).cpu().numpy()
            ref = op[k].astype(np.float64)
            sel = valid if k in ("M", "cov_screen") else np.ones(len(valid), bool)
            # float64 restatement vs the float32 path: fp32 rounding noise only
            assert G.floored_rel(got[sel], ref[sel]) <= 1e-4, k
        assert pr.n_degenerate == op["n_degenerate"]
    with pytest.raises(ValueError):
        sb.project_scene(scene, cam, dtype=np.float64)


@pytest.mark.parametrize("fname,prefix", [("golden_A.npz", ""), ("golden_edge.npz", "e2_")])
def test_compact_arrays_vs_reference(fname, prefix):
    """compact_arrays: the visible clusters' rows and the compact map."""
    sb = _sb()
    d = G.load(fname)
    scene, cam = _scene(d, prefix), G.camera(d, prefix)
    n = scene.n
    vis = torch.from_numpy(d[f"{prefix}vis_mask"]).cuda() if f"{prefix}vis_mask" in d else \
        torch.ones((n + 127) // 128, dtype=torch.bool, device="cuda")
    pr = sb.project_scene(scene, cam)
    out, cmap = sb.compact_arrays({"xy": pr.xy, "radius": pr.radius}, vis, 128, n)
    assert np.array_equal(cmap.cpu().numpy(), d[f"{prefix}compact_map"])
    assert torch.equal(out["xy"], pr.xy[cmap]) and torch.equal(out["radius"], pr.radius[cmap])
    obj, cmap2 = sb.compact_arrays(pr, vis, 128, n)
    assert torch.equal(cmap, cmap2) and torch.equal(obj.depth, pr.depth[cmap])


@pytest.mark.parametrize("fname,prefix", [("golden_A.npz", ""), ("golden_edge.npz", "e1_")])
def test_blend_tile_vs_reference(fname, prefix):
    """blend_tile / half_path_blend (forward.py:161-230) through the device's
    warp kernel, tile by tile, against the reference's full-image fixtures
    (the image is the assembly of the tiles, forward.py:240-255)."""
    sb = _sb()
    d = G.load(fname)
    scene, cam = _scene(d, prefix), G.camera(d, prefix)
    bg = tuple(float(b) for b in d[f"{prefix}cfg_bg"])
    cfg = sb.RasterConfig(background=bg)
    out, ctx = sb.forward(scene, cam, cfg)
    proj = ctx.projected
    res = cam.resolution
    tiles = ctx.tiles
    assert tiles
    for tile in tiles[:: max(1, len(tiles) // 12)]:
        rgb, T, fr, valid = sb.blend_tile(tile, proj, cfg, res)
        x0, y0 = tile.origin
        for lane in range(32):
            for i in range(4):
                x, y = x0 + lane % 16, y0 + 4 * (lane // 16) + i
                if not bool(valid[lane, i]):
                    assert torch.equal(rgb[lane, i].cpu(), torch.tensor(bg, dtype=torch.float32))
                    continue
                assert np.abs(rgb[lane, i].cpu().numpy() - d[f"{prefix}fwd_color"][y, x]).max() <= 1e-3
                assert abs(float(T[lane, i]) - float(d[f"{prefix}fwd_T"][y, x])) <= 1e-3
        rgb_h, T_h, fr_h, _ = sb.half_path_blend(tile, proj, cfg, res)
        vv = valid.cpu().numpy()
        ys = (y0 + 4 * (np.arange(32) // 16))[:, None] + np.arange(4)[None, :]
        xs = (x0 + np.arange(32) % 16)[:, None].repeat(4, 1)
        ref_h = d[f"{prefix}fwdh_color"][ys[vv], xs[vv]]
        assert np.abs(rgb_h.cpu().numpy()[vv] - ref_h).max() <= 2e-3


def test_activate_and_compose_cov3d():
    """scene.py:46-126 restatements (float64, device) against numpy."""
    sb = _sb()
    rng = np.random.default_rng(3)
    n = 500
    pos, ls, q = rng.normal(size=(n, 3)), rng.normal(size=(n, 3)), rng.normal(size=(n, 4))
    col, op = rng.normal(size=(n, 3)) * 4, rng.normal(size=n) * 4
    p, s, u, c, o = sb.activate(*(torch.from_numpy(a).cuda() for a in (pos, ls, q, col, op)))
    np.testing.assert_allclose(s.cpu().numpy(), np.exp(ls), rtol=4e-16)   # CUDA vs numpy exp: <= 1 ulp
    np.testing.assert_allclose(u.cpu().numpy(), q / np.linalg.norm(q, axis=1, keepdims=True), rtol=1e-15)
    ref_sig = lambda x: np.where(x >= 0, 1 / (1 + np.exp(-np.abs(x))), np.exp(-np.abs(x)) / (1 + np.exp(-np.abs(x))))  # noqa
    np.testing.assert_allclose(c.cpu().numpy(), ref_sig(col), rtol=1e-15)
    np.testing.assert_allclose(o.cpu().numpy(), ref_sig(op), rtol=1e-15)
    with pytest.raises(sb.ValidationError):
        bad = q.copy()
        bad[7] = 0.0
        sb.activate(pos, ls, bad, col, op)
    cov = sb.compose_cov3d(s, u).cpu().numpy()
    R = sb.quat_to_rotmat(u).cpu().numpy()
    ref = np.einsum("nij,nj,nkj->nik", R, np.exp(ls) ** 2, R)
    np.testing.assert_allclose(cov, 0.5 * (ref + ref.transpose(0, 2, 1)), rtol=1e-12, atol=1e-15)
    ev = np.linalg.eigvalsh(cov)
    np.testing.assert_allclose(np.sort(ev, 1), np.sort(np.exp(ls) ** 2, 1), rtol=1e-9)
