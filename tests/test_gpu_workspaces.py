"""The launch chain keeps no memsets between kernels: the tile queues, the
projection look-back, the bin count arrays and the loss accumulator reset
themselves, the screen-gradient rows are zeroed by the forward's projection
and handed to exactly one backward.  These
tests drive the orders in which that state could leak between calls --
interleaved contexts, renders in between, resolution and scene-size
changes -- and require results identical to a fresh, isolated call.
"""
import numpy as np
import pytest
import torch

from tests import goldens as G

pytestmark = pytest.mark.gpu


def _sb():
    import paper_2503_01199_b200 as sb
    return sb


def _scene(d, prefix=""):
    sc = G.scene(d, prefix)
    return _sb().SceneSoA(*[sc[k] for k in G.CH], device="cuda")


def _grads(scene, ctx, dI):
    sb = _sb()
    res = sb.backward(scene, ctx, dI, sb.DensifyStats.zeros(scene.n))
    torch.cuda.synchronize()
    return res.grads.packed.cpu().numpy().copy()


def _second_camera(cam, w=96, h=72):
    """Same pose, another tile grid (its own bin state, same sgrad rows)."""
    sb = _sb()
    c = sb.CameraView.from_any(cam)
    W, H = c.resolution
    return sb.CameraView(c.world_to_camera, c.focal * (w / W), c.principal_point * (w / W), (w, h), c.near, c.far)


def _close(a, b):
    # atomics make the sums order-nondeterministic at the ulp level
    return np.allclose(a, b, rtol=1e-4, atol=1e-7 * max(1.0, float(np.abs(b).max())))


def test_interleaved_contexts_match_isolated_backward():
    """forward A, forward B, backward A, backward B: B's forward re-zeroes the
    shared screen-gradient rows after A's, so A's backward must zero them
    itself and B's must not reuse A's leftovers."""
    sb = _sb()
    d = G.load("golden_A.npz")
    scene = _scene(d)
    cams = [G.camera(d), _second_camera(G.camera(d))]
    dIs = [torch.from_numpy(d["dL_dI"]).cuda(), torch.rand(72, 96, 3, device="cuda") - 0.5]
    ref = []
    for cam, dI in zip(cams, dIs):        # isolated: forward + backward each
        _, ctx = sb.forward(scene, cam)
        ref.append(_grads(scene, ctx, dI))
    _, ca = sb.forward(scene, cams[0])
    _, cb = sb.forward(scene, cams[1])
    ga = _grads(scene, ca, dIs[0])
    gb = _grads(scene, cb, dIs[1])
    assert _close(ga, ref[0])
    assert _close(gb, ref[1])


def test_render_between_forward_and_backward():
    sb = _sb()
    d = G.load("golden_A.npz")
    scene, cam = _scene(d), G.camera(d)
    dI = torch.from_numpy(d["dL_dI"]).cuda()
    _, ctx = sb.forward(scene, cam)
    ref = _grads(scene, ctx, dI)
    _, ctx = sb.forward(scene, cam)
    img = sb.render(scene, cam)           # must not disturb ctx's backward state
    assert _close(_grads(scene, ctx, dI), ref)
    out, _ = sb.forward(scene, cam)
    assert torch.equal(img.color, out.color)


def test_repeated_calls_bit_identical_forward():
    """Self-resetting queues / counters: many back-to-back forwards give the
    same tile lists and image as the first."""
    sb = _sb()
    d = G.load("golden_A.npz")
    scene, cam = _scene(d), G.camera(d)
    out0, ctx0 = sb.forward(scene, cam)
    for _ in range(5):
        out, ctx = sb.forward(scene, cam)
        assert torch.equal(ctx.tile_offsets, ctx0.tile_offsets)
        assert torch.equal(ctx.tile_prims, ctx0.tile_prims)
        assert torch.equal(out.color, out0.color)
        assert (ctx.n_compact, ctx.n_pairs, ctx.visible_clusters) == (ctx0.n_compact, ctx0.n_pairs,
                                                                        ctx0.visible_clusters)
    _, l0 = sb.loss_and_grad(out0.color, torch.zeros_like(out0.color), 0.2)
    for _ in range(3):
        loss1, _ = sb.loss_and_grad(out0.color, torch.zeros_like(out0.color), 0.2)
        loss0, _ = sb.loss_and_grad(out0.color, torch.zeros_like(out0.color), 0.2)
        assert loss0 == loss1             # the accumulator is left zeroed


def test_resolution_and_scene_size_changes():
    """Alternating tile grids (per-grid bin state) and a growing scene (the
    projection workspace's look-back words move) reproduce isolated runs."""
    sb = _sb()
    d = G.load("golden_A.npz")
    scene = _scene(d)
    cam = G.camera(d)
    cams = [cam, _second_camera(cam)]
    first = [sb.forward(scene, c)[0].color.clone() for c in cams]
    for _ in range(2):
        for c, img in zip(cams, first):
            assert torch.equal(sb.forward(scene, c)[0].color, img)
    # grow the scene (append copies) and shrink it back
    n = scene.n
    raw = [getattr(scene, k).detach().cpu().numpy()[: n // 2] for k in G.CH]
    scene.append_raw(*raw)
    grown = sb.forward(scene, cam)[0].color.clone()
    assert torch.equal(sb.forward(scene, cam)[0].color, grown)
    scene.keep(torch.arange(scene.n, device=scene.device) < n)
    assert torch.equal(sb.forward(scene, cam)[0].color, first[0])
