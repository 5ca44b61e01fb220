"""View-parallel training through the device path: two ranks
(gloo, sharing the one GPU of the test box -- a functional check, never a
timing) run train() with a ViewParallel; every step sums the two ranks'
view gradients with one all-reduce and takes one identical Adam step, so the
ranks' parameters must stay bit-identical and the fit must progress."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import goldens as G

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, zero1=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2503_01199_b200 as sb
        from paper_2503_01199_b200.parallel import ViewParallel
        from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, random_scene_arrays
        spec = SyntheticSceneSpec(n_gaussians=600, n_views=5, view_resolution=(64, 64), seed=2)
        gt = random_scene_arrays(spec)
        cams = camera_ring(spec)
        gt_scene = sb.SceneSoA(*[gt[k] for k in G.CH], device="cuda")
        views = [(c, sb.render(gt_scene, c).color.clone()) for c in cams]
        init = {k: v.copy() for k, v in gt.items()}
        init["color"] = np.zeros_like(init["color"])
        scene = sb.SceneSoA(*[init[k] for k in G.CH], device="cuda")
        cfg = sb.TrainConfig(epochs=8, lrs=sb.LearningRates(color=2e-2),
                             densify=sb.DensifyConfig(start_epoch=2, densify_interval_epochs=3, budget=660))
        vp = ViewParallel(zero1=zero1)
        res = sb.train(cfg, scene, views, parallel=vp)
        st = sb.DensifyStats.from_scene(scene)     # rank-local since the last densify
        S = st.S.clone()
        vp.reduce_stats(S, st.M.clone(), st.C.clone())
        out[rank] = dict(data=scene.data.cpu().numpy(), S=S.cpu().numpy(), S_local=st.S.cpu().numpy(),
                         m=scene.extras["adam_m"].cpu().numpy(), step=scene.extras["adam_step"].cpu().numpy(),
                         losses=[m.loss for m in res.metrics], n=scene.n, log=len(res.densify_log))
    finally:
        dist.destroy_process_group()


def test_view_parallel_train_two_ranks():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True, start_method="spawn")
    a, b = out[0], out[1]
    assert a["n"] == b["n"] and a["n"] > 600          # densified identically (5 views: one idle rank per epoch)
    assert np.array_equal(a["data"], b["data"])        # one identical Adam step per rank per step
    assert np.array_equal(a["S"], b["S"]) and a["S"].any()
    assert not np.array_equal(a["S_local"], b["S_local"])   # reduced only when read
    assert a["losses"] == b["losses"]
    assert a["losses"][-1] < 0.7 * a["losses"][0]


def test_view_parallel_train_two_ranks_zero1():
    """ViewParallel(zero1=True): reduce-scatter + sharded Adam + all-gather
    gives the same parameters and (after the final sync) the same optimiser
    state as the all-reduce step."""
    world = 2
    res = {}
    for z in (False, True):
        mgr = mp.Manager()
        out = mgr.dict()
        mp.start_processes(_worker, args=(world, _free_port(), out, z), nprocs=world, join=True,
                           start_method="spawn")
        res[z] = (out[0], out[1])
    for r in range(2):
        assert np.array_equal(res[True][r]["data"], res[False][r]["data"])
        assert np.array_equal(res[True][r]["m"], res[False][r]["m"])
        assert np.array_equal(res[True][r]["step"], res[False][r]["step"])
    assert res[True][0]["losses"] == res[False][0]["losses"]


def _overlap_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2503_01199_b200 as sb
        from paper_2503_01199_b200.parallel import ViewParallel
        from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, random_scene_arrays
        spec = SyntheticSceneSpec(n_gaussians=3000, n_views=4, view_resolution=(96, 72), seed=4)
        arrays = random_scene_arrays(spec)
        cams = camera_ring(spec)
        cfg = sb.RasterConfig(deterministic=True)
        rng = np.random.default_rng(7)
        targets = [torch.from_numpy(rng.uniform(0, 1, (72, 96, 3))).float().cuda() for _ in cams]
        lrs = sb.LearningRates().at(0.0, position_scale=1.0)
        vp = ViewParallel()
        got = {}
        for mode in ("plain", "overlap"):
            scene = sb.SceneSoA(*[arrays[k] for k in G.CH], device="cuda")
            sb.morton_sort(scene)
            state = sb.AdamState(scene)
            stats = sb.DensifyStats.zeros(scene.n).attach(scene) or sb.DensifyStats.from_scene(scene)
            for step in range(3):
                v = (2 * step + rank) % len(cams)
                out_, ctx = sb.forward(scene, cams[v], cfg)
                _, dI = sb.loss_and_grad(out_.color, targets[v], 0.2, return_tensor=True)
                st = sb.DensifyStats.from_scene(scene)
                if mode == "plain":
                    res = sb.backward(scene, ctx, dI, st)
                    mask = vp.reduce_grads(res.grads.packed, res.cluster_mask)
                    sb.adam_step(scene, res.grads, state, mask, lrs)
                else:
                    vp.overlapped_step(scene, ctx, dI, state, lrs, st, chunks=3)
            torch.cuda.synchronize()
            got[mode] = (scene.data.cpu().numpy(), state.m_rows.cpu().numpy(), state.step.cpu().numpy())
        out[rank] = got
    finally:
        dist.destroy_process_group()


def test_overlapped_step_matches_plain_two_ranks():
    """ViewParallel.overlapped_step (chunked async all-reduce interleaved
    with the chain and Adam) == backward + reduce_grads + adam_step, bit for
    bit, on two ranks (fixed-order backward so runs are comparable), and the
    ranks stay identical."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_overlap_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    a, b = out[0], out[1]
    for x, y in zip(a["plain"], a["overlap"]):
        assert np.array_equal(x, y)
    for x, y in zip(a["overlap"], b["overlap"]):
        assert np.array_equal(x, y)
