"""world_size-2 gloo tests of the view-parallel exchange (CPU tensors):
sums of grads / S / M / C, OR of cluster masks, round-robin view shards."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2503_01199_b200.parallel import ViewParallel
        vp = ViewParallel()
        n, k = 300, 3
        g = torch.full((n, 16), float(rank + 1))
        S = torch.arange(n, dtype=torch.float64) * (rank + 1)
        M = -S.clone()
        C = torch.full((n,), rank + 2, dtype=torch.int32)
        mask = torch.tensor([rank == 0, rank == 1, False])
        m = vp.reduce(g, S, M, C, mask)
        # one-collective step: mask in the padding column, stats reduced lazily
        g2 = torch.zeros((n, 16))
        g2[:, :14] = float(rank + 1)
        m2 = vp.reduce_grads(g2, mask)
        S2 = torch.arange(n, dtype=torch.float64) * (rank + 1)
        M2 = -S2.clone()
        C2 = torch.full((n,), rank + 2, dtype=torch.int32)
        vp.reduce_stats(S2, M2, C2)
        out[rank] = dict(g=float(g[0, 0]), g_all=bool((g == 3.0).all()), S=float(S[10]), M=float(M[10]),
                         C=int(C[5]), mask=m.tolist(), views=[vp.views_for_step(s, 8) for s in range(4)],
                         g2_ok=bool((g2[:, :14] == 3.0).all()) and bool((g2[:, 14:] == 0).all()), mask2=m2.tolist(),
                         S2=float(S2[10]), M2=float(M2[10]), C2=int(C2[5]), C2_dtype=str(C2.dtype))
    finally:
        dist.destroy_process_group()


def test_view_parallel_reduce_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        o = out[r]
        assert o["g_all"] and o["g"] == 3.0
        assert o["S"] == 30.0 and o["M"] == -30.0
        assert o["C"] == 5
        assert o["mask"] == [True, True, False]
        assert o["g2_ok"] and o["mask2"] == [True, True, False]
        assert o["S2"] == 30.0 and o["M2"] == -30.0 and o["C2"] == 5 and o["C2_dtype"] == "torch.int32"
    # every view of an 8-view ring is rendered exactly once per 4 steps
    seen = sorted(v for r in range(world) for step in out[r]["views"] for v in step)
    assert seen == sorted(list(range(8)))


def test_single_process_is_identity():
    from paper_2503_01199_b200.parallel import ViewParallel
    vp = ViewParallel()
    g = torch.ones(4, 16)
    m = vp.reduce(g, torch.zeros(4, dtype=torch.float64), torch.zeros(4, dtype=torch.float64),
                  torch.zeros(4, dtype=torch.int32), torch.tensor([1], dtype=torch.uint8))
    assert m.tolist() == [True] and float(g.sum()) == 64.0


def _zero1_worker(rank, world, port, out):
    """ZeRO-1 step on CPU tensors with a torch stand-in for the device Adam:
    reduce-scatter of cluster-aligned shards (mask in the padding column),
    each rank updates only its rows, all-gather of the parameters, then a
    sync of the per-shard optimiser state."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import types
        import paper_2503_01199_b200.optim as optim
        from paper_2503_01199_b200.parallel import ViewParallel

        def fake_adam(scene, grads, state, mask, lrs, rows=None):
            r0, r1 = rows
            m = torch.repeat_interleave(mask, 128)[: r1 - r0]
            g = grads.packed if hasattr(grads, "packed") else grads
            upd = torch.where(m[:, None], -0.5 * torch.sign(g), torch.zeros_like(g))
            scene.data[r0:r1] += upd
            state.m_rows[r0:r1] += torch.where(m[:, None], g, torch.zeros_like(g))
            state.step[r0:r1] += m.to(torch.int32)
        optim.adam_step = fake_adam
        vp = ViewParallel(zero1=True)
        n = 700                                      # 6 clusters, shards of 3 clusters = 384 rows
        assert vp.shard_rows(n) == 384 and vp.padded_rows(n) == 768
        scene = types.SimpleNamespace(n=n, data=torch.zeros((n, 16)))
        state = types.SimpleNamespace(scene=scene, m_rows=torch.zeros((n, 16)), v_rows=torch.zeros((n, 16)),
                                      step=torch.zeros(n, dtype=torch.int32))
        gb = vp.grad_buffer(n, "cpu")
        gb[:n, :14] = float(rank + 1)
        mask = torch.zeros(6, dtype=torch.bool)
        mask[rank] = True                              # rank 0 sees cluster 0, rank 1 cluster 1
        mask[4] = True
        vp.zero1_step(scene, gb, mask, state, {})
        vp.sync_optimizer_state(state)
        out[rank] = dict(data=scene.data.clone(), m=state.m_rows.clone(), step=state.step.clone())
    finally:
        dist.destroy_process_group()


def test_zero1_shards_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_zero1_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    a, b = out[0], out[1]
    assert torch.equal(a["data"], b["data"]) and torch.equal(a["m"], b["m"]) and torch.equal(a["step"], b["step"])
    rows_upd = torch.zeros(700, dtype=torch.bool)
    for c in (0, 1, 4):                               # OR of the masks
        rows_upd[c * 128:(c + 1) * 128] = True
    assert torch.equal(a["step"], rows_upd.to(torch.int32))
    assert (a["data"][rows_upd, :14] == -0.5).all() and (a["data"][~rows_upd] == 0).all()
    assert (a["m"][rows_upd, :14] == 3.0).all()      # summed gradients (1 + 2)
    assert (a["data"][:, 14:] == 0).all()
