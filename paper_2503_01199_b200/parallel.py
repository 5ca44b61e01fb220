"""View-sharded data parallelism across GPUs.

The reference trains one view at a time (train.py:95-104) and has no
distributed code.  Views are independent given replicated
Gaussians, so each rank rasterises its own views; the only exchange per
optimiser step is a SUM of the per-view results:

  grads (N, 16) float32      ->  one float32 all-reduce
  S, M (float64), C (int32),
  cluster mask (K, uint8)    ->  one float64 all-reduce over [S | M | C | mask]
                                 (C and the mask are exact in float64; the
                                 mask is OR-ed as "sum > 0")

followed by one identical cluster-sparse Adam step on every rank.  Multi-view
semantics are SUM_v backward(scene, ctx_v, dI_v) plus summed statistics and
OR-ed masks, then a single adam_step -- the SURVEY 8(e) definition.
Works with any torch.distributed backend (NCCL over NVLink on the GPU box,
gloo for the CPU tests).

The training step uses the leaner pair reduce_grads / reduce_stats (or
overlapped_step, which splits the gradient exchange into cluster-aligned
row chunks so each chunk's all-reduce runs under the next chunk's chain and
the previous chunk's Adam):
  - per step ONE all-reduce of the (N, 16) float32 gradient rows, with the
    cluster mask riding in padding column 14 of each cluster's first row
    (the chain writes zeros there and Adam never reads columns 14-15);
  - the statistics stay rank-local, accumulated in place by every backward,
    and are summed over ranks only when they are read (before a densify
    step).  The sum is linear, so sum_ranks(sum_steps) equals the per-step
    reduction's sum_steps(sum_ranks): 20 B/Gaussian less traffic per step.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

CLUSTER_SIZE = 128
MASK_COL = 14     # padding column of the gradient rows that carries the cluster mask


class ViewParallel:
    """zero1=True: the optimiser step is sharded (ZeRO stage 1) -- the
    gradient rows are REDUCE-SCATTERED in cluster-aligned row shards (mask in
    the padding column), each rank runs the sparse Adam on its shard only
    (the 400 B/row Adam traffic splits by the world size), and the updated
    parameter rows are ALL-GATHERED.  Same bytes on the wire as one
    all-reduce (which is a reduce-scatter + all-gather); the moments of other
    ranks' shards are stale until sync_optimizer_state(), which every
    restructuring (densify, Morton re-sort, checkpoint) must be preceded by."""

    def __init__(self, group=None, zero1: bool = False):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.zero1 = bool(zero1) and self.world > 1
        self._bufs = {}

    # ---- ZeRO-1 ---------------------------------------------------------------
    def shard_rows(self, n: int) -> int:
        """Rows per rank: equal, cluster-aligned shards covering n rows."""
        k = (n + CLUSTER_SIZE - 1) // CLUSTER_SIZE
        return ((k + self.world - 1) // self.world) * CLUSTER_SIZE

    def padded_rows(self, n: int) -> int:
        return self.shard_rows(n) * self.world

    def grad_buffer(self, n: int, device) -> torch.Tensor:
        """Padded (world x shard, 16) gradient rows for backward(grads_out=);
        rows >= n stay zero."""
        key = ("grads", n, str(device))
        if key not in self._bufs:
            self._bufs = {k: v for k, v in self._bufs.items() if k[1] == n}
            self._bufs[key] = torch.zeros((self.padded_rows(n), 16), dtype=torch.float32, device=device)
        return self._bufs[key]

    def zero1_step(self, scene, grads_padded: torch.Tensor, cluster_mask: torch.Tensor, state, lrs: dict):
        """Reduce-scatter the (padded) gradient rows, sharded sparse Adam,
        all-gather the parameter rows.  grads_padded: grad_buffer(n) whose
        first n rows hold this rank's gradient sum; cluster_mask: (K,)."""
        from .backward import SceneGrads
        from .optim import adam_step
        n = scene.n
        per = self.shard_rows(n)
        if grads_padded.shape[0] != per * self.world:
            raise ValueError("grads_padded must come from grad_buffer(scene.n)")
        heads = grads_padded[:n:CLUSTER_SIZE, MASK_COL]
        heads.copy_(cluster_mask.to(grads_padded.dtype))
        shard = torch.empty((per, 16), dtype=grads_padded.dtype, device=grads_padded.device)
        dist.reduce_scatter_tensor(shard, grads_padded, group=self.group)
        r0 = self.rank * per
        r1 = min(r0 + per, n)
        m = max(r1 - r0, 0)
        mask = shard[::CLUSTER_SIZE, MASK_COL] > 0
        shard[::CLUSTER_SIZE, MASK_COL] = 0.0
        if m:
            adam_step(scene, SceneGrads(shard[:m].contiguous()), state,
                      mask[:(m + CLUSTER_SIZE - 1) // CLUSTER_SIZE], lrs, rows=(r0, r1))
        send = torch.zeros((per, 16), dtype=scene.data.dtype, device=scene.data.device)
        if m:
            send[:m] = scene.data[r0:r1]
        full = torch.empty((per * self.world, 16), dtype=scene.data.dtype, device=scene.data.device)
        dist.all_gather_into_tensor(full, send, group=self.group)
        scene.data.copy_(full[:n])

    def sync_optimizer_state(self, state):
        """All-gather every rank's Adam moment / step shards (ZeRO-1), so all
        ranks hold the full optimiser state before a restructuring."""
        if not self.zero1:
            return
        scene = state.scene
        n = scene.n
        per = self.shard_rows(n)
        r0, r1 = self.rank * per, min(self.rank * per + per, n)
        for t in (state.m_rows, state.v_rows, state.step.view(-1, 1)):
            width = t.shape[1]
            send = torch.zeros((per, width), dtype=t.dtype, device=t.device)
            if r1 > r0:
                send[:r1 - r0] = t[r0:r1]
            full = torch.empty((per * self.world, width), dtype=t.dtype, device=t.device)
            dist.all_gather_into_tensor(full, send, group=self.group)
            t.copy_(full[:n])

    # ---- all-reduce overlapped with the chain and Adam -----------------------
    def chunk_bounds(self, n: int, chunks: int) -> list:
        """Cluster-aligned row ranges [r0, r1) covering n rows."""
        k = (n + CLUSTER_SIZE - 1) // CLUSTER_SIZE
        per = max(1, (k + chunks - 1) // chunks) * CLUSTER_SIZE
        return [(r0, min(r0 + per, n)) for r0 in range(0, n, per)]

    def overlapped_step(self, scene, ctx, dL_dI, state, lrs: dict, stats=None, chunks: int = 4):
        """One data-parallel training step after the forward: raster backward,
        then per cluster-aligned row chunk the projection chain, an ASYNC
        all-reduce of that chunk's gradient rows (the cluster mask rides in
        padding column 14, which the chain sets to 1.0 on a visible
        cluster's first row) and, once its reduction has landed, that chunk's
        sparse Adam step.  The collective of chunk c overlaps the chain of
        chunk c + 1 and the Adam of chunk c - 1 (NCCL runs on its own
        stream).  Same sums and the same Adam arithmetic as backward +
        reduce_grads + adam_step; on one rank it is exactly that."""
        from .backward import SceneGrads, backward
        from .optim import adam_step
        n = scene.n
        key = ("rows", n, str(scene.device))
        if key not in self._bufs:
            self._bufs = {k: v for k, v in self._bufs.items() if k[1] == n}
            self._bufs[key] = torch.empty((max(n, 1), 16), dtype=torch.float32, device=scene.device)
        g = self._bufs[key]
        bounds = self.chunk_bounds(n, chunks)
        works = []

        def schedule(chain, grads):
            for r0, r1 in bounds:
                chain(r0, r1)
                if self.world > 1:
                    works.append(dist.all_reduce(grads[r0:r1], group=self.group, async_op=True))

        res = backward(scene, ctx, dL_dI, stats, grads_out=g, chain_chunks=schedule)
        for i, (r0, r1) in enumerate(bounds):
            sub = g[r0:r1]
            if self.world > 1:
                works[i].wait()
                mask = sub[::CLUSTER_SIZE, MASK_COL] > 0
            else:
                mask = res.cluster_mask[r0 // CLUSTER_SIZE:(r1 + CLUSTER_SIZE - 1) // CLUSTER_SIZE]
            adam_step(scene, SceneGrads(sub), state, mask, lrs, rows=(r0, r1))
        return res

    def views_for_step(self, step: int, n_views: int, views_per_rank: int = 1) -> list:
        """Indices of the views this rank renders at `step` (round robin)."""
        base = (step * self.world + self.rank) * views_per_rank
        return [(base + j) % n_views for j in range(views_per_rank)]

    def reduce(self, grads: torch.Tensor, S: torch.Tensor, M: torch.Tensor, C: torch.Tensor,
               cluster_mask: torch.Tensor):
        """In place: grads, S, M, C become the sums over ranks; returns the
        OR-ed cluster mask (bool)."""
        if self.world == 1:
            return cluster_mask.bool()
        n, k = S.numel(), cluster_mask.numel()
        flat = torch.empty(2 * n + n + k, dtype=torch.float64, device=S.device)
        flat[:n] = S
        flat[n:2 * n] = M
        flat[2 * n:3 * n] = C.to(torch.float64)
        flat[3 * n:] = cluster_mask.to(torch.float64)
        w1 = dist.all_reduce(grads, group=self.group, async_op=True)
        dist.all_reduce(flat, group=self.group)
        w1.wait()
        S.copy_(flat[:n])
        M.copy_(flat[n:2 * n])
        C.copy_(flat[2 * n:3 * n].round().to(C.dtype))
        return flat[3 * n:] > 0

    def reduce_grads(self, grads: torch.Tensor, cluster_mask: torch.Tensor) -> torch.Tensor:
        """In place: the (N, 16) float32 gradient rows become the sum over
        ranks (padding columns left zero); returns the OR-ed cluster mask
        (bool).  One all-reduce."""
        if self.world == 1:
            return cluster_mask.bool()
        n, k = grads.shape[0], cluster_mask.numel()
        if k != (n + CLUSTER_SIZE - 1) // CLUSTER_SIZE or grads.shape[1] != 16:
            raise ValueError(f"grads {tuple(grads.shape)} do not match {k} clusters")
        heads = grads[::CLUSTER_SIZE, MASK_COL]
        heads.copy_(cluster_mask.to(grads.dtype))
        dist.all_reduce(grads, group=self.group)
        mask = grads[::CLUSTER_SIZE, MASK_COL] > 0
        grads[::CLUSTER_SIZE, MASK_COL] = 0.0
        return mask

    def reduce_stats(self, S: torch.Tensor, M: torch.Tensor, C: torch.Tensor):
        """In place: rank-local accumulated statistics become their sum over
        ranks (call before reading them, e.g. before densify_step; the ranks'
        local accumulators must then be reset together)."""
        if self.world == 1:
            return
        w1 = dist.all_reduce(S, group=self.group, async_op=True)
        w2 = dist.all_reduce(M, group=self.group, async_op=True)
        dist.all_reduce(C, group=self.group)
        w1.wait()
        w2.wait()

    def all_sum(self, t: torch.Tensor):
        """In place sum over ranks (small host-side metrics)."""
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
