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

The training step uses the leaner pair reduce_grads / reduce_stats:
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
    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

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
