"""Throughput of BASELINE.json's other configs on one B200.

bench.py's headline is config B.  This tool measures the rest, device-timed
with CUDA events (inputs resident in HBM), one JSON line per config:

  A  10K Gaussians, 128x128, full training iteration
  C  3M Gaussians, 1920x1080, 100-view ring (1 epoch = 100 iterations),
     densification at every epoch boundary (DensifyConfig(start_epoch=1,
     densify_interval_epochs=1, budget=1.05 N)); timed over whole epochs so
     the densify events are inside the timed region
  D  1M Gaussians, 8 views per optimiser step on one GPU (the N=1 point of
     the view-sharded run): per view forward + loss + backward, grads summed,
     statistics accumulated, masks OR-ed, one sparse Adam step
  E  6M Gaussians, 3840x2160, 8-view ring, Morton re-sort every 500
     iterations; timed over 500 iterations including one re-sort

    python tools/bench_configs.py [A C D E]
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2503_01199_b200 as sb  # noqa: E402
from paper_2503_01199_b200 import _lib  # noqa: E402
from paper_2503_01199_b200.synthetic import (SyntheticSceneSpec, camera_ring, random_scene_arrays,  # noqa: E402
                                             scaled_scene_arrays)

CH = ("position", "log_scale", "rotation", "color", "opacity_logit")
DEV = torch.device("cuda", 0)


def make(n, res, n_views, scaled=True, n_targets=8):
    if scaled:
        arr = scaled_scene_arrays(n, 7, res)
    else:
        arr = random_scene_arrays(SyntheticSceneSpec(n_gaussians=n, n_views=1, view_resolution=res, seed=7))
    scene = sb.SceneSoA(*[arr[k] for k in CH], device=DEV)
    state = sb.AdamState(scene)
    sb.DensifyStats.zeros(scene.n, DEV).attach(scene)
    sb.morton_sort(scene)
    views = camera_ring(SyntheticSceneSpec(n_gaussians=n, n_views=n_views, view_resolution=res, seed=7))
    rng = np.random.default_rng(1234)
    W, H = res
    targets = [torch.from_numpy(rng.integers(0, 256, (H, W, 3), dtype=np.uint8)).to(DEV)
               for _ in range(min(n_targets, n_views))]
    return scene, state, views, targets


def device_time(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b), (time.perf_counter() - t0) * 1e3


def iteration(scene, state, cam, target, lrs):
    out, ctx = sb.forward(scene, cam)
    loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True)
    res = sb.backward(scene, ctx, dI)
    sb.adam_step(scene, res.grads, state, res.cluster_mask, lrs)
    return ctx


def stage_times(scene, state, views, targets, lrs, iters=3):
    _lib.enable_call_timing(True)
    for i in range(iters):
        ctx = iteration(scene, state, views[i % len(views)], targets[i % len(targets)], lrs)
    torch.cuda.synchronize()
    tim = _lib.call_timings()
    _lib.enable_call_timing(False)
    return {k: statistics.mean(v) for k, v in tim.items()}, ctx


def line(name, workload, value, unit, ms, extra):
    d = {"config": name, "workload": workload, "value": value, "unit": unit, "ms_timed": ms,
         "data": "synthetic (reference generator, seed 7)", "dtype": "f32", "n_gpus": 1}
    d.update(extra)
    print(json.dumps(d), flush=True)


def config_A(steps=200):
    scene, state, views, targets = make(10_000, (128, 128), 1, scaled=False)
    lrs = sb.LearningRates().at(0.0, position_scale=3.2)
    for _ in range(5):
        iteration(scene, state, views[0], targets[0], lrs)
    def run():
        for _ in range(steps):      # (contexts not retained: no allocator growth inside the timed loop)
            iteration(scene, state, views[0], targets[0], lrs)

    ms, wall = device_time(run)
    stages, ctx = stage_times(scene, state, views, targets, lrs)
    line("A", "10K Gaussians, 128x128, full training iteration", steps / (ms / 1e3), "iters/s", ms,
         {"steps": steps, "wall_ms": wall, "stages_ms": stages, "P_pairs": ctx.n_pairs,
          "note": "launch/host bound at this size (12 launches + one counter read per iteration)"})


def warm_densify():
    """One densify event on a small scene first: the surgery's torch kernels
    load lazily on first use (~140 ms once per process), which is not a
    per-event cost."""
    scene, state, views, targets = make(20_000, (256, 256), 2, scaled=False)
    lrs = sb.LearningRates().at(0.0, position_scale=3.2)
    for v in range(2):
        iteration(scene, state, views[v], targets[v], lrs)
    sb.densify_step(scene, sb.DensifyStats.from_scene(scene),
                    sb.DensifyConfig(start_epoch=1, densify_interval_epochs=1, budget=int(1.05 * scene.n)), 1)
    torch.cuda.synchronize()


PREGROW_GB = 4


def pregrow_allocator(gb=PREGROW_GB):
    """One large block through torch's caching allocator, freed at once: the
    allocator keeps the segment and carves later allocations from it.  The
    first densify event otherwise grows the allocator by ~1.2 GB in six
    cudaMalloc segments, 13-133 ms once per process (tools/probes/
    densify_alloc_probe.py), against a 1.6-2.2 ms event."""
    x = torch.empty(gb << 30, dtype=torch.uint8, device=DEV)
    del x


def config_C(epochs=2):
    n0 = 3_000_000
    warm_densify()
    pregrow_allocator()
    scene, state, views, targets = make(n0, (1920, 1080), 100)
    dcfg = sb.DensifyConfig(start_epoch=1, densify_interval_epochs=1, budget=int(1.05 * n0))
    lrs = sb.LearningRates().at(0.0, position_scale=3.2)
    for i in range(5):
        iteration(scene, state, views[i], targets[i % len(targets)], lrs)
    log = []
    dens_ms = []

    def run():
        for e in range(1, epochs + 1):
            for vi in range(len(views)):
                iteration(scene, state, views[vi], targets[vi % len(targets)], lrs)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            row = sb.densify_step(scene, sb.DensifyStats.from_scene(scene), dcfg, e)
            b.record()
            dens_ms.append((a, b))
            log.append(row)

    ms, wall = device_time(run)
    iters = epochs * len(views)
    stages, ctx = stage_times(scene, state, views, targets, lrs)
    line("C", "3M Gaussians, 1920x1080, 100-view epochs, densify every 100 iterations",
         iters / (ms / 1e3), "iters/s", ms,
         {"iterations": iters, "densify_events": len(log), "wall_ms": wall,
          "allocator": f"pre-grown by one {PREGROW_GB} GB block before timing (first-growth cudaMalloc is a "
                       "once-per-process cost: 13-133 ms)",
          "densify_ms": [a.elapsed_time(b) for a, b in dens_ms],
          "n_after": scene.n, "densify_log": [r.__dict__ if r is not None else None for r in log],
          "stages_ms": stages, "P_pairs": ctx.n_pairs, "n_compact": ctx.n_compact})


def config_D(steps=10, streams=int(os.environ.get("SB_VIEW_STREAMS", "2"))):
    n = 1_000_000
    scene, state, views, targets = make(n, (1920, 1080), 8)
    lrs = sb.LearningRates().at(0.0, position_scale=3.2)
    batch = [(views[v], targets[v]) for v in range(8)]

    def step():
        # the library's multi-view step: each view's chain adds its rows into
        # one running sum (sb_chain_projection_bwd_accumulate), masks OR-ed,
        # one Adam step; the losses stay on the device (no per-step sync)
        sb.multiview_step(scene, state, batch, lrs, return_tensor=True, streams=streams)

    for _ in range(3):
        step()
    ms, wall = device_time(lambda: [step() for _ in range(steps)])
    line("D", "1M Gaussians, 1920x1080, 8 views per optimiser step on 1 GPU (grads summed, one Adam step)",
         8 * steps / (ms / 1e3), "views/s", ms,
         {"steps": steps, "steps_per_s": steps / (ms / 1e3), "wall_ms": wall, "view_streams": streams,
          "note": "N=1 point of the view-sharded run; N=2/4/8 add one all-reduce per step (bench.py --gpus N)"})


def config_E(iters=500):
    n = 6_000_000
    scene, state, views, targets = make(n, (3840, 2160), 8)
    lrs = sb.LearningRates().at(0.0, position_scale=3.2)
    for i in range(5):
        iteration(scene, state, views[i % 8], targets[i % len(targets)], lrs)
    sort_ev = []

    def run():
        for i in range(iters):
            iteration(scene, state, views[i % 8], targets[i % len(targets)], lrs)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        sb.morton_sort(scene)
        b.record()
        sort_ev.append((a, b))

    ms, wall = device_time(run)
    stages, ctx = stage_times(scene, state, views, targets, lrs)
    line("E", "6M Gaussians, 3840x2160, 8-view ring, Morton re-sort every 500 iterations",
         iters / (ms / 1e3), "iters/s", ms,
         {"iterations": iters, "wall_ms": wall, "resort_ms": [a.elapsed_time(b) for a, b in sort_ev],
          "stages_ms": stages, "P_pairs": ctx.n_pairs, "n_compact": ctx.n_compact,
          "raster_fwd_bwd_ms_per_view": stages.get("sb_raster_fwd", 0) + stages.get("sb_raster_bwd", 0)})


if __name__ == "__main__":
    which = sys.argv[1:] or ["A", "C", "D", "E"]
    for w in which:
        globals()[f"config_{w}"]()
        torch.cuda.empty_cache()
