"""Benchmark: LiteGS training iteration on B200 (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload ("config B"): 1,000,000 synthetic Gaussians (reference generator,
seed 7, footprints shrunk by (N/512)^(1/3) per SURVEY 8(d)), Morton-sorted,
1920x1080 views on the reference's camera ring.  One step = one full training
iteration per GPU: project + cluster cull + compact + bin + per-tile sort +
raster forward + L1/D-SSIM loss + raster backward + projection chain +
cluster-sparse Adam (N > 1: the gradient rows and cluster masks are
all-reduced over NCCL in four cluster-aligned chunks, each overlapping the
next chunk's chain and the previous chunk's Adam; densification statistics
stay rank-local until read).
Each rank rasterises its own view against replicated Gaussians (weak scaling).

`value`  whole-job views/s with inputs resident in HBM, device-timed with CUDA
         events over K steps, max over ranks.
`e2e`    the same through the public API with host buffers: every step copies
         its target image (uint8, pinned) host->device and reads the loss back.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "raster fwd+bwd ms/view & train iters/s @1M Gaussians 1080p; HBM roofline frac"
N_GAUSS = 1_000_000
RES = (1920, 1080)
N_VIEWS = 8
CH = ("position", "log_scale", "rotation", "color", "opacity_logit")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def setup_dist():
    """One process per GPU over NCCL.  If ranks outnumber the visible GPUs
    (a functional check of the multi-rank path on a 1-GPU box), ranks share
    devices and exchange over gloo instead -- never used for timing claims."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL's own report of the communicator (ranks, NVLink / NVLS paths)
        # on stderr, for the driver's multi-GPU records
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        ndev = max(torch.cuda.device_count(), 1)
        if ws <= ndev:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            local = local % ndev
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
    return ws, rank, local


def build_workload(device):
    import paper_2503_01199_b200 as sb
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays
    arr = scaled_scene_arrays(N_GAUSS, 7, RES)
    scene = sb.SceneSoA(*[arr[k] for k in CH], device=device)
    state = sb.AdamState(scene)
    sb.DensifyStats.zeros(scene.n, device).attach(scene)
    sb.morton_sort(scene)
    views = camera_ring(SyntheticSceneSpec(n_gaussians=N_GAUSS, n_views=N_VIEWS, view_resolution=RES, seed=7))
    rng = np.random.default_rng(1234)
    W, H = RES
    targets_host = [torch.from_numpy(rng.integers(0, 256, (H, W, 3), dtype=np.uint8)).pin_memory()
                    for _ in range(N_VIEWS)]
    return scene, state, views, targets_host


class Trainer:
    """One training iteration through the public API (train.py:95-104)."""

    def __init__(self, scene, state, views, ws, rank, zero1=False):
        import paper_2503_01199_b200 as sb
        from paper_2503_01199_b200.parallel import ViewParallel
        self.sb = sb
        self.scene, self.state, self.views = scene, state, views
        self.ws, self.rank = ws, rank
        self.vp = ViewParallel(zero1=zero1)
        self.lrs = sb.LearningRates().at(0.0, position_scale=3.2)

    def view_index(self, it):
        return self.vp.views_for_step(it, len(self.views))[0]

    def step(self, it, target, loss_out=None):
        sb = self.sb
        cam = self.views[self.view_index(it)]
        out, ctx = sb.forward(self.scene, cam)
        loss, dI = sb.loss_and_grad(out.color, target, 0.2, return_tensor=True, loss_out=loss_out)
        # statistics accumulate rank-locally in the scene (summed over ranks
        # only when read: ViewParallel.reduce_stats before a densify step)
        if self.vp.zero1:
            # ZeRO-1: reduce-scatter the gradient rows, sharded Adam, all-gather
            gbuf = self.vp.grad_buffer(self.scene.n, self.scene.device)
            res = sb.backward(self.scene, ctx, dI, sb.DensifyStats.from_scene(self.scene), grads_out=gbuf)
            self.vp.zero1_step(self.scene, gbuf, res.cluster_mask, self.state, self.lrs)
            return loss, ctx
        if self.ws > 1:
            # sum the views' grads over ranks, OR the masks --
            # the gradient rows (mask in a padding column) all-reduced in
            # cluster-aligned chunks, each under the next chunk's chain and
            # the previous chunk's Adam step
            self.vp.overlapped_step(self.scene, ctx, dI, self.state, self.lrs,
                                    sb.DensifyStats.from_scene(self.scene), chunks=4)
            return loss, ctx
        res = sb.backward(self.scene, ctx, dI, sb.DensifyStats.from_scene(self.scene))
        sb.adam_step(self.scene, res.grads, self.state, res.cluster_mask, self.lrs)
        return loss, ctx


def timed(fn, steps, ws):
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    t0 = time.perf_counter()
    fn()
    b.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if ws > 1:
        dist.barrier()
    ms = a.elapsed_time(b)
    if ws > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, wall


# algorithmic bytes per launch; P pairs, Nc compact, Npix pixels
# kernels timed by back-to-back replay (bench's roofline and raster line)
REPLAYED = ("sb_raster_fwd", "sb_raster_bwd")
K_REPLAY = 20


def algorithmic_bytes(name, n, nc, P, npix):
    return {
        "sb_project_cull_compact": 56 * n + 48 * nc,
        "sb_bin_emit": 12 * nc + 8 * P,
        "sb_tile_sort": 8 * P + 4 * P,
        "sb_raster_fwd": 40 * P + 20 * npix,
        "sb_raster_bwd": 96 * P + 20 * npix,
        "sb_chain_projection_bwd": 188 * nc,
        "sb_adam_sparse": 400 * nc,
    }.get(name)


def cpu_baseline_oracle(sample_iters=1):
    """The CPU oracle (C port of the reference, all host threads) on config B."""
    from oracle import oracle as O
    from paper_2503_01199_b200.synthetic import SyntheticSceneSpec, camera_ring, scaled_scene_arrays
    arr = scaled_scene_arrays(N_GAUSS, 7, RES)
    _, perm = O.morton_perm(arr["position"])
    arr = {k: np.ascontiguousarray(v[perm]) for k, v in arr.items()}
    views = camera_ring(SyntheticSceneSpec(n_gaussians=N_GAUSS, n_views=N_VIEWS, view_resolution=RES, seed=7))
    rng = np.random.default_rng(1234)
    p14 = np.ascontiguousarray(O.pack14(arr))
    m = np.zeros_like(p14); v = np.zeros_like(p14); st = np.zeros(len(p14), np.int64)
    lr = [1.6e-4 * 3.2, 5e-3, 1e-3, 2.5e-3, 5e-2]
    times = []
    for it in range(sample_iters):
        target = rng.integers(0, 256, (RES[1], RES[0], 3)).astype(np.float64) / 255.0
        t0 = time.perf_counter()
        col, T, fr, ctx = O.forward(arr, views[it % N_VIEWS])
        _, dI = O.loss_and_grad(col, target, 0.2)
        b = O.backward(arr, ctx, dI.astype(np.float32))
        O.adam_step(p14, np.ascontiguousarray(b["grads"]), m, v, st, b["cluster_mask"], lr)
        times.append(time.perf_counter() - t0)
    return times


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cores = os.cpu_count()
    # torchrun pre-sets OMP_NUM_THREADS=1; the baseline uses every host thread
    os.environ["OMP_NUM_THREADS"] = str(cores)
    from oracle import oracle as O
    O.build() if not os.path.exists(O.LIB_PATH) else None
    # the driver's own step / warm-up counts (one config-B iteration is ~3 s
    # on 16 host threads); only a very long request is capped, and the line
    # then says so ("steps_requested")
    w = min(args.warmup, 2)
    k = max(1, min(args.steps, 40))
    cpu_baseline_oracle(w) if w else None
    times = cpu_baseline_oracle(k)
    ms = 1e3 * sum(times) / len(times)
    val = 1e3 / ms
    sample = (f"{k} full config-B iterations (1M Gaussians, 1920x1080: project, cull, compact, bin, forward, "
              f"fp64 L1+SSIM loss, backward, Adam) of the C oracle port, OpenMP over tiles")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": "iters/s", "n_gpus": ws, "steps": k,
        "warmup": w, "steps_requested": args.steps, "warmup_requested": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32+f64", "data": "synthetic",
        "config": {"workload": "config B: 1M Gaussians, 1920x1080, full train iteration", "n_gaussians": N_GAUSS,
                   "resolution": list(RES)},
        "cpu_baseline": {"value": val, "unit": "iters/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": val, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--zero1", action="store_true", help="N > 1: reduce-scatter + sharded Adam + all-gather")
    args = ap.parse_args()
    ws, rank, local = setup_dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    args.warmup = max(args.warmup, 3)
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    import paper_2503_01199_b200 as sb
    from paper_2503_01199_b200 import _lib
    scene, state, views, targets_host = build_workload(device)
    trainer = Trainer(scene, state, views, ws, rank, zero1=args.zero1)
    # targets stay uint8 (the dataset format); the fused loss reads them directly
    targets_dev = [t.to(device) for t in targets_host]

    it = {"i": 0}

    def run(k):
        for _ in range(k):
            i = it["i"]
            trainer.step(i, targets_dev[trainer.view_index(i)])
            it["i"] += 1

    run(args.warmup)
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = _lib.launch_count["n"]
    ms, wall = timed(lambda: run(args.steps), args.steps, ws)
    launches = _lib.launch_count["n"] - launches0
    clk = clocks.stop()
    ms_step = ms / args.steps
    value = ws * args.steps / (ms / 1e3)

    # e2e: public API with host buffers -- every step copies its uint8 target
    # from pinned host memory (prefetched on a copy stream while the previous
    # step computes) and reads its loss back (the loss kernel stores it into
    # mapped pinned memory); the timed region ends after the last has landed
    W, H = RES
    h2d = H * W * 3
    copy_stream = torch.cuda.Stream(device)
    loss_host = torch.empty(max(args.steps, 2), dtype=torch.float64, pin_memory=True)

    def fetch(i):
        with torch.cuda.stream(copy_stream):
            t = targets_host[trainer.view_index(i)].to(device, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_stream)
        return t, ev

    def run_e2e(k):
        nxt = fetch(it["i"])
        for j in range(k):
            i = it["i"]
            tgt, ev = nxt
            torch.cuda.current_stream(device).wait_event(ev)
            tgt.record_stream(torch.cuda.current_stream(device))
            if j + 1 < k:
                nxt = fetch(i + 1)
            # the loss kernel writes the step's loss straight into pinned
            # host memory (mapped): the device-to-host read of the result
            trainer.step(i, tgt, loss_out=loss_host[j:j + 1])
            it["i"] += 1

    run_e2e(2)
    e2e_ms, _ = timed(lambda: run_e2e(args.steps), args.steps, ws)
    losses = loss_host[:args.steps].tolist()
    e2e_val = ws * args.steps / (e2e_ms / 1e3)

    # per-kernel durations (CUDA events on the launching stream, separate pass)
    # (a) in-step: events around every call of 3 training steps.  The host
    #     sizes each view's pair buffers from one counter read, so a call's
    #     start event can fire while the host is still issuing it: these
    #     include host launch gaps.
    # (b) replayed: the raster kernels of the last step re-issued K_REPLAY
    #     times back to back on their stream with the same buffers, events
    #     around the batch: the kernels' own average launch duration.
    _lib.enable_call_timing(True)
    _lib.keep_last_args(REPLAYED)
    ctxs = []
    for _ in range(3):
        _, ctx = trainer.step(it["i"], targets_dev[0])
        ctxs.append(ctx)
        it["i"] += 1
    torch.cuda.synchronize()
    tim = _lib.call_timings()
    _lib.enable_call_timing(False)
    replayed = {k: _lib.replay_time(k, K_REPLAY) for k in REPLAYED}
    _lib.keep_last_args(None)
    ctx = ctxs[-1]
    n, nc, P, npix = scene.n, ctx.n_compact, ctx.n_pairs, W * H
    stages_in_step = {k: statistics.mean(v) for k, v in tim.items()}
    stages = dict(stages_in_step)
    stages.update(replayed)
    dominant = max(stages, key=stages.get)
    peak, peak_kind = peaks()
    ab = algorithmic_bytes(dominant, n, nc, P, npix)
    achieved = ab / (stages[dominant] * 1e-3) / 1e9 if ab else None
    # DRAM traffic and warp instructions of the dominant call from the
    # round's committed ncu capture (profiles/traffic.json names it); ncu
    # cannot run inside the timed bench.  The issue roofline: those warp
    # instructions at one issue per cycle on the 4 x 148 schedulers at the
    # clock sampled during the timed region, against this run's duration.
    traffic = traffic_source = issue = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            ent = tj.get(dominant) or {}
            traffic = ent.get("dram_bytes")
            traffic_source = tj.get("_source")
            wi = ent.get("warp_instructions")
            f_sm = (clk.get("sm_mhz") or 1965.0) * 1e6
            if wi:
                floor_ms = wi / (4 * 148 * f_sm) * 1e3
                issue = {"warp_instructions": wi, "floor_ms": floor_ms, "achieved_ms": stages[dominant],
                         "frac": floor_ms / stages[dominant]}
        except Exception:
            traffic = None
    raster_ms = stages.get("sb_raster_fwd", 0.0) + stages.get("sb_raster_bwd", 0.0)
    raster_bytes = algorithmic_bytes("sb_raster_fwd", n, nc, P, npix) + algorithmic_bytes("sb_raster_bwd", n, nc, P,
                                                                                          npix)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        os.environ["OMP_NUM_THREADS"] = str(os.cpu_count())
        try:
            t = cpu_baseline_oracle(1)
            cpu = {"value": 1.0 / t[0], "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": "1 full config-B iteration of the C oracle port (OpenMP over tiles, all host threads)"}
        except Exception as e:  # the baseline must not take down the bench line
            cpu = {"value": None, "unit": "iters/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {e}"}

    # rank consistency: every rank must hold bit-identical parameters after
    # the timed steps (one identical Adam step per step on every rank)
    consistency = None
    if ws > 1:
        h = scene.data.contiguous().view(torch.int32).to(torch.int64)
        w = torch.arange(1, h.numel() + 1, device=h.device, dtype=torch.int64).view_as(h) % 1000003
        ck = torch.stack([(h * w).sum() % (1 << 61), h.sum()])
        allck = [torch.zeros_like(ck) for _ in range(ws)]
        dist.all_gather(allck, ck)
        vals = [tuple(int(v) for v in c.tolist()) for c in allck]
        consistency = {"param_checksums": [v[0] for v in vals], "ranks_identical": len(set(vals)) == 1}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference generator, seed 7, N-scaled)",
            "config": {"workload": "config B: 1M Gaussians, 1920x1080, full train iteration per view per GPU",
                       "n_gaussians": N_GAUSS, "resolution": list(RES), "views_per_gpu_per_step": 1,
                       "parallelism": f"view-parallel dp{ws}" if ws > 1 else "single GPU",
                       "l2": "inputs larger than L2 (params 64 MB + pairs ~165 MB + records 45 MB per view)",
                       "P_pairs": P, "n_compact": nc},
            "raster_fwd_bwd_ms_per_view": raster_ms,
            "raster_fwd_bwd_roofline_frac": (raster_bytes / (raster_ms * 1e-3) / 1e9) / peak if raster_ms else None,
            "stages_ms": stages,
            "stages_ms_in_step": stages_in_step,
            "stage_timing": ("stages_ms: raster fwd / bwd = average of %d back-to-back replays of the step's launch "
                             "(CUDA events on its stream); the other stages and stages_ms_in_step = events around "
                             "each call inside 3 training steps (include host launch gaps)" % K_REPLAY),
            "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak if achieved else None, "traffic": traffic,
                         "traffic_source": traffic_source, "algorithmic_bytes": ab, "peak_kind": peak_kind,
                         "issue_roofline": issue},
            "e2e": {"value": e2e_val, "unit": "iters/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": loss_host.element_size()},
            "gpu_launches": launches,
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        if consistency is not None:
            line["rank_consistency"] = consistency
            line["config"]["optimizer_step"] = "zero1 (reduce-scatter, sharded Adam, all-gather)" if args.zero1 \
                else "all-reduce of the gradient rows in 4 chunks overlapped with the chain and Adam, replicated Adam"
        print(json.dumps(line))
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
