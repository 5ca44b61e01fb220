import sys, os, time, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
from bench_configs import make, iteration, warm_densify
import paper_2503_01199_b200 as sb
pre = int(sys.argv[1])
warm_densify()
if pre:
    x = torch.empty(pre << 30, dtype=torch.uint8, device="cuda"); del x
n0 = 3_000_000
scene, state, views, targets = make(n0, (1920, 1080), 10)
dcfg = sb.DensifyConfig(start_epoch=1, densify_interval_epochs=1, budget=int(1.05 * n0))
lrs = sb.LearningRates().at(0.0, position_scale=3.2)
for e in range(1, 4):
    for vi in range(10):
        iteration(scene, state, views[vi], targets[vi % len(targets)], lrs)
    torch.cuda.synchronize()
    s0 = torch.cuda.memory_stats()
    t = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    row = sb.densify_step(scene, sb.DensifyStats.from_scene(scene), dcfg, e)
    b.record(); torch.cuda.synchronize()
    s1 = torch.cuda.memory_stats()
    print(f"pre={pre} event {e}: {a.elapsed_time(b):.2f} ms device, {1e3*(time.perf_counter()-t):.2f} ms wall, "
          f"segments +{s1['segment.all.allocated']-s0['segment.all.allocated']}, "
          f"alloc bytes +{(s1['reserved_bytes.all.allocated']-s0['reserved_bytes.all.allocated'])/1e6:.0f} MB, n={scene.n}")
