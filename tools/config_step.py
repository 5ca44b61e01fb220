"""A few training iterations of one BASELINE config, for ncu launch lists:
    ncu --metrics gpu__time_duration.sum --csv ... python tools/config_step.py C
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_configs as b  # noqa: E402
import paper_2503_01199_b200 as sb  # noqa: E402

SHAPES = {"A": (10_000, (128, 128), False), "B": (1_000_000, (1920, 1080), True),
          "C": (3_000_000, (1920, 1080), True), "E": (6_000_000, (3840, 2160), True)}

if __name__ == "__main__":
    n, res, scaled = SHAPES[sys.argv[1] if len(sys.argv) > 1 else "C"]
    scene, state, views, targets = b.make(n, res, 8, scaled=scaled)
    lrs = sb.LearningRates().at(0.0, position_scale=3.2)
    for i in range(3):
        b.iteration(scene, state, views[0], targets[0], lrs)
