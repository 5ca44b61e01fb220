"""Golden PLY fixture from the reference's own save_ply (scene.py:275-287).

    PYTHONPATH=/root/reference/pkg/src python tools/make_golden_ply.py

Writes tests/golden/small_scene.ply (200 seeded Gaussians, rounded through
float32 first so both packages hold identical values) and the raw arrays it
was made from (tests/golden/small_scene.npz)."""
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from tinysplat.scene import SceneSoA, save_ply  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "tests", "golden")

rng = np.random.default_rng(2503)
n = 200
arr = {
    "position": rng.uniform(-1, 1, (n, 3)),
    "log_scale": np.log(rng.uniform(0.01, 0.1, (n, 3))),
    "rotation": rng.normal(size=(n, 4)),
    "color": rng.uniform(-1.5, 1.5, (n, 3)),
    "opacity_logit": rng.uniform(-0.5, 2.0, n),
}
arr = {k: v.astype(np.float32).astype(np.float64) for k, v in arr.items()}
scene = SceneSoA(arr["position"], arr["log_scale"], arr["rotation"], arr["color"], arr["opacity_logit"])
save_ply(scene, os.path.join(OUT, "small_scene.ply"))
np.savez(os.path.join(OUT, "small_scene.npz"), **arr)
print("wrote", os.path.join(OUT, "small_scene.ply"))
