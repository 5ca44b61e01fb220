"""Scene PLY import/export and training checkpoints with optimiser state.

Reference: pkg/src/tinysplat/scene.py:266-314 (save_ply / load_ply: binary
little-endian, one float32 row of 14 raw-space values per Gaussian) and
train.py:152-181 (write_metrics_csv, write_densify_csv, checkpoint).  The
PLY bytes are the reference's exactly (same header, same column order), so
files move between the two packages in both directions.

Beyond the reference: `save_checkpoint` /
`load_checkpoint` also keep every scene extra (Adam moments and step
counters, densification statistics, ...) and the scene generation, so a run
resumes bit-for-bit where it stopped; the reference checkpoints parameters
only.
"""
from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np
import torch

from .scene import CHANNEL_COLS, SceneSoA

PLY_PROPS = (
    "x", "y", "z",
    "f_dc_0", "f_dc_1", "f_dc_2",
    "opacity",
    "scale_0", "scale_1", "scale_2",
    "rot_0", "rot_1", "rot_2", "rot_3",
)
# PLY column -> (channel, column inside the channel)
_PLY_COLS = (("position", 0, 3), ("color", 3, 6), ("opacity_logit", 6, 7), ("log_scale", 7, 10),
             ("rotation", 10, 14))


def _rows(scene: SceneSoA) -> np.ndarray:
    data = scene.data.detach().to("cpu")
    rows = np.empty((scene.n, len(PLY_PROPS)), dtype="<f4")
    for ch, a, b in _PLY_COLS:
        c0, c1 = CHANNEL_COLS[ch]
        rows[:, a:b] = data[:, c0:c1].numpy()
    return rows


def save_ply(scene: SceneSoA, path) -> None:
    """scene.py:275-287: header, then n x 14 little-endian float32 rows."""
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {scene.n}"]
    header += [f"property float {p}" for p in PLY_PROPS]
    header.append("end_header")
    with open(path, "wb") as f:
        f.write(("\n".join(header) + "\n").encode("ascii"))
        f.write(_rows(scene).tobytes())


def load_ply(path, device=None) -> SceneSoA:
    """scene.py:290-314, with the reference's error messages."""
    with open(path, "rb") as f:
        data = f.read()
    end = data.find(b"end_header\n")
    if end < 0:
        raise ValueError(f"{path}: not a ply file (missing end_header)")
    header = data[:end].decode("ascii").splitlines()
    body = data[end + len(b"end_header\n"):]
    n = None
    props = []
    for line in header:
        parts = line.split()
        if parts[:2] == ["element", "vertex"]:
            n = int(parts[2])
        elif parts and parts[0] == "property":
            if parts[1] != "float":
                raise ValueError(f"{path}: unsupported property type {parts[1]}")
            props.append(parts[2])
    if n is None:
        raise ValueError(f"{path}: missing vertex element")
    if tuple(props) != PLY_PROPS:
        raise ValueError(f"{path}: unexpected property layout {props}")
    rows = np.frombuffer(body, dtype="<f4", count=n * len(PLY_PROPS)).reshape(n, len(PLY_PROPS))
    return SceneSoA(rows[:, 0:3], rows[:, 7:10], rows[:, 10:14], rows[:, 3:6], rows[:, 6], device=device)


def write_metrics_csv(rows, path) -> None:
    """train.py:152-159."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["epoch", "loss", "psnr", "n_primitives", "visible_clusters", "culled_clusters", "wall_time"])
        for r in rows:
            w.writerow([r.epoch, repr(r.loss), repr(r.psnr), r.n_primitives, repr(r.visible_clusters),
                        repr(r.culled_clusters), repr(r.wall_time)])


def write_densify_csv(rows, path) -> None:
    """train.py:162-170."""
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["epoch", "n_before", "n_after", "n_split", "n_clone", "n_pruned", "max_score", "mean_score"])
        for r in rows:
            w.writerow([r.epoch, r.n_before, r.n_after, r.n_split, r.n_clone, r.n_pruned, repr(r.max_score),
                        repr(r.mean_score)])


def save_checkpoint(scene: SceneSoA, out_dir, meta: dict | None = None) -> Path:
    """scene.ply (the reference's format) + extras.npz (every registered
    extra: Adam m / v / step, densification S / M / C, ...) + state.json
    (generation, caller metadata such as the epoch)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    save_ply(scene, out / "scene.ply")
    np.savez(out / "extras.npz", **{k: v.detach().to("cpu").numpy() for k, v in scene.extras.items()})
    (out / "state.json").write_text(json.dumps({"n": scene.n, "generation": scene.generation,
                                                "meta": meta or {}}, indent=1))
    return out


def load_checkpoint(out_dir, device=None) -> tuple[SceneSoA, dict]:
    """Inverse of save_checkpoint: the scene with its extras and generation
    restored (an AdamState(scene) built from it would reset the moments, so
    use `adam_state_from(scene)`), and the caller metadata."""
    out = Path(out_dir)
    scene = load_ply(out / "scene.ply", device=device)
    state = json.loads((out / "state.json").read_text())
    if state["n"] != scene.n:
        raise ValueError(f"{out}: state.json says {state['n']} primitives, scene.ply has {scene.n}")
    with np.load(out / "extras.npz") as z:
        for k in z.files:
            t = torch.from_numpy(np.array(z[k])).to(scene.data.device)
            if t.shape[0] != scene.n:
                raise ValueError(f"{out}: extra '{k}' has {t.shape[0]} rows, scene has {scene.n}")
            scene.extras[k] = t
    scene.generation = int(state["generation"])
    return scene, state["meta"]


def adam_state_from(scene: SceneSoA):
    """An AdamState over moments already registered on the scene (resume)."""
    from .optim import AdamState
    st = AdamState.__new__(AdamState)
    for k in ("adam_m", "adam_v", "adam_step"):
        if k not in scene.extras:
            raise KeyError(f"scene has no '{k}' extra: not a checkpoint with optimiser state")
    st.scene = scene
    return st


def checkpoint(result, out_dir, manifest_text: str | None = None) -> Path:
    """train.py:173-181 (scene.ply, metrics.csv, densify.csv, manifest.cfg),
    plus the optimiser state of save_checkpoint."""
    out = save_checkpoint(result.scene, out_dir)
    write_metrics_csv(result.metrics, out / "metrics.csv")
    write_densify_csv(result.densify_log, out / "densify.csv")
    if manifest_text is not None:
        (out / "manifest.cfg").write_text(manifest_text)
    return out
