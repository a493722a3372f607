"""Reference numbers for tests/test_gpu_acceptance.py: the REAL reference
(voxsplat) runs the desk-scale pipeline on the same data the GPU test uses --
64^3 shells volume, two basic transfer functions, a 42-view Fibonacci rig at
128^2, TrainConfig(stage1_iters=3000, stage2_iters=1000, seed=0) -- and
records the held-out PSNRs (20 other directions) and primitive counts.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_desk_reference.py

(~20 min on 8 cores).  Writes tests/golden/desk_reference.json.
"""
import json
import os
import sys
import time

import numpy as np

for p in ("/root/reference/pkg/src",):
    if p not in sys.path:
        sys.path.insert(0, p)

from voxsplat import dvr  # noqa: E402
from voxsplat.gaussians import Camera  # noqa: E402
from voxsplat.metrics import psnr  # noqa: E402
from voxsplat.shading import LightConfig  # noqa: E402
from voxsplat.trainer import TrainConfig, render_model, train_base, train_editable  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
RES = 128


def fibonacci_dirs(n, offset=0.5):
    i = np.arange(n, dtype=np.float64) + offset
    z = 1.0 - 2.0 * i / n
    r = np.sqrt(np.maximum(1.0 - z * z, 0.0))
    phi = np.pi * (3.0 - np.sqrt(5.0)) * i
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def main():
    vol = dvr.make_shells_volume((64, 64, 64))
    tfs = [dvr.TransferFunction1D.basic_bump(0.35, 0.55, (0.2, 0.5, 0.9), 0.8),
           dvr.TransferFunction1D.basic_bump(0.60, 0.80, (0.9, 0.4, 0.15), 0.8)]
    light = LightConfig()
    lo, hi = vol.bbox
    radius = 1.1 * float(np.linalg.norm(np.asarray(hi) - np.asarray(lo)))
    cams = [Camera.look_at(radius * d, np.zeros(3), 0.8, RES, RES) for d in fibonacci_dirs(42)]
    held = [Camera.look_at(radius * d, np.zeros(3), 0.8, RES, RES)
            for d in fibonacci_dirs(20, 0.25)]
    out = {"rig": "42-view Fibonacci train, 20-view Fibonacci (offset 0.25) held out, 128^2",
           "config": "TrainConfig(stage1_iters=3000, stage2_iters=1000, seed=0)", "scenes": []}
    t0 = time.time()
    for tf in tfs:
        imgs = [dvr.render_view(vol, tf, c, light) for c in cams]
        ds = dvr.VolumeDataset(list(cams), imgs, light, {"volume": vol.descriptor(), "cameras": []})
        cfg = TrainConfig(stage1_iters=3000, stage2_iters=1000, seed=0)
        base, _ = train_base(ds, cfg)
        ed, _ = train_editable(base, ds, cfg)
        gts = [dvr.render_view(vol, tf, c, light) for c in held]
        b = float(np.mean([psnr(render_model(base, c, None, dtype=np.float64), g)
                           for c, g in zip(held, gts)]))
        e = float(np.mean([psnr(render_model(ed, c, light, dtype=np.float64), g)
                           for c, g in zip(held, gts)]))
        out["scenes"].append({"base_psnr": b, "editable_psnr": e,
                              "base_count": int(len(base.geometry.mu)),
                              "editable_count": int(len(ed.geometry.mu))})
        print(out["scenes"][-1], f"{time.time() - t0:.0f}s", flush=True)
    with open(os.path.join(HERE, "desk_reference.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
