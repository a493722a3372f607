"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): one C1 frame (10k Gaussians, 128x128; FAST and EXACT blends,
eager and as a captured FrameGraph), one stage-2 training step (K=15, every
loss term, K4a/K4b, Adam), one inverse iteration (InverseGraph), a
deterministic K4a backward, VQ assign / decode.

    compute-sanitizer --tool racecheck python tools/sanitize_once.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17954_b200 import ComposedScene, DeviceScene, LightConfig  # noqa: E402
from paper_2504_17954_b200.inverse import InverseFitter, InverseGraph, init_transform  # noqa: E402
from paper_2504_17954_b200.scene import FrameGraph  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays, editable_model  # noqa: E402
from paper_2504_17954_b200.trainer import EditableTrainer, _stage2_init  # noqa: E402
from paper_2504_17954_b200.vq import assign_device, decode_device  # noqa: E402

W = H = 128
scene = ComposedScene.compose([editable_model(s, 5000, density=10_000) for s in range(2)],
                              LightConfig("orbital", 0.45, 0.9))
cam = bench_camera(W, H)
ds = DeviceScene(scene)
for exact in (True, False):
    ds.render(cam, fast=not exact, exact=exact)
fg = FrameGraph(ds, W, H, warm_cam=cam)
fg.replay(bench_camera(W, H, 0.3))
torch.cuda.synchronize()
print("render ok")

a = editable_arrays(0, 10_000, density=10_000)
p = {k: a[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
p.update(_stage2_init(10_000))
tr = EditableTrainer(p, a["palette"], LightConfig("orbital", 0.45, 0.9))
gt = torch.rand((H, W, 4), dtype=torch.float64, device="cuda")
loss, grads, stat = tr.step(cam, gt)
tr.apply(grads, 1, 100)
os.environ["IVR_DETERMINISTIC"] = "1"
tr.step(cam, gt)
os.environ["IVR_DETERMINISTIC"] = "0"
torch.cuda.synchronize()
print("train ok")

fit0 = InverseFitter(scene, [], [])
ref = fit0.render(init_transform(scene), cam).out64.clone() * 0.9
fit = InverseFitter(scene, [ref], [cam], ds=fit0.ds)
G = InverseGraph(fit, init_transform(scene), 4)
G.run()
torch.cuda.synchronize()
print("inverse ok")

vals = torch.from_numpy(np.random.default_rng(0).normal(size=200_000)).cuda()
cents = torch.sort(torch.from_numpy(np.random.default_rng(1).normal(size=4096)).cuda()).values
idx = assign_device(vals, cents)
decode_device(idx, cents)
torch.cuda.synchronize()
print("vq ok")
