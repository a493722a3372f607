"""One C3 StepGraph replay between cudaProfilerStart/Stop (ncu profiles the
graph's kernel nodes): the launch list of the product training step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_17954_b200 import LightConfig  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays  # noqa: E402
from paper_2504_17954_b200.trainer import EditableTrainer, StepGraph, _stage2_init  # noqa: E402

a = editable_arrays(0, 300_000, density=300_000)
light = LightConfig("orbital", 0.45, 0.9)
cam = bench_camera(800, 800, 0.3)
gt = EditableTrainer(a, a["palette"], light).render_rgba(cam).clone()
p = {k: a[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
p.update(_stage2_init(300_000))
tr = EditableTrainer(p, a["palette"], light)
G = StepGraph(tr, cam, gt)
for it in range(1, 4):
    G.step(cam, gt, it, 1000)
G.flush()
torch.cuda.synchronize()
torch.cuda.profiler.start()
G.step(cam, gt, 4, 1000)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
G.flush()
