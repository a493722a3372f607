"""One C3 stage-2 training step between cudaProfilerStart/Stop (for ncu with
--profile-from-start off)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_17954_b200 import LightConfig  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays  # noqa: E402
from paper_2504_17954_b200.trainer import EditableTrainer, _stage2_init  # noqa: E402

a = editable_arrays(0, 300_000, density=300_000)
light = LightConfig("orbital", 0.45, 0.9)
cam = bench_camera(800, 800, 0.3)
gt = EditableTrainer(a, a["palette"], light).render_rgba(cam).clone()
p = {k: a[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
p.update(_stage2_init(300_000))
tr = EditableTrainer(p, a["palette"], light)
for _ in range(3):
    loss, grads, _ = tr.step(cam, gt)
    tr.apply(grads, 1, 100)
torch.cuda.synchronize()
torch.cuda.profiler.start()
loss, grads, _ = tr.step(cam, gt)
tr.apply(grads, 1, 100)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
