"""One C2 frame between cudaProfilerStart/Stop, for an ncu launch list:

    ncu --profile-from-start off --metrics gpu__time_duration.sum \
        --clock-control none --csv python tools/frame_launches.py [--graph]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_17954_b200 import DeviceScene, FrameGraph  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, c2_scene  # noqa: E402

ds = DeviceScene(c2_scene())
cam = bench_camera()
ds.render_frame(cam, fast=False)
for _ in range(3):
    ds.render_frame(cam, fast=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
if "--graph" in sys.argv:
    fg = FrameGraph(ds, cam.width, cam.height)
    fg.replay(cam)
else:
    ds.render_frame(cam, fast=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
