"""One C4 inverse iteration between cudaProfilerStart/Stop (ncu): one replay
of the InverseGraph (render + loss + backward + pack + device Adam); ncu
profiles the graph's kernel nodes one by one."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_17954_b200.inverse import InverseFitter, InverseGraph, init_transform  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, c2_scene  # noqa: E402

sc = c2_scene()
cam = bench_camera(800, 800, 0.8)
p0 = init_transform(sc)
fit0 = InverseFitter(sc, [], [])
ref = fit0.render(p0, cam).out64.clone() * 0.95
fit = InverseFitter(sc, [ref], [cam], ds=fit0.ds)
G = InverseGraph(fit, p0, 1000)
for _ in range(3):
    G.replay()
torch.cuda.synchronize()
torch.cuda.profiler.start()
G.replay()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
