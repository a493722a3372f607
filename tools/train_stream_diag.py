import sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_2504_17954_b200 import LightConfig
from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays
from paper_2504_17954_b200.trainer import EditableTrainer, _stage2_init, StepGraph
a = editable_arrays(0, 300_000, density=300_000)
light = LightConfig("orbital", 0.45, 0.9)
cams = [bench_camera(800, 800, az) for az in np.linspace(-3.0, 3.0, 8)]
gt_tr = EditableTrainer(a, a["palette"], light)
gts = [gt_tr.render_rgba(c).clone() for c in cams]
p = {k: a[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
p.update(_stage2_init(300_000))
tr = EditableTrainer(p, a["palette"], light)
G = StepGraph(tr, cams[0], gts[0])
it = [0]
def step():
    v = it[0] % len(cams); it[0] += 1
    G.step(cams[v], gts[v], it[0], 10000)
for _ in range(5): step()
torch.cuda.synchronize()
# host cost of staging alone
t0 = time.perf_counter()
for _ in range(20): G._stage(cams[1], gts[1], 5, 10000)
torch.cuda.synchronize()
print("stage host us", (time.perf_counter() - t0) / 20 * 1e6)
for mode in ("same_view", "rotating"):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for i in range(30):
        if mode == "same_view":
            G.step(cams[0], gts[0], it[0], 10000); it[0] += 1
        else:
            step()
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(mode, "device ms/step", e0.elapsed_time(e1) / 30, "host submit ms/step", (t1 - t0) / 30 * 1e3)
# replay only
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(30): G.g.replay()
e1.record(); torch.cuda.synchronize()
print("replay only ms", e0.elapsed_time(e1) / 30)
G.flush()
