"""K3 schedule trace for the C2 frame: per (tile, 8x4 block) unit start/end
times and SM, to see how much of the kernel is load-imbalance tail.

    python tools/blend_trace.py            (IVR_BLEND_QUEUE=0 for static CTAs)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17954_b200 import DeviceScene, _lib as L  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, c2_scene  # noqa: E402

ds = DeviceScene(c2_scene())
cam = bench_camera()
ds.render_frame(cam, fast=False)
for _ in range(3):
    ds.render_frame(cam, fast=True)
ntiles = 50 * 50
buf = torch.zeros(ntiles * 8 * 4, dtype=torch.int64, device="cuda")
torch.cuda.synchronize()
L.lib().ivr_debug_blend_trace(buf.data_ptr())
F = ds.render_frame(cam, fast=True, want_state=True)
torch.cuda.synchronize()
L.lib().ivr_debug_blend_trace(None)
tf = F.t_final.cpu().numpy()
lp = F.last_pos.cpu().numpy()
tr_all = buf.view(-1, 4).cpu().numpy()
idx = np.nonzero(tr_all[:, 3] > 0)[0]
tr = tr_all[idx]
t0 = tr[:, 2].min()
s, e = (tr[:, 2] - t0) / 1e3, (tr[:, 3] - t0) / 1e3
dur = e - s
span = e.max()
print(f"units {len(tr)}  span {span:.1f} us  sum {dur.sum():.0f} us  mean {dur.mean():.2f} "
      f"p99 {np.percentile(dur, 99):.1f} max {dur.max():.1f} us")
order = np.argsort(-dur)[:8]
tiles = F.tile_ranges.cpu().numpy()
blk_of = {}
for i in order:
    t = int(tr[i, 0])
    ty, tx = divmod(t, 50)
    b = int(idx[i] % 8)
    bx, by = (b % 2) * 8, (b // 2) * 4
    y0, x0 = ty * 16 + by, tx * 16 + bx
    tt = tf[y0:y0 + 4, x0:x0 + 8]
    ll = lp[y0:y0 + 4, x0:x0 + 8] - tiles[t]
    print(f"  tile {t:5d} pairs {tiles[t + 1] - tiles[t]:6d} sm {int(tr[i, 1]):3d} "
          f"start {s[i]:7.1f} dur {dur[i]:7.1f}  lanes stopped {(tt < 1e-4).sum():2d}/32 "
          f"max last {ll.max()}")
# busy-warp profile over time (units in flight)
grid = np.linspace(0, span, 21)
inflight = [int(((s <= g) & (e > g)).sum()) for g in grid]
print("units in flight at 5% steps:", inflight)
sm_busy_end = np.zeros(148)
for i in range(len(tr)):
    sm_busy_end[int(tr[i, 1])] = max(sm_busy_end[int(tr[i, 1])], e[i])
print("per-SM last finish: min %.1f median %.1f max %.1f us" % (sm_busy_end.min(), np.median(sm_busy_end), sm_busy_end.max()))
