"""Per-tile work distribution of the C2 frame (load-balance diagnostics)."""
import numpy as np
import torch

from paper_2504_17954_b200 import DeviceScene
from paper_2504_17954_b200.synthetic import bench_camera, c2_scene

sc = c2_scene()
ds = DeviceScene(sc)
cam = bench_camera()
F = ds.render_frame(cam, fast=False, want_state=True, exact=False)
torch.cuda.synchronize()
tr = F.tile_ranges.cpu().numpy().astype(np.int64)
cnt = np.diff(tr)
contrib = F.contrib.cpu().numpy()
last = F.last_pos.cpu().numpy().astype(np.int64)
ntx = F.ntx
H, W = contrib.shape
ty, tx = np.divmod(np.arange(len(cnt)), ntx)
# per-tile walked length = max over its pixels of (last_pos - start)
walk = np.zeros(len(cnt), np.int64)
for t in range(len(cnt)):
    y0, x0 = ty[t] * 16, tx[t] * 16
    lp = last[y0:y0 + 16, x0:x0 + 16]
    walk[t] = max(int(lp.max()) - tr[t], 0)
print("tiles", len(cnt), "pairs", cnt.sum())
for name, v in (("pairs/tile", cnt), ("walked/tile", walk)):
    q = np.percentile(v, [50, 90, 99, 100])
    print(name, "mean %.0f" % v.mean(), "p50/p90/p99/max", q.astype(int).tolist())
slots = 148 * 3
srt = np.sort(walk)[::-1]
print("max walk / (sum walk / %d slots) = %.2f" % (slots, srt[0] / (srt.sum() / slots)))
print("contrib mean %.1f max %d" % (contrib.mean(), contrib.max()))
