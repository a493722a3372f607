"""Lloyd step timing at k = 4096 on N(0,1) values: the atomic form
(ivr_kmeans_lloyd_step, float64 sums privatised in shared memory) and the
sorted form (ivr_kmeans_lloyd_step_sorted: segment sums between midpoints)
for 1 and 5 centroid sets."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17954_b200 import _lib as L  # noqa: E402
from paper_2504_17954_b200 import device as D  # noqa: E402
from paper_2504_17954_b200 import vq  # noqa: E402


def dev_us(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


K = 4096
for n in (4_000_000, 16_000_000):
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    xs = torch.sort(x).values
    seeds = vq._seed_restarts(x, K, np.random.default_rng(0), 5)
    c = torch.sort(seeds, dim=1).values.contiguous()
    nb = L.lib().ivr_kmeans_lloyd_workspace_size(K)
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    sh = torch.empty(5, dtype=torch.float64, device="cuda")
    new = torch.empty_like(c)
    t_atomic = dev_us(lambda: L.lib().ivr_kmeans_lloyd_step(
        D.ptr(x), n, D.ptr(c), K, D.ptr(new), D.ptr(sh), D.ptr(ws), nb, D.stream_handle()))
    res = {"atomic_1set_us": round(t_atomic, 1)}
    for sets in (1, 5):
        nb2 = int(L.lib().ivr_kmeans_lloyd_sorted_workspace_size(K, sets))
        ws2 = torch.empty(nb2, dtype=torch.uint8, device="cuda")
        res[f"sorted_{sets}set_us"] = round(dev_us(lambda: L.lib().ivr_kmeans_lloyd_step_sorted(
            D.ptr(xs), n, D.ptr(c), K, sets, D.ptr(new), D.ptr(sh), D.ptr(ws2), nb2,
            D.stream_handle())), 1)
    print(n, res)
