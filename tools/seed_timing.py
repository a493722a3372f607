"""k-means++ seeding timing (ivr_kmeans_seed_sorted vs the full-pass
ivr_kmeans_seed) on N(0,1) values, k = 4096, with the sorted kernel's
per-phase split (CTA 0's clock: pick, wait for the pick, d2 update, grid
barrier, block re-sums, arrival)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17954_b200 import _lib as L  # noqa: E402
from paper_2504_17954_b200 import device as D  # noqa: E402


def al(v):
    return (v + 255) & ~255


K = 4096
for n in (4_000_000, 12_000_000, 16_000_000):
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    order = torch.argsort(x).to(torch.int32)
    for R in (1, 5):
        rng = np.random.default_rng(0)
        first = torch.tensor([int(rng.integers(n)) for _ in range(R)], dtype=torch.int64,
                             device="cuda")
        u = torch.from_numpy(rng.random(R * (K - 1))).cuda()
        c = torch.empty((R, K), dtype=torch.float64, device="cuda")
        nb = int(L.lib().ivr_kmeans_seed_sorted_workspace_size(n, R))
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.check(L.lib().ivr_kmeans_seed_sorted(D.ptr(x), D.ptr(order), n, K, R, D.ptr(first),
                                                   D.ptr(u), D.ptr(c), D.ptr(ws), nb,
                                                   D.stream_handle()), "s")
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
        # phase_ns sits after dcount [2 * 8] and ctl [4 * 8] and the arrival word
        ph = ws[nb - al(8 * 8 + 32 * 8 + 8 + 48) + 40 * 8 + 8:][:48].cpu().numpy().view(np.uint64)
        ph = ph / 1e3 / (K - 1)
        names = ("pick", "wait", "update", "barrier", "resum", "arrive")
        print(n, R, "seedings ms", round(ms, 1), "us/centre", round(ms * 1e3 / (K - 1), 2),
              {a: round(float(b), 2) for a, b in zip(names, ph)})
    first = int(first[0].item())
    u = u[:K - 1]
    c = c[0]
    wf = torch.empty(int(L.lib().ivr_kmeans_seed_workspace_size(n)), dtype=torch.uint8,
                     device="cuda")
    c2 = torch.empty_like(c)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.check(L.lib().ivr_kmeans_seed(D.ptr(x), n, K, first, D.ptr(u), D.ptr(c2), D.ptr(wf),
                                    wf.numel(), D.stream_handle()), "f")
    torch.cuda.synchronize()
    ms2 = (time.perf_counter() - t0) * 1e3
    print("   full-pass seeding ms", round(ms2, 1), "same centres", bool(torch.equal(c, c2)))
