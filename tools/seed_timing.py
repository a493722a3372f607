"""k-means++ seeding timing on N(0,1) values, k = 4096: ivr_kmeans_seed_sorted
for 1 and 5 seedings of one attribute per launch (with CTA 0's per-phase
split: pick, wait for the picks, d2 update, grid barrier, block re-sums,
arrival) against the full-pass ivr_kmeans_seed, which must pick the same
centres."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17954_b200 import _lib as L  # noqa: E402
from paper_2504_17954_b200 import device as D  # noqa: E402
from paper_2504_17954_b200 import vq  # noqa: E402

K = 4096
for n in (4_000_000, 12_000_000, 16_000_000):
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    order = torch.argsort(x).to(torch.int32)
    for R in (1, 5):
        draws = vq._draw_seeds(n, K, np.random.default_rng(0), R)
        u = torch.from_numpy(np.concatenate([d[1] for d in draws])).cuda()
        c = torch.empty((R, K), dtype=torch.float64, device="cuda")
        arr = (L.SeedProblem_t * R)()
        for i, (f, _) in enumerate(draws):
            arr[i].values, arr[i].order, arr[i].n, arr[i].first = D.ptr(x), D.ptr(order), n, f
            arr[i].u, arr[i].centers = u.data_ptr() + 8 * (K - 1) * i, D.ptr(c[i])
        nb = int(L.lib().ivr_kmeans_seed_sorted_workspace_size(arr, R))
        ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
        for rep in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            L.check(L.lib().ivr_kmeans_seed_sorted(arr, R, K, D.ptr(ws), nb, D.stream_handle()),
                    "s")
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
        ph = ws[64:64 + 48].cpu().numpy().view(np.uint64) / 1e3 / (K - 1)
        names = ("pick", "wait", "update", "barrier", "resum", "arrive")
        print(n, R, "seedings ms", round(ms, 1), "us/centre", round(ms * 1e3 / (K - 1), 2),
              {a: round(float(b), 2) for a, b in zip(names, ph)})
    first, u0 = draws[0]
    wf = torch.empty(int(L.lib().ivr_kmeans_seed_workspace_size(n)), dtype=torch.uint8,
                     device="cuda")
    c2 = torch.empty(K, dtype=torch.float64, device="cuda")
    uu = torch.from_numpy(u0).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.check(L.lib().ivr_kmeans_seed(D.ptr(x), n, K, first, D.ptr(uu), D.ptr(c2), D.ptr(wf),
                                    wf.numel(), D.stream_handle()), "f")
    torch.cuda.synchronize()
    ms2 = (time.perf_counter() - t0) * 1e3
    print("   full-pass seeding ms", round(ms2, 1), "same centres", bool(torch.equal(c[0], c2)))

# every attribute's 5 restart seedings of a 4M editable model in one launch,
# as quantize_attributes makes them
from paper_2504_17954_b200.synthetic import editable_model  # noqa: E402

m = editable_model(0, 4_000_000, density=4_000_000)
probs, keep = [], []
for name, owner in vq.QUANTIZED_ATTRIBUTES:
    xa = D.to_dev(np.asarray(getattr(getattr(m, owner), name), dtype=np.float64).reshape(-1))
    o = vq._value_order(xa)
    keep.append((xa, o))
    probs.extend((xa, o, f, u) for f, u in vq._draw_seeds(xa.numel(), K, np.random.default_rng(0), 5))
u = torch.from_numpy(np.concatenate([p[3] for p in probs])).cuda()
c = torch.empty((len(probs), K), dtype=torch.float64, device="cuda")
arr = (L.SeedProblem_t * len(probs))()
for i, (xa, o, f, _) in enumerate(probs):
    arr[i].values, arr[i].order, arr[i].n, arr[i].first = D.ptr(xa), D.ptr(o), xa.numel(), f
    arr[i].u, arr[i].centers = u.data_ptr() + 8 * (K - 1) * i, D.ptr(c[i])
nb = int(L.lib().ivr_kmeans_seed_sorted_workspace_size(arr, len(probs)))
ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L.check(L.lib().ivr_kmeans_seed_sorted(arr, len(probs), K, D.ptr(ws), nb, D.stream_handle()),
            "s")
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
ph = ws[64:64 + 48].cpu().numpy().view(np.uint64) / 1e3 / (K - 1)
print("4M model,", len(probs), "seedings in one launch: ms", round(ms, 1), "us/centre",
      round(ms * 1e3 / (K - 1), 2),
      {a: round(float(b), 2) for a, b in zip(("pick", "wait", "update", "barrier", "resum",
                                              "arrive"), ph)})
