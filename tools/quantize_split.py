"""C5 quantize_model (4M editable model, K=4096) with the host wall time split
into seeding, Lloyd, value sort, SSE, assign, decode, uploads and the rest."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_17954_b200 import vq  # noqa: E402
from paper_2504_17954_b200.synthetic import editable_model  # noqa: E402

acc = collections.defaultdict(float)


def timed(name, fn):
    def w(*a, **k):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        acc[name] += time.perf_counter() - t
        return r
    return w


vq._seed_plusplus = timed("seed", vq._seed_plusplus)
vq._seed_batch = timed("seed", vq._seed_batch)
vq._lloyd = timed("lloyd", vq._lloyd)
vq._lloyd_sets = timed("lloyd", vq._lloyd_sets)
vq._value_order = timed("sort", vq._value_order)
vq._sse = timed("sse", vq._sse)
vq.assign_device = timed("assign", vq.assign_device)
vq.Codebook.decode = timed("decode", vq.Codebook.decode)
vq.D.to_dev = timed("upload", vq.D.to_dev)
m = editable_model(0, 4_000_000, density=4_000_000)
vq.quantize_model(m, k=64, seed=0)  # warm-up (kernels, allocator)
acc.clear()
torch.cuda.synchronize()
t0 = time.perf_counter()
vq.quantize_model(m, k=4096, seed=0)
torch.cuda.synchronize()
tot = time.perf_counter() - t0
print({"total_s": round(tot, 3), **{k: round(v, 3) for k, v in acc.items()},
       "rest": round(tot - sum(acc.values()), 3)})
