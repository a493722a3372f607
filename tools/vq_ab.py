"""K5 assign / K6 decode timing on the C5 values (8 attributes of a 4M model,
K=4096), L2 flushed before each call, with a bit-equality check of the
indices against torch.searchsorted on the float64 midpoints.

    python tools/vq_ab.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2504_17954_b200.device import to_dev  # noqa: E402
from paper_2504_17954_b200.synthetic import editable_arrays  # noqa: E402
from paper_2504_17954_b200.vq import QUANTIZED_ATTRIBUTES, assign_device, decode_device  # noqa: E402

v = editable_arrays(0, 4_000_000, density=4_000_000)
host = np.concatenate([np.ascontiguousarray(v[nm]).reshape(-1) for nm, _ in QUANTIZED_ATTRIBUTES])
vals = to_dev(host)
cents = to_dev(np.sort(np.quantile(host[::97], np.linspace(0.0, 1.0, 4096))))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=6):
    ts = []
    for _ in range(reps):
        flush.zero_()
        ev[0].record()
        r = fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return min(ts[1:]), r


n = vals.numel()
a_ms, idx = timed(lambda: assign_device(vals, cents))
d_ms, (out, _) = timed(lambda: decode_device(idx, cents))
mids = 0.5 * (cents[1:] + cents[:-1])
ref = torch.searchsorted(mids, vals, side="left")
print(f"assign {a_ms * 1e3:.1f} us  {n * 10 / (a_ms * 1e-3) / 1e9:.0f} GB/s (10 B/value)  "
      f"equal to searchsorted {bool(torch.equal(idx.long(), ref))}")
print(f"decode {d_ms * 1e3:.1f} us  {n * 10 / (d_ms * 1e-3) / 1e9:.0f} GB/s (10 B/value)  "
      f"equal to gather {bool(torch.equal(out, cents[idx.long()]))}")
