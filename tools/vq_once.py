"""One K5 assign + K6 decode over 60M values (K=4096) between
cudaProfilerStart/Stop, for ncu --profile-from-start off."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2504_17954_b200.vq import assign_device, decode_device  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
vals = torch.randn(60_000_000, dtype=torch.float64, device="cuda", generator=g)
cents = torch.sort(torch.randn(4096, dtype=torch.float64, device="cuda", generator=g)).values
idx = assign_device(vals, cents)
decode_device(idx, cents)
torch.cuda.synchronize()
torch.cuda.profiler.start()
idx = assign_device(vals, cents)
decode_device(idx, cents)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
