"""C3 stage-2 step timing (bench.py's train leg: StepGraph replays, FAST and
EXACT blends, eager per-stage split) for A/B runs of library builds.
    IVR_LIB_PATH=... python tools/train_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.bench_train(None)
print(os.environ.get("IVR_LIB_PATH", "in-tree").split("/")[-1], round(r["ms_per_it"], 4),
      "exact", round(r["exact_blend"]["ms_per_it"], 4),
      {k.split("(")[0].strip(): round(v, 4) for k, v in r["split_ms_eager"].items()})
