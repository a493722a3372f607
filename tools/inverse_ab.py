"""C4 inverse-iteration timing (bench.py's inverse leg) for A/B runs.
    python tools/inverse_ab.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2504_17954_b200.synthetic import c2_scene  # noqa: E402

r = bench.bench_inverse(c2_scene())
print("inverse", round(r["ms_per_it"], 4), {k: round(v, 4) for k, v in r["split_ms_eager"].items()})
