"""Warp-stall samples of one kernel launch in an ncu report, aggregated per
CUDA source line (needs a -lineinfo build and --import-source on).

    python tools/ncu_hot.py rep.ncu-rep [launch_skip] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(skip), "--launch-count",
       "1", "--print-source", "cuda,sass"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
per_line = defaultdict(int)
text = {}
fname, func = "?", "?"
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        iss = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= iss:
        continue
    try:
        s = int(r[iss] or 0)
    except ValueError:
        continue
    key = (fname, r[0])
    per_line[key] += s
    if r[1].strip():
        text[key] = r[1].strip()
tot = sum(per_line.values()) or 1
print(func[:110])
print("total samples", tot)
for (f, ln), s in sorted(per_line.items(), key=lambda x: -x[1])[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}%  {f}:{ln:5s} {text.get((f, ln), '')[:95]}")
