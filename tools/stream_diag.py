"""C2 stream diagnostics: host submit cost and device throughput per slot
count.  Usage: python tools/stream_diag.py [frames]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2504_17954_b200 import DeviceScene  # noqa: E402
from paper_2504_17954_b200.scene import FrameGraph  # noqa: E402
from paper_2504_17954_b200.synthetic import bench_camera, c2_scene  # noqa: E402


def main(nf):
    ds = DeviceScene(c2_scene(bench.PER_MODEL, bench.N_MODELS, bench.DENSITY))
    cams = [bench_camera(bench.W_IMG, bench.H_IMG, bench.view_azimuth(0, s)) for s in range(nf)]
    F = ds.render_frame(cams[0], fast=False)
    torch.cuda.synchronize()
    for slots in (1, 2, 3, 4, 6, 8):
        fg = FrameGraph(ds, bench.W_IMG, bench.H_IMG, warm_cam=cams[0], slots=slots)
        for s in range(2 * slots):
            fg.submit(s % slots, cams[s])
        torch.cuda.synchronize()
        s0 = fg.stream(0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s0)
        for k in range(1, slots):
            fg.stream(k).wait_event(a)
        t0 = time.perf_counter()
        for s in range(nf):
            fg.submit(s % slots, cams[s])
        t1 = time.perf_counter()
        for k in range(1, slots):
            j = torch.cuda.Event()
            j.record(fg.stream(k))
            s0.wait_event(j)
        b.record(s0)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / nf
        print(f"slots {slots}: device {1000 / ms:7.1f} FPS ({ms * 1000:6.1f} us/frame), "
              f"host submit {(t1 - t0) / nf * 1e6:6.1f} us/frame", flush=True)
        del fg
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 120)
