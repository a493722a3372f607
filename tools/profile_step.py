"""Kernel-time breakdown (torch.profiler) of one C3 training step or one C4
inverse iteration.  Usage: python tools/profile_step.py [train|inverse|inverse_host]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main(which):
    from paper_2504_17954_b200 import LightConfig
    from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays, c2_scene
    from paper_2504_17954_b200.trainer import EditableTrainer, _stage2_init
    if which == "train":
        a = editable_arrays(0, 300_000, density=300_000)
        light = LightConfig("orbital", 0.45, 0.9)
        cam = bench_camera(800, 800, 0.3)
        gt = EditableTrainer(a, a["palette"], light).render_rgba(cam).clone()
        p = {k: a[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
        p.update(_stage2_init(300_000))
        tr = EditableTrainer(p, a["palette"], light)

        def step():
            loss, grads, _ = tr.step(cam, gt)
            tr.apply(grads, 1, 100)
    else:
        from paper_2504_17954_b200.inverse import InverseFitter, init_transform
        sc = c2_scene()
        cam = bench_camera(800, 800, 0.8)
        p0 = init_transform(sc)
        fit = InverseFitter(sc, [], [])
        ref = fit.render(p0, cam).out64.clone() * 0.95
        fit = InverseFitter(sc, [ref], [cam], ds=fit.ds)

        if which == "inverse_host":
            def step():
                fit.view_grads(p0, 0)
        else:  # the product path: one InverseGraph replay per iteration
            from paper_2504_17954_b200.inverse import InverseGraph
            step = InverseGraph(fit, p0, 100_000).replay
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for _ in range(10):
        step()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 10
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(5):
            step()
        torch.cuda.synchronize()
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=35))
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    busy = sum(e.device_time for e in ev) / 5 / 1e3
    print(f"wall {wall * 1e3:.2f} ms/step, GPU kernel time {busy:.2f} ms/step, "
          f"{len(ev) / 5:.0f} kernels/step")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "train")
