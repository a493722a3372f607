#!/usr/bin/env python
"""Benchmark: 800x800 render FPS of the composed ~1M-Gaussian editable model
(BASELINE.json configs[1]) on the B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one frame of the hot path over the resident composed model: K1
(edits + projection + Blinn-Phong) -> K2 (bit-exact bin/sort) -> K3 (tile
blend), with the C2 edit sequence applied.  Under torchrun each rank renders
its own views of a full replica (views are independent: weak scaling, no
data-path collective).  Rank 0 prints ONE JSON line.

``--impl reference`` times the reference algorithm on the host cores through
the CPU port in oracle/ (the reference is a Python/numba package that cannot
be built into a library here), on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "800x800 render FPS (composed 1M Gaussians), train it/s, % HBM roofline, 1-8 GPU"
W_IMG = H_IMG = 800
PER_MODEL, N_MODELS, DENSITY = 200_000, 5, 1_000_000
# our kernels per frame: K1 (1) + K2 (init, minmax, coarse key, 4x3 radix, fix-up,
# fallback gate, 3 scan, tile hist, tile rowscan, tile ranges, placement, tile order
# = 25) + K3 (1)
def launches_per_frame(n):
    """Kernels in one captured frame: K1; K2 = init + minmax + 3 per radix
    pass (the first upsweep also maps the coarse keys) + fix-up + fallback
    gate + hist + rowscan + tile ranges (also P) + placement; tile order; K3
    (sort.cu / blend.cu)."""
    lg = 1
    while (1 << lg) < n:
        lg += 1
    passes = min(max((lg + 4 + 7) // 8, 2), 4)
    return 1 + (2 + 3 * passes + 2 + 4) + 1 + 1


SLOTS = int(os.environ.get("IVR_SLOTS", "6"))  # concurrent frame slots (FrameGraph / FramePipeline)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=2)
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the C3 train / C4 inverse / C5 VQ secondary measurements")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), ws


def view_azimuth(rank, step):
    """Camera views: rank r renders its own orbit azimuths (independent views)."""
    base = 0.8 + 0.7 * rank
    return float(np.arctan2(np.sin(base + 0.01 * step), np.cos(base + 0.01 * step)))


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled every 2 ms through
    NVML (the data behind nvidia-smi's clocks.sm / clocks_event_reasons.*)
    on a background thread during the timed region."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4),
               ("hw_power_brake_slowdown", 0x80))

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            visible = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(visible.split(",")[self.gpu]) if visible else self.gpu
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
        except Exception:
            return

        def loop():
            while not self._stop.is_set():
                try:
                    self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                    r = int(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
                    for nm, bit in self.REASONS:
                        if r & bit:
                            self.reasons.add(nm)
                except Exception:
                    pass
                time.sleep(0.002)

        self.t = threading.Thread(target=loop, daemon=True)
        self.t.start()

    def stop(self):
        self._stop.set()
        if self.t is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        self.t.join(timeout=2)
        return {"sm_mhz": float(np.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ CPU side
def cpu_frames(scene_arrays, cam, frames, nthreads=0):
    """The reference algorithm for one C2 frame on the host (oracle/ port:
    numpy per-Gaussian math + C/OpenMP compositor).  Returns (sec/frame, threads)."""
    import oracle as O
    a = scene_arrays
    times = []
    for _ in range(frames):
        t0 = time.perf_counter()
        o_eff = O.effective_o_logit(a["o_logit"], a["opacity_scale"])
        rgb, _ = O.shade(a["mu"], a["n_raw"], a["delta_c"], a["k_a_raw"], a["k_d_raw"],
                         a["k_s_raw"], a["log_beta"], a["palette_rgb"], a["light"], cam)
        st = O.rasterize(a["mu"], a["q_raw"], a["log_s"], o_eff, a["n_raw"], rgb, cam,
                         dtype=np.float32, nthreads=nthreads)
        O.maps(st)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), O.max_threads() if nthreads <= 0 else nthreads


def host_scene_arrays(scene):
    models = scene.models
    cat = {k: np.concatenate([getattr(m.geometry, k) for m in models])
           for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
    cat.update({k: np.concatenate([getattr(m.shading, k) for m in models])
                for k in ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")})
    cat["palette_rgb"] = np.concatenate([
        np.broadcast_to(e.palette_override if e.palette_override is not None else m.palette.c_p,
                        (len(m), 3)) for m, e in zip(models, scene.edits)])
    cat["opacity_scale"] = np.concatenate([np.full(len(m), e.opacity_scale)
                                           for m, e in zip(models, scene.edits)])
    lt = scene.light
    cat["light"] = (lt.mode, lt.polar, lt.azimuth, lt.term_scales)
    return cat


def config_dict(n, extra=None):
    d = {"workload": "C2: composed 5x200k editable Gaussians (density 1M), 800x800 fwd + "
                     "relight/TF edit (palette override, opacity 0.5, orbital light, term scales)",
         "n_gaussians": n, "width": W_IMG, "height": H_IMG, "channels": "rgba",
         "dtype_mode": "float32 (reference default)",
         "l2": "inputs larger than L2 (scene 168 MB float64 > 126 MB); frames streamed on "
               "6 concurrent slots; frame_ms_isolated = each frame alone after an L2 flush"}
    if extra:
        d.update(extra)
    return d


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    from paper_2504_17954_b200.synthetic import bench_camera, c2_scene
    scene = c2_scene(PER_MODEL, N_MODELS, DENSITY)
    arrays = host_scene_arrays(scene)
    cam = bench_camera(W_IMG, H_IMG, view_azimuth(0, 0))
    cpu_frames(arrays, cam, 1)  # warm (first-touch, thread pool)
    steps = max(1, min(args.steps, 3))
    sec, thr = cpu_frames(arrays, cam, steps)
    fps = 1.0 / sec
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": 1, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": config_dict(len(arrays["mu"])),
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": thr, "kind": "port",
                             "sample": f"{steps} full C2 frames (1M Gaussians, 800x800) through "
                                       "oracle/ (numpy + C/OpenMP compositor)"},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _device_time(fn, steps, warmup=2):
    """Mean device ms of fn() over `steps` calls (CUDA events, L2 flushed)."""
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.mean(ts)), float(np.median(ts))


def _max_over_ranks(x, dist):
    import torch
    if dist is None:
        return x
    t = torch.tensor([x], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def bench_train(scene, dist=None, world=1, rank=0):
    """C3: stage-2 training step (K=15 channels, fwd + all losses + bwd +
    Adam) on one 300k-Gaussian basic model at 800x800, one view / iteration.
    With N ranks every rank trains its own basic TF (independent seeds, no
    communication): aggregate it/s = N / slowest rank's ms per iteration."""
    from paper_2504_17954_b200 import LightConfig
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays
    from paper_2504_17954_b200.trainer import EditableTrainer, _stage2_init
    a = editable_arrays(rank, 300_000, density=300_000)
    light = LightConfig("orbital", 0.45, 0.9)
    cams = [bench_camera(W_IMG, H_IMG, az) for az in np.linspace(-3.0, 3.0, 8)]
    gt_tr = EditableTrainer(a, a["palette"], light)
    gts = [gt_tr.render_rgba(c).clone() for c in cams]
    p = {k: a[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
    p.update(_stage2_init(300_000))
    tr = EditableTrainer(p, a["palette"], light)
    it = [0]
    # the product path: the whole step (fwd, losses, bwd, Adam) as one CUDA graph
    from paper_2504_17954_b200.trainer import StepGraph
    G = StepGraph(tr, cams[0], gts[0])

    def step():
        v = it[0] % len(cams)
        it[0] += 1
        G.step(cams[v], gts[v], it[0], 10000)
    mean_ms, med_ms = _device_time(step, 10)
    G.flush()
    mean_ms = _max_over_ranks(mean_ms, dist)
    return {"metric": "stage-2 train it/s (300k Gaussians, 800x800, K=15, 1 view/it)",
            "value": world * 1000.0 / mean_ms, "unit": "it/s", "ms_per_it": mean_ms,
            "ms_per_it_median": med_ms, "n_gaussians": 300_000, "n_gpus": world,
            "scaling": "weak (one basic TF per GPU)",
            "note": "StepGraph replay: fwd (K1-K3), L1+SSIM + normal/offset/bilateral/opacity "
                    "terms, K4a+K4b, gradient assembly, Adam; densify excluded"}


def bench_inverse(scene, dist=None, world=1, rank=0):
    """C4: one inverse-exploration iteration on the composed 1M scene (render
    f64-semantics + loss + transform-only backward + Adam).  N ranks shard N
    views (one each); the packed transform gradient is all-reduced (NCCL,
    4S+12 float64) every iteration and every rank applies the same Adam."""
    from paper_2504_17954_b200.inverse import InverseFitter, InverseGraph, init_transform
    from paper_2504_17954_b200.synthetic import bench_camera
    cam = bench_camera(W_IMG, H_IMG, 0.8 + 0.7 * rank)
    p_true = init_transform(scene)
    p_true.lam = np.array([1.2, 0.8, 1.0, 1.0])
    fit0 = InverseFitter(scene, [], [])
    ref = fit0.render(p_true, cam).out64.clone()
    fit = InverseFitter(scene, [ref], [cam], ds=fit0.ds)
    params = init_transform(scene)
    # the product path: whole iterations replayed as CUDA graphs (InverseGraph:
    # device Adam + table refresh, no host round trip); with N ranks one
    # stream-ordered NCCL all-reduce of the packed gradient per iteration
    step = InverseGraph(fit, params, 100_000, dist=dist, view_div=float(world)).replay
    note = ("whole iterations replayed as CUDA graphs (InverseGraph: device Adam)" +
            ("; views sharded, one NCCL all-reduce per iteration between the compute "
             "and update graphs" if dist is not None else ""))
    mean_ms, med_ms = _device_time(step, 10)
    mean_ms = _max_over_ranks(mean_ms, dist)
    return {"metric": "inverse exploration it/s (composed 1M, 800x800, 1 view per GPU)",
            "value": 1000.0 / mean_ms, "unit": "it/s", "views_per_s": world * 1000.0 / mean_ms,
            "ms_per_it": mean_ms, "ms_per_it_median": med_ms, "n_gpus": world,
            "scaling": "weak (views sharded, one NCCL all-reduce of 4S+12 float64 per iteration)",
            "note": note}


def bench_vq(scene):
    """C5: K5 assign + K6 decode over the 60M scalar attribute values of a 4M
    editable model with a 4096-entry codebook (HBM-bound)."""
    import torch
    from paper_2504_17954_b200.vq import assign_device, decode_device
    n_vals = 4_000_000 * 15
    g = torch.Generator(device="cuda").manual_seed(0)
    vals = torch.randn(n_vals, dtype=torch.float64, device="cuda", generator=g)
    cents = torch.sort(torch.randn(4096, dtype=torch.float64, device="cuda", generator=g)).values
    out = {}
    a_ms, _ = _device_time(lambda: out.__setitem__("idx", assign_device(vals, cents)), 5)
    d_ms, _ = _device_time(lambda: decode_device(out["idx"], cents), 5)
    hbm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6650.0)) \
        if os.path.exists(os.path.join(REPO, "MEASURED_PEAKS.json")) else 6650.0
    a_gbs = n_vals * 10 / (a_ms * 1e-3) / 1e9
    d_gbs = n_vals * 10 / (d_ms * 1e-3) / 1e9
    return {"metric": "VQ assign/decode over 60M values, K=4096", "assign_ms": a_ms,
            "decode_ms": d_ms, "assign_gbs": a_gbs, "decode_gbs": d_gbs,
            "assign_hbm_frac": a_gbs / hbm, "decode_hbm_frac": d_gbs / hbm,
            "alg_bytes_per_value": 10}


def bench_service(scene):
    """§8(f) service frame path: one 800x800 'shaded' frame rendered (float64
    semantics, as render_mode_image) and delivered as PNG bytes / raw uint8 on
    the host (device display + PNG assembly, one D2H per frame)."""
    import time as _t
    from paper_2504_17954_b200.render_modes import DisplayRenderer
    from paper_2504_17954_b200.synthetic import bench_camera
    R = DisplayRenderer(scene)
    cams = [bench_camera(W_IMG, H_IMG, 0.1 * i) for i in range(12)]
    res = {}
    for fmt in ("png", "raw"):
        for c in cams[:2]:
            R.frame_bytes(c, "shaded", fmt)
        t0 = _t.perf_counter()
        nb = 0
        for c in cams:
            nb = len(R.frame_bytes(c, "shaded", fmt))
        dt = (_t.perf_counter() - t0) / len(cams)
        res[fmt] = {"frames_per_s": 1.0 / dt, "bytes_per_frame": nb}
    return {"metric": "service frames/s (800x800 shaded, float64 render, bytes on the host)",
            "png": res["png"], "raw": res["raw"],
            "note": "host wall clock per synchronous frame (render + display kernel + device PNG "
                    "+ D2H); reference: render_mode_image + PIL png_bytes on the CPU"}


def bench_dvr(scene):
    """§8(f) 4: ground-truth volume rendering for dataset generation, one
    800x800 view of a 128^3 'lobes' volume (float64 ray march on the GPU)."""
    from paper_2504_17954_b200 import LightConfig, orbit_camera
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.dvr import (TransferFunction1D, make_volume, render_view_device,
                                           union_transfer_functions)
    vol = make_volume("lobes", (128, 128, 128))
    tf = union_transfer_functions([TransferFunction1D.basic_bump(0.2, 0.45, (0.9, 0.3, 0.2), 0.8),
                                   TransferFunction1D.basic_bump(0.55, 0.8, (0.2, 0.5, 0.9), 0.6)])
    vals = to_dev(vol.values)
    cams = [orbit_camera(np.zeros(3), 330.0, 0.3, a, 0.8, W_IMG, H_IMG) for a in np.linspace(0, 6, 6)]
    it = [0]

    def one():
        render_view_device(vol, tf, cams[it[0] % len(cams)], LightConfig(), dev_values=vals)
        it[0] += 1
    mean_ms, med_ms = _device_time(one, 5)
    return {"metric": "DVR views/s (800x800, 128^3 volume, float64 ray march)",
            "value": 1000.0 / mean_ms, "unit": "views/s", "ms_per_view": mean_ms}


def run_ours(args):
    import torch
    rank, local_rank, world = dist_env()
    dev_idx = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev_idx)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("IVR_DIST_BACKEND", "nccl")  # gloo: functional test only
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev_idx))
        else:
            dist.init_process_group(backend)
    from paper_2504_17954_b200 import DeviceScene
    from paper_2504_17954_b200.synthetic import bench_camera, c2_scene

    scene = c2_scene(PER_MODEL, N_MODELS, DENSITY)
    ds = DeviceScene(scene)
    n = ds.n
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    cams = [bench_camera(W_IMG, H_IMG, view_azimuth(rank, s))
            for s in range(max(args.steps, 10) + args.warmup)]

    # warm-up: first frame learns the pair capacity (one sync), then fast frames
    F = ds.render_frame(cams[0], fast=False)
    for s in range(args.warmup):
        F = ds.render_frame(cams[s], fast=True)
    torch.cuda.synchronize()
    assert not ds.check_overflow(F)

    # ---- per-kernel split (instrumented, un-captured launches; L2 flushed per frame)
    n_split = max(3, min(args.steps, 10))
    sev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n_split)]
    for s in range(n_split):
        flush.zero_()
        ds.render_frame(cams[args.warmup + s], fast=True, events=sev[s])
    torch.cuda.synchronize()
    stage = np.array([[sev[s][i].elapsed_time(sev[s][i + 1]) for i in range(3)]
                      for s in range(n_split)])

    # ---- the product path: the whole frame captured once as a CUDA graph
    from paper_2504_17954_b200.scene import FrameGraph
    fg = FrameGraph(ds, W_IMG, H_IMG, warm_cam=cams[0], slots=SLOTS)
    for s in range(args.warmup):
        fg.submit(s % SLOTS, cams[s])
    torch.cuda.synchronize()

    # ---- (diagnostic) each frame alone: L2 flushed before it, slot 0 only
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    for s in range(args.steps):
        flush.zero_()                      # L2 flush between timed frames (not timed)
        fg.stage(cams[args.warmup + s])    # this frame's camera/edit upload (not timed)
        ev[s][0].record()
        fg.launch()
        ev[s][1].record()
    torch.cuda.synchronize()
    overflow = fg.overflowed()
    frame_ms = np.array([ev[s][0].elapsed_time(ev[s][1]) for s in range(args.steps)])

    # ---- the headline: a stream of K views, consecutive frames on SLOTS
    # slots (own streams / workspaces) so later frames' K1/K2 overlap earlier
    # frames' K3 tails; the scene (168 MB float64) exceeds the 126 MB L2
    s0 = fg.stream(0)
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local_rank)
    sampler.start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(s0)
    for k in range(1, SLOTS):
        fg.stream(k).wait_event(t_start)
    for s in range(args.steps):
        fg.submit(s % SLOTS, cams[args.warmup + s])
    for k in range(1, SLOTS):
        j = torch.cuda.Event()
        j.record(fg.stream(k))
        s0.wait_event(j)
    t_end.record(s0)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()
    overflow = overflow or any(int(F.n_pairs.item()) > fg.capacity for _, F in fg.graphs)
    frames = [fg.F]
    ms = t_start.elapsed_time(t_end) / args.steps
    t_tot = ms * args.steps / 1e3
    if dist:
        tt = torch.tensor([t_tot], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_tot = float(tt.item())
    fps_total = world * args.steps / t_tot

    # ---- end-to-end through the public API with host buffers: every frame
    # uploads its camera/light/edit tables from pinned memory and its RGBA +
    # per-pixel contribution counts land in pinned host buffers; frame i+1's
    # upload + compute overlaps frame i's device->host copy (FramePipeline)
    from collections import deque

    from paper_2504_17954_b200.scene import FramePipeline
    pipe = FramePipeline(fg)
    e2e_steps = max(10, min(args.steps, 50))
    for s in range(3):
        pipe.result(pipe.submit(cams[s]))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    inflight = deque()
    for s in range(e2e_steps):
        inflight.append(pipe.submit(cams[s % len(cams)]))
        if len(inflight) >= fg.slots:
            pipe.result(inflight.popleft())
    while inflight:
        pipe.result(inflight.popleft())
    t_e2e = time.perf_counter() - t0
    if dist:
        tt = torch.tensor([t_e2e], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e_fps = world * e2e_steps / t_e2e

    # ---- roofline of the dominant kernel (stage with the largest time)
    import json as _json
    with open(os.path.join(REPO, "MEASURED_PEAKS.json")) if os.path.exists(
            os.path.join(REPO, "MEASURED_PEAKS.json")) else open(os.devnull) as f:
        try:
            peaks = _json.load(f)
        except Exception:
            peaks = {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    P = int(frames[-1].n_pairs.item())
    K = 4
    stage_ms = stage.mean(axis=0)
    names = ["preprocess(K1)", "bin_sort(K2)", "blend(K3)"]
    # algorithmic bytes per launch: K1 reads 168 B/Gaussian
    # (float64 SoA + shading) + 4 B scene id, writes 8+4+8+32+4K B; K2 moves ~176 B per
    # Gaussian (min/max, coarse key, 4 radix passes, fix-up, count scan, 2 placement
    # walks incl. the 32 B record for the tile cull) + 4 B per pair written; K3 reads
    # 4 B pair id + 32 B record + 4K B values per pair, writes 4K+4 B per pixel.
    alg = [n * (172 + 52 + 4 * K), n * 176 + P * 4,
           P * (4 + 32 + 4 * K) + W_IMG * H_IMG * (4 * K + 4)]
    dom = int(np.argmax(stage_ms))
    achieved = alg[dom] / (stage_ms[dom] * 1e-3) / 1e9
    # DRAM traffic per launch and issue utilisation of the dominant kernel from
    # the committed ncu --set full capture of one C2 frame (profiles/)
    traffic, issue = None, None
    ncu_path = os.path.join(REPO, "profiles", "r01_ncu_c2_frame.json")
    if os.path.exists(ncu_path):
        kern = {"preprocess(K1)": "preprocess_kernel", "bin_sort(K2)": "pair_place_kernel",
                "blend(K3)": "blend_fwd_kernel"}[names[dom]]
        for rec in _json.load(open(ncu_path))["kernels"]:
            if kern in rec["kernel"]:
                traffic = rec["dram_read_bytes"] + rec["dram_write_bytes"]
                issue = {"issue_active_pct": rec["issue_active_pct"],
                         "sm_active_over_elapsed": rec["sm_active_over_elapsed"],
                         "source": "profiles/r01_ncu_c2_frame.json (ncu --set full, cold)"}
    roofline = {"kernel": names[dom], "bound": "hbm", "achieved": achieved, "peak": hbm_peak,
                "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic,
                "peak_source": peak_src,
                "note": "K3 is bound by FP32/MUFU instruction issue and the longest 8x4 block "
                        "walk, not HBM: its pair lists and records are L2-resident "
                        "(traffic << algorithmic bytes); see 'issue'",
                "issue": issue,
                "stage_ms_uncaptured": {nm: float(v) for nm, v in zip(names, stage_ms)},
                "frame_ms_isolated_min_med_max": [float(frame_ms.min()), float(np.median(frame_ms)),
                                         float(frame_ms.max())],
                "alg_bytes": {nm: int(v) for nm, v in zip(names, alg)}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arrays = host_scene_arrays(scene)
        cam = cams[0]
        sec, thr = cpu_frames(arrays, cam, max(1, args.cpu_frames))
        cpu = {"value": 1.0 / sec, "unit": "frames/s", "cores": thr, "kind": "port",
               "sample": f"{max(1, args.cpu_frames)} full C2 frames (1M Gaussians, 800x800) "
                         "via oracle/ (numpy + C/OpenMP)"}

    extra = None
    if not args.no_extra:
        extra = {}
        jobs = [("train_c3", lambda: bench_train(scene, dist, world, rank)),
                ("inverse_c4", lambda: bench_inverse(scene, dist, world, rank))]
        if world == 1:  # VQ / service frames: replicas only, reported at N = 1
            jobs.append(("vq_c5", lambda: bench_vq(scene)))
            jobs.append(("service_frames", lambda: bench_service(scene)))
            jobs.append(("dvr_views", lambda: bench_dvr(scene)))
        for name, fn in jobs:
            try:
                extra[name] = fn()
            except Exception as e:  # report, never hide the headline line
                extra[name] = {"error": f"{type(e).__name__}: {e}"}
            torch.cuda.empty_cache()

    if rank == 0:
        line = {"metric": METRIC, "value": fps_total, "unit": "frames/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded editable Gaussians, SURVEY.md 8(d))",
                "config": config_dict(n, {"pairs": P, "parallelism": f"replicas x{world} (views)"}),
                "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": e2e_fps, "unit": "frames/s",
                        "h2d_bytes_per_step": pipe.h2d_bytes_per_frame(),
                        "d2h_bytes_per_step": pipe.d2h_bytes_per_frame(),
                        "pipelined": "frames on 6 concurrent slots; each frame's D2H overlaps "
                                     "later frames' upload+compute; host wall clock over all frames"},
                "gpu_launches": launches_per_frame(n) * args.steps, "overflow": overflow,
                "extra": extra}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
