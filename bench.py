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
def launches_per_frame(n):
    """Kernels in one captured frame (sort.cu / blend.cu): K1; K2 = bucket
    count, bucket scan, bucket scatter, bucket sort (+ long-run fallback in
    its last block), tile histogram, tile scan (+ ranges / P / schedule /
    re-arm in its last block), placement; K3.  Plus one memset node (K2's
    control block)."""
    del n
    return 1 + 7 + 1


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
    numpy per-Gaussian math + C/OpenMP compositor).  Returns (sec/frame,
    threads, last frame's state)."""
    import oracle as O
    a = scene_arrays
    times = []
    st = None
    for _ in range(frames):
        t0 = time.perf_counter()
        o_eff = O.effective_o_logit(a["o_logit"], a["opacity_scale"])
        rgb, _ = O.shade(a["mu"], a["n_raw"], a["delta_c"], a["k_a_raw"], a["k_d_raw"],
                         a["k_s_raw"], a["log_beta"], a["palette_rgb"], a["light"], cam)
        st = O.rasterize(a["mu"], a["q_raw"], a["log_s"], o_eff, a["n_raw"], rgb, cam,
                         dtype=np.float32, nthreads=nthreads)
        st["maps"] = O.maps(st)
        times.append(time.perf_counter() - t0)
    return float(np.mean(times)), O.max_threads() if nthreads <= 0 else nthreads, st


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
    cat["scene_ids"] = np.concatenate([np.full(len(m), i) for i, m in enumerate(models)])
    lt = scene.light
    cat["light"] = (lt.mode, lt.polar, lt.azimuth, lt.term_scales)
    return cat


C3_N = 300_000
C3_LIGHT = ("orbital", 0.45, 0.9)


def c3_params(seed=0):
    """The C3 workload: a 300k basic model (geometry of the seeded scene,
    neutral stage-2 shading, trainer.py:562-577) -- the parameters the GPU
    training bench steps."""
    from paper_2504_17954_b200.synthetic import editable_arrays
    from paper_2504_17954_b200.trainer import _stage2_init
    a = editable_arrays(seed, C3_N, density=C3_N)
    p = {k: a[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")}
    p.update(_stage2_init(C3_N))
    return a, p


def cpu_extras(scene, arrays):
    """Same-run CPU baselines of the other configs on the host cores
    (BASELINE.md 4): the oracle's stage-2 step + Adam at 300k (C3), one
    inverse step on the composed 1M scene in float64 (C4), assign + decode
    over the 60M values of a 4M model at K=4096 (C5; k-means++ seeding timed
    on a 1M subsample and extrapolated)."""
    import oracle as O
    from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays
    res = {}
    cores = O.max_threads()
    # C3
    a, p = c3_params(0)
    cam = bench_camera(W_IMG, H_IMG, 0.3)
    gt = np.random.default_rng(5).uniform(0.0, 1.0, (H_IMG, W_IMG, 4))
    light = C3_LIGHT + (np.ones(4),)
    adam = O.Adam()
    t0 = time.perf_counter()
    _, g, _ = O.stage2_step(p, a["palette"], light, cam, gt)
    t1 = time.perf_counter()
    for k, v in g.items():
        adam.step(k, p[k], v, 1e-3)
    t2 = time.perf_counter()
    res["train_c3"] = {"value": 1.0 / (t2 - t0), "unit": "it/s", "step_s": t1 - t0,
                       "adam_s": t2 - t1, "cores": cores, "kind": "port",
                       "sample": "1 stage-2 step (oracle.stage2_step: K=15 render, all losses, "
                                 "backward) + Adam over the 10 groups, 300k Gaussians, 800x800"}
    del a, p, g
    # C4
    cam = bench_camera(W_IMG, H_IMG, 0.8)
    geom = tuple(arrays[k] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw"))
    shad = tuple(arrays[k] for k in ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta"))
    ids = arrays["scene_ids"]
    S = int(ids.max()) + 1
    c_p = np.stack([arrays["palette_rgb"][np.argmax(ids == s)] for s in range(S)])
    sc = np.array([arrays["opacity_scale"][np.argmax(ids == s)] for s in range(S)])
    o_raw = O.inv_softplus(np.maximum(sc, 1e-6))
    mode, pol, az, ts = arrays["light"]
    ref = np.random.default_rng(6).uniform(0.0, 1.0, (H_IMG, W_IMG, 4))
    t0 = time.perf_counter()
    O.inverse_step(geom, shad, ids, arrays["light"], c_p, o_raw, np.ones(4), np.zeros(4), pol, az,
                   cam, ref)
    dt = time.perf_counter() - t0
    res["inverse_c4"] = {"value": 1.0 / dt, "unit": "it/s", "cores": cores, "kind": "port",
                         "sample": "1 inverse step (oracle.inverse_step: float64 render, L1+SSIM, "
                                   "backward, per-scene reductions), composed 1M, 800x800"}
    # C5
    v = editable_arrays(0, 4_000_000, density=4_000_000)
    from paper_2504_17954_b200.vq import QUANTIZED_ATTRIBUTES
    vals = np.concatenate([np.ascontiguousarray(v[nm]).reshape(-1) for nm, _ in QUANTIZED_ATTRIBUTES])
    del v
    cents = np.sort(np.quantile(vals[::97], np.linspace(0.0, 1.0, 4096)))
    t0 = time.perf_counter()
    idx = O.vq_assign(vals, cents)
    t1 = time.perf_counter()
    O.vq_decode(idx.astype(np.uint16), cents)
    t2 = time.perf_counter()
    # k-means++ seeding (vq.py:60-72): 32 steps on a 1M subsample, per-step cost
    rng = np.random.default_rng(0)
    x = vals[:1_000_000].copy()
    d2 = (x - x[0]) ** 2
    t3 = time.perf_counter()
    for _ in range(32):
        c = x[rng.choice(x.size, p=d2 / d2.sum())]
        d2 = np.minimum(d2, (x - c) ** 2)
    step = (time.perf_counter() - t3) / 32
    res["vq_c5"] = {"assign_s": t1 - t0, "decode_s": t2 - t1, "values": int(vals.size),
                    "assign_gbs_alg": vals.size * 6 / (t1 - t0) / 1e9,
                    "cores": cores, "kind": "port",
                    "kmeans_seed_step_s_per_1M": step,
                    "kmeans_full_estimate_s": step * 4095 * (vals.size / 1e6) * 5,
                    "sample": "assign (C/OpenMP searchsorted on float64 mids) + decode over all "
                              "60M values of the 8 attributes of a 4M model, K=4096; k-means "
                              "extrapolated from 32 k-means++ steps on 1M samples x 4095 steps x "
                              "60 (M values) x 5 restarts"}
    return res


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
    sec, thr, _ = cpu_frames(arrays, cam, steps)
    fps = 1.0 / sec
    extra = None if args.no_extra else cpu_extras(scene, arrays)
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": 1, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference", "config": config_dict(len(arrays["mu"])),
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": thr, "kind": "port",
                             "sample": f"{steps} full C2 frames (1M Gaussians, 800x800) through "
                                       "oracle/ (numpy + C/OpenMP compositor)"},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "extra": extra}
    print(json.dumps(line), flush=True)


NCU_FILES = ("r02_ncu_c2_frame", "r02_ncu_c3_train_step", "r02_ncu_c4_inverse_step", "r02_ncu_c5_vq",
             "r01_ncu_c2_frame", "r01_ncu_c3_train_step", "r01_ncu_c4_inverse_step", "r01_ncu_c5_vq")


def load_ncu():
    """Kernel-name substring -> the first matching record of the committed
    ncu --set full summaries (profiles/, newest round first)."""
    recs = []
    for f in NCU_FILES:
        path = os.path.join(REPO, "profiles", f + ".json")
        if os.path.exists(path):
            for r in json.load(open(path))["kernels"]:
                r = dict(r)
                r["source"] = "profiles/" + f + ".json"
                recs.append(r)

    class Lookup(dict):
        def get(self, key, default=None):
            for r in recs:
                if key in r["kernel"]:
                    return r
            return default
    return Lookup()


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


def _split_events(fn, n_ev, reps=5):
    """Mean device ms between consecutive events of fn(events) over `reps`
    calls (L2 flushed before each)."""
    import torch
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(2):  # warm-up: workspaces and caching-allocator blocks
        fn([torch.cuda.Event(enable_timing=True) for _ in range(n_ev)])
    torch.cuda.synchronize()
    rows = []
    for _ in range(reps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
        fn(ev)
        torch.cuda.synchronize()
        rows.append([ev[i].elapsed_time(ev[i + 1]) for i in range(n_ev - 1)])
    return np.mean(np.array(rows), axis=0)


def bench_train(scene, dist=None, world=1, rank=0):
    """C3: stage-2 training step (K=15 channels, fwd + all losses + bwd +
    Adam) on one 300k-Gaussian basic model at 800x800, one view / iteration.
    With N ranks every rank trains its own basic TF (independent seeds, no
    communication): aggregate it/s = N / slowest rank's ms per iteration.
    Also: the eager step split by CUDA events (per-kernel table) and the
    EXACT-blend step (bit-faithful maps) for comparison."""
    import torch
    from paper_2504_17954_b200 import LightConfig
    from paper_2504_17954_b200.synthetic import bench_camera
    from paper_2504_17954_b200.trainer import EditableTrainer, StepGraph
    a, p = c3_params(rank)
    light = LightConfig(*C3_LIGHT)
    cams = [bench_camera(W_IMG, H_IMG, az) for az in np.linspace(-3.0, 3.0, 8)]
    gt_tr = EditableTrainer(a, a["palette"], light)
    gts = [gt_tr.render_rgba(c).clone() for c in cams]
    del gt_tr
    res = {}
    for exact in (False, True):
        tr = EditableTrainer(p, a["palette"], light)
        tr.exact = exact
        it = [0]
        # the product path: the whole step (fwd, losses, bwd, Adam) as one CUDA graph
        G = StepGraph(tr, cams[0], gts[0])

        def step():
            v = it[0] % len(cams)
            it[0] += 1
            G.step(cams[v], gts[v], it[0], 10000)
        mean_ms, med_ms = _device_time(step, 10)
        G.flush()
        res[exact] = (_max_over_ranks(mean_ms, dist), med_ms, tr)
    mean_ms, med_ms, tr = res[False]
    # per-kernel split of the (eager) FAST step
    tr.exact = False

    def eager(ev):
        loss, grads, stat = tr.step(cams[1], gts[1], events=ev[:6])
        tr.apply(grads, 1, 10000)
        ev[6].record()
    split = _split_events(eager, 7)
    P = int(tr._last_pairs.item())
    parts = dict(zip(("forward(K14 attrs, K1, K2, K3)", "losses(K7 L1+SSIM, K10 regularizers)",
                      "K4a blend_bwd", "K4b preprocess_bwd", "K14 assemble+loss", "K11 adam"),
                     [float(x) for x in split]))
    return {"metric": "stage-2 train it/s (300k Gaussians, 800x800, K=15, 1 view/it)",
            "value": world * 1000.0 / mean_ms, "unit": "it/s", "ms_per_it": mean_ms,
            "ms_per_it_median": med_ms, "n_gaussians": C3_N, "n_gpus": world, "pairs": P,
            "exact_blend": {"value": world * 1000.0 / res[True][0], "ms_per_it": res[True][0],
                            "note": "same StepGraph with the EXACT (bit-faithful float64) blend"},
            "split_ms_eager": parts,
            "scaling": "weak (one basic TF per GPU)",
            "note": "StepGraph replay: fwd (K1-K3), L1+SSIM + normal/offset/bilateral/opacity "
                    "terms, K4a+K4b, gradient assembly, Adam; densify excluded; FAST blend"}


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
    G = InverseGraph(fit, params, 100_000, dist=dist, view_div=float(world))
    step = G.replay
    note = ("whole iterations replayed as CUDA graphs (InverseGraph: device Adam)" +
            ("; views sharded, one NCCL all-reduce per iteration between the compute "
             "and update graphs" if dist is not None else ""))
    mean_ms, med_ms = _device_time(step, 10)
    mean_ms = _max_over_ranks(mean_ms, dist)
    # the graph's launch sequence run eagerly with events between the kernels
    split = _split_events(lambda ev: G._views(events=ev), 7)
    P = int(G._last_pairs.item())
    parts = dict(zip(("K1 preprocess (float64 semantics)", "K2 bin/sort", "K3 blend_fwd",
                      "loss(K7)", "K4a blend_bwd", "K4b preprocess_bwd (transform only) + pack"),
                     [float(x) for x in split]))
    return {"metric": "inverse exploration it/s (composed 1M, 800x800, 1 view per GPU)",
            "value": 1000.0 / mean_ms, "unit": "it/s", "views_per_s": world * 1000.0 / mean_ms,
            "ms_per_it": mean_ms, "ms_per_it_median": med_ms, "n_gpus": world, "pairs": P,
            "split_ms_eager": parts,
            "scaling": "weak (views sharded, one NCCL all-reduce of 4S+12 float64 per iteration)",
            "note": note}


def bench_vq(scene):
    """C5: K5 assign + K6 decode over the 60M scalar attribute values of a 4M
    editable model (the 8 quantized attributes, vq.py:19-28) with a
    4096-entry codebook (HBM-bound)."""
    import torch
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.synthetic import editable_arrays
    from paper_2504_17954_b200.vq import QUANTIZED_ATTRIBUTES, assign_device, decode_device
    v = editable_arrays(0, 4_000_000, density=4_000_000)
    host = np.concatenate([np.ascontiguousarray(v[nm]).reshape(-1) for nm, _ in QUANTIZED_ATTRIBUTES])
    del v
    vals = to_dev(host)
    cents = to_dev(np.sort(np.quantile(host[::97], np.linspace(0.0, 1.0, 4096))))
    n_vals = vals.numel()
    out = {}
    a_ms, _ = _device_time(lambda: out.__setitem__("idx", assign_device(vals, cents)), 5)
    d_ms, _ = _device_time(lambda: decode_device(out["idx"], cents), 5)
    del vals, out
    torch.cuda.empty_cache()
    res = {"metric": "VQ assign/decode over 60M values (8 attributes of a 4M model), K=4096",
           "values": int(n_vals), "assign_ms": a_ms, "decode_ms": d_ms,
           "assign_values_per_s": n_vals / (a_ms * 1e-3), "decode_values_per_s": n_vals / (d_ms * 1e-3)}
    if os.environ.get("IVR_BENCH_QUANTIZE", "1") != "0":
        res["quantize_e2e"] = bench_quantize()
    return res


def bench_quantize():
    """C5 end to end: quantize_model of a 4M editable model at K=4096
    (vq.py:150-176: per attribute k-means++ seeding from the reference's
    numpy stream + Lloyd, 5 restarts, then encode) on the device, and the
    decoded model rendered at 800x800 (FAST frames, device time)."""
    import torch
    from paper_2504_17954_b200 import ComposedScene, DeviceScene, LightConfig
    from paper_2504_17954_b200.synthetic import bench_camera, editable_model
    from paper_2504_17954_b200.vq import quantize_model
    m = editable_model(0, 4_000_000, density=4_000_000)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    qm = quantize_model(m, k=4096, seed=0)
    torch.cuda.synchronize()
    t_q = time.perf_counter() - t0
    ks = {name: cb.k for name, (cb, _) in qm.quantized.items()}
    ds = DeviceScene(ComposedScene.compose([qm], LightConfig("orbital", 0.45, 0.9)))
    cams = [bench_camera(W_IMG, H_IMG, 0.8 + 0.1 * i) for i in range(8)]
    ds.render_frame(cams[0], fast=False)
    it = [0]

    def frame():
        ds.render_frame(cams[it[0] % len(cams)], fast=True)
        it[0] += 1
    f_ms, _ = _device_time(frame, 5)
    P = int(ds.render_frame(cams[0], fast=False).n_pairs.item())
    del ds, qm, m
    torch.cuda.empty_cache()
    return {"quantize_model_s": t_q, "codebook_sizes": ks, "gaussians": 4_000_000,
            "decoded_render_ms": f_ms, "decoded_render_fps": 1000.0 / f_ms, "decoded_pairs": P,
            "note": "host wall clock around quantize_model (8 attributes, K=4096, 5 restarts); "
                    "decoded model rendered eagerly (K1-K3, FAST) at 800x800, L2 flushed"}


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

    peaks = {}
    pk_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(pk_path):
        try:
            peaks = json.load(open(pk_path))
        except Exception:
            peaks = {}
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "hbm_gbs" in peaks else \
        "fallback (B200_PROFILING.md 6.65 TB/s)"
    P = int(frames[-1].n_pairs.item())
    stage_ms = stage.mean(axis=0)
    WH = W_IMG * H_IMG

    # ---- parity of the headline path with the CPU reference, same camera
    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arrays = host_scene_arrays(scene)
        cam = cams[0]
        sec, thr, ref = cpu_frames(arrays, cam, max(1, args.cpu_frames))
        cpu = {"value": 1.0 / sec, "unit": "frames/s", "cores": thr, "kind": "port",
               "sample": f"{max(1, args.cpu_frames)} full C2 frames (1M Gaussians, 800x800) "
                         "via oracle/ (numpy + C/OpenMP)"}
        Fg = fg.submit(0, cam)  # the captured headline frame (FAST blend) of this camera
        torch.cuda.synchronize()
        Fe = ds.render_frame(cam, fast=True, want_state=True)  # + last_pos / t_final
        torch.cuda.synchronize()
        rgba = np.concatenate([ref["maps"]["color"], ref["maps"]["alpha"][..., None]], axis=-1)
        img = Fg.out.cpu().numpy()
        parity = {"camera": "cams[0] (orbit azimuth 0.8)", "mode": "FAST (headline FrameGraph)",
                  "pairs": int(ref["pair_splat"].size),
                  "pairs_equal": bool(int(Fg.n_pairs.item()) == ref["pair_splat"].size and
                                      np.array_equal(Fg.pairs(), ref["pair_splat"])),
                  "tile_ranges_equal": bool(np.array_equal(Fg.tile_ranges.cpu().numpy(),
                                                           ref["tile_ranges"])),
                  "contrib_equal": bool(np.array_equal(Fg.contrib.cpu().numpy(), ref["contrib"])),
                  "last_pos_equal": bool(np.array_equal(Fe.last_pos.cpu().numpy(), ref["last_pos"])),
                  "max_abs": float(np.abs(img - rgba).max()),
                  "identical_values": float(np.mean(img == rgba)),
                  "tolerance": 1e-4}

    # ---- per-kernel roofline table (CUDA-event times from this run; algorithmic
    # bytes per SURVEY 8(d) for the C2 kernels, DESIGN.md 3 for the others;
    # DRAM traffic / issue from the committed ncu captures, same kernel scope)
    ncu = load_ncu()
    kern = []

    def row(name, ms, alg, basis, ncu_key=None, launches=1, bound="hbm", note=None):
        ach = alg / (ms * 1e-3) / 1e9
        r = {"kernel": name, "us": ms * 1e3, "alg_bytes": int(alg), "alg_basis": basis,
             "achieved_gbs": ach, "frac": ach / hbm_peak, "bound": bound}
        rec = ncu.get(ncu_key) if ncu_key else None
        if rec:
            r["traffic"] = (rec["dram_read_bytes"] + rec["dram_write_bytes"]) * launches
            r["traffic_over_alg"] = r["traffic"] / alg
            r["ncu"] = {k: rec[k] for k in ("duration_us", "issue_active_pct",
                                            "sm_active_over_elapsed", "warps_active_pct")}
            if "pipe_pct" in rec:  # FP32 FMA / ALU / XU / FP64 pipe, % of peak (active cycles)
                r["ncu"]["pipe_pct"] = rec["pipe_pct"]
            r["ncu"]["source"] = rec["source"]
        if note:
            r["note"] = note
        kern.append(r)
        return r

    row("K1 preprocess (C2)", stage_ms[0], 136 * n, "SURVEY 8(d): 136 B/Gaussian (in 88 + out 48)",
        "preprocess_kernel")
    row("K2 bin/sort stage (C2, all launches)", stage_ms[1], 24 * n + 12 * P,
        "SURVEY 8(d): 24 B/Gaussian (depth-rank sort) + 12 B/pair (key gen / placement)",
        None, note="whole ivr_bin_sort_cull + ivr_tile_order stage")
    k3 = row("K3 blend_fwd (C2)", stage_ms[2], 40 * P + 16 * WH,
             "SURVEY 8(d): 40 B/pair (id + record + rgba gather) + 16 B/pixel (RGBA f32 out)",
             "blend_fwd_kernel<4, 0, 1>", bound="issue (FP32/MUFU) + longest 8x4 block walk")

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
        t3 = extra.get("train_c3", {})
        if "split_ms_eager" in t3:
            sp, P3, N3, K3 = t3["split_ms_eager"], t3["pairs"], C3_N, 15
            row("K4a blend_bwd (C3, K=15)", sp["K4a blend_bwd"],
                P3 * (4 + 32 + 4 * K3) + WH * (4 * K3 + 12) + N3 * (K3 + 6) * 4,
                "DESIGN 3: 96 B/pair gather + 72 B/pixel (d_out, last_pos, t_final) + "
                "84 B/Gaussian accumulators", "blend_bwd_kernel<16, 0, 1>")
            row("K4b preprocess_bwd (C3)", sp["K4b preprocess_bwd"], N3 * (168 + 84 + 224),
                "DESIGN 3: 168 B params + 84 B accumulators in, 224 B gradients out per Gaussian",
                "preprocess_bwd_kernel<1>")
            row("losses K7+K10 (C3)", sp["losses(K7 L1+SSIM, K10 regularizers)"],
                WH * 4 * 56 + WH * (4 * K3 * 2 + 64),
                "DESIGN 3: K7 56 B/pixel-channel (4 ch) + K10 (maps in, d_out out, normals)")
            row("K11 adam (C3)", sp["K11 adam"], N3 * 24 * 8 * 7,
                "DESIGN 3: 24 float64 parameters x 7 accesses per Gaussian "
                "(SURVEY 8(d) counts 672 B at float32)", "adam_kernel")
        t4 = extra.get("inverse_c4", {})
        if "split_ms_eager" in t4:
            sp, P4 = t4["split_ms_eager"], t4["pairs"]
            row("K3 blend_fwd (C4, float64 semantics)", sp["K3 blend_fwd"], 40 * P4 + 16 * WH,
                "SURVEY 8(d): 40 B/pair + 16 B/pixel", "blend_fwd_kernel<4, 1, 1>")
            row("K4a blend_bwd (C4, no geometry)", sp["K4a blend_bwd"], 40 * P4 + 16 * WH,
                "SURVEY 8(d) C4: 40 P + 16 WH read", "blend_bwd_kernel<4, 1, 0>")
            row("K4b preprocess_bwd (C4, transform only)", sp["K4b preprocess_bwd (transform only) + pack"],
                (16 + 100) * n, "SURVEY 8(d) C4: 16 B/Gaussian atomics + 100 B shade-bwd read",
                "preprocess_bwd_kernel<0>")
        v5 = extra.get("vq_c5", {})
        if "assign_ms" in v5:
            row("K5 vq_assign (C5)", v5["assign_ms"], 6 * v5["values"],
                "SURVEY 8(d) C5: 4 B in + 2 B out per value (float64 storage moves 10 B)",
                "vq_assign_win_kernel", note="implementation bytes 10/value: frac x 10/6")
            row("K6 vq_decode (C5)", v5["decode_ms"], 6 * v5["values"],
                "SURVEY 8(d) C5: 2 B in + 4 B out per value (float64 storage moves 10 B)",
                "vq_decode_kernel", note="implementation bytes 10/value: frac x 10/6")

    roofline = {"kernel": "K3 blend_fwd (C2)", "bound": "hbm", "achieved": k3["achieved_gbs"],
                "peak": hbm_peak, "unit": "GB/s", "frac": k3["frac"],
                "traffic": k3.get("traffic"), "peak_source": peak_src,
                "alg_bytes": k3["alg_bytes"], "alg_basis": k3["alg_basis"], "us": k3["us"],
                "why_dominant": "largest single kernel by CUDA-event time (and ncu share) of a C2 frame",
                "note": "K3 is bound by FP32/MUFU issue and the longest 8x4 block walk, not HBM "
                        "(its lists and records are L2-resident); see kernels[] / ncu",
                "frame_bytes_survey": int(160 * n + 52 * P + 16 * WH),
                "frame_frac_isolated": (160 * n + 52 * P + 16 * WH) / (float(np.median(frame_ms)) * 1e-3) / 1e9 / hbm_peak,
                "stage_ms_uncaptured": {"K1": float(stage_ms[0]), "K2": float(stage_ms[1]),
                                        "K3": float(stage_ms[2])},
                "frame_ms_isolated_min_med_max": [float(frame_ms.min()), float(np.median(frame_ms)),
                                                  float(frame_ms.max())]}
    if cpu is not None and extra is not None and world == 1:
        try:
            cpu["extra"] = cpu_extras(scene, host_scene_arrays(scene))
        except Exception as e:
            cpu["extra"] = {"error": f"{type(e).__name__}: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": fps_total, "unit": "frames/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f32 blend (certified decisions); f64 keys / preprocess",
                "data": "synthetic (seeded editable Gaussians, SURVEY.md 8(d))",
                "config": config_dict(n, {"pairs": P, "parallelism": f"replicas x{world} (views)"}),
                "clocks": clocks, "roofline": roofline, "kernels": kern, "parity": parity,
                "cpu_baseline": cpu,
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
