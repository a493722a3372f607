"""Scene models, composition, edits and the resident GPU renderer.

Host containers mirror voxsplat/scene.py:56-228 (BasicSceneModel, EditState,
ComposedScene, EffectiveScene, apply_edits).  Rendering goes through
``DeviceScene``: the composed model is concatenated ONCE into HBM (float64
SoA + per-splat scene id), and every frame passes the edits as per-scene
tables (palette, opacity scale) plus the global light, which K1 resolves in
registers -- instead of the reference's re-concatenation of every array on
each render (scene.py:206-212).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .errors import MixedStage, OutOfRange, ShapeMismatch
from .gaussians import GaussianGeometry, ShColor
from .rasterizer import RenderOutput, _channel_layout, _cols, _unpack, workspace
from .shading import LightConfig, Palette, ShadingAttributes

STAGE_BASE = "base"
STAGE_EDITABLE = "editable"


@dataclass
class BasicSceneModel:
    """One trained basic scene (base stage: SH colours; editable stage:
    shading attributes + palette; optionally quantized)."""

    stage: str
    geometry: GaussianGeometry
    sh: ShColor = None
    shading: ShadingAttributes = None
    palette: Palette = None
    quantized: dict = None
    metadata: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.stage not in (STAGE_BASE, STAGE_EDITABLE):
            raise OutOfRange(f"unknown stage {self.stage!r}")
        n = len(self.geometry)
        if self.stage == STAGE_BASE:
            if self.sh is None or self.shading is not None:
                raise MixedStage("base stage carries SH colors only")
            if self.sh.coefficients.shape[0] != n:
                raise ShapeMismatch("SH coefficient count != primitive count")
        else:
            if self.sh is not None:
                raise MixedStage("editable stage must not carry SH data")
            if self.palette is None:
                raise MixedStage("editable stage requires a palette")
            if self.quantized is None and (self.shading is None or len(self.shading) != n):
                raise ShapeMismatch("shading attribute count != primitive count")

    def __len__(self):
        return len(self.geometry)

    @property
    def is_quantized(self):
        return self.quantized is not None

    def copy(self):
        from .vq import Codebook
        return BasicSceneModel(
            stage=self.stage, geometry=self.geometry.copy(),
            sh=ShColor(self.sh.coefficients.copy(), self.sh.degree) if self.sh is not None else None,
            shading=self.shading.copy() if self.shading is not None else None,
            palette=self.palette.copy() if self.palette is not None else None,
            quantized={k: (Codebook(cb.name, cb.centroids.copy()), idx.copy())
                       for k, (cb, idx) in self.quantized.items()} if self.quantized else None,
            metadata=dict(self.metadata))


@dataclass
class EditState:
    """Per-scene edits: optional palette recolour and an opacity scale."""

    palette_override: np.ndarray = None
    opacity_scale: float = 1.0

    def __post_init__(self):
        if self.palette_override is not None:
            self.palette_override = np.asarray(self.palette_override, dtype=np.float64).reshape(3)
            if np.any((self.palette_override < 0) | (self.palette_override > 1)):
                raise OutOfRange("palette override components must lie in [0, 1]")
        self.opacity_scale = float(self.opacity_scale)
        if self.opacity_scale < 0:
            raise OutOfRange("opacity scale must be >= 0")

    def copy(self):
        return EditState(None if self.palette_override is None else self.palette_override.copy(),
                         self.opacity_scale)

    def to_dict(self):
        return {"palette_override": None if self.palette_override is None
                else self.palette_override.tolist(), "opacity_scale": self.opacity_scale}

    @classmethod
    def from_dict(cls, d):
        return cls(d.get("palette_override"), d.get("opacity_scale", 1.0))


@dataclass
class ComposedScene:
    """Ordered editable models with per-scene edits and one global light."""

    models: list
    edits: list
    light: LightConfig
    transform: dict = None

    def __post_init__(self):
        if len(self.edits) != len(self.models):
            raise ShapeMismatch("one edit state per basic model required")

    @classmethod
    def compose(cls, models, light=None):
        """Concatenate editable models (quantized inputs are decoded first;
        scene.py:160-167).  No re-optimisation."""
        from .vq import dequantize_model
        if any(m.stage != STAGE_EDITABLE for m in models):
            raise MixedStage("only editable-stage models compose")
        models = [dequantize_model(m) if m.is_quantized else m.copy() for m in models]
        return cls(models, [EditState() for _ in models], light or LightConfig())

    @property
    def count(self):
        return sum(len(m) for m in self.models)

    @property
    def scene_ids(self):
        return np.concatenate([np.full(len(m), i, dtype=np.int64)
                               for i, m in enumerate(self.models)])

    def copy(self):
        return ComposedScene([m.copy() for m in self.models], [e.copy() for e in self.edits],
                             self.light.copy(),
                             dict(self.transform) if self.transform is not None else None)


@dataclass
class EffectiveScene:
    """Edit-resolved snapshot (host), scene.py:188-196."""

    geometry: GaussianGeometry
    shading: ShadingAttributes
    palette_rgb: np.ndarray
    light: LightConfig
    scene_ids: np.ndarray


def _sigmoid(x):
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def apply_edits(scene):
    """Resolve edits into effective primitives on the host (scene.py:199-228).

    The GPU render path does not call this: K1 resolves the same edits per
    splat from the per-scene tables."""
    geometry = GaussianGeometry.concat([m.geometry for m in scene.models])
    shading = ShadingAttributes.concat([m.shading for m in scene.models])
    palette_rgb = np.concatenate([
        np.broadcast_to(e.palette_override if e.palette_override is not None else m.palette.c_p,
                        (len(m), 3)) for m, e in zip(scene.models, scene.edits)], axis=0)
    scales = np.concatenate([np.full(len(m), e.opacity_scale)
                             for m, e in zip(scene.models, scene.edits)])
    if not np.all(scales == 1.0):
        geometry = geometry.copy()
        p = np.clip(scales * _sigmoid(geometry.o_logit), 1e-12, 1.0 - 1e-9)
        geometry.o_logit = np.log(p / (1.0 - p))
    return EffectiveScene(geometry, shading, palette_rgb, scene.light.copy(), scene.scene_ids)


class DeviceScene:
    """A composed editable scene resident in HBM, rendered by K1-K3.

    ``scene`` may be a ComposedScene or a single editable BasicSceneModel.
    Edits, light and camera are read at render time, so edits applied to the
    host ComposedScene are picked up by the next frame without re-upload."""

    def __init__(self, scene, device=None, dg=None):
        if isinstance(scene, BasicSceneModel):
            scene = ComposedScene.compose([scene])
        self.scene = scene
        models = scene.models
        if dg is None:
            geom = {k: np.concatenate([getattr(m.geometry, k) for m in models], axis=0)
                    for k in D.DeviceGaussians.GEOM}
            shad = {k: np.concatenate([getattr(m.shading, k) for m in models], axis=0)
                    for k in D.DeviceGaussians.SHADE}
            ids = np.concatenate([np.full(len(m), i, dtype=np.int32) for i, m in enumerate(models)])
            dg = D.DeviceGaussians(geom, shad, ids, device)
        self.dg = dg  # or arrays already resident (ivrg.load_device)
        if os.environ.get("IVR_STATIC_CACHE", "1") != "0":
            dg.build_cache()  # frozen scene: camera-independent work done once
        self.n = self.dg.n
        self.n_scenes = len(models)
        self.ws = D.Workspace(self.dg.device)
        dev = self.dg.device
        # per-frame edit tables: a ring of pinned host staging buffers (the
        # host may run ahead of the GPU) + device copies
        self._ring = 8
        self._h_tabs = [torch.empty(4 * self.n_scenes, dtype=torch.float64, pin_memory=True)
                        for _ in range(self._ring)]
        self._d_tabs = [torch.empty(4 * self.n_scenes, dtype=torch.float64, device=dev)
                        for _ in range(self._ring)]
        self._events = [None] * self._ring
        self._slot = 0

    # ------------------------------------------------------------ per frame
    def _tables(self, light=None, palettes=None, opacity_scales=None):
        """Fill the per-scene palette / opacity tables for this frame."""
        sc = self.scene
        S = self.n_scenes
        pal = np.empty((S, 3))
        osc = np.empty(S)
        for i, (m, e) in enumerate(zip(sc.models, sc.edits)):
            pal[i] = e.palette_override if e.palette_override is not None else m.palette.c_p
            osc[i] = e.opacity_scale
        if palettes is not None:
            pal = np.asarray(palettes, dtype=np.float64).reshape(S, 3)
        if opacity_scales is not None:
            osc = np.asarray(opacity_scales, dtype=np.float64).reshape(S)
        k = self._slot
        self._slot = (k + 1) % self._ring
        if self._events[k] is not None:
            self._events[k].synchronize()
        h_tab, d_tab = self._h_tabs[k], self._d_tabs[k]
        h = h_tab.numpy()
        h[:3 * S] = pal.reshape(-1)
        h[3 * S:] = osc
        d_tab.copy_(h_tab, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._events[k] = ev
        self._d_tab = d_tab
        light = light or sc.light
        shading = D.shading_struct(self.dg, d_tab[:3 * S], False, light)
        edits = L.Edits_t()
        edits.scene_id = self.dg.scene_id.data_ptr()
        edits.opacity_scale = d_tab[3 * S:].data_ptr()
        edits.rescale_opacity = 0 if np.all(osc == 1.0) else 1
        return shading, edits

    def h2d_bytes_per_frame(self):
        return 8 * 4 * self.n_scenes

    def render_frame(self, cam, channels=("color", "alpha"), attrs=None, dtype=np.float32,
                     want_state=False, debug=False, light=None, lam=None, b=None,
                     palettes=None, opacity_scales=None, fast=False, out=None, stream=None,
                     events=None, exact=None):
        """Enqueue one frame; returns the Frame of device tensors.

        fast=True skips the pair-count readback (no host sync): the pair
        capacity learned on earlier frames is reused and overflow must be
        checked later with ``check_overflow(frame)``.  exact=None picks the
        certified float32 blend for fast frames and the bit-faithful float64
        blend otherwise."""
        if exact is None:
            exact = not fast
        layout = _channel_layout(channels, attrs)
        cols, attr_cols, K = _cols(layout)
        shading, edits = self._tables(light, palettes, opacity_scales)
        if lam is not None or b is not None:
            shading = D.shading_struct(self.dg, self._d_tab[:3 * self.n_scenes], False,
                                       light or self.scene.light, lam, b)
        attrs_dev = [(D.to_dev(np.asarray(attrs[name], dtype=np.float64).reshape(self.n, w)), c, w)
                     for name, c, w in attr_cols]
        f64 = np.dtype(dtype) == np.float64
        if not fast or self.ws.pair_capacity == 0:
            F = D.rasterize_device(self.dg, cam, K, cols, self.ws, shading, edits, None, attrs_dev,
                                   f64, want_state, debug, stream, exact=exact)
        else:
            if events:
                events[0].record()
            F = D.preprocess(self.dg, cam, K, cols, self.ws, shading, edits, None, attrs_dev, f64,
                             debug, stream, exact_rgb=exact)
            if events:
                events[1].record()
            D.bin_sort(F, self.ws, stream)
            if events:
                events[2].record()
            D.blend(F, self.ws, want_state, stream, out=out, exact=exact)
            if events:
                events[3].record()
            F.empty = False
        F.layout = layout
        F.dtype = dtype
        F._keep_tabs = (shading, edits)
        return F

    def render_host(self, cam, host_out, host_contrib, **kw):
        """Render and copy the maps into caller-provided pinned host tensors
        (the end-to-end path: per-frame H2D edit tables in, D2H image out)."""
        F = self.render_frame(cam, fast=True, **kw)
        host_out.copy_(F.out, non_blocking=True)
        host_contrib.copy_(F.contrib, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if self.check_overflow(F):  # capacity grew: redo synchronously
            F = self.render_frame(cam, fast=False, **kw)
            host_out.copy_(F.out)
            host_contrib.copy_(F.contrib)
        return _unpack(host_out.numpy(), F.layout, host_contrib.numpy())

    @staticmethod
    def check_overflow(F):
        return int(F.n_pairs.item()) > F.capacity

    def render(self, cam, channels=("color", "alpha"), attrs=None, dtype=np.float32, **kw):
        """Synchronous render returning host RenderOutput (numpy)."""
        F = self.render_frame(cam, channels, attrs, dtype, **kw)
        if F.empty and self.n == 0:
            H, W = cam.height, cam.width
            K = sum(w for _, w in F.layout)
            return _unpack(np.zeros((H, W, K), dtype=dtype), F.layout, np.zeros((H, W), np.int32))
        out = D.to_host(F.out64 if F.f64 else F.out).astype(dtype, copy=False)
        return _unpack(out, F.layout, D.to_host(F.contrib))


class FrameGraph:
    """A whole frame (K1 -> K2 -> K3) captured once as a CUDA graph.

    Per frame the host writes the camera / light / edit tables into pinned
    staging (a ring, so the host can run ahead), one small H2D copy lands
    them in fixed device buffers, and the graph replays: one launch instead of
    ~27, and no host gaps inside the frame.  Resolution, channel layout and
    mode are fixed per graph.  The pair capacity learned on the warm-up frame
    is reused (with 30% headroom); ``overflowed()`` reports whether a replay
    needed more, in which case ``recapture()`` grows it.

    ``slots`` > 1 captures independent copies of the frame -- each with its
    own workspace, parameter buffers, outputs and CUDA stream -- so
    consecutive frames (different views) run concurrently: frame i+1's
    preprocess and sort fill the SMs that frame i's blend tail leaves idle.
    Slot 0 on the current stream is what ``stage/launch/replay`` use.
    """

    RING = 8

    def __init__(self, ds, width, height, exact=False, headroom=1.3, warm_cam=None, slots=1):
        self.ds, self.W, self.H, self.exact = ds, int(width), int(height), exact
        self.slots = max(1, int(slots))
        dev = ds.dg.device
        S = ds.n_scenes
        nb = ctypes.sizeof(L.FrameParams_t)
        self._h = [torch.empty(nb + 8 * 4 * S, dtype=torch.uint8, pin_memory=True)
                   for _ in range(self.RING)]
        self._ev = [None] * self.RING
        self._slot = 0
        self.nb = nb
        self.res = []
        for k in range(self.slots):
            self.res.append({
                # every slot owns its workspace: an eager render on ds.ws at
                # another size must never reallocate buffers a graph replays
                "ws": D.Workspace(dev),
                # one device block per slot (one H2D per frame): params | tables
                "d_stage": torch.empty(nb + 8 * 4 * S, dtype=torch.uint8, device=dev),
                "stream": torch.cuda.current_stream(dev) if k == 0 else torch.cuda.Stream(device=dev),
            })
        for r in self.res:  # views of the slot's staging block
            r["d_params"] = r["d_stage"][:nb]
            r["d_tab"] = r["d_stage"][nb:].view(torch.float64)
        self.d_params, self.d_tab = self.res[0]["d_params"], self.res[0]["d_tab"]
        from .synthetic import bench_camera
        cam = warm_cam or bench_camera(self.W, self.H)
        F = ds.render_frame(cam, fast=False, exact=exact)  # learns the pair capacity
        self.capacity = max(int(int(F.n_pairs.item()) * headroom) + 4096, 1 << 16)
        self._capture(cam)

    def _stage(self, cam, light=None, palettes=None, opacity_scales=None, slot=0):
        """Write this frame's parameters into the slot's device buffers (H2D
        on the slot's stream)."""
        sc = self.ds.scene
        S = self.ds.n_scenes
        pal = np.empty((S, 3))
        osc = np.empty(S)
        for i, (m, e) in enumerate(zip(sc.models, sc.edits)):
            pal[i] = e.palette_override if e.palette_override is not None else m.palette.c_p
            osc[i] = e.opacity_scale
        if palettes is not None:
            pal = np.asarray(palettes, dtype=np.float64).reshape(S, 3)
        if opacity_scales is not None:
            osc = np.asarray(opacity_scales, dtype=np.float64).reshape(S)
        if int(cam.width) != self.W or int(cam.height) != self.H:
            raise ValueError("FrameGraph resolution is fixed at capture time")
        k = self._slot
        self._slot = (k + 1) % self.RING
        if self._ev[k] is not None:
            self._ev[k].synchronize()
        h = self._h[k]
        P = D.frame_params(cam, light or sc.light, rescale_opacity=not np.all(osc == 1.0))
        ctypes.memmove(h.data_ptr(), ctypes.addressof(P), self.nb)
        tab = np.frombuffer(h.numpy(), dtype=np.float64, count=4 * S, offset=self.nb)
        tab[:3 * S] = pal.reshape(-1)
        tab[3 * S:] = osc
        r = self.res[slot]
        with torch.cuda.stream(r["stream"]):
            r["d_stage"].copy_(h, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(r["stream"])
        self._ev[k] = ev

    def _capture(self, cam):
        ds = self.ds
        S = ds.n_scenes
        layout = _channel_layout(("color", "alpha"), None)
        cols, _, K = _cols(layout)
        self.graphs = []
        self._keep = []
        torch.cuda.synchronize()
        for k, r in enumerate(self.res):
            self._stage(cam, slot=k)
            torch.cuda.synchronize()
            shading = D.shading_struct(ds.dg, r["d_tab"][:3 * S], False, ds.scene.light)
            edits = L.Edits_t()
            edits.scene_id = ds.dg.scene_id.data_ptr()
            edits.opacity_scale = r["d_tab"][3 * S:].data_ptr()
            edits.rescale_opacity = 0  # taken from d_params
            ws = r["ws"]
            with torch.cuda.stream(r["stream"]):
                # allocate every workspace buffer at its final size before capture
                F = D.preprocess(ds.dg, cam, K, cols, ws, shading, edits, params_dev=r["d_params"],
                                 exact_rgb=self.exact)
                D.bin_sort(F, ws, capacity=self.capacity)
                D.blend(F, ws, want_state=False, exact=self.exact)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):  # captured on torch's side stream, replayed on the slot's
                F = D.preprocess(ds.dg, cam, K, cols, ws, shading, edits, params_dev=r["d_params"],
                                 exact_rgb=self.exact)
                D.bin_sort(F, ws, capacity=self.capacity)
                D.blend(F, ws, want_state=False, exact=self.exact)
            F.layout = layout
            self.graphs.append((g, F))
            self._keep.append((shading, edits))
        torch.cuda.synchronize()
        self.g, self.F = self.graphs[0]
        self.K = K

    def stage(self, cam, **edits):
        """Enqueue this frame's camera / light / edit upload (async)."""
        self._stage(cam, **edits)

    def launch(self):
        """Enqueue the captured frame; returns the Frame whose .out holds RGBA."""
        self.g.replay()
        return self.F

    def replay(self, cam, **edits):
        """stage() + launch()."""
        self._stage(cam, **edits)
        self.g.replay()
        return self.F

    def submit(self, slot, cam, **edits):
        """Stage + replay on the slot's own stream; returns the slot's Frame."""
        self._stage(cam, slot=slot, **edits)
        g, F = self.graphs[slot]
        with torch.cuda.stream(self.res[slot]["stream"]):
            g.replay()
        return F

    def stream(self, slot):
        return self.res[slot]["stream"]

    def render_host(self, cam, host_out, host_contrib=None, **edits):
        """End-to-end frame: H2D inputs, replay, D2H image (synchronous)."""
        F = self.replay(cam, **edits)
        host_out.copy_(F.out, non_blocking=True)
        if host_contrib is not None:
            host_contrib.copy_(F.contrib, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if self.overflowed():  # pair capacity too small for this view: grow and redo
            self.recapture(cam)
            return self.render_host(cam, host_out, host_contrib, **edits)
        return host_out

    def overflowed(self):
        return int(self.F.n_pairs.item()) > self.capacity

    def recapture(self, cam, n_pairs=None):
        n = int(self.F.n_pairs.item()) if n_pairs is None else int(n_pairs)
        self.capacity = int(n * 1.3) + 4096
        self._capture(cam)


class FramePipeline:
    """End-to-end frames: frames on alternating slots (own streams) run
    concurrently, and each frame's device->host copy overlaps later frames.

    ``submit(cam, **edits)`` stages the frame's parameters (pinned ring, one
    H2D) and replays the next slot's captured graph on that slot's stream,
    then enqueues the RGBA / contribution-count / pair-count copies into the
    slot's pinned host buffers on a copy stream; ``result(ticket)`` waits for
    that frame's copies and returns its RenderOutput (views of the slot's
    pinned buffers, valid until the slot is reused ``slots`` submits later).
    A frame whose pair count outgrew the captured capacity is re-rendered
    synchronously after growing the capacity."""

    def __init__(self, fg: FrameGraph):
        self.fg = fg
        n = fg.slots
        H, W, K = fg.H, fg.W, fg.K
        self.copy_stream = torch.cuda.Stream(device=fg.ds.dg.device)
        self.h_out = [torch.empty((H, W, K), dtype=torch.float32, pin_memory=True) for _ in range(n)]
        self.h_cnt = [torch.empty((H, W), dtype=torch.int32, pin_memory=True) for _ in range(n)]
        self.h_np = [torch.empty(1, dtype=torch.int32, pin_memory=True) for _ in range(n)]
        self.done = [None] * n
        self.k = 0

    def h2d_bytes_per_frame(self):
        return self.fg.nb + 8 * 4 * self.fg.ds.n_scenes

    def d2h_bytes_per_frame(self):
        return self.h_out[0].numel() * 4 + self.h_cnt[0].numel() * 4 + 4

    def submit(self, cam, **edits):
        fg = self.fg
        k = self.k
        self.k = (k + 1) % fg.slots
        st = fg.stream(k)
        if self.done[k] is not None:  # the slot's previous image must have left the device
            st.wait_event(self.done[k])
        F = fg.submit(k, cam, **edits)
        ev = torch.cuda.Event()
        ev.record(st)
        cs = self.copy_stream
        cs.wait_event(ev)
        with torch.cuda.stream(cs):
            self.h_out[k].copy_(F.out, non_blocking=True)
            self.h_cnt[k].copy_(F.contrib, non_blocking=True)
            self.h_np[k].copy_(F.n_pairs[:1], non_blocking=True)
            d = torch.cuda.Event()
            d.record(cs)
        self.done[k] = d
        return (k, cam, edits)

    def result(self, ticket):
        k, cam, edits = ticket
        self.done[k].synchronize()
        fg = self.fg
        if int(self.h_np[k][0]) > fg.capacity:  # this view needed more pairs: grow, redo
            torch.cuda.synchronize()
            fg.recapture(cam, n_pairs=int(self.h_np[k][0]))
            fg.render_host(cam, self.h_out[k], self.h_cnt[k], **edits)
        return _unpack(self.h_out[k].numpy(), fg.F.layout, self.h_cnt[k].numpy())


def compose_device(models, palettes, light=None, metadata=None):
    """ComposedScene.compose for models already resident in HBM
    (scene.py:147-186): one batched device copy per attribute (ivr_concat)
    into the concatenated SoA + scene ids; returns a DeviceScene.  ``models``
    are DeviceGaussians with shading attributes, ``palettes`` their c_p."""
    from .ivrg import ResidentModel
    if not models:
        raise ShapeMismatch("compose needs at least one model")
    if any(not m.has_shading for m in models):
        raise MixedStage("only editable-stage models compose")
    dev = models[0].device
    rows = [m.n for m in models]
    N = sum(rows)
    widths = {"mu": 3, "q_raw": 4, "log_s": 3, "o_logit": 1, "n_raw": 3, "delta_c": 3,
              "k_a_raw": 1, "k_d_raw": 1, "k_s_raw": 1, "log_beta": 1}
    out = {}
    ids = torch.empty(N, dtype=torch.int32, device=dev)
    c_rows = (ctypes.c_int64 * len(models))(*rows)
    for j, (name, w) in enumerate(widths.items()):
        dst = torch.empty((N, w) if w > 1 else (N,), dtype=torch.float64, device=dev)
        srcs = (ctypes.c_void_p * len(models))(*[m.t[name].data_ptr() for m in models])
        L.check(L.lib().ivr_concat(srcs, c_rows, len(models), w, D.ptr(dst),
                                   D.ptr(ids) if j == 0 else None, D.stream_handle()),
                "ivr_concat")
        out[name] = dst
    dg = D.DeviceGaussians({k: out[k] for k in D.DeviceGaussians.GEOM},
                           {k: out[k] for k in D.DeviceGaussians.SHADE}, None, dev)
    dg.scene_id = ids
    stubs, row = [], 0
    for i, m in enumerate(models):
        stubs.append(ResidentModel(STAGE_EDITABLE, m.n, dict((metadata or {}).get(i, {})),
                                   Palette(np.asarray(palettes[i], np.float64)), None,
                                   (row, row + m.n)))
        row += m.n
    sc = ComposedScene(stubs, [EditState() for _ in models], light or LightConfig())
    return DeviceScene(sc, dg=dg)


def render_composed(scene, cam, channels=("color", "alpha"), attrs=None, dtype=np.float32,
                    sequential=False):
    """Shade and rasterize a composed scene for one camera (scene.py:231-239).

    Uploads the scene for this one call; keep a ``DeviceScene`` to render
    many frames of the same scene without re-uploading."""
    del sequential
    return DeviceScene(scene).render(cam, channels, attrs, dtype)


def save_model(model, path):
    """scene.save_model (scene.py:242-347): the IVRG writer (ivrg.py)."""
    from .ivrg import save_model as _save
    return _save(model, path)


def load_model(path):
    """scene.load_model (scene.py:349-436): the IVRG reader (ivrg.py)."""
    from .ivrg import load_model as _load
    return _load(path)
