"""Device plumbing: torch-owned HBM buffers, C-ABI structs, kernel launches.

PyTorch provides device memory (caching allocator) and the current CUDA
stream; every compute step is a ``libivrgs.so`` call (include/ivrgs.h).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import _lib as L

TILE = 16


def cuda_device():
    if not torch.cuda.is_available():
        raise L.NativeLibraryMissing("no CUDA device: the editable-Gaussian path is GPU-only")
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _pinned_copy(t):
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)  # torch's cached page-locked blocks
    h.copy_(t)
    return h


def to_host(t):
    """Device tensor -> (ordinary) numpy array through a page-locked staging
    block from torch's caching host allocator: a pageable D2H runs at ~2 GB/s
    on these hosts (128 MB: 57 ms), a pinned one at ~55 GB/s (2.3 ms) plus the
    host copy out of the staging block; the block goes back to the cache, so
    no page-locked memory stays attached to the returned array."""
    if t.device.type != "cuda":
        return t.numpy()
    h = _pinned_copy(t)
    out = np.empty(tuple(t.shape), dtype=h.numpy().dtype)
    np.copyto(out, h.numpy())
    return out


def to_host_bytes(t):
    """Device tensor -> bytes through a page-locked staging block (to_host)."""
    if t.device.type != "cuda":
        return t.numpy().tobytes()
    return _pinned_copy(t).numpy().tobytes()


def to_dev(a, dtype=torch.float64, device=None):
    """Host array -> contiguous device tensor (no copy if already on device)."""
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        return a.to(device=device or cuda_device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(np.asarray(a))
    t = torch.from_numpy(arr)
    if t.dtype != dtype:
        t = t.to(dtype)
    return t.to(device or cuda_device(), non_blocking=False).contiguous()


def camera_struct(cam) -> L.Camera_t:
    c = L.Camera_t()
    pos = np.asarray(cam.position, dtype=np.float64).reshape(3)
    rot = np.asarray(cam.rotation, dtype=np.float64).reshape(9)
    for i in range(3):
        c.position[i] = float(pos[i])
    for i in range(9):
        c.rotation[i] = float(rot[i])
    # Camera.focal / center_px evaluated exactly as the reference does
    c.focal = float(0.5 * cam.height / np.tan(0.5 * cam.fov_y))
    c.cx = float((cam.width - 1) / 2.0)
    c.cy = float((cam.height - 1) / 2.0)
    c.width = int(cam.width)
    c.height = int(cam.height)
    return c


def light_direction(polar, azimuth):
    """light_direction_from_angles (shading.py:179-183), host float64."""
    cp, sp = np.cos(polar), np.sin(polar)
    ca, sa = np.cos(azimuth), np.sin(azimuth)
    return np.array([cp * ca, cp * sa, sp])


class DeviceGaussians:
    """Float64 SoA geometry (+ optional shading attributes) resident in HBM."""

    GEOM = ("mu", "q_raw", "log_s", "o_logit", "n_raw")
    SHADE = ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")

    def __init__(self, geom, shading=None, scene_id=None, device=None):
        dev = device or cuda_device()
        self.n = len(geom.mu) if hasattr(geom, "mu") else int(geom["mu"].shape[0])
        get = (lambda o, k: getattr(o, k)) if not isinstance(geom, dict) else (lambda o, k: o[k])
        self.t = {k: to_dev(get(geom, k), device=dev) for k in self.GEOM}
        if shading is not None:
            gs = (lambda o, k: getattr(o, k)) if not isinstance(shading, dict) else (lambda o, k: o[k])
            for k in self.SHADE:
                self.t[k] = to_dev(gs(shading, k), device=dev)
        self.has_shading = shading is not None
        self.scene_id = to_dev(scene_id, torch.int32, dev) if scene_id is not None else None
        self.device = dev
        self.cache = None

    def build_cache(self):
        """Camera-/edit-independent per-Gaussian values (ivr_preprocess_static)
        for a scene rendered many times; later frames read them instead of
        recomputing (bit-identical).  Invalidate with ``drop_cache`` if the
        arrays change."""
        self.cache = torch.empty((max(self.n, 1), 16), dtype=torch.float64, device=self.device)
        self.cache_ok = False
        g = self.struct()
        sh = None
        if self.has_shading:
            sh = L.Shading_t()
            for k in self.SHADE:
                setattr(sh, k, self.t[k].data_ptr())
        L.check(L.lib().ivr_preprocess_static(ctypes.byref(g), ctypes.byref(sh) if sh is not None
                                              else None, ptr(self.cache), stream_handle()),
                "ivr_preprocess_static")
        self.cache_ok = True
        return self

    def drop_cache(self):
        self.cache = None
        self.cache_ok = False

    def struct(self) -> L.Gaussians_t:
        g = L.Gaussians_t()
        g.n = self.n
        for k in self.GEOM:
            setattr(g, k, self.t[k].data_ptr())
        c = getattr(self, "cache", None)
        g.cache = c.data_ptr() if c is not None and getattr(self, "cache_ok", False) else None
        return g


def shading_struct(dg: DeviceGaussians, palette_dev, per_splat, light, lam=None, b=None):
    """ivr_shading for DeviceGaussians + palette tensor + LightConfig."""
    s = L.Shading_t()
    for k in DeviceGaussians.SHADE:
        setattr(s, k, dg.t[k].data_ptr())
    s.palette = palette_dev.data_ptr()
    s.per_splat_palette = 1 if per_splat else 0
    s.orbital = 1 if light.mode == "orbital" else 0
    ld = light_direction(light.polar, light.azimuth) if s.orbital else np.zeros(3)
    for i in range(3):
        s.light_dir[i] = float(ld[i])
    ts = np.asarray(light.term_scales, dtype=np.float64).reshape(4)
    lam = np.ones(4) if lam is None else np.asarray(lam, dtype=np.float64).reshape(4)
    b = np.zeros(4) if b is None else np.asarray(b, dtype=np.float64).reshape(4)
    for i in range(4):
        s.term_scales[i] = float(ts[i])
        s.lam[i] = float(lam[i])
        s.b[i] = float(b[i])
    return s


class Workspace:
    """Grow-only cache of device buffers keyed by name (one per renderer)."""

    def __init__(self, device=None):
        self.device = device or cuda_device()
        self.bufs = {}
        self.pair_capacity = 0

    def get(self, name, numel, dtype):
        numel = max(int(numel), 1)
        t = self.bufs.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(int(numel * 1.0) if t is None else max(numel, int(t.numel() * 1.25)),
                            dtype=dtype, device=self.device)
            self.bufs[name] = t
        return t[:numel]

    def depth_minmax(self):
        """K1 -> K2 depth-range words, armed to {~0, 0} once; K2 re-arms them
        after every frame (ivr_bin_sort_frame)."""
        t = self.bufs.get("depth_mm")
        if t is None:
            t = self.bufs["depth_mm"] = torch.tensor([-1, 0], dtype=torch.int64, device=self.device)
        return t


class Frame:
    """Device outputs of one rasterization (kept alive for the backward)."""

    def pairs(self):
        """The reference's per-tile pair list (pair_splat without the cull bit)."""
        P = int(self.n_pairs.item())
        return (self.pair_splat[:P] & 0x7fffffff).cpu().numpy()


def preprocess(dg: DeviceGaussians, cam, K, cols, ws: Workspace, shading=None, edits=None,
               colors=None, attrs=(), f64=False, debug=False, stream=None, params_dev=None,
               exact_rgb=False):
    """Launch K1; returns a Frame with the per-splat buffers.  With
    ``params_dev`` (a device tensor holding an ivr_frame_params) the camera
    and light come from device memory (CUDA-graph replay); ``cam`` then only
    supplies width/height."""
    n = dg.n
    F = Frame()
    F.n, F.K, F.f64, F.cam = n, K, f64, cam
    F.depth_key = ws.get("depth_key", n, torch.int64)
    F.count = ws.get("count", n, torch.int32)
    F.rect = ws.get("rect", 4 * n, torch.int16)
    F.rec = ws.get("rec", 8 * n, torch.float32)
    F.values = ws.get("values", K * n, torch.float32)
    F.rec64 = ws.get("rec64", 8 * n, torch.float64) if f64 else None
    F.values64 = ws.get("values64", K * n, torch.float64) if f64 else None
    lay = L.Layout_t()
    lay.k = K
    lay.col_color, lay.col_alpha, lay.col_depth, lay.col_normal = cols
    lay.colors = colors.data_ptr() if colors is not None else None
    F._keep = [colors]
    lay.n_attr = len(attrs)
    for i, (t, col, w) in enumerate(attrs):
        lay.attr[i] = t.data_ptr()
        lay.attr_col[i] = col
        lay.attr_width[i] = w
        F._keep.append(t)
    out = L.ProjOut_t()
    out.depth_key, out.count, out.rect = F.depth_key.data_ptr(), F.count.data_ptr(), F.rect.data_ptr()
    F.depth_mm = ws.depth_minmax()
    out.depth_minmax = F.depth_mm.data_ptr()
    out.rec, out.values = F.rec.data_ptr(), F.values.data_ptr()
    if f64:
        out.rec64, out.values64 = F.rec64.data_ptr(), F.values64.data_ptr()
    if debug:
        dev = dg.device
        F.dbg = {"mean2d": torch.empty(2 * n, dtype=torch.float64, device=dev),
                 "conic": torch.empty(3 * n, dtype=torch.float64, device=dev),
                 "cov2d": torch.empty(4 * n, dtype=torch.float64, device=dev),
                 "depth": torch.empty(n, dtype=torch.float64, device=dev),
                 "opacity": torch.empty(n, dtype=torch.float64, device=dev),
                 "rgb": torch.zeros(3 * n, dtype=torch.float64, device=dev),
                 "radius": torch.empty(n, dtype=torch.float64, device=dev),
                 "valid": torch.empty(n, dtype=torch.uint8, device=dev)}
        for k, v in F.dbg.items():
            setattr(out, k, v.data_ptr())
    g = dg.struct()
    sh = ctypes.byref(shading) if shading is not None else None
    ed = ctypes.byref(edits) if edits is not None else None
    mode = (L.PRE_F64 if f64 else 0) | (L.PRE_EXACT_RGB if exact_rgb else 0)
    if params_dev is not None:
        L.check(L.lib().ivr_preprocess_fwd_params(
            ctypes.byref(g), sh, ed, ptr(params_dev), int(cam.width), int(cam.height),
            ctypes.byref(lay), ctypes.byref(out), mode, stream_handle(stream)),
            "ivr_preprocess_fwd_params")
    else:
        cs = camera_struct(cam)
        L.check(L.lib().ivr_preprocess_fwd(ctypes.byref(g), sh, ed, ctypes.byref(cs),
                                           ctypes.byref(lay), ctypes.byref(out), mode,
                                           stream_handle(stream)), "ivr_preprocess_fwd")
    return F


def frame_params(cam, light=None, lam=None, b=None, rescale_opacity=False) -> L.FrameParams_t:
    """Host ivr_frame_params for one frame (camera + light + transform)."""
    P = L.FrameParams_t()
    P.cam = camera_struct(cam)
    if light is not None:
        P.orbital = 1 if light.mode == "orbital" else 0
        ld = light_direction(light.polar, light.azimuth) if P.orbital else np.zeros(3)
        ts = np.asarray(light.term_scales, dtype=np.float64).reshape(4)
    else:
        P.orbital, ld, ts = 0, np.zeros(3), np.ones(4)
    lam = np.ones(4) if lam is None else np.asarray(lam, dtype=np.float64).reshape(4)
    b = np.zeros(4) if b is None else np.asarray(b, dtype=np.float64).reshape(4)
    for i in range(3):
        P.light_dir[i] = float(ld[i])
    for i in range(4):
        P.term_scales[i], P.lam[i], P.b[i] = float(ts[i]), float(lam[i]), float(b[i])
    P.rescale_opacity = 1 if rescale_opacity else 0
    if P.orbital:
        dp, da = light_direction_derivatives(light.polar, light.azimuth)
        for i in range(3):
            P.dl_dp[i], P.dl_da[i] = float(dp[i]), float(da[i])
    return P


def light_direction_derivatives(polar, azimuth):
    """d light_direction / d polar, d azimuth (host float64)."""
    p, a = polar, azimuth
    return ((-np.sin(p) * np.cos(a), -np.sin(p) * np.sin(a), np.cos(p)),
            (-np.cos(p) * np.sin(a), np.cos(p) * np.cos(a), 0.0))


def bin_sort(F: Frame, ws: Workspace, stream=None, capacity=None):
    """Launch K2 into F (pair_splat, tile_ranges, n_pairs)."""
    cam = F.cam
    ntx, nty = (cam.width + TILE - 1) // TILE, (cam.height + TILE - 1) // TILE
    F.ntx, F.nty = ntx, nty
    n = F.n
    cap = capacity or max(ws.pair_capacity, 4 * n, 1 << 16)
    ws.pair_capacity = cap
    nbytes = L.lib().ivr_bin_sort_workspace_size(n, cap, ntx * nty)
    scratch = ws.get("sort_ws", nbytes, torch.uint8)
    F.pair_splat = ws.get("pair_splat", cap, torch.int32)
    F.tile_ranges = ws.get("tile_ranges", ntx * nty + 1, torch.int32)
    F.n_pairs = ws.get("n_pairs", 1, torch.int32)
    F.capacity = cap
    # K2; the per-(splat, tile) cull runs in K3/K4 staging (precull=False) or
    # here as bit 31 of pair_splat (precull=True; masked in .pairs()).  K1's
    # depth range and the K3/K4 tile schedule ride along (ivr_bin_sort_frame).
    precull = os.environ.get("IVR_PRECULL", "0") == "1"
    F.tile_order = None
    if os.environ.get("IVR_TILE_ORDER", "1") != "0":
        F.tile_order = ws.get("tile_order", ntx * nty, torch.int32)
    mm = getattr(F, "depth_mm", None)
    L.check(L.lib().ivr_bin_sort_frame(n, ptr(F.depth_key), ptr(mm), ptr(F.count), ptr(F.rect),
                                       ptr(F.rec) if precull else None, ntx, nty, cam.width,
                                       cam.height, cap, ptr(scratch), nbytes, ptr(F.pair_splat),
                                       ptr(F.tile_ranges), ptr(F.n_pairs), ptr(F.tile_order),
                                       stream_handle(stream)), "ivr_bin_sort_frame")
    F.preculled = precull
    return F


def blend(F: Frame, ws: Workspace, want_state=True, stream=None, out=None, exact=False):
    """Launch K3.  exact=True: bit-faithful float64 evaluation of every
    candidate pair (IVR_BLEND_EXACT); otherwise certified float32 (FAST)."""
    cam = F.cam
    H, W, K = cam.height, cam.width, F.K
    dev = F.depth_key.device
    if F.f64:
        F.out64 = out if out is not None else torch.empty((H, W, K), dtype=torch.float64, device=dev)
        F.out = None
    else:
        F.out = out if out is not None else torch.empty((H, W, K), dtype=torch.float32, device=dev)
        F.out64 = None
    F.contrib = torch.empty((H, W), dtype=torch.int32, device=dev)
    F.last_pos = torch.empty((H, W), dtype=torch.int32, device=dev) if want_state else None
    F.t_final = torch.empty((H, W), dtype=torch.float64, device=dev) if want_state else None
    L.check(L.lib().ivr_blend_fwd(ptr(F.tile_ranges), ptr(F.pair_splat), F.ntx, F.nty, ptr(F.rec),
                                  ptr(F.values), ptr(F.rec64), ptr(F.values64), K, W, H, ptr(F.out),
                                  ptr(F.out64), ptr(F.contrib), ptr(F.last_pos), ptr(F.t_final),
                                  ptr(getattr(F, "tile_order", None)),
                                  (L.BLEND_EXACT if exact else 0) |
                                  (L.BLEND_PRECULLED if getattr(F, "preculled", False) else 0),
                                  stream_handle(stream)),
            "ivr_blend_fwd")
    F.exact = exact
    return F


def blend_backward(F: Frame, d_out, stream=None, deterministic=None, geometry=True):
    """K4a: per-Gaussian float32 accumulators from the upstream image gradient
    d_out (H,W,K float32 device tensor).  deterministic (default: env
    IVR_DETERMINISTIC=1): fixed-order reduction, identical on every run.
    geometry=False: only the value and opacity accumulators (transform fits;
    mean2d / conic stay zero)."""
    if deterministic is None:
        deterministic = os.environ.get("IVR_DETERMINISTIC", "0") == "1"
    n, K = F.n, F.K
    dev = F.depth_key.device
    arena = torch.zeros(n * (K + 6), dtype=torch.float32, device=dev)  # one memset
    g = {"values": arena[:n * K], "mean2d": arena[n * K:n * (K + 2)],
         "conic": arena[n * (K + 2):n * (K + 5)], "opacity": arena[n * (K + 5):]}
    if F.t_final is None:
        raise ValueError("blend_backward needs the forward state (render with want_state=True)")
    # float64 upstream gradients (the photometric loss's) are read in place
    dflag = L.BLEND_DOUT_F64 if d_out.dtype == torch.float64 else 0
    d_out = d_out.contiguous() if dflag else d_out.to(torch.float32).contiguous()
    cam = F.cam
    if deterministic:
        nb = int(L.lib().ivr_blend_bwd_det_workspace_size(F.capacity, K))
        ws = torch.empty(max(nb, 8), dtype=torch.uint8, device=dev)
        L.check(L.lib().ivr_blend_bwd_deterministic(
            ptr(F.tile_ranges), ptr(F.pair_splat), F.ntx, F.nty, ptr(F.rec), ptr(F.values),
            ptr(F.rec64), K, cam.width, cam.height, ptr(F.t_final), ptr(F.last_pos), ptr(d_out), n,
            ptr(F.depth_key), ptr(F.count), ptr(F.rect), F.capacity, ptr(ws), nb,
            ptr(g["values"]), ptr(g["mean2d"]), ptr(g["conic"]), ptr(g["opacity"]),
            ptr(getattr(F, "tile_order", None)),
            (L.BLEND_PRECULLED if getattr(F, "preculled", False) else 0) |
            (0 if geometry else L.BLEND_NO_GEOMETRY) | dflag,
            stream_handle(stream)), "ivr_blend_bwd_deterministic")
        return g
    L.check(L.lib().ivr_blend_bwd(ptr(F.tile_ranges), ptr(F.pair_splat), F.ntx, F.nty, ptr(F.rec),
                                  ptr(F.values), ptr(F.rec64), K, cam.width, cam.height,
                                  ptr(F.t_final), ptr(F.last_pos), ptr(d_out), ptr(g["values"]),
                                  ptr(g["mean2d"]),
                                  ptr(g["conic"]), ptr(g["opacity"]),
                                  ptr(getattr(F, "tile_order", None)),
                                  (L.BLEND_PRECULLED if getattr(F, "preculled", False) else 0) |
                                  (0 if geometry else L.BLEND_NO_GEOMETRY) | dflag,
                                  stream_handle(stream)), "ivr_blend_bwd")
    return g


GRAD_SHAPES = {"d_mu": 3, "d_q_raw": 4, "d_log_s": 3, "d_o_logit": 1, "d_n_raw": 3, "d_colors": 3,
               "d_mean2d": 2, "d_delta_c": 3, "d_k_a_raw": 1, "d_k_d_raw": 1, "d_k_s_raw": 1,
               "d_log_beta": 1}


def preprocess_backward(dg: DeviceGaussians, cam, K, cols, g=None, shading=None, edits=None,
                        params_dev=None, d_rgb=None, geometry=True, want=(), per_scene=0,
                        per_splat_c_p=False, light=None, stream=None):
    """K4b: float64 per-Gaussian gradients.  Returns (dict of device tensors,
    bad-row tensor)."""
    n = dg.n
    dev = dg.device
    out = {}
    R = L.Grads_t()
    if g is not None:
        R.g_values, R.g_mean2d = g["values"].data_ptr(), g["mean2d"].data_ptr()
        R.g_conic, R.g_opacity = g["conic"].data_ptr(), g["opacity"].data_ptr()
    if d_rgb is not None:
        R.d_rgb_extra = d_rgb.data_ptr()
    # outputs K4b stores for every Gaussian in this configuration share one
    # uninitialised arena; the atomically reduced ones (per-scene d_c_p,
    # d_scale, d_globals) and any the kernel would not reach live in a small
    # zeroed arena
    stored = {"d_colors", "d_mean2d", "d_o_logit", "d_mu", "d_n_raw"}
    if g is not None:
        stored.add("d_values")
    if geometry:
        stored.update(("d_q_raw", "d_log_s"))
    if shading is not None:
        stored.update(("d_delta_c", "d_k_a_raw", "d_k_d_raw", "d_k_s_raw", "d_log_beta"))
        if per_splat_c_p:
            stored.add("d_c_p")
    sizes = [(name, n * GRAD_SHAPES[name]) for name in want if name in GRAD_SHAPES]
    if "d_values" in want:
        sizes.append(("d_values", n * K))
    if "d_c_p" in want:
        sizes.append(("d_c_p", (n if per_splat_c_p else max(per_scene, 1)) * 3))
    if "d_scale" in want:
        sizes.append(("d_scale", max(per_scene, 1)))
    if shading is not None and "d_globals" in want:
        sizes.append(("d_globals", 10))
    for part, alloc in (([x for x in sizes if x[0] in stored], torch.empty),
                        ([x for x in sizes if x[0] not in stored], torch.zeros)):
        if not part:
            continue
        arena = alloc(sum(sz for _, sz in part), dtype=torch.float64, device=dev)
        o = 0
        for name, sz in part:
            out[name] = arena[o:o + sz]
            setattr(R, name, out[name].data_ptr())
            o += sz
    R.per_scene = 0 if per_splat_c_p else int(per_scene)
    if light is not None and light.mode == "orbital":
        dp, da = light_direction_derivatives(light.polar, light.azimuth)
        for i in range(3):
            R.dl_dp[i], R.dl_da[i] = float(dp[i]), float(da[i])
    bad = torch.full((16,), -1, dtype=torch.int64, device=dev)  # ~0 as uint64
    R.bad = bad.data_ptr()
    if ("d_globals" in out or R.per_scene > 0) and \
            os.environ.get("IVR_DETERMINISTIC", "0") == "1":
        # fixed-order sums of the per-block transform-gradient partials
        ns = int(L.lib().ivr_preprocess_bwd_scratch_len(n, R.per_scene))
        scratch = torch.empty(max(ns, 1), dtype=torch.float64, device=dev)
        R.scratch, R.scratch_len = scratch.data_ptr(), ns  # stream-ordered reuse is safe
    lay = L.Layout_t()
    lay.k = K
    lay.col_color, lay.col_alpha, lay.col_depth, lay.col_normal = cols
    gs = dg.struct()
    cs = camera_struct(cam)
    L.check(L.lib().ivr_preprocess_bwd(
        ctypes.byref(gs), ctypes.byref(shading) if shading is not None else None,
        ctypes.byref(edits) if edits is not None else None, ptr(params_dev), ctypes.byref(cs),
        ctypes.byref(lay), ctypes.byref(R), 1 if geometry else 0, stream_handle(stream)),
        "ivr_preprocess_bwd")
    return out, bad


def raise_if_bad(bad, n, order):
    """NonFiniteGradient(first tensor in `order` with a bad row, that row)."""
    b = bad.cpu().numpy().view(np.uint64)
    for name in order:
        if name in L.BAD_IDS:
            v = int(b[L.BAD_IDS.index(name)])
            if v != 0xFFFFFFFFFFFFFFFF and v < n:
                from .errors import NonFiniteGradient
                raise NonFiniteGradient(name, v)


def rasterize_device(dg, cam, K, cols, ws, shading=None, edits=None, colors=None, attrs=(),
                     f64=False, want_state=True, debug=False, stream=None, exact=True,
                     params_dev=None, capacity=None):
    """K1 + K2 + K3 with pair-capacity overflow handling (synchronizes once to
    read the pair count).  With ``capacity`` (CUDA-graph capture) there is no
    host synchronisation: the caller checks ``F.n_pairs`` against it later;
    ``params_dev`` takes the camera / light from device memory."""
    F = preprocess(dg, cam, K, cols, ws, shading, edits, colors, attrs, f64, debug, stream,
                   params_dev=params_dev, exact_rgb=exact)
    if dg.n == 0:
        F.empty = True
        return F
    if capacity is not None:
        bin_sort(F, ws, stream, capacity=capacity)
        F.P, F.empty = None, False
        blend(F, ws, want_state, stream, exact=exact)
        return F
    bin_sort(F, ws, stream)
    P = int(F.n_pairs.item())
    if P > F.capacity:
        F.depth_mm = None  # consumed (re-armed) by the first pass: K2 reduces the range itself
        bin_sort(F, ws, stream, capacity=int(P * 1.25) + 4096)
        P = int(F.n_pairs.item())
    F.P = P
    F.empty = False
    blend(F, ws, want_state, stream, exact=exact)
    return F
