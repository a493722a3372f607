"""Display rendering and the service frame path (drop-in for
voxsplat/render_modes.py, and the per-frame work of service.py:169-187,
255-275).

``render_mode_image`` / ``to_uint8`` / ``png_bytes`` keep the reference's
host API.  ``DisplayRenderer`` is the B200 frame path behind the interactive
UI: the scene stays resident, each frame renders on the device, the display
map and uint8 conversion run in one kernel (``ivr_display_u8``) and the PNG
is assembled on the device (``ivr_png_encode``: stored deflate blocks,
parallel adler32 / CRC-32), so a frame leaves the GPU as its final bytes.
"""

from __future__ import annotations

import ctypes
import io

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .errors import MixedStage, OutOfRange
from .rasterizer import _channel_layout, _cols, rasterize_forward
from .scene import STAGE_EDITABLE, ComposedScene, DeviceScene
from .shading import LightConfig

RENDER_MODES = ("shaded", "normal", "ambient", "diffuse", "specular", "depth", "alpha")
_DISPLAY_MODE = {"shaded": 0, "alpha": 1, "normal": 2, "depth": 3,
                 "ambient": 0, "diffuse": 0, "specular": 0}


def as_composed(model):
    """View any loaded model as a composed scene (render_modes.py:23-29)."""
    if isinstance(model, ComposedScene):
        return model
    light = LightConfig.from_dict(model.metadata["light"]) \
        if model.metadata.get("light") else LightConfig()
    return ComposedScene.compose([model], light)


def _display_map(out, mode):
    """render_modes.py:75-92 on host maps (float64)."""
    if mode == "alpha":
        return out.alpha
    if mode == "normal":
        n = np.asarray(out.normal, dtype=np.float64)
        norm = np.linalg.norm(n, axis=-1, keepdims=True)
        unit = np.where(norm > 1e-8, n / np.maximum(norm, 1e-8), 0.0)
        return 0.5 * (unit + 1.0)
    alpha = np.asarray(out.alpha, dtype=np.float64)
    covered = alpha > 1e-6
    d = np.zeros_like(alpha)
    d[covered] = out.depth[covered] / alpha[covered]
    if covered.any():
        lo, hi = d[covered].min(), d[covered].max()
        d[covered] = (d[covered] - lo) / (hi - lo) if hi > lo else 1.0
    return d


def render_mode_image(model, cam, mode):
    """Float image in [0, 1] for one render mode (render_modes.py:31-72);
    every render runs on the GPU."""
    if mode not in RENDER_MODES:
        raise OutOfRange(f"unknown render mode {mode!r}")
    from .trainer import render_model
    if not isinstance(model, ComposedScene) and model.stage != STAGE_EDITABLE:
        if mode in ("ambient", "diffuse", "specular"):
            raise MixedStage(f"mode {mode!r} needs an editable-stage model")
        rgba = render_model(model, cam, dtype=np.float64)
        if mode == "shaded":
            return rgba
        if mode == "alpha":
            return rgba[..., 3]
        out, _ = rasterize_forward(model.geometry, np.zeros((len(model.geometry), 3)), cam,
                                   channels=("alpha", "depth", "normal"), dtype=np.float64)
        return _display_map(out, mode)
    scene = as_composed(model)
    if scene.transform is not None and mode == "shaded":
        from .inverse import TransformParams, render_with_transform
        return render_with_transform(scene, TransformParams.from_dict(scene.transform), cam,
                                     dtype=np.float64)
    R = DisplayRenderer(scene)
    img = R.float_image(cam, mode)
    return img


def to_uint8(img):
    """render_modes.py:93-95."""
    return np.clip(np.round(np.asarray(img, dtype=np.float64) * 255.0), 0, 255).astype(np.uint8)


def to_pil(img):
    from PIL import Image
    img8 = to_uint8(img)
    if img8.ndim == 2:
        return Image.fromarray(img8, mode="L")
    return Image.fromarray(img8, mode="RGBA" if img8.shape[-1] == 4 else "RGB")


def png_bytes(img):
    """PIL-encoded PNG (render_modes.py:106-110)."""
    buf = io.BytesIO()
    to_pil(img).save(buf, format="PNG")
    return buf.getvalue()


class DisplayRenderer:
    """Resident scene + device display / PNG encoding for a stream of frames."""

    def __init__(self, scene, device=None):
        self.scene = as_composed(scene) if not isinstance(scene, DeviceScene) else scene.scene
        self.ds = scene if isinstance(scene, DeviceScene) else DeviceScene(self.scene, device)
        self.dev = self.ds.dg.device
        self._ws = torch.empty(64, dtype=torch.uint8, device=self.dev)

    def _render(self, cam, mode):
        """float64 maps (H,W,K) on the device and their column map."""
        if mode in ("ambient", "diffuse", "specular"):
            return self._render_term(cam, mode)
        channels = ("color", "alpha") if mode == "shaded" else ("color", "alpha", "depth", "normal")
        F = self.ds.render_frame(cam, channels=channels, dtype=np.float64)
        cols, _, K = _cols(_channel_layout(channels, None))
        return F.out64, cols, K

    def _render_term(self, cam, mode):
        """One lighting term as the colour (render_modes.py:55-60): K1's
        shading terms on the device, then the colour path of K1-K3 with the
        scene's opacity edits."""
        ds = self.ds
        shading, edits = ds._tables()
        n = ds.n
        rgb = torch.empty(3 * n, dtype=torch.float64, device=self.dev)
        terms = torch.empty(9 * n, dtype=torch.float64, device=self.dev)
        g = ds.dg.struct()
        cs = D.camera_struct(cam)
        L.check(L.lib().ivr_shade_fwd(ctypes.byref(g), ctypes.byref(shading),
                                      D.ptr(ds.dg.scene_id), ctypes.byref(cs), D.ptr(rgb),
                                      D.ptr(terms), D.stream_handle()), "ivr_shade_fwd")
        j = {"ambient": 0, "diffuse": 1, "specular": 2}[mode]
        col = terms.view(n, 9)[:, 3 * j:3 * j + 3].contiguous()
        channels = ("color", "alpha")
        cols, _, K = _cols(_channel_layout(channels, None))
        F = D.rasterize_device(ds.dg, cam, K, cols, ds.ws, None, edits, col, (), f64=True,
                               want_state=False, exact=True)
        return F.out64, cols, K

    def frame_u8(self, cam, mode="shaded"):
        """uint8 display image (H,W[,C]) as a device tensor."""
        if mode not in RENDER_MODES:
            raise OutOfRange(f"unknown render mode {mode!r}")
        out, cols, K = self._render(cam, mode)
        H, W = cam.height, cam.width
        dm = _DISPLAY_MODE[mode]
        C = {0: 4, 1: 1, 2: 3, 3: 1}[dm]
        dst = torch.empty((H, W, C) if C > 1 else (H, W), dtype=torch.uint8, device=self.dev)
        c4 = (ctypes.c_int32 * 4)(*cols)
        L.check(L.lib().ivr_display_u8(D.ptr(out), H, W, K, c4, dm, D.ptr(dst), D.ptr(self._ws),
                                       D.stream_handle()), "ivr_display_u8")
        return dst

    def float_image(self, cam, mode="shaded"):
        """The float image render_mode_image returns (host float64)."""
        out, cols, K = self._render(cam, mode)
        o = D.to_host(out)
        cc, ca, cd, cn = cols
        if mode in ("shaded", "ambient", "diffuse", "specular"):
            return np.concatenate([np.clip(o[..., cc:cc + 3], 0, 1), o[..., ca:ca + 1]], axis=-1)
        if mode == "alpha":
            return o[..., ca]
        from types import SimpleNamespace
        m = SimpleNamespace(alpha=o[..., ca], depth=o[..., cd], normal=o[..., cn:cn + 3])
        return _display_map(m, mode)

    def frame_bytes(self, cam, mode="shaded", fmt="png"):
        """One service frame: the raw uint8 bytes or a PNG, encoded on the
        device and copied to the host once."""
        img = self.frame_u8(cam, mode)
        if fmt == "raw":
            return D.to_host_bytes(img)
        if fmt != "png":
            raise OutOfRange(f"unknown format {fmt!r}")
        H, W = img.shape[0], img.shape[1]
        C = 1 if img.dim() == 2 else img.shape[2]
        size = int(L.lib().ivr_png_size(H, W, C))
        buf = torch.empty(size, dtype=torch.uint8, device=self.dev)
        ws = torch.empty(64, dtype=torch.uint8, device=self.dev)
        L.check(L.lib().ivr_png_encode(D.ptr(img), H, W, C, D.ptr(buf), size, D.ptr(ws),
                                       D.stream_handle()), "ivr_png_encode")
        return D.to_host_bytes(buf)
