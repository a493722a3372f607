"""Tile rasterizer entry points (drop-in for voxsplat/rasterizer.py).

``rasterize_forward`` / ``rasterize_backward`` keep the reference signatures
(rasterizer.py:53-55, 185) and return host numpy maps, but every stage runs
on the GPU: K1 preprocess, K2 bit-exact bin/sort, K3 tile blend (and K4 for
the backward).  The returned ``state`` owns the device buffers the backward
needs (the reference's state dict of numpy arrays, rasterizer.py:74-78).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import device as D
from .errors import ShapeMismatch

TILE_SIZE = 16
_WS = {}


def workspace():
    dev = D.cuda_device()
    ws = _WS.get(dev.index)
    if ws is None:
        ws = _WS[dev.index] = D.Workspace(dev)
    return ws


@dataclass
class RenderOutput:
    """Per-pixel maps of one rasterization (all H x W [x k])."""

    color: np.ndarray | None
    alpha: np.ndarray
    depth: np.ndarray | None
    normal: np.ndarray | None
    attr: dict = field(default_factory=dict)
    per_pixel_contrib_count: np.ndarray | None = None


def _channel_layout(channels, attrs):
    """Ordered (name, width): color, alpha, depth, normal, then attrs
    (rasterizer.py:39-50)."""
    widths = {"color": 3, "alpha": 1, "depth": 1, "normal": 3}
    layout = [(c, widths[c]) for c in ("color", "alpha", "depth", "normal") if c in channels]
    for name, vals in (attrs or {}).items():
        vals = np.asarray(vals) if not isinstance(vals, torch.Tensor) else vals
        layout.append((name, 1 if vals.ndim == 1 else int(vals.shape[1])))
    return layout


def _cols(layout):
    cols = {"color": -1, "alpha": -1, "depth": -1, "normal": -1}
    attr_cols = []
    c = 0
    for name, w in layout:
        if name in cols:
            cols[name] = c
        else:
            attr_cols.append((name, c, w))
        c += w
    return (cols["color"], cols["alpha"], cols["depth"], cols["normal"]), attr_cols, c


def _unpack(out, layout, contrib):
    maps, col = {}, 0
    for name, w in layout:
        m = out[:, :, col:col + w]
        maps[name] = m[:, :, 0] if w == 1 else m
        col += w
    return RenderOutput(
        color=maps.get("color"),
        alpha=maps.get("alpha", np.zeros(out.shape[:2], dtype=out.dtype)),
        depth=maps.get("depth"), normal=maps.get("normal"),
        attr={k: v for k, v in maps.items() if k not in ("color", "alpha", "depth", "normal")},
        per_pixel_contrib_count=contrib)


def rasterize_forward(geom, colors, cam, channels=("color", "alpha"), attrs=None,
                      dtype=np.float32, sequential=False, *, exact=True):
    """Rasterize on the GPU; returns (RenderOutput, state-for-backward).

    Same contract as rasterizer.py:53-164: ``colors`` are per-splat rgb
    already resolved for this camera, ``attrs`` maps names to (N,) or (N,k)
    values; outputs are deterministic (``sequential`` is accepted and has no
    effect, exactly as in the reference).  ``exact`` (extension) selects the
    bit-faithful float64 blend (default) or the certified float32 blend."""
    del sequential
    dtype = np.dtype(dtype).type
    H, W = int(cam.height), int(cam.width)
    layout = _channel_layout(channels, attrs)
    cols, attr_cols, K = _cols(layout)
    n = len(geom)
    state = {"geom": geom, "cam": cam, "layout": layout, "dtype": dtype, "colors": colors,
             "attrs": attrs or {}, "n": n}
    if n == 0:
        out = np.zeros((H, W, K), dtype=dtype)
        state["empty"] = True
        return _unpack(out, layout, np.zeros((H, W), np.int32)), state
    f64 = dtype == np.float64
    dg = D.DeviceGaussians(geom)
    colors_dev = D.to_dev(np.asarray(colors).reshape(n, 3)) if cols[0] >= 0 else None
    attrs_dev = [(D.to_dev(np.asarray(attrs[name], dtype=np.float64).reshape(n, w)), c, w)
                 for name, c, w in attr_cols]
    # the returned state owns its buffers (a later call must not overwrite them)
    F = D.rasterize_device(dg, cam, K, cols, D.Workspace(dg.device), colors=colors_dev,
                           attrs=attrs_dev, f64=f64, want_state=True, exact=exact)
    out = D.to_host(F.out64 if f64 else F.out).astype(dtype, copy=False)
    contrib = D.to_host(F.contrib)
    state.update(frame=F, dg=dg, empty=False)
    return _unpack(out, layout, contrib), state


def render_attribute_map(geom, attr_values, cam, dtype=np.float32):
    """Composite a per-splat attribute with the colour weights
    (rasterizer.py:289-297)."""
    out, _ = rasterize_forward(geom, None, cam, channels=("alpha",),
                               attrs={"attr": np.asarray(attr_values)}, dtype=dtype)
    return out.attr["attr"]


def _project_only(geom, cam):
    """Run K1 with its float64 parity outputs (used by project_gaussians)."""
    n = len(geom)
    dg = D.DeviceGaussians(geom)
    F = D.preprocess(dg, cam, 1, (-1, 0, -1, -1), workspace(), debug=True)
    g = {k: v.cpu().numpy() for k, v in F.dbg.items()}
    return {"mean2d": g["mean2d"].reshape(n, 2), "cov2d": g["cov2d"].reshape(n, 2, 2),
            "conic": g["conic"].reshape(n, 3), "depth": g["depth"],
            "valid": g["valid"].astype(bool), "radius": g["radius"]}


def d_out_tensor(state, d_maps, device):
    """Pack the named upstream map gradients into one (H, W, K) float32 tensor
    (rasterizer.py:209-219)."""
    _check_dmaps(state, d_maps)
    cam = state["cam"]
    H, W = cam.height, cam.width
    K = sum(w for _, w in state["layout"])
    d_out = torch.zeros((H, W, K), dtype=torch.float32, device=device)
    col = 0
    for name, w in state["layout"]:
        g = d_maps.get(name)
        if g is not None:
            t = g if isinstance(g, torch.Tensor) else torch.from_numpy(np.asarray(g, np.float64))
            d_out[:, :, col:col + w] = t.to(device=device, dtype=torch.float32).reshape(H, W, w)
        col += w
    return d_out


def rasterize_backward(state, d_maps):
    """Exact-decision gradients of the forward pass on the GPU (K4a + K4b).

    Same contract as rasterizer.py:185-286: returns d_mu, d_q_raw, d_log_s,
    d_o_logit, d_n_raw, d_colors, d_attrs, d_mean2d (host float64) and raises
    NonFiniteGradient(key, row) for the first non-finite key."""
    geom, n = state["geom"], state["n"]
    grads = {"d_mean2d": np.zeros((n, 2)), "d_mu": np.zeros((n, 3)), "d_q_raw": np.zeros((n, 4)),
             "d_log_s": np.zeros((n, 3)), "d_o_logit": np.zeros(n), "d_n_raw": np.zeros((n, 3)),
             "d_colors": np.zeros((n, 3)),
             "d_attrs": {k: np.zeros(np.asarray(v).shape) for k, v in state["attrs"].items()}}
    if state.get("empty"):
        _check_dmaps(state, d_maps)
        return grads
    F, dg = state["frame"], state["dg"]
    layout = state["layout"]
    cols, attr_cols, K = _cols(layout)
    d_out = d_out_tensor(state, d_maps, dg.device)
    g = D.blend_backward(F, d_out)
    want = ("d_mu", "d_q_raw", "d_log_s", "d_o_logit", "d_n_raw", "d_colors", "d_mean2d",
            "d_values")
    out, bad = D.preprocess_backward(dg, state["cam"], K, cols, g=g, geometry=True, want=want)
    D.raise_if_bad(bad, n, ("d_mu", "d_q_raw", "d_log_s", "d_o_logit", "d_n_raw", "d_colors"))
    for key, w in (("d_mu", 3), ("d_q_raw", 4), ("d_log_s", 3), ("d_n_raw", 3), ("d_colors", 3),
                   ("d_mean2d", 2)):
        grads[key] = D.to_host(out[key]).reshape(n, w)
    grads["d_o_logit"] = D.to_host(out["d_o_logit"])
    dv = D.to_host(out["d_values"]).reshape(n, K)
    for name, c, w in attr_cols:
        grads["d_attrs"][name] = dv[:, c:c + w].reshape(np.asarray(state["attrs"][name]).shape).copy()
    return grads


def _check_dmaps(state, d_maps):
    cam = state["cam"]
    H, W = cam.height, cam.width
    for name, w in state["layout"]:
        g = d_maps.get(name)
        if g is None:
            continue
        want = (H, W) if w == 1 else (H, W, w)
        if tuple(np.shape(g)) != want:
            raise ShapeMismatch(f"gradient for {name}: {tuple(np.shape(g))} != {want}")
