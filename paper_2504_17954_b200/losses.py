"""Training / fitting objectives on the GPU (drop-in for voxsplat/losses.py).

Every function takes numpy arrays or CUDA tensors, computes in float64 on the
device and returns the reference's (loss, gradient) pairs with the analytic
gradients of losses.py:45-268.  L1 + SSIM (value and gradient) run in two
fused tiled kernels (csrc/ssim.cu); the small regularizers are torch ops.
Inputs given as numpy come back as numpy.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from .errors import ShapeMismatch

SSIM_SIGMA = 1.5
SSIM_RADIUS = 5
SSIM_C1 = 0.01 ** 2
SSIM_C2 = 0.03 ** 2

_offs = np.arange(-SSIM_RADIUS, SSIM_RADIUS + 1, dtype=np.float64)
_K1D = np.exp(-(_offs ** 2) / (2.0 * SSIM_SIGMA ** 2))
_K1D /= _K1D.sum()


@dataclass
class LossWeights:
    """Default weighting of the total objective (losses.py:28-42)."""

    l1_weight: float = 0.8
    ssim_weight: float = 0.2
    normal_consistency: float = 0.01
    opacity_l1: float = 0.1
    offset_sparsity: float = 0.01
    bilateral_smoothness: float = 0.01

    def __post_init__(self):
        for f in self.__dataclass_fields__:
            if getattr(self, f) < 0:
                raise ValueError(f"loss weight {f} must be >= 0")


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _t(x):
    if isinstance(x, torch.Tensor):
        return x.to(device=_dev(), dtype=torch.float64)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, dtype=np.float64))).to(_dev())


def _out(ref, t):
    return t if isinstance(ref, torch.Tensor) else t.cpu().numpy()


_WS = {}


def _window_ptr():
    w = np.ascontiguousarray(_K1D, dtype=np.float64)
    return w, w.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _photometric_dev(x, y, a, b, with_ssim):
    """csrc/ssim.cu on (H, W, C) float64 device tensors: returns
    (sums = [sum of SSIM over windows and channels, sum |x - y|],
    d = a * sign(x - y) + b * d(mean SSIM)/dx)."""
    from . import _lib as L
    from . import device as D
    if x.dtype != torch.float64 or y.dtype != torch.float64 or x.dim() != 3 or x.shape != y.shape:
        raise ShapeMismatch(f"prediction / ground truth must be float64 (H, W, C) tensors of one "
                            f"shape, got {x.dtype} {tuple(x.shape)} and {y.dtype} {tuple(y.shape)}")
    x, y = x.contiguous(), y.contiguous()
    h, w, nc = x.shape
    nbytes = L.lib().ivr_photometric_workspace_size(h, w, nc)
    key = (x.device, nbytes)
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=x.device)
    d = torch.empty_like(x)
    sums = torch.empty(2, dtype=torch.float64, device=x.device)
    keep, wp = _window_ptr()
    L.check(L.lib().ivr_photometric_loss(D.ptr(x), D.ptr(y), h, w, nc, wp, float(a), float(b),
                                         1 if with_ssim else 0, D.ptr(d), D.ptr(sums), D.ptr(ws),
                                         nbytes, D.stream_handle()), "ivr_photometric_loss")
    del keep
    return sums, d


def _photometric_frame_dev(frame, cols, y, a, b, with_ssim):
    """``_photometric_dev`` with the prediction read in place from K3's
    float32 (H, W, k) frame at columns ``cols`` (ivr_photometric_loss_frame):
    the same sums and d as on ``frame[..., cols].double()``, without the
    gather and the float64 copy."""
    import ctypes
    from . import _lib as L
    from . import device as D
    if frame.dtype != torch.float32 or frame.dim() != 3:
        raise ShapeMismatch(f"frame must be a float32 (H, W, k) tensor, got {frame.dtype} "
                            f"{tuple(frame.shape)}")
    frame, y = frame.contiguous(), y.contiguous()
    h, w, k = frame.shape
    nc = len(cols)
    if any(not 0 <= int(c) < k for c in cols):
        raise ShapeMismatch(f"columns {list(cols)} outside the frame's {k} channels")
    if tuple(y.shape) != (h, w, nc) or y.dtype != torch.float64:
        raise ShapeMismatch(f"prediction {(h, w, nc)} vs ground truth {y.dtype} "
                            f"{tuple(y.shape)} (float64 expected)")
    nbytes = L.lib().ivr_photometric_workspace_size(h, w, nc)
    key = (y.device, nbytes)
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = torch.empty(max(nbytes, 8), dtype=torch.uint8, device=y.device)
    d = torch.empty((h, w, nc), dtype=torch.float64, device=y.device)
    sums = torch.empty(2, dtype=torch.float64, device=y.device)
    keep, wp = _window_ptr()
    cm = (ctypes.c_int32 * nc)(*[int(c) for c in cols])
    L.check(L.lib().ivr_photometric_loss_frame(D.ptr(frame), k, cm, D.ptr(y), h, w, nc, wp,
                                               float(a), float(b), 1 if with_ssim else 0,
                                               D.ptr(d), D.ptr(sums), D.ptr(ws), nbytes,
                                               D.stream_handle()), "ivr_photometric_loss_frame")
    del keep
    return sums, d


def regularize_t(out, cols, gt=None, d_rgba=None, cam_params=None, w_normal=0.0, w_offset=0.0,
                 w_bil=0.0, bil_cols=()):
    """Fused map terms of a training step (csrc/regularize.cu): returns
    (terms = [normal loss, mean |delta_c|, bilateral sum], d_out float32
    (H,W,K)).  ``out`` is K3's float32 (H,W,K) map stack, ``cols`` =
    (color, alpha, depth, normal, delta_c) columns (-1 absent), ``cam_params``
    a device float64 block (focal, cx, cy, rotation[9])."""
    from . import _lib as L
    from . import device as D
    h, w, k = out.shape
    nbytes = L.lib().ivr_regularize_workspace_size(h, w)
    key = ("reg", out.device, nbytes)
    ws = _WS.get(key)
    if ws is None:
        ws = _WS[key] = torch.empty(nbytes, dtype=torch.uint8, device=out.device)
    d_out = torch.empty_like(out)
    terms = torch.empty(3, dtype=torch.float64, device=out.device)
    c5 = (ctypes.c_int32 * 5)(*cols)
    nb = len(bil_cols)
    bc = (ctypes.c_int32 * max(nb, 1))(*(list(bil_cols) or [0]))
    L.check(L.lib().ivr_regularize(D.ptr(out), k, h, w, c5, bc, nb, D.ptr(gt), D.ptr(d_rgba),
                                   D.ptr(cam_params), float(w_normal), float(w_offset), float(w_bil),
                                   D.ptr(d_out), D.ptr(terms), D.ptr(ws), nbytes,
                                   D.stream_handle()), "ivr_regularize")
    return terms, d_out


def ssim_t(x, y):
    """Mean SSIM over channels and its gradient w.r.t. x (float64 device
    tensors (H, W, C)); one fused window pass + one adjoint pass (csrc/ssim.cu)."""
    if x.shape != y.shape:
        raise ShapeMismatch(f"ssim inputs differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    h, w, nc = x.shape
    win = 2 * SSIM_RADIUS + 1
    if h < win or w < win:
        raise ShapeMismatch(f"image {h}x{w} smaller than the {win}x{win} ssim window")
    sums, d = _photometric_dev(x, y, 0.0, 1.0, True)
    return sums[0] / float((h - win + 1) * (w - win + 1) * nc), d


def ssim(x, y):
    """losses.ssim (losses.py:57-115): (value, d_value/d_x); (H,W) or (H,W,C)."""
    xt, yt = _t(x), _t(y)
    sq = xt.dim() == 2
    if sq:
        xt, yt = xt[..., None], yt[..., None]
    v, d = ssim_t(xt, yt)
    if sq:
        d = d[..., 0]
    return float(v), _out(x, d)


def photometric_loss_t(pred, gt, weights=None):
    """0.8 L1 + 0.2 (1 - SSIM) on device tensors; returns (loss tensor, d_pred).
    L1, SSIM and both gradients come from the fused kernels (csrc/ssim.cu)."""
    weights = weights or LossWeights()
    if pred.shape != gt.shape:
        raise ShapeMismatch(f"prediction {tuple(pred.shape)} vs ground truth {tuple(gt.shape)}")
    x = pred if pred.dim() == 3 else pred[..., None]
    y = gt if gt.dim() == 3 else gt[..., None]
    h, w, nc = x.shape
    win = 2 * SSIM_RADIUS + 1
    with_ssim = weights.ssim_weight > 0.0
    if with_ssim and (h < win or w < win):
        raise ShapeMismatch(f"image {h}x{w} smaller than the {win}x{win} ssim window")
    numel = x.numel()
    sums, d = _photometric_dev(x.to(torch.float64), y.to(torch.float64),
                               weights.l1_weight / numel, -weights.ssim_weight, with_ssim)
    loss = weights.l1_weight * (sums[1] / numel)
    if with_ssim:
        s = sums[0] / float((h - win + 1) * (w - win + 1) * nc)
        loss = loss + weights.ssim_weight * (1.0 - s)
    return loss, (d if pred.dim() == 3 else d[..., 0])


def photometric_loss(pred_rgba, gt_rgba, weights=None):
    """losses.photometric_loss (losses.py:118-138): (loss, d_pred)."""
    loss, d = photometric_loss_t(_t(pred_rgba), _t(gt_rgba), weights)
    return float(loss), _out(pred_rgba, d)


def pseudo_normal_from_depth(depth, alpha, cam, alpha_threshold=1e-3):
    """losses.py:141-181: camera-oriented pseudo-normals from a depth map."""
    d, a = _t(depth), _t(alpha)
    if d.shape != a.shape:
        raise ShapeMismatch(f"depth {tuple(d.shape)} vs alpha {tuple(a.shape)}")
    h, w = d.shape
    py, px = torch.meshgrid(torch.arange(h, dtype=torch.float64, device=d.device),
                            torch.arange(w, dtype=torch.float64, device=d.device), indexing="ij")
    cx, cy = (cam.width - 1) / 2.0, (cam.height - 1) / 2.0
    f = 0.5 * cam.height / np.tan(0.5 * cam.fov_y)
    pts = torch.stack([(px - cx) * d / f, (py - cy) * d / f, d], dim=-1)
    dx = torch.empty_like(pts)
    dx[:, :-1] = pts[:, 1:] - pts[:, :-1]
    dx[:, -1] = pts[:, -1] - pts[:, -2]
    dy = torch.empty_like(pts)
    dy[:-1] = pts[1:] - pts[:-1]
    dy[-1] = pts[-1] - pts[-2]
    n = torch.linalg.cross(dx, dy, dim=-1)
    norms = torch.linalg.norm(n, dim=-1, keepdim=True)
    good = norms[..., 0] > 1e-12
    n = torch.where(good[..., None], n / torch.clamp(norms, min=1e-12), torch.zeros_like(n))
    away = (n * pts).sum(-1) > 0.0
    n = torch.where(away[..., None], -n, n)
    rot = torch.from_numpy(np.asarray(cam.rotation, dtype=np.float64)).to(d.device)
    nw = n @ rot
    mask = (a > alpha_threshold) & good
    nw = torch.where(mask[..., None], nw, torch.zeros_like(nw))
    return _out(depth, nw), _out(depth, mask)


def normal_consistency_t(n, t, m):
    """Device form of normal_consistency_loss (no host sync): (loss tensor,
    gradient); n, t (H,W,3) float64, m (H,W) bool."""
    cnt = m.sum().clamp(min=1).to(n.dtype)
    diff = (n - t) * m[..., None]
    norms = torch.linalg.norm(diff, dim=-1)
    loss = norms.sum() / cnt
    safe = norms > 1e-12
    g = torch.where(safe[..., None], diff / torch.where(safe, norms, 1.0)[..., None], 0.0) / cnt
    return loss, g


def normal_consistency_loss(normal_map, target, mask):
    """losses.py:184-206: mean L2 distance over masked pixels, gradient to the map."""
    n, t = _t(normal_map), _t(target)
    m = mask.to(_dev()).bool() if isinstance(mask, torch.Tensor) else \
        torch.from_numpy(np.asarray(mask, bool)).to(_dev())
    if n.shape != t.shape:
        raise ShapeMismatch(f"normal maps differ: {tuple(n.shape)} vs {tuple(t.shape)}")
    loss, d_n = normal_consistency_t(n, t, m)
    return float(loss), _out(normal_map, d_n)


def _fdiff_abs(img):
    img = img if img.dim() == 3 else img[..., None]
    gx = torch.zeros(img.shape[:2], dtype=img.dtype, device=img.device)
    gy = torch.zeros_like(gx)
    gx[:, :-1] = (img[:, 1:] - img[:, :-1]).abs().sum(-1)
    gy[:-1] = (img[1:] - img[:-1]).abs().sum(-1)
    return gx + gy


def bilateral_smoothness_t(k, c, m=None):
    """Device form of bilateral_smoothness (no host sync): (loss tensor, d_k)."""
    if m is None:
        m = torch.ones(k.shape[:2], dtype=torch.bool, device=k.device)
    cnt = m.sum().clamp(min=1).to(k.dtype)
    d_k = torch.zeros_like(k)
    weight = torch.exp(-_fdiff_abs(c)) * m / cnt
    k3 = k if k.dim() == 3 else k[..., None]
    d3 = d_k if d_k.dim() == 3 else d_k[..., None]
    gx = k3[:, 1:] - k3[:, :-1]
    gy = k3[1:] - k3[:-1]
    loss = (gx.abs().sum(-1) * weight[:, :-1]).sum() + (gy.abs().sum(-1) * weight[:-1]).sum()
    sx = torch.sign(gx) * weight[:, :-1, None]
    sy = torch.sign(gy) * weight[:-1, :, None]
    d3[:, 1:] += sx
    d3[:, :-1] -= sx
    d3[1:] += sy
    d3[:-1] -= sy
    return loss, d_k


def bilateral_smoothness(attr_map, gt_color, mask=None):
    """losses.py:219-253: edge-aware smoothness and its gradient."""
    k, c = _t(attr_map), _t(gt_color)
    if k.shape[:2] != c.shape[:2]:
        raise ShapeMismatch(f"attribute {tuple(k.shape)} vs color {tuple(c.shape)}")
    m = None if mask is None else _t(mask).bool()
    loss, d_k = bilateral_smoothness_t(k, c, m)
    return float(loss), _out(attr_map, d_k)


def offset_sparsity_loss(offset_map):
    """losses.py:256-260."""
    m = _t(offset_map)
    return float(m.abs().mean()), _out(offset_map, torch.sign(m) / m.numel())


def opacity_l1_loss(o_logit):
    """losses.py:263-268: mean mapped opacity, gradient w.r.t. the logits."""
    x = _t(o_logit)
    o = torch.sigmoid(x)
    return float(o.mean()), _out(o_logit, o * (1.0 - o) / o.numel())
