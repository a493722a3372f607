"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the reference hot path.

Every function cites the reference lines it restates (paths relative to
``/root/reference/pkg/src/voxsplat/``).  The restatement keeps the reference's
float64 evaluation order operation by operation (numpy ufuncs and ``matmul``
for the per-Gaussian math; ``composite.c`` for the numba loops), because the
hot path's contract is bit-exact sort keys / tile lists and the f32 kernel
records are rounded from these float64 values.

Checked against golden vectors generated from the real reference by
``tests/golden/make_golden.py`` (``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

__all__ = [
    "ALPHA_CAP", "ALPHA_SKIP", "T_STOP", "TILE", "NEAR_PLANE", "COV2D_DILATION",
    "OCam", "ocam", "orbit", "look_at", "sigmoid", "inv_sigmoid", "softplus",
    "inv_softplus", "normalize", "normalize_backward", "quat_rot", "project",
    "shade", "effective_o_logit", "channel_layout", "rasterize",
    "maps", "light_dir", "rasterize_backward", "project_backward", "shade_backward", "vq_assign",
    "vq_decode", "kmeans", "sh_basis", "sh_colors", "sh_colors_backward", "ssim", "photometric_loss", "inverse_step", "Adam",
    "pseudo_normal_from_depth", "normal_consistency_loss", "bilateral_smoothness", "stage2_step",
    "naive_composite",
    "lib", "max_threads",
]

# _kernels.py:14-16, rasterizer.py:24, gaussians.py:21-22
ALPHA_CAP = 0.99
ALPHA_SKIP = 1.0 / 255.0
T_STOP = 1e-4
TILE = 16
NEAR_PLANE = 0.01
COV2D_DILATION = 0.3


# --------------------------------------------------------------- C library
_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libivr_oracle.so")
_lib = None


def lib():
    """Load (building on first use) the oracle's C restatement."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.orc_composite_forward.argtypes = [P, I64, P, P, P, P, P, I64, I64, I64, I64,
                                            I64, ctypes.c_int, P, P, P, P, ctypes.c_int]
        L.orc_composite_backward.argtypes = [P, I64, P, P, P, P, P, I64, I64, I64, I64,
                                             I64, P, P, P, P, P, P, P, ctypes.c_int]
        L.orc_vq_assign.argtypes = [P, I64, P, I64, P, ctypes.c_int]
        L.orc_max_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def max_threads():
    return int(lib().orc_max_threads())


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------- helpers
def sigmoid(x):
    """_mathutil.py:6-13 (branch on sign for stability)."""
    x = np.asarray(x)
    out = np.empty_like(x, dtype=np.result_type(x, np.float32))
    nonneg = x >= 0
    out[nonneg] = 1.0 / (1.0 + np.exp(-x[nonneg]))
    e = np.exp(x[~nonneg])
    out[~nonneg] = e / (1.0 + e)
    return out


def inv_sigmoid(y):
    """_mathutil.py:16-18."""
    y = np.asarray(y)
    return np.log(y / (1.0 - y))


def softplus(x):
    """inverse.py:23-25."""
    return np.logaddexp(0.0, np.asarray(x, dtype=np.float64))


def inv_softplus(y):
    """inverse.py:28-32."""
    y = np.asarray(y, dtype=np.float64)
    return y + np.log1p(-np.exp(-y))


def normalize(v, eps=0.0):
    """_mathutil.py:31-36."""
    nrm = np.linalg.norm(v, axis=-1, keepdims=True)
    if eps:
        nrm = np.maximum(nrm, eps)
    return v / nrm


def normalize_backward(v, d_unit):
    """_mathutil.py:39-44."""
    nrm = np.linalg.norm(v, axis=-1, keepdims=True)
    u = v / nrm
    return (d_unit - np.sum(d_unit * u, axis=-1, keepdims=True) * u) / nrm


# --------------------------------------------------------------- camera
@dataclass
class OCam:
    """Pinhole camera, gaussians.py:139-164 (+z forward, +y down)."""

    position: np.ndarray
    rotation: np.ndarray
    fov_y: float
    width: int
    height: int

    @property
    def focal(self):
        return 0.5 * self.height / np.tan(0.5 * self.fov_y)

    @property
    def center_px(self):
        return ((self.width - 1) / 2.0, (self.height - 1) / 2.0)


def ocam(cam) -> OCam:
    """Adapt any camera-like object (reference or product) to OCam."""
    return OCam(np.asarray(cam.position, dtype=np.float64).reshape(3),
                np.asarray(cam.rotation, dtype=np.float64).reshape(3, 3),
                float(cam.fov_y), int(cam.width), int(cam.height))


def look_at(position, target, fov_y, width, height, up=(0.0, 0.0, 1.0)):
    """gaussians.py:166-181."""
    position = np.asarray(position, dtype=np.float64)
    fwd = normalize(np.asarray(target, dtype=np.float64) - position)
    right = np.cross(np.asarray(up, dtype=np.float64), fwd)
    nr = np.linalg.norm(right)
    if nr < 1e-8:
        right = np.cross(np.array([1.0, 0.0, 0.0]), fwd)
        nr = np.linalg.norm(right)
    right /= nr
    down = np.cross(fwd, right)
    return OCam(position, np.stack([right, down, fwd], axis=0), fov_y, width, height)


def orbit(center, radius, polar, azimuth, fov_y, width, height):
    """gaussians.py:203-215."""
    d = np.array([np.cos(polar) * np.cos(azimuth), np.cos(polar) * np.sin(azimuth),
                  np.sin(polar)])
    return look_at(np.asarray(center, dtype=np.float64) + radius * d, center, fov_y,
                   width, height)


# --------------------------------------------------------------- projection
def quat_rot(q):
    """gaussians.py:222-236 (w-first unit quaternion -> R)."""
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    R = np.empty((q.shape[0], 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - w * z)
    R[:, 0, 2] = 2 * (x * z + w * y)
    R[:, 1, 0] = 2 * (x * y + w * z)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - w * x)
    R[:, 2, 0] = 2 * (x * z - w * y)
    R[:, 2, 1] = 2 * (y * z + w * x)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def project(mu, q_raw, log_s, cam):
    """EWA projection, gaussians.py:296-346; returns the reference's cache."""
    cam = ocam(cam)
    q = normalize(q_raw)
    s = np.exp(log_s)
    W = cam.rotation
    t = (mu - cam.position[None, :]) @ W.T
    tz = t[:, 2]
    valid = tz > NEAR_PLANE
    tzs = np.where(valid, tz, 1.0)
    f = cam.focal
    cx, cy = cam.center_px
    mean2d = np.stack([f * t[:, 0] / tzs + cx, f * t[:, 1] / tzs + cy], axis=1)
    R = quat_rot(q)
    M3 = R * s[:, None, :]
    cov3d = M3 @ np.swapaxes(M3, 1, 2)
    n = mu.shape[0]
    J = np.zeros((n, 2, 3))
    J[:, 0, 0] = f / tzs
    J[:, 1, 1] = f / tzs
    J[:, 0, 2] = -f * t[:, 0] / tzs ** 2
    J[:, 1, 2] = -f * t[:, 1] / tzs ** 2
    M = J @ W[None, :, :]
    cov2d = M @ cov3d @ np.swapaxes(M, 1, 2)
    cov2d[:, 0, 0] += COV2D_DILATION
    cov2d[:, 1, 1] += COV2D_DILATION
    a, b, c = cov2d[:, 0, 0], cov2d[:, 0, 1], cov2d[:, 1, 1]
    det = a * c - b * b
    dets = np.where(det > 0, det, 1.0)
    conic = np.stack([c / dets, -b / dets, a / dets], axis=1)
    valid = valid & (det > 0)
    return {"t": t, "tz": tzs, "valid": valid, "mean2d": mean2d, "cov2d": cov2d,
            "conic": conic, "depth": tz, "q": q, "s": s, "R": R, "cov3d": cov3d,
            "J": J, "M": M, "q_raw": q_raw, "cam": cam}


def project_backward(proj, d_mean2d, d_cov2d, d_depth):
    """gaussians.py:349-400 (with covariance_backward :278-289 and
    quat_to_rot_backward :239-264)."""
    cam = proj["cam"]
    t, tz, J, M, cov3d = proj["t"], proj["tz"], proj["J"], proj["M"], proj["cov3d"]
    q, s = proj["q"], proj["s"]
    W = cam.rotation
    f = cam.focal
    n = t.shape[0]
    bad = ~proj["valid"]
    d_mean2d = np.where(bad[:, None], 0.0, d_mean2d)
    d_cov2d = np.where(bad[:, None, None], 0.0, d_cov2d)
    d_depth = np.where(bad, 0.0, d_depth)
    d_cov3d = np.swapaxes(M, 1, 2) @ d_cov2d @ M
    dM = d_cov2d @ M @ np.swapaxes(cov3d, 1, 2) + np.swapaxes(d_cov2d, 1, 2) @ M @ cov3d
    dJ = dM @ W.T[None, :, :]
    dt = np.zeros((n, 3))
    dt[:, 0] += dJ[:, 0, 2] * (-f / tz ** 2)
    dt[:, 1] += dJ[:, 1, 2] * (-f / tz ** 2)
    dt[:, 2] += (dJ[:, 0, 0] * (-f / tz ** 2) + dJ[:, 1, 1] * (-f / tz ** 2)
                 + dJ[:, 0, 2] * (2 * f * t[:, 0] / tz ** 3)
                 + dJ[:, 1, 2] * (2 * f * t[:, 1] / tz ** 3))
    dt[:, 0] += d_mean2d[:, 0] * f / tz
    dt[:, 1] += d_mean2d[:, 1] * f / tz
    dt[:, 2] += -d_mean2d[:, 0] * f * t[:, 0] / tz ** 2 - d_mean2d[:, 1] * f * t[:, 1] / tz ** 2
    dt[:, 2] += d_depth
    d_mu = dt @ W
    # covariance_backward
    R = quat_rot(q)
    M3 = R * s[:, None, :]
    dM3 = (d_cov3d + np.swapaxes(d_cov3d, 1, 2)) @ M3
    ds = np.einsum("nik,nik->nk", dM3, R)
    g = dM3 * s[:, None, :]
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    dw = 2 * (-z * g[:, 0, 1] + y * g[:, 0, 2] + z * g[:, 1, 0] - x * g[:, 1, 2]
              - y * g[:, 2, 0] + x * g[:, 2, 1])
    dx = 2 * (y * g[:, 0, 1] + z * g[:, 0, 2] + y * g[:, 1, 0] - 2 * x * g[:, 1, 1]
              - w * g[:, 1, 2] + z * g[:, 2, 0] + w * g[:, 2, 1] - 2 * x * g[:, 2, 2])
    dy = 2 * (-2 * y * g[:, 0, 0] + x * g[:, 0, 1] + w * g[:, 0, 2] + x * g[:, 1, 0]
              + z * g[:, 1, 2] - w * g[:, 2, 0] + z * g[:, 2, 1] - 2 * y * g[:, 2, 2])
    dz = 2 * (-2 * z * g[:, 0, 0] - w * g[:, 0, 1] + x * g[:, 0, 2] + w * g[:, 1, 0]
              - 2 * z * g[:, 1, 1] + y * g[:, 1, 2] + x * g[:, 2, 0] + y * g[:, 2, 1])
    dq = np.stack([dw, dx, dy, dz], axis=1)
    return {"d_mu": d_mu, "d_q_raw": normalize_backward(proj["q_raw"], dq),
            "d_log_s": ds * s}


# --------------------------------------------------------------- shading
def light_dir(polar, azimuth):
    """shading.py:179-183."""
    cp, sp = np.cos(polar), np.sin(polar)
    ca, sa = np.cos(azimuth), np.sin(azimuth)
    return np.array([cp * ca, cp * sa, sp])


def shade(mu, n_raw, delta_c, k_a_raw, k_d_raw, k_s_raw, log_beta, palette, light,
          cam, coeff_transform=None):
    """Blinn-Phong editable shading, shading.py:225-329.

    ``light`` is (mode, polar, azimuth, term_scales); ``palette`` is (3,) or
    per-splat (N, 3).  Returns (rgb, cache)."""
    mode, polar, azimuth, ts = light
    ts = np.asarray(ts, dtype=np.float64).reshape(4)
    cam = ocam(cam)
    nrm = normalize(n_raw, eps=1e-12)
    w_cam = np.asarray(cam.position) - mu
    v = normalize(w_cam, eps=1e-12)
    head = mode == "headlight"
    if head:
        l = h = v
        u = None
    else:
        l = np.broadcast_to(light_dir(polar, azimuth), mu.shape)
        u = v + l
        h = normalize(u, eps=1e-12)
    sa, sd, ss = sigmoid(k_a_raw), sigmoid(k_d_raw), sigmoid(k_s_raw)
    beta1 = np.exp(log_beta) + 1.0
    if coeff_transform is None:
        lam, b = np.ones(4), np.zeros(4)
    else:
        lam = np.asarray(coeff_transform[0], dtype=np.float64).reshape(4)
        b = np.asarray(coeff_transform[1], dtype=np.float64).reshape(4)
    ta, td, tsp = lam[0] * sa + b[0], lam[1] * sd + b[1], lam[2] * ss + b[2]
    tb = lam[3] * beta1 + b[3]
    gates = ((ta > 0.0) & (ta < 1.0), (td > 0.0) & (td < 1.0), (tsp > 0.0) & (tsp < 1.0),
             tb > 1.0)
    k_a = ts[0] * np.clip(ta, 0.0, 1.0)
    k_d = ts[1] * np.clip(td, 0.0, 1.0)
    k_s = ts[2] * np.clip(tsp, 0.0, 1.0)
    beta = ts[3] * np.maximum(tb, 1.0)
    c_p = np.asarray(palette, dtype=np.float64)
    per_splat = c_p.ndim == 2
    c_pre = (c_p if per_splat else c_p[None, :]) + delta_c
    c_v = np.clip(c_pre, 0.0, 1.0)
    ndl = np.sum(nrm * l, axis=-1)
    ndh = np.sum(nrm * h, axis=-1)
    a_ndl, a_ndh = np.abs(ndl), np.abs(ndh)
    gate = a_ndl > 0.0
    spow = np.where(a_ndh > 0.0, np.power(np.maximum(a_ndh, 1e-300), beta), 0.0)
    spow = np.where(gate, spow, 0.0)
    amb = k_a[:, None] * c_v
    dif = (k_d * a_ndl)[:, None] * c_v
    spec = (k_s * spow)[:, None] * np.ones(3)
    rgb = amb + dif + spec
    cache = dict(head=head, n=nrm, l=l, v=v, h=h, u=u, w_cam=w_cam, sig=(sa, sd, ss),
                 beta1=beta1, lam=lam, b=b, ts=ts, gates=gates, k=(k_a, k_d, k_s, beta),
                 c_v=c_v, per_splat=per_splat, open=(c_pre > 0.0) & (c_pre < 1.0),
                 ndl=ndl, ndh=ndh, a_ndl=a_ndl, a_ndh=a_ndh, gate=gate, spow=spow,
                 polar=polar, azimuth=azimuth, n_raw=n_raw,
                 terms={"ambient": amb, "diffuse": dif, "specular": spec})
    return rgb, cache


def shade_backward(cache, d_rgb):
    """shading.py:332-445."""
    d_rgb = np.asarray(d_rgb, dtype=np.float64)
    n, l, h = cache["n"], cache["l"], cache["h"]
    sa, sd, ss = cache["sig"]
    beta1, lam, ts = cache["beta1"], cache["lam"], cache["ts"]
    k_a, k_d, k_s, beta = cache["k"]
    c_v, a_ndl, a_ndh = cache["c_v"], cache["a_ndl"], cache["a_ndh"]
    gate, spow = cache["gate"], cache["spow"]
    s3 = d_rgb.sum(axis=-1)
    dot_cv = np.sum(d_rgb * c_v, axis=-1)
    d_c_v = (k_a + k_d * a_ndl)[:, None] * d_rgb
    d_k_a, d_k_d, d_k_s = dot_cv, a_ndl * dot_cv, spow * s3
    d_spow = k_s * s3
    safe = a_ndh > 0.0
    log_andh = np.log(np.where(safe, a_ndh, 1.0))
    d_a_ndh = np.where(gate & safe, d_spow * beta * np.exp((beta - 1.0) * log_andh), 0.0)
    d_beta = np.where(gate & safe, d_spow * spow * log_andh, 0.0)
    d_a_ndl = k_d * dot_cv
    d_ndl = np.sign(cache["ndl"]) * d_a_ndl
    d_ndh = np.sign(cache["ndh"]) * d_a_ndh
    d_n_unit = d_ndl[:, None] * l + d_ndh[:, None] * h
    d_l = d_ndl[:, None] * n
    d_h = d_ndh[:, None] * n
    if cache["head"]:
        d_v = d_h + d_l
    else:
        d_u = normalize_backward(cache["u"], d_h)
        d_v = d_u
        d_l = d_l + d_u
    d_mu = -normalize_backward(cache["w_cam"], d_v)
    if cache["head"]:
        d_polar = d_azimuth = 0.0
    else:
        p, a = cache["polar"], cache["azimuth"]
        dl_dp = np.array([-np.sin(p) * np.cos(a), -np.sin(p) * np.sin(a), np.cos(p)])
        dl_da = np.array([-np.cos(p) * np.sin(a), np.cos(p) * np.cos(a), 0.0])
        d_polar = float(np.sum(d_l * dl_dp))
        d_azimuth = float(np.sum(d_l * dl_da))
    ga, gd, gs, gb = cache["gates"]
    ea, ed, es, eb = d_k_a * ts[0] * ga, d_k_d * ts[1] * gd, d_k_s * ts[2] * gs, d_beta * ts[3] * gb
    d_lam = np.array([np.sum(ea * sa), np.sum(ed * sd), np.sum(es * ss), np.sum(eb * beta1)])
    d_b = np.array([np.sum(ea), np.sum(ed), np.sum(es), np.sum(eb)])
    d_open = np.where(cache["open"], d_c_v, 0.0)
    return {
        "d_delta_c": d_open,
        "d_k_a_raw": ea * lam[0] * sa * (1.0 - sa),
        "d_k_d_raw": ed * lam[1] * sd * (1.0 - sd),
        "d_k_s_raw": es * lam[2] * ss * (1.0 - ss),
        "d_log_beta": eb * lam[3] * (beta1 - 1.0),
        "d_n_raw": normalize_backward(cache["n_raw"], d_n_unit),
        "d_c_p": d_open if cache["per_splat"] else d_open.sum(axis=0),
        "d_mu": d_mu, "d_lam": d_lam, "d_b": d_b,
        "d_polar": d_polar, "d_azimuth": d_azimuth,
    }


def effective_o_logit(o_logit, scales):
    """Opacity edit, scene.py:214-220: logit(clip(scale*sigmoid(o))) applied to
    every splat as soon as ANY per-splat scale differs from 1."""
    if np.all(scales == 1.0):
        return o_logit
    return inv_sigmoid(np.clip(scales * sigmoid(o_logit), 1e-12, 1.0 - 1e-9))


# --------------------------------------------------------------- rasterizer
def channel_layout(channels, attrs):
    """rasterizer.py:39-50."""
    widths = {"color": 3, "alpha": 1, "depth": 1, "normal": 3}
    out = [(c, widths[c]) for c in ("color", "alpha", "depth", "normal") if c in channels]
    for name, vals in (attrs or {}).items():
        vals = np.asarray(vals)
        out.append((name, 1 if vals.ndim == 1 else vals.shape[1]))
    return out


def rasterize(mu, q_raw, log_s, o_logit, n_raw, colors, cam, channels=("color", "alpha"),
              attrs=None, dtype=np.float32, nthreads=0):
    """rasterize_forward, rasterizer.py:53-164 (binning :88-132, packing
    :134-153, compositor _kernels.py:19-72).  Returns a state dict holding the
    maps and every intermediate the parity tests compare."""
    cam = ocam(cam)
    H, W = cam.height, cam.width
    lay = channel_layout(channels, attrs)
    K = sum(w for _, w in lay)
    n = mu.shape[0]
    st = {"layout": lay, "dtype": dtype, "n": n, "cam": cam, "attrs": attrs or {}, "n_raw": n_raw,
          "colors": colors, "empty": True}
    out = np.zeros((H, W, K))
    st.update(out=out, contrib=np.zeros((H, W), np.int32),
              last_pos=np.zeros((H, W), np.int64), t_final=np.ones((H, W)))
    if n == 0:
        return st
    proj = project(mu, q_raw, log_s, cam)
    opacity = sigmoid(o_logit)
    mean2d, conic, depth, cov = proj["mean2d"], proj["conic"], proj["depth"], proj["cov2d"]
    half_tr = 0.5 * (cov[:, 0, 0] + cov[:, 1, 1])
    lam_max = half_tr + np.sqrt(np.maximum(
        0.25 * (cov[:, 0, 0] - cov[:, 1, 1]) ** 2 + cov[:, 0, 1] ** 2, 0.0))
    with np.errstate(invalid="ignore", divide="ignore"):
        cut = np.sqrt(2.0 * np.log(np.maximum(opacity / ALPHA_SKIP, 1.0)))
    radius = np.ceil(np.sqrt(np.maximum(lam_max, 0.0)) * cut) + 1
    visible = proj["valid"] & (opacity >= ALPHA_SKIP) & (radius > 0)
    ntx, nty = (W + TILE - 1) // TILE, (H + TILE - 1) // TILE
    tx0 = np.clip(np.floor((mean2d[:, 0] - radius) / TILE), 0, ntx - 1).astype(np.int64)
    tx1 = np.clip(np.floor((mean2d[:, 0] + radius) / TILE), 0, ntx - 1).astype(np.int64)
    ty0 = np.clip(np.floor((mean2d[:, 1] - radius) / TILE), 0, nty - 1).astype(np.int64)
    ty1 = np.clip(np.floor((mean2d[:, 1] + radius) / TILE), 0, nty - 1).astype(np.int64)
    visible &= ((mean2d[:, 0] + radius >= 0) & (mean2d[:, 0] - radius < W)
                & (mean2d[:, 1] + radius >= 0) & (mean2d[:, 1] - radius < H))
    st.update(proj=proj, opacity=opacity, radius=radius, visible=visible, ntx=ntx, nty=nty,
              rect=np.stack([tx0, tx1, ty0, ty1], axis=1))
    if not visible.any():
        return st
    counts = np.where(visible, (tx1 - tx0 + 1) * (ty1 - ty0 + 1), 0)
    # fill_pairs (_kernels.py:19-28): splat-major, then ty, then tx
    splat = np.repeat(np.arange(n, dtype=np.int64), counts)
    offsets = np.zeros(n, np.int64)
    np.cumsum(counts[:-1], out=offsets[1:])
    k = np.arange(splat.size, dtype=np.int64) - offsets[splat]
    wdt = (tx1 - tx0 + 1)[splat]
    tile = (ty0[splat] + k // wdt) * ntx + (tx0[splat] + k % wdt)
    order = np.lexsort((depth[splat], tile))  # rasterizer.py:129
    tile, splat = tile[order], splat[order]
    ranges = np.searchsorted(tile, np.arange(ntx * nty + 1)).astype(np.int64)
    vals = np.zeros((n, K), dtype=dtype)
    col = 0
    for name, w in lay:
        if name == "color":
            vals[:, col:col + 3] = np.asarray(colors, dtype=dtype)
        elif name == "alpha":
            vals[:, col] = 1.0
        elif name == "depth":
            vals[:, col] = depth.astype(dtype)
        elif name == "normal":
            vals[:, col:col + 3] = normalize(n_raw, eps=1e-12).astype(dtype)
        else:
            vals[:, col:col + w] = np.asarray(attrs[name], dtype=dtype).reshape(n, w)
        col += w
    km, kc, ko = mean2d.astype(dtype), conic.astype(dtype), opacity.astype(dtype)
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    st.update(pair_splat=splat, pair_tile=tile, tile_ranges=ranges, values=vals,
              kmean2d=km, kconic=kc, kopacity=ko, counts=counts, empty=False,
              _k=(f64(km), f64(kc), f64(ko), f64(vals)))
    lp = st["last_pos"]
    lib().orc_composite_forward(
        _p(ranges), ntx * nty, _p(splat), _p(st["_k"][0]), _p(st["_k"][1]), _p(st["_k"][2]),
        _p(st["_k"][3]), K, W, H, TILE, ntx, int(np.dtype(dtype) == np.float32), _p(out),
        _p(st["contrib"]), _p(lp), _p(st["t_final"]), int(nthreads))
    return st


def naive_composite(mean2d, conic, opacity, depth, values, width, height):
    """The reference's independent test compositor (pkg/tests/oracles.py:16-43):
    ALL splats sorted globally by depth (stable), every pixel composited
    vectorised with the same cap / skip / stop constants; no tiles, no lists.
    Returns (out (H,W,K), contributor count (H,W))."""
    n, k = values.shape
    ys, xs = np.mgrid[0:height, 0:width]
    xs, ys = xs.astype(np.float64), ys.astype(np.float64)
    out = np.zeros((height, width, k))
    T = np.ones((height, width))
    alive = np.ones((height, width), bool)
    count = np.zeros((height, width), np.int64)
    for i in np.argsort(depth, kind="stable"):
        dx, dy = xs - mean2d[i, 0], ys - mean2d[i, 1]
        a, b, c = conic[i]
        sig = 0.5 * (a * dx * dx + c * dy * dy) + b * dx * dy
        al = np.minimum(np.where(sig >= 0, opacity[i] * np.exp(-sig), 0.0), ALPHA_CAP)
        m = alive & (al >= ALPHA_SKIP)
        w = np.where(m, T * al, 0.0)
        out += w[:, :, None] * values[i][None, None, :]
        T = np.where(m, T * (1.0 - al), T)
        count += m
        alive &= T >= T_STOP
    return out, count


def maps(st):
    """Unpack the packed output like rasterizer.py:167-182 (in ``dtype``)."""
    out = st["out"].astype(st["dtype"])
    res, col = {}, 0
    for name, w in st["layout"]:
        m = out[:, :, col:col + w]
        res[name] = m[:, :, 0] if w == 1 else m
        col += w
    return res


def rasterize_backward(st, d_maps, nthreads=0):
    """rasterize_backward, rasterizer.py:185-286."""
    n, cam = st["n"], st["cam"]
    H, W = cam.height, cam.width
    g = {"d_mean2d": np.zeros((n, 2)), "d_mu": np.zeros((n, 3)), "d_q_raw": np.zeros((n, 4)),
         "d_log_s": np.zeros((n, 3)), "d_o_logit": np.zeros(n), "d_n_raw": np.zeros((n, 3)),
         "d_colors": np.zeros((n, 3)),
         "d_attrs": {k: np.zeros(np.asarray(v).shape) for k, v in st["attrs"].items()}}
    if st["empty"]:
        return g
    K = st["values"].shape[1]
    d_out = np.zeros((H, W, K))
    col = 0
    for name, w in st["layout"]:
        if d_maps.get(name) is not None:
            d_out[:, :, col:col + w] = np.asarray(d_maps[name], np.float64).reshape(H, W, w)
        col += w
    P = st["pair_splat"].size
    pdv, pdm, pdc, pdo = np.zeros((P, K)), np.zeros((P, 2)), np.zeros((P, 3)), np.zeros(P)
    km, kc, ko, kv = st["_k"]
    lib().orc_composite_backward(
        _p(st["tile_ranges"]), st["ntx"] * st["nty"], _p(st["pair_splat"]), _p(km), _p(kc),
        _p(ko), _p(kv), K, W, H, TILE, st["ntx"], _p(d_out), _p(st["last_pos"]),
        _p(st["t_final"]), _p(pdv), _p(pdm), _p(pdc), _p(pdo), int(nthreads))
    ps = st["pair_splat"]
    d_values, d_mean2d, d_conic, d_op = np.zeros((n, K)), np.zeros((n, 2)), np.zeros((n, 3)), np.zeros(n)
    np.add.at(d_values, ps, pdv)
    np.add.at(d_mean2d, ps, pdm)
    np.add.at(d_conic, ps, pdc)
    np.add.at(d_op, ps, pdo)
    conic = st["proj"]["conic"]
    Q = np.empty((n, 2, 2))
    Q[:, 0, 0], Q[:, 0, 1], Q[:, 1, 0], Q[:, 1, 1] = conic[:, 0], conic[:, 1], conic[:, 1], conic[:, 2]
    dQ = np.empty((n, 2, 2))
    dQ[:, 0, 0] = d_conic[:, 0]
    dQ[:, 0, 1] = dQ[:, 1, 0] = 0.5 * d_conic[:, 1]
    dQ[:, 1, 1] = d_conic[:, 2]
    d_cov2d = -Q @ dQ @ Q
    d_depth = np.zeros(n)
    col = 0
    for name, w in st["layout"]:
        sl = d_values[:, col:col + w]
        if name == "color":
            g["d_colors"] = sl.copy()
        elif name == "depth":
            d_depth = sl[:, 0].copy()
        elif name == "normal":
            g["d_n_raw"] += normalize_backward(st["n_raw"], sl)
        elif name != "alpha":
            g["d_attrs"][name] = sl.reshape(np.asarray(st["attrs"][name]).shape).copy()
        col += w
    g["d_mean2d"] = d_mean2d
    g["d_values"] = d_values
    g["d_conic"] = d_conic
    g["d_opacity"] = d_op
    pg = project_backward(st["proj"], d_mean2d, d_cov2d, d_depth)
    g["d_mu"] += pg["d_mu"]
    g["d_q_raw"] += pg["d_q_raw"]
    g["d_log_s"] += pg["d_log_s"]
    o = st["opacity"]
    g["d_o_logit"] += d_op * o * (1.0 - o)
    return g


# --------------------------------------------------------------- SH colour
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
         -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
         -0.5900435899266435)


def sh_basis(d, degree):
    """Real SH basis (N,B) and d basis / d dir (N,B,3), gaussians.py:427-494."""
    x, y, z = d[:, 0], d[:, 1], d[:, 2]
    n, nb = d.shape[0], (degree + 1) ** 2
    B, D = np.zeros((n, nb)), np.zeros((n, nb, 3))
    B[:, 0] = SH_C0
    if degree >= 1:
        B[:, 1], B[:, 2], B[:, 3] = -SH_C1 * y, SH_C1 * z, -SH_C1 * x
        D[:, 1, 1], D[:, 2, 2], D[:, 3, 0] = -SH_C1, SH_C1, -SH_C1
    if degree >= 2:
        xx, yy, zz = x * x, y * y, z * z
        c = SH_C2
        B[:, 4], B[:, 5] = c[0] * x * y, c[1] * y * z
        B[:, 6], B[:, 7], B[:, 8] = c[2] * (2 * zz - xx - yy), c[3] * x * z, c[4] * (xx - yy)
        D[:, 4, 0], D[:, 4, 1], D[:, 5, 1], D[:, 5, 2] = c[0] * y, c[0] * x, c[1] * z, c[1] * y
        D[:, 6, 0], D[:, 6, 1], D[:, 6, 2] = c[2] * (-2 * x), c[2] * (-2 * y), c[2] * (4 * z)
        D[:, 7, 0], D[:, 7, 2] = c[3] * z, c[3] * x
        D[:, 8, 0], D[:, 8, 1] = c[4] * (2 * x), c[4] * (-2 * y)
    if degree >= 3:
        xx, yy, zz = x * x, y * y, z * z
        c = SH_C3
        B[:, 9] = c[0] * y * (3 * xx - yy)
        B[:, 10] = c[1] * x * y * z
        B[:, 11] = c[2] * y * (4 * zz - xx - yy)
        B[:, 12] = c[3] * z * (2 * zz - 3 * xx - 3 * yy)
        B[:, 13] = c[4] * x * (4 * zz - xx - yy)
        B[:, 14] = c[5] * z * (xx - yy)
        B[:, 15] = c[6] * x * (xx - 3 * yy)
        D[:, 9, 0], D[:, 9, 1] = c[0] * 6 * x * y, c[0] * (3 * xx - 3 * yy)
        D[:, 10, 0], D[:, 10, 1], D[:, 10, 2] = c[1] * y * z, c[1] * x * z, c[1] * x * y
        D[:, 11, 0] = c[2] * (-2 * x * y)
        D[:, 11, 1] = c[2] * (4 * zz - xx - 3 * yy)
        D[:, 11, 2] = c[2] * (8 * y * z)
        D[:, 12, 0], D[:, 12, 1] = c[3] * (-6 * x * z), c[3] * (-6 * y * z)
        D[:, 12, 2] = c[3] * (6 * zz - 3 * xx - 3 * yy)
        D[:, 13, 0] = c[4] * (4 * zz - 3 * xx - yy)
        D[:, 13, 1], D[:, 13, 2] = c[4] * (-2 * x * y), c[4] * (8 * x * z)
        D[:, 14, 0], D[:, 14, 1], D[:, 14, 2] = c[5] * (2 * x * z), c[5] * (-2 * y * z), c[5] * (xx - yy)
        D[:, 15, 0], D[:, 15, 1] = c[6] * (3 * xx - 3 * yy), c[6] * (-6 * x * y)
    return B, D


def sh_colors(mu, coeffs, degree, cam_pos):
    """view_dirs + eval_sh (gaussians.py:497-508, 521-524): (rgb, cache)."""
    v = mu - np.asarray(cam_pos)[None, :]
    d = normalize(v, eps=1e-12)
    B, D = sh_basis(d, degree)
    raw = np.einsum("nb,nbc->nc", B, coeffs) + 0.5
    return np.maximum(raw, 0.0), {"B": B, "D": D, "raw": raw, "coeffs": coeffs, "v": v}


def sh_colors_backward(cache, d_rgb):
    """eval_sh_backward + view_dirs_backward (gaussians.py:511-518, 527-529):
    (d_coeffs, d_mu)."""
    g = d_rgb * (cache["raw"] > 0)
    d_coeffs = cache["B"][:, :, None] * g[:, None, :]
    inner = np.einsum("nbc,nc->nb", cache["coeffs"], g)
    d_dir = np.einsum("nb,nbk->nk", inner, cache["D"])
    return d_coeffs, normalize_backward(cache["v"], d_dir)


# --------------------------------------------------------------- VQ
def vq_assign(values, centroids, nthreads=0):
    """assign_nearest, vq.py:90-96 (searchsorted over float64 mids)."""
    v = np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    c = np.ascontiguousarray(centroids, dtype=np.float64).reshape(-1)
    out = np.empty(v.size, np.int64)
    lib().orc_vq_assign(_p(v), v.size, _p(c), c.size, _p(out), int(nthreads))
    return out.reshape(np.shape(values))


def vq_decode(indices, centroids):
    """Codebook.decode, vq.py:128-134 (raises on out-of-range index)."""
    idx = np.asarray(indices)
    if idx.size and int(idx.max()) >= centroids.size:
        raise IndexError(f"index {int(idx.max())} >= K={centroids.size}")
    return np.asarray(centroids, np.float64)[idx.astype(np.int64)]


def kmeans(samples, k, seed=0, restarts=5, max_iters=50, tol=1e-6):
    """Scalar k-means, vq.py:31-87 (k-means++ seeding + Lloyd, best SSE)."""
    x = np.asarray(samples, dtype=np.float64).reshape(-1)
    distinct = np.unique(x)
    if distinct.size <= k:
        return distinct
    rng = np.random.default_rng(seed)
    best, best_sse = None, np.inf
    for _ in range(restarts):
        c = np.empty(k)
        c[0] = x[rng.integers(x.size)]
        d2 = (x - c[0]) ** 2
        for i in range(1, k):
            tot = d2.sum()
            if tot <= 0.0:
                c[i:] = c[0]
                break
            c[i] = x[rng.choice(x.size, p=d2 / tot)]
            d2 = np.minimum(d2, (x - c[i]) ** 2)
        scale = max(float(np.abs(x).max()), 1e-12)
        for _it in range(max_iters):
            c = np.sort(c)
            idx = np.searchsorted(0.5 * (c[1:] + c[:-1]), x) if c.size > 1 else np.zeros(x.size, np.int64)
            sums = np.bincount(idx, weights=x, minlength=c.size)
            cnt = np.bincount(idx, minlength=c.size)
            new = np.where(cnt > 0, sums / np.maximum(cnt, 1), c)
            shift = np.abs(new - c).max() / scale
            c = new
            if shift < tol:
                break
        c = np.sort(c)
        idx = np.searchsorted(0.5 * (c[1:] + c[:-1]), x)
        sse = float(np.sum((x - c[idx]) ** 2))
        if sse < best_sse:
            best, best_sse = c, sse
    return np.unique(best)


# --------------------------------------------------------------- losses
_SSIM_R = 5
_o = np.arange(-_SSIM_R, _SSIM_R + 1, dtype=np.float64)
_K1D = np.exp(-(_o ** 2) / (2.0 * 1.5 ** 2))
_K1D /= _K1D.sum()


def _filt(img, mode):
    from scipy.signal import convolve
    return convolve(convolve(img, _K1D[:, None], mode=mode), _K1D[None, :], mode=mode)


def ssim(x, y):
    """losses.py:45-115 (valid-window Gaussian SSIM + analytic gradient)."""
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    sq = x.ndim == 2
    if sq:
        x, y = x[..., None], y[..., None]
    h, w, nc = x.shape
    C1, C2 = 0.01 ** 2, 0.03 ** 2
    nv = (h - 2 * _SSIM_R) * (w - 2 * _SSIM_R)
    total, dx = 0.0, np.zeros_like(x)
    for c in range(nc):
        xc, yc = x[..., c], y[..., c]
        ux, uy = _filt(xc, "valid"), _filt(yc, "valid")
        uxx, uyy, uxy = _filt(xc * xc, "valid"), _filt(yc * yc, "valid"), _filt(xc * yc, "valid")
        vx, vy, vxy = uxx - ux * ux, uyy - uy * uy, uxy - ux * uy
        a1, a2 = 2.0 * ux * uy + C1, 2.0 * vxy + C2
        b1, b2 = ux * ux + uy * uy + C1, vx + vy + C2
        s = (a1 * a2) / (b1 * b2)
        total += s.mean()
        up = 1.0 / (nv * nc)
        da1, da2 = a2 / (b1 * b2) * up, a1 / (b1 * b2) * up
        db1, db2 = -s / b1 * up, -s / b2 * up
        d_uxy = 2.0 * da2
        d_uxx = db2
        d_ux = 2.0 * uy * da1 + 2.0 * ux * db1 - 2.0 * ux * db2 - uy * d_uxy
        dx[..., c] = _filt(d_ux, "full") + 2.0 * xc * _filt(d_uxx, "full") + yc * _filt(d_uxy, "full")
    return total / nc, (dx[..., 0] if sq else dx)


def photometric_loss(pred, gt, l1_w=0.8, ssim_w=0.2):
    """losses.py:118-138."""
    pred, gt = np.asarray(pred, np.float64), np.asarray(gt, np.float64)
    diff = pred - gt
    loss = l1_w * np.mean(np.abs(diff))
    d = l1_w * np.sign(diff) / diff.size
    if ssim_w > 0.0:
        s, ds = ssim(pred, gt)
        loss += ssim_w * (1.0 - s)
        d = d - ssim_w * ds
    return loss, d


def pseudo_normal_from_depth(depth, alpha, cam, alpha_threshold=1e-3):
    """losses.py:141-186: camera-space points from the depth map, forward
    differences (backward on the last row/column), cross product, oriented to
    the camera, rotated to world; mask = alpha > threshold and |n| > 1e-12."""
    cam = ocam(cam)
    depth, alpha = np.asarray(depth, np.float64), np.asarray(alpha, np.float64)
    h, w = depth.shape
    px, py = np.meshgrid(np.arange(w, dtype=np.float64), np.arange(h, dtype=np.float64))
    cx, cy = cam.center_px
    f = cam.focal
    pts = np.stack([(px - cx) * depth / f, (py - cy) * depth / f, depth], axis=-1)
    dx = np.empty_like(pts)
    dx[:, :-1] = pts[:, 1:] - pts[:, :-1]
    dx[:, -1] = pts[:, -1] - pts[:, -2]
    dy = np.empty_like(pts)
    dy[:-1] = pts[1:] - pts[:-1]
    dy[-1] = pts[-1] - pts[-2]
    nrm = np.cross(dx, dy)
    ln = np.linalg.norm(nrm, axis=-1, keepdims=True)
    good = ln[..., 0] > 1e-12
    nrm = np.where(good[..., None], nrm / np.maximum(ln, 1e-12), 0.0)
    away = np.sum(nrm * pts, axis=-1) > 0.0
    nrm[away] = -nrm[away]
    n_world = nrm @ cam.rotation
    mask = (alpha > alpha_threshold) & good
    n_world[~mask] = 0.0
    return n_world, mask


def normal_consistency_loss(normal_map, target, mask):
    """losses.py:189-206: mean L2 distance over the mask; gradient to the map."""
    n, t = np.asarray(normal_map, np.float64), np.asarray(target, np.float64)
    count = int(mask.sum())
    d_n = np.zeros_like(n)
    if count == 0:
        return 0.0, d_n
    diff = (n - t)[mask]
    ln = np.linalg.norm(diff, axis=-1)
    safe = ln > 1e-12
    g = np.zeros_like(diff)
    g[safe] = diff[safe] / ln[safe, None] / count
    d_n[mask] = g
    return ln.sum() / count, d_n


def bilateral_smoothness(attr_map, gt_color):
    """losses.py:219-253 (no mask): mean |grad K| exp(-|grad c_gt|), forward
    differences, L1 over components and directions."""
    k, c = np.asarray(attr_map, np.float64), np.asarray(gt_color, np.float64)
    c3 = c if c.ndim == 3 else c[..., None]
    gxc = np.zeros(c3.shape[:2])
    gyc = np.zeros(c3.shape[:2])
    gxc[:, :-1] = np.sum(np.abs(c3[:, 1:] - c3[:, :-1]), axis=-1)
    gyc[:-1] = np.sum(np.abs(c3[1:] - c3[:-1]), axis=-1)
    count = k.shape[0] * k.shape[1]
    weight = np.exp(-(gxc + gyc)) * np.ones(k.shape[:2], bool) / count
    d_k = np.zeros_like(k)
    k3 = k if k.ndim == 3 else k[..., None]
    d3 = d_k if d_k.ndim == 3 else d_k[..., None]
    gx = k3[:, 1:] - k3[:, :-1]
    gy = k3[1:] - k3[:-1]
    loss = float(np.sum(np.abs(gx).sum(-1) * weight[:, :-1]) + np.sum(np.abs(gy).sum(-1) * weight[:-1]))
    sx = np.sign(gx) * weight[:, :-1, None]
    sy = np.sign(gy) * weight[:-1, :, None]
    d3[:, 1:] += sx
    d3[:, :-1] -= sx
    d3[1:] += sy
    d3[:-1] -= sy
    return loss, d_k


def stage2_step(params, palette, light, cam, gt, nthreads=0, w_nc=0.01, w_off=0.01, w_bil=0.01,
                w_op=0.1, aux=None):
    """trainer._stage2_step, trainer.py:397-444 with LossWeights defaults
    (losses.py:28-37): K=15 render (colour, alpha, depth, normal, delta_c,
    k_a, k_d, k_s, beta), photometric + normal consistency + offset sparsity +
    bilateral smoothness x4 + opacity L1, full backward.
    Returns (loss, grads, stat)."""
    p = params
    rgb, cache = shade(p["mu"], p["n_raw"], p["delta_c"], p["k_a_raw"], p["k_d_raw"],
                       p["k_s_raw"], p["log_beta"], palette, light, cam)
    k_a, k_d, k_s = sigmoid(p["k_a_raw"]), sigmoid(p["k_d_raw"]), sigmoid(p["k_s_raw"])
    beta = np.exp(p["log_beta"]) + 1.0
    attrs = {"delta_c": p["delta_c"], "k_a": k_a, "k_d": k_d, "k_s": k_s, "beta": beta}
    st = rasterize(p["mu"], p["q_raw"], p["log_s"], p["o_logit"], p["n_raw"], rgb, cam,
                   channels=("color", "alpha", "depth", "normal"), attrs=attrs,
                   dtype=np.float32, nthreads=nthreads)
    mp = maps(st)
    rgba = np.concatenate([mp["color"].astype(np.float64),
                           mp["alpha"].astype(np.float64)[..., None]], axis=-1)
    loss, d_rgba = photometric_loss(rgba, gt)
    d_maps = {"color": d_rgba[..., :3], "alpha": d_rgba[..., 3]}
    tgt, mask = pseudo_normal_from_depth(mp["depth"], mp["alpha"], cam)
    nl, d_n = normal_consistency_loss(mp["normal"], tgt, mask)
    d_maps["normal"] = w_nc * d_n
    loss += w_nc * nl
    off = np.asarray(mp["delta_c"], np.float64)
    loss += w_off * float(np.mean(np.abs(off)))
    d_maps["delta_c"] = w_off * (np.sign(off) / off.size)
    gt_rgb = np.asarray(gt)[..., :3]
    for name in ("k_a", "k_d", "k_s", "beta"):
        bl, dm = bilateral_smoothness(mp[name], gt_rgb)
        loss += w_bil * bl
        d_maps[name] = w_bil * dm
    g = rasterize_backward(st, d_maps, nthreads=nthreads)
    sg = shade_backward(cache, g["d_colors"])
    da = g["d_attrs"]
    o = sigmoid(p["o_logit"])
    loss += w_op * float(o.mean())
    d_o_logit = g["d_o_logit"] + w_op * (o * (1.0 - o) / o.size)
    grads = {"mu": g["d_mu"] + sg["d_mu"], "q_raw": g["d_q_raw"], "log_s": g["d_log_s"],
             "o_logit": d_o_logit, "n_raw": g["d_n_raw"] + sg["d_n_raw"],
             "delta_c": sg["d_delta_c"] + da["delta_c"],
             "k_a_raw": sg["d_k_a_raw"] + da["k_a"] * k_a * (1.0 - k_a),
             "k_d_raw": sg["d_k_d_raw"] + da["k_d"] * k_d * (1.0 - k_d),
             "k_s_raw": sg["d_k_s_raw"] + da["k_s"] * k_s * (1.0 - k_s),
             "log_beta": sg["d_log_beta"] + da["beta"] * (beta - 1.0)}
    stat = np.linalg.norm(g["d_mean2d"], axis=1) + np.linalg.norm(grads["n_raw"], axis=1)
    if aux is not None:  # intermediates for diagnostics
        aux.update(raster=g, d_maps=d_maps, state=st)
    return loss, grads, stat


class Adam:
    """trainer.py:100-128."""

    def __init__(self, eps=1e-15, betas=(0.9, 0.999)):
        self.eps, (self.b1, self.b2), self.state = eps, betas, {}

    def step(self, name, param, grad, lr):
        st = self.state.setdefault(name, {"m": np.zeros_like(param), "v": np.zeros_like(param), "t": 0})
        st["t"] += 1
        st["m"] = self.b1 * st["m"] + (1.0 - self.b1) * grad
        st["v"] = self.b2 * st["v"] + (1.0 - self.b2) * grad * grad
        mh = st["m"] / (1.0 - self.b1 ** st["t"])
        vh = st["v"] / (1.0 - self.b2 ** st["t"])
        param -= lr * mh / (np.sqrt(vh) + self.eps)
        return param

    def remap(self, parents, is_new):
        """trainer.py:122-128: re-index moment rows; new rows reset to 0."""
        for st in self.state.values():
            for key in ("m", "v"):
                arr = st[key][parents].copy()
                arr[is_new] = 0.0
                st[key] = arr


def inverse_step(geom, shading, scene_ids, light, c_p, opacity_raw, lam, b, polar, azimuth,
                 cam, reference, nthreads=0):
    """inverse._step, inverse.py:118-190: returns (loss, grads, rgba)."""
    mu, q_raw, log_s, o_logit, n_raw = geom
    dc, ka, kd, ks, lb = shading
    mode, _, _, ts = light
    scale = softplus(opacity_raw)[scene_ids]
    o_base = sigmoid(o_logit)
    if np.all(scale == 1.0):
        o_eff_logit, p, gate = o_logit, o_base, np.ones(o_base.shape, bool)
    else:
        p = np.clip(scale * o_base, 1e-12, 1.0 - 1e-9)
        gate = (scale * o_base > 1e-12) & (scale * o_base < 1.0 - 1e-9)
        o_eff_logit = inv_sigmoid(p)
    rgb, cache = shade(mu, n_raw, dc, ka, kd, ks, lb, np.asarray(c_p)[scene_ids],
                       (mode, polar, azimuth, ts), cam, coeff_transform=(lam, b))
    st = rasterize(mu, q_raw, log_s, o_eff_logit, n_raw, rgb, cam, dtype=np.float64,
                   nthreads=nthreads)
    mp = maps(st)
    rgba = np.concatenate([mp["color"], mp["alpha"][..., None]], axis=-1)
    loss, d = photometric_loss(rgba, reference)
    g = rasterize_backward(st, {"color": d[..., :3], "alpha": d[..., 3]}, nthreads=nthreads)
    sg = shade_backward(cache, g["d_colors"])
    S = np.asarray(c_p).shape[0]
    d_cp = np.zeros((S, 3))
    np.add.at(d_cp, scene_ids, sg["d_c_p"])
    d_p = g["d_o_logit"] / (p * (1.0 - p))
    d_sc = np.zeros(S)
    np.add.at(d_sc, scene_ids, np.where(gate, d_p * o_base, 0.0))
    grads = {"c_p": d_cp, "opacity_raw": d_sc * sigmoid(opacity_raw), "lam": sg["d_lam"],
             "b": sg["d_b"], "angles": np.array([sg["d_polar"], sg["d_azimuth"]])}
    return loss, grads, rgba
