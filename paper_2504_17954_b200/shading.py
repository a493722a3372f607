"""Editable Blinn-Phong shading (drop-in for voxsplat/shading.py).

Host containers mirror the reference types (Palette, LightConfig,
ShadingAttributes; shading.py:27-176).  ``shade_gaussians`` runs the float64
shading kernel on the GPU (ivr_shade_fwd) and returns the reference's
(rgb, terms, cache) triple; ``shade_backward`` runs K4's shading backward.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from . import device as D
from .errors import OutOfRange, ShapeMismatch

WHITE = np.ones(3)
HEADLIGHT = "headlight"
ORBITAL = "orbital"


def _sig(x):
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def _logit(y):
    y = np.asarray(y, dtype=np.float64)
    return np.log(y / (1.0 - y))


@dataclass
class Palette:
    """Base colour shared by every splat of one basic scene."""

    c_p: np.ndarray

    def __post_init__(self):
        self.c_p = np.asarray(self.c_p, dtype=np.float64).reshape(3)
        if not np.all(np.isfinite(self.c_p)):
            raise OutOfRange("palette color must be finite")

    def copy(self):
        return Palette(self.c_p.copy())


@dataclass
class LightConfig:
    """Headlight (camera-attached) or orbital (fixed direction) light plus
    the global (ambient, diffuse, specular, shininess) term scales."""

    mode: str = HEADLIGHT
    polar: float = 0.0
    azimuth: float = 0.0
    term_scales: np.ndarray = field(default_factory=lambda: np.ones(4))

    def __post_init__(self):
        if self.mode not in (HEADLIGHT, ORBITAL):
            raise OutOfRange(f"unknown light mode: {self.mode!r}")
        self.polar = float(self.polar)
        self.azimuth = float(self.azimuth)
        if not -np.pi / 2 <= self.polar <= np.pi / 2:
            raise OutOfRange(f"polar angle {self.polar} outside [-pi/2, pi/2]")
        if not -np.pi <= self.azimuth <= np.pi:
            raise OutOfRange(f"azimuth angle {self.azimuth} outside [-pi, pi]")
        self.term_scales = np.asarray(self.term_scales, dtype=np.float64).reshape(4)
        if not np.all(self.term_scales > 0):
            raise OutOfRange("term_scales must be strictly positive")

    def copy(self):
        return LightConfig(self.mode, self.polar, self.azimuth, self.term_scales.copy())

    def to_dict(self):
        return {"mode": self.mode, "polar": self.polar, "azimuth": self.azimuth,
                "term_scales": self.term_scales.tolist()}

    @classmethod
    def from_dict(cls, d):
        return cls(mode=d.get("mode", HEADLIGHT), polar=d.get("polar", 0.0),
                   azimuth=d.get("azimuth", 0.0),
                   term_scales=np.asarray(d.get("term_scales", [1.0, 1.0, 1.0, 1.0])))


@dataclass
class ShadingAttributes:
    """Per-splat material in storage form: delta_c (N,3), k_a/k_d/k_s logits
    (N,), log_beta (N,) with beta = exp(log_beta) + 1."""

    delta_c: np.ndarray
    k_a_raw: np.ndarray
    k_d_raw: np.ndarray
    k_s_raw: np.ndarray
    log_beta: np.ndarray

    def __post_init__(self):
        self.delta_c = np.atleast_2d(np.asarray(self.delta_c, dtype=np.float64))
        n = self.delta_c.shape[0]
        for name in ("k_a_raw", "k_d_raw", "k_s_raw", "log_beta"):
            arr = np.atleast_1d(np.asarray(getattr(self, name), dtype=np.float64))
            if arr.shape != (n,):
                raise ShapeMismatch(f"{name} must have shape ({n},), got {arr.shape}")
            setattr(self, name, arr)
        if self.delta_c.shape[1] != 3:
            raise ShapeMismatch(f"delta_c must be (N, 3), got {self.delta_c.shape}")

    def __len__(self):
        return self.delta_c.shape[0]

    @property
    def k_a(self):
        return _sig(self.k_a_raw)

    @property
    def k_d(self):
        return _sig(self.k_d_raw)

    @property
    def k_s(self):
        return _sig(self.k_s_raw)

    @property
    def beta(self):
        return np.exp(self.log_beta) + 1.0

    @classmethod
    def from_natural(cls, delta_c, k_a, k_d, k_s, beta):
        beta = np.atleast_1d(np.asarray(beta, dtype=np.float64))
        if np.any(beta <= 1.0):
            raise OutOfRange("shininess must be > 1 to admit a log parameterization")
        return cls(delta_c, _logit(k_a), _logit(k_d), _logit(k_s), np.log(beta - 1.0))

    def copy(self):
        return ShadingAttributes(self.delta_c.copy(), self.k_a_raw.copy(), self.k_d_raw.copy(),
                                 self.k_s_raw.copy(), self.log_beta.copy())

    def select(self, idx):
        return ShadingAttributes(self.delta_c[idx], self.k_a_raw[idx], self.k_d_raw[idx],
                                 self.k_s_raw[idx], self.log_beta[idx])

    @staticmethod
    def concat(parts):
        return ShadingAttributes(*(np.concatenate([getattr(p, k) for p in parts], axis=0)
                                   for k in ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw",
                                             "log_beta")))


def resolve_light_direction(light, cam, mu):
    """Per-point unit light direction (shading.py:186-196): from the camera
    towards each point for a headlight, the constant orbital direction
    otherwise."""
    mu = np.asarray(mu, dtype=np.float64)
    if light.mode != ORBITAL:
        d = np.asarray(cam.position, dtype=np.float64) - mu
        return d / np.maximum(np.linalg.norm(d, axis=-1, keepdims=True), 1e-12)
    l = light_direction_from_angles(light.polar, light.azimuth)
    return np.broadcast_to(l, mu.shape).copy() if mu.ndim > 1 else l


def blinn_phong(c_v, n, l, v, k_a, k_d, k_s, beta):
    """The reflection formula shared by splat shading and volume rendering
    (shading.py:199-222), on host arrays with numpy broadcasting over the
    leading axes: ambient k_a c_v, diffuse k_d |n.l| c_v, white specular
    k_s |n.h|^beta with h = normalize(v + l) (eps 1e-12), gated on |n.l| > 0.
    Returns (rgb, ambient, diffuse, specular).  A host utility: the GPU
    paths evaluate the same expression inside K1 / K13."""
    c_v = np.asarray(c_v, dtype=np.float64)
    n, l, v = (np.asarray(x, dtype=np.float64) for x in (n, l, v))
    k_a, k_d, k_s, beta = (np.asarray(x, dtype=np.float64) for x in (k_a, k_d, k_s, beta))
    u = v + l
    h = u / np.maximum(np.linalg.norm(u, axis=-1, keepdims=True), 1e-12)
    a_ndl = np.abs(np.sum(n * l, axis=-1))
    a_ndh = np.abs(np.sum(n * h, axis=-1))
    spow = np.where(a_ndh > 0.0, np.power(np.maximum(a_ndh, 1e-300), beta), 0.0)
    spow = np.where(a_ndl > 0.0, spow, 0.0)
    ambient = k_a[..., None] * c_v
    diffuse = (k_d * a_ndl)[..., None] * c_v
    specular = (k_s * spow)[..., None] * WHITE
    return ambient + diffuse + specular, ambient, diffuse, specular


def light_direction_from_angles(polar, azimuth):
    return D.light_direction(polar, azimuth)


def _palette_array(palette):
    c_p = palette.c_p if isinstance(palette, Palette) else np.asarray(palette, dtype=np.float64)
    return np.asarray(c_p, dtype=np.float64)


def shade_gaussians(geom, attrs, palette, light, cam, coeff_transform=None):
    """Per-splat rgb under the editable reflection model (GPU, float64).

    Same contract as shading.py:225-329: returns (rgb (N,3), terms dict with
    ambient/diffuse/specular, cache for ``shade_backward``)."""
    n = len(geom)
    c_p = _palette_array(palette)
    per_splat = c_p.ndim == 2
    lam, b = (None, None) if coeff_transform is None else coeff_transform
    if n == 0:
        z = np.zeros((0, 3))
        return z, {"ambient": z, "diffuse": z, "specular": z}, {"n": 0}
    dg = D.DeviceGaussians(geom, attrs)
    pal = D.to_dev(c_p.reshape(-1, 3))
    S = D.shading_struct(dg, pal, per_splat, light, lam, b)
    dev = dg.device
    import torch
    rgb = torch.empty(3 * n, dtype=torch.float64, device=dev)
    terms = torch.empty(9 * n, dtype=torch.float64, device=dev)
    g = dg.struct()
    cs = D.camera_struct(cam)
    L.check(L.lib().ivr_shade_fwd(ctypes.byref(g), ctypes.byref(S), None, ctypes.byref(cs),
                                  D.ptr(rgb), D.ptr(terms), D.stream_handle()), "ivr_shade_fwd")
    rgb_h = rgb.cpu().numpy().reshape(n, 3)
    t = terms.cpu().numpy().reshape(n, 9)
    terms_h = {"ambient": t[:, 0:3], "diffuse": t[:, 3:6], "specular": t[:, 6:9]}
    cache = {"geom": geom, "attrs": attrs, "palette": c_p, "per_splat_palette": per_splat,
             "light": light.copy(), "cam": cam,
             "lam": np.ones(4) if lam is None else np.asarray(lam, dtype=np.float64).reshape(4),
             "b": np.zeros(4) if b is None else np.asarray(b, dtype=np.float64).reshape(4),
             "dg": dg, "pal_dev": pal, "n": n}
    return rgb_h, terms_h, cache


def shade_backward(cache, d_rgb):
    """Gradients of the shaded colour w.r.t. every learnable input on the GPU
    (float64; shading.py:332-445): d_delta_c, d_k_a_raw, d_k_d_raw, d_k_s_raw,
    d_log_beta, d_n_raw, d_c_p (per splat for per-splat palettes, else summed),
    d_mu, d_lam, d_b, d_polar, d_azimuth.  Raises NonFiniteGradient."""
    import torch
    n = cache["n"]
    if n == 0:
        z = np.zeros((0, 3))
        return {"d_delta_c": z, "d_k_a_raw": np.zeros(0), "d_k_d_raw": np.zeros(0),
                "d_k_s_raw": np.zeros(0), "d_log_beta": np.zeros(0), "d_n_raw": z,
                "d_c_p": z if cache["per_splat_palette"] else np.zeros(3), "d_mu": z,
                "d_lam": np.zeros(4), "d_b": np.zeros(4), "d_polar": 0.0, "d_azimuth": 0.0}
    dg = cache["dg"]
    light = cache["light"]
    S = D.shading_struct(dg, cache["pal_dev"], cache["per_splat_palette"], light, cache["lam"],
                         cache["b"])
    d_rgb_dev = D.to_dev(np.asarray(d_rgb, dtype=np.float64).reshape(n, 3))
    want = ("d_mu", "d_n_raw", "d_delta_c", "d_k_a_raw", "d_k_d_raw", "d_k_s_raw", "d_log_beta",
            "d_c_p", "d_globals")
    out, bad = D.preprocess_backward(dg, cache["cam"], 1, (-1, -1, -1, -1), shading=S,
                                     d_rgb=d_rgb_dev, geometry=False, want=want, per_scene=1,
                                     per_splat_c_p=cache["per_splat_palette"], light=light)
    D.raise_if_bad(bad, n, ("d_delta_c", "d_k_a_raw", "d_k_d_raw", "d_k_s_raw", "d_log_beta",
                            "d_n_raw", "d_mu"))
    h = {k: v.cpu().numpy() for k, v in out.items()}
    gl = h["d_globals"]
    res = {"d_delta_c": h["d_delta_c"].reshape(n, 3), "d_k_a_raw": h["d_k_a_raw"],
           "d_k_d_raw": h["d_k_d_raw"], "d_k_s_raw": h["d_k_s_raw"], "d_log_beta": h["d_log_beta"],
           "d_n_raw": h["d_n_raw"].reshape(n, 3),
           "d_c_p": h["d_c_p"].reshape(n, 3) if cache["per_splat_palette"] else h["d_c_p"][:3],
           "d_mu": h["d_mu"].reshape(n, 3), "d_lam": gl[0:4].copy(), "d_b": gl[4:8].copy(),
           "d_polar": float(gl[8]) if light.mode == ORBITAL else 0.0,
           "d_azimuth": float(gl[9]) if light.mode == ORBITAL else 0.0}
    for name in ("d_lam", "d_b"):
        if not np.all(np.isfinite(res[name])):
            from .errors import NonFiniteGradient
            raise NonFiniteGradient(name, int(np.flatnonzero(~np.isfinite(res[name]))[0]))
    return res
