"""Gaussian storage, camera model and projection entry points.

Host-side containers mirror voxsplat's public types (gaussians.py:29-215):
structure-of-arrays float64 storage in the unconstrained domain and a pinhole
camera (+z forward, +x right, +y down).  Host properties (``opacity``,
``normals`` ...) are conveniences for callers; every render/gradient path
runs on the GPU through ``libivrgs.so``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import CulledBehindCamera

NEAR_PLANE = 0.01       # gaussians.py:21
COV2D_DILATION = 0.3    # gaussians.py:22


def _sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    e = np.exp(x[~pos])
    out[~pos] = e / (1.0 + e)
    return out


def _unit_rows(v, eps=0.0):
    n = np.linalg.norm(v, axis=-1, keepdims=True)
    if eps:
        n = np.maximum(n, eps)
    return v / n


@dataclass
class GaussianGeometry:
    """Primitive geometry in storage form: mu (N,3), q_raw (N,4) w-first,
    log_s (N,3), o_logit (N,), n_raw (N,3)."""

    mu: np.ndarray
    q_raw: np.ndarray
    log_s: np.ndarray
    o_logit: np.ndarray
    n_raw: np.ndarray

    def __post_init__(self):
        self.mu = np.atleast_2d(np.asarray(self.mu, dtype=np.float64))
        self.q_raw = np.atleast_2d(np.asarray(self.q_raw, dtype=np.float64))
        self.log_s = np.atleast_2d(np.asarray(self.log_s, dtype=np.float64))
        self.o_logit = np.atleast_1d(np.asarray(self.o_logit, dtype=np.float64))
        self.n_raw = np.atleast_2d(np.asarray(self.n_raw, dtype=np.float64))

    @classmethod
    def from_natural(cls, mu, q, s, opacity, n):
        q = np.atleast_2d(np.asarray(q, dtype=np.float64))
        s = np.atleast_2d(np.asarray(s, dtype=np.float64))
        o = np.clip(np.atleast_1d(np.asarray(opacity, dtype=np.float64)), 1e-6, 1.0 - 1e-6)
        return cls(mu=mu, q_raw=q, log_s=np.log(s), o_logit=np.log(o / (1.0 - o)), n_raw=n)

    def __len__(self):
        return self.mu.shape[0]

    @property
    def quat(self):
        return _unit_rows(self.q_raw)

    @property
    def scales(self):
        return np.exp(self.log_s)

    @property
    def opacity(self):
        return _sigmoid(self.o_logit)

    @property
    def normals(self):
        return _unit_rows(self.n_raw, eps=1e-12)

    def copy(self):
        return GaussianGeometry(self.mu.copy(), self.q_raw.copy(), self.log_s.copy(),
                                self.o_logit.copy(), self.n_raw.copy())

    def select(self, idx):
        return GaussianGeometry(self.mu[idx], self.q_raw[idx], self.log_s[idx],
                                self.o_logit[idx], self.n_raw[idx])

    @staticmethod
    def concat(parts):
        return GaussianGeometry(*(np.concatenate([getattr(p, k) for p in parts], axis=0)
                                  for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")))


SH_C0 = 0.28209479177387814


@dataclass
class ShColor:
    """Spherical-harmonic colour coefficients (N, (L+1)^2, 3), DC first."""

    coefficients: np.ndarray
    degree: int

    def __post_init__(self):
        self.coefficients = np.asarray(self.coefficients, dtype=np.float64)
        want = (self.degree + 1) ** 2
        if self.coefficients.shape[-2] != want or self.coefficients.shape[-1] != 3:
            raise ValueError(f"degree {self.degree} needs (*, {want}, 3) coefficients, "
                             f"got {self.coefficients.shape}")

    @classmethod
    def from_dc(cls, rgb, degree=0):
        rgb = np.atleast_2d(np.asarray(rgb, dtype=np.float64))
        c = np.zeros((rgb.shape[0], (degree + 1) ** 2, 3))
        c[:, 0, :] = (rgb - 0.5) / SH_C0
        return cls(c, degree)


@dataclass
class Camera:
    """Pinhole camera; ``rotation`` is world-to-camera, row-orthonormal."""

    position: np.ndarray
    rotation: np.ndarray
    fov_y: float
    width: int
    height: int

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        if not (0.0 < self.fov_y < np.pi):
            raise ValueError(f"fov_y out of (0, pi): {self.fov_y}")
        err = np.abs(self.rotation @ self.rotation.T - np.eye(3)).max()
        if err > 1e-6:
            raise ValueError(f"rotation not orthonormal (err {err:.2e})")

    @property
    def focal(self):
        return 0.5 * self.height / np.tan(0.5 * self.fov_y)

    @property
    def center_px(self):
        return ((self.width - 1) / 2.0, (self.height - 1) / 2.0)

    @classmethod
    def look_at(cls, position, target, fov_y, width, height, up=(0.0, 0.0, 1.0)):
        position = np.asarray(position, dtype=np.float64)
        fwd = _unit_rows(np.asarray(target, dtype=np.float64) - position)
        right = np.cross(np.asarray(up, dtype=np.float64), fwd)
        nr = np.linalg.norm(right)
        if nr < 1e-8:  # looking along the up axis: use +x as the reference
            right = np.cross(np.array([1.0, 0.0, 0.0]), fwd)
            nr = np.linalg.norm(right)
        right /= nr
        down = np.cross(fwd, right)
        return cls(position, np.stack([right, down, fwd], axis=0), fov_y, width, height)

    def to_dict(self):
        return {"position": [float(v) for v in self.position],
                "rotation": [float(v) for v in self.rotation.reshape(-1)],
                "fov_y": float(self.fov_y), "width": int(self.width), "height": int(self.height)}

    @classmethod
    def from_dict(cls, d):
        return cls(np.array(d["position"], dtype=np.float64),
                   np.array(d["rotation"], dtype=np.float64).reshape(3, 3),
                   float(d["fov_y"]), int(d["width"]), int(d["height"]))


def orbit_camera(center, radius, polar, azimuth, fov_y, width, height):
    """Camera on a sphere around ``center`` (x = cos cos, y = cos sin, z = sin)."""
    d = np.array([np.cos(polar) * np.cos(azimuth), np.cos(polar) * np.sin(azimuth),
                  np.sin(polar)])
    return Camera.look_at(np.asarray(center, dtype=np.float64) + radius * d, center, fov_y,
                          width, height)


def project_gaussians(geom, cam, near=NEAR_PLANE):
    """EWA projection on the GPU (gaussians.py:296-346 semantics).

    Returns a dict with mean2d (N,2), cov2d (N,2,2), conic (N,3), depth (N,),
    valid (N,) as host float64 arrays (the kernel's float64 parity outputs).
    """
    if near != NEAR_PLANE:
        raise ValueError("the GPU projection uses the reference near plane 0.01")
    from .rasterizer import _project_only
    return _project_only(geom, cam)


def project_gaussian(geom, cam, index=0):
    """Single-primitive projection; raises CulledBehindCamera when culled."""
    p = project_gaussians(geom, cam)
    if not p["valid"][index]:
        raise CulledBehindCamera(f"primitive {index} at camera-space z <= near")
    a, b, c = p["conic"][index]
    return {"mean2d": p["mean2d"][index], "cov2d": p["cov2d"][index],
            "conic": np.array([[a, b], [b, c]]), "depth": p["depth"][index]}


def view_dirs(mu, cam_position):
    """Unit directions from the camera to each primitive."""
    return _unit_rows(mu - np.asarray(cam_position)[None, :], eps=1e-12)
