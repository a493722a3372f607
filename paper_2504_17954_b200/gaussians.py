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
    out = _project_only(geom, cam)
    out["geom"], out["cam"] = geom, cam  # what project_backward needs
    return out


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


# ---------------------------------------------------------------------------
# per-Gaussian building blocks of the projection / colour (gaussians.py:222-289,
# 349-400, 429-529) as array functions.  The render and training paths run
# them fused inside K1 / K4b / K8; these entry points evaluate the same
# expressions batched on the GPU (torch float64) for API compatibility.

def _dev(x):
    from . import device as D
    return D.to_dev(np.ascontiguousarray(np.asarray(x, dtype=np.float64)))


def _rot_t(q):
    w, x, y, z = q.unbind(1)
    return __import__("torch").stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1).view(-1, 3, 3)


def _rot_backward_t(q, g):
    import torch
    w, x, y, z = q.unbind(1)
    G = lambda r, c: g[:, r, c]  # noqa: E731
    dw = 2 * (-z * G(0, 1) + y * G(0, 2) + z * G(1, 0) - x * G(1, 2) - y * G(2, 0) + x * G(2, 1))
    dx = 2 * (y * G(0, 1) + z * G(0, 2) + y * G(1, 0) - 2 * x * G(1, 1) - w * G(1, 2)
              + z * G(2, 0) + w * G(2, 1) - 2 * x * G(2, 2))
    dy = 2 * (-2 * y * G(0, 0) + x * G(0, 1) + w * G(0, 2) + x * G(1, 0) + z * G(1, 2)
              - w * G(2, 0) + z * G(2, 1) - 2 * y * G(2, 2))
    dz = 2 * (-2 * z * G(0, 0) - w * G(0, 1) + x * G(0, 2) + w * G(1, 0) - 2 * z * G(1, 1)
              + y * G(1, 2) + x * G(2, 0) + y * G(2, 1))
    return torch.stack([dw, dx, dy, dz], 1)


def quat_to_rot(q):
    """Unit quaternions (N,4) w-first -> rotations (N,3,3) (gaussians.py:222-236)."""
    return _rot_t(_dev(np.atleast_2d(q))).cpu().numpy()


def quat_to_rot_backward(q, dR):
    """d/dq of quat_to_rot for the upstream dR (N,3,3) (gaussians.py:239-264)."""
    return _rot_backward_t(_dev(np.atleast_2d(q)), _dev(dR).view(-1, 3, 3)).cpu().numpy()


def build_covariance(q, s):
    """Sigma = R diag(s)^2 R^T (gaussians.py:267-275); a single q gives (3,3)."""
    single = np.asarray(q).ndim == 1
    R = _rot_t(_dev(np.atleast_2d(q)))
    M = R * _dev(np.atleast_2d(s))[:, None, :]
    cov = (M @ M.transpose(1, 2)).cpu().numpy()
    return cov[0] if single else cov


def covariance_backward(q, s, d_cov):
    """(dq, ds) of build_covariance for the full dL/dSigma (gaussians.py:278-289)."""
    import torch
    qt, st = _dev(np.atleast_2d(q)), _dev(np.atleast_2d(s))
    R = _rot_t(qt)
    M = R * st[:, None, :]
    dc = _dev(d_cov).view(-1, 3, 3)
    dM = (dc + dc.transpose(1, 2)) @ M
    ds = torch.einsum("nik,nik->nk", dM, R)
    dq = _rot_backward_t(qt, dM * st[:, None, :])
    return dq.cpu().numpy(), ds.cpu().numpy()


def sh_basis(dirs, degree):
    """Real SH basis (N,B) and its direction derivatives (N,B,3) for unit
    directions (gaussians.py:429-494), from csrc/sh.cu (ivr_sh_basis)."""
    import torch
    from . import _lib as L
    from . import device as D
    d = _dev(np.atleast_2d(dirs)).contiguous()
    n, nb = d.shape[0], (int(degree) + 1) ** 2
    B = torch.empty((n, nb), dtype=torch.float64, device=d.device)
    dB = torch.empty((n, nb, 3), dtype=torch.float64, device=d.device)
    L.check(L.lib().ivr_sh_basis(n, int(degree), D.ptr(d), D.ptr(B), D.ptr(dB),
                                 D.stream_handle()), "ivr_sh_basis")
    return B.cpu().numpy(), dB.cpu().numpy()


def eval_sh(color, view_dirs):
    """SH colour along unit ``view_dirs`` with the +0.5 offset, clamped at 0
    from below (gaussians.py:497-507).  Returns (rgb (N,3), cache)."""
    B, dB = sh_basis(view_dirs, color.degree)
    coeffs = np.asarray(color.coefficients, np.float64)
    raw = np.einsum("nb,nbc->nc", B, coeffs) + 0.5
    return np.maximum(raw, 0.0), {"basis": B, "dbasis": dB, "raw": raw, "coeffs": coeffs}


def eval_sh_backward(cache, d_rgb):
    """(d_coeffs (N,B,3), d_dir (N,3)) of eval_sh (gaussians.py:510-518)."""
    g = np.asarray(d_rgb, np.float64) * (cache["raw"] > 0)
    d_coeffs = cache["basis"][:, :, None] * g[:, None, :]
    inner = np.einsum("nbc,nc->nb", cache["coeffs"], g)
    return d_coeffs, np.einsum("nb,nbk->nk", inner, cache["dbasis"])


def view_dirs_backward(mu, cam_position, d_dir):
    """d/dmu of view_dirs (gaussians.py:527-529)."""
    from ._mathutil import normalize_rows_backward
    v = np.asarray(mu, np.float64) - np.asarray(cam_position, np.float64)[None, :]
    return normalize_rows_backward(v, np.asarray(d_dir, np.float64))


def project_backward(cache, d_mean2d, d_cov2d, d_depth):
    """Chain d_mean2d (N,2), the full d_cov2d (N,2,2) and d_depth (N,) back to
    (d_mu, d_q_raw, d_log_s) (gaussians.py:349-400), batched on the GPU.
    ``cache`` is the dict project_gaussians returns."""
    import torch
    geom, cam = cache["geom"], cache["cam"]
    q_raw = _dev(geom.q_raw)
    qn = q_raw / torch.linalg.norm(q_raw, dim=1, keepdim=True)
    s = torch.exp(_dev(geom.log_s))
    R = _rot_t(qn)
    M3 = R * s[:, None, :]
    cov3d = M3 @ M3.transpose(1, 2)
    Wr = _dev(cam.rotation)
    f = float(cam.focal)
    t = (_dev(geom.mu) - _dev(cam.position)[None, :]) @ Wr.T
    valid = torch.from_numpy(np.asarray(cache["valid"], bool)).to(t.device)
    tz = torch.where(valid, t[:, 2], torch.ones_like(t[:, 2]))
    n = t.shape[0]
    J = torch.zeros((n, 2, 3), dtype=torch.float64, device=t.device)
    J[:, 0, 0] = f / tz
    J[:, 0, 2] = -f * t[:, 0] / tz ** 2
    J[:, 1, 1] = f / tz
    J[:, 1, 2] = -f * t[:, 1] / tz ** 2
    M = J @ Wr
    dm = torch.where(valid[:, None], _dev(d_mean2d).view(n, 2), 0.0)
    dc = torch.where(valid[:, None, None], _dev(d_cov2d).view(n, 2, 2), 0.0)
    dd = torch.where(valid, _dev(d_depth).view(n), 0.0)
    d_cov3d = M.transpose(1, 2) @ dc @ M
    dM = dc @ M @ cov3d.transpose(1, 2) + dc.transpose(1, 2) @ M @ cov3d
    dJ = dM @ Wr.T
    dt = torch.zeros((n, 3), dtype=torch.float64, device=t.device)
    dt[:, 0] = dJ[:, 0, 2] * (-f / tz ** 2) + dm[:, 0] * f / tz
    dt[:, 1] = dJ[:, 1, 2] * (-f / tz ** 2) + dm[:, 1] * f / tz
    dt[:, 2] = (dJ[:, 0, 0] * (-f / tz ** 2) + dJ[:, 1, 1] * (-f / tz ** 2)
                + dJ[:, 0, 2] * (2 * f * t[:, 0] / tz ** 3) + dJ[:, 1, 2] * (2 * f * t[:, 1] / tz ** 3)
                - dm[:, 0] * f * t[:, 0] / tz ** 2 - dm[:, 1] * f * t[:, 1] / tz ** 2 + dd)
    d_mu = dt @ Wr
    dMc = (d_cov3d + d_cov3d.transpose(1, 2)) @ M3
    ds = torch.einsum("nik,nik->nk", dMc, R)
    dq_unit = _rot_backward_t(qn, dMc * s[:, None, :])
    nq = torch.linalg.norm(q_raw, dim=1, keepdim=True)
    u = q_raw / nq
    d_q_raw = (dq_unit - (dq_unit * u).sum(1, keepdim=True) * u) / nq
    return {"d_mu": d_mu.cpu().numpy(), "d_q_raw": d_q_raw.cpu().numpy(),
            "d_log_s": (ds * s).cpu().numpy()}
