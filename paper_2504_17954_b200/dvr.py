"""Ground-truth direct volume rendering for dataset generation (drop-in for
voxsplat/dvr.py).

Volumes, transfer functions and materials are the reference's host types;
``render_view`` ray-marches on the GPU (csrc/dvr.cu, float64, the reference's
per-sample arithmetic), so generating a multi-view training set no longer
costs CPU minutes per view.  ``generate_dataset`` / ``load_dataset`` keep the
reference's on-disk layout (PNG views + manifest.json).
"""

from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .errors import OutOfRange, ShapeMismatch
from .gaussians import Camera
from .shading import LightConfig, light_direction_from_angles
from .trainer import ViewDataset

T_STOP = 1e-4
FLAT_GRADIENT = 1e-6
MANIFEST_VERSION = 1


@dataclass
class VolumeGrid:
    """Scalar field on a regular grid centred on the origin (dvr.py:30-66)."""

    values: np.ndarray
    spacing: np.ndarray = field(default_factory=lambda: np.ones(3))
    kind: str = "custom"

    def __post_init__(self):
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        if self.values.ndim != 3 or min(self.values.shape) < 2:
            raise ShapeMismatch(f"volume must be 3-d with dims >= 2, got {self.values.shape}")
        if not np.all(np.isfinite(self.values)):
            raise OutOfRange("volume contains non-finite values")
        self.spacing = np.asarray(self.spacing, dtype=np.float64).reshape(3)
        if np.any(self.spacing <= 0):
            raise OutOfRange("voxel spacing must be positive")

    @property
    def dims(self):
        return self.values.shape

    @property
    def origin(self):
        return -(np.array(self.dims) - 1) * self.spacing / 2.0

    @property
    def bbox(self):
        lo = self.origin
        return lo, lo + (np.array(self.dims) - 1) * self.spacing

    def descriptor(self):
        return {"kind": self.kind, "dims": list(self.dims), "spacing": self.spacing.tolist()}


def _grid_coords(dims):
    axes = [np.linspace(-1.0, 1.0, d) for d in dims]
    return np.meshgrid(*axes, indexing="ij")


def make_shells_volume(dims=(64, 64, 64)):
    x, y, z = _grid_coords(dims)
    r = np.sqrt(x * x + y * y + z * z) / np.sqrt(3.0)
    return VolumeGrid(np.clip(r, 0.0, 1.0), kind="shells")


def make_lobes_volume(dims=(64, 64, 64), lobes=4.0, alpha=0.25):
    x, y, z = _grid_coords(dims)
    rho_r = np.cos(2.0 * np.pi * lobes * np.cos(np.pi * np.sqrt(x * x + y * y) / 2.0))
    v = (1.0 - np.sin(np.pi * z / 2.0) + alpha * (1.0 + rho_r)) / (2.0 * (1.0 + alpha))
    return VolumeGrid(np.clip(v, 0.0, 1.0), kind="lobes")


def make_swirl_volume(dims=(64, 64, 64)):
    x, y, z = _grid_coords(dims)
    v = (np.sin(np.pi * x) * np.cos(np.pi * y) + np.sin(np.pi * y) * np.cos(np.pi * z)
         + np.sin(np.pi * z) * np.cos(np.pi * x))
    return VolumeGrid((v + 3.0) / 6.0, kind="swirl")


VOLUME_GENERATORS = {"shells": make_shells_volume, "lobes": make_lobes_volume,
                     "swirl": make_swirl_volume}


def make_volume(kind, dims=(64, 64, 64)):
    if kind not in VOLUME_GENERATORS:
        raise OutOfRange(f"unknown volume kind {kind!r}; choose from {sorted(VOLUME_GENERATORS)}")
    return VOLUME_GENERATORS[kind](tuple(dims))


@dataclass
class TransferFunction1D:
    """Piecewise-linear scalar -> (rgb, opacity) map (dvr.py:111-170)."""

    values: np.ndarray
    colors: np.ndarray
    opacities: np.ndarray

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64).reshape(-1)
        self.colors = np.asarray(self.colors, dtype=np.float64).reshape(-1, 3)
        self.opacities = np.asarray(self.opacities, dtype=np.float64).reshape(-1)
        n = self.values.size
        if n < 2 or self.colors.shape[0] != n or self.opacities.size != n:
            raise ShapeMismatch("transfer function needs >= 2 aligned control points")
        if np.any(np.diff(self.values) < 0):
            raise OutOfRange("transfer function control values must be sorted")
        if np.any((self.opacities < 0) | (self.opacities > 1)):
            raise OutOfRange("transfer function opacities must lie in [0, 1]")

    @classmethod
    def basic_bump(cls, v_lo, v_hi, color, max_opacity):
        if not v_lo < v_hi:
            raise OutOfRange("bump needs v_lo < v_hi")
        mid = 0.5 * (v_lo + v_hi)
        color = np.asarray(color, dtype=np.float64)
        return cls([v_lo, mid, v_hi], [color, color, color], [0.0, float(max_opacity), 0.0])

    def support(self):
        nz = np.flatnonzero(self.opacities > 0)
        if nz.size == 0:
            return None
        return (self.values[max(nz[0] - 1, 0)], self.values[min(nz[-1] + 1, self.values.size - 1)])

    def lookup(self, v):
        v = np.clip(np.asarray(v, dtype=np.float64), self.values[0], self.values[-1])
        rgb = np.stack([np.interp(v, self.values, self.colors[:, c]) for c in range(3)], axis=-1)
        return rgb, np.interp(v, self.values, self.opacities)

    def to_dict(self):
        return {"values": self.values.tolist(), "colors": self.colors.tolist(),
                "opacities": self.opacities.tolist()}

    @classmethod
    def from_dict(cls, d):
        return cls(d["values"], d["colors"], d["opacities"])


def transfer_functions_disjoint(tfs):
    supports = sorted(s for s in (tf.support() for tf in tfs) if s is not None)
    return all(a[1] <= b[0] for a, b in zip(supports, supports[1:]))


def union_transfer_functions(tfs):
    if not transfer_functions_disjoint(tfs):
        raise OutOfRange("transfer function supports overlap; union is undefined")
    order = np.argsort([tf.values[0] for tf in tfs], kind="stable")
    parts = [tfs[i] for i in order]
    return TransferFunction1D(np.concatenate([p.values for p in parts]),
                              np.concatenate([p.colors for p in parts], axis=0),
                              np.concatenate([p.opacities for p in parts]))


@dataclass
class Material:
    """Global Blinn-Phong coefficients of the volume (dvr.py:164-171)."""

    k_a: float = 0.4
    k_d: float = 0.6
    k_s: float = 0.3
    beta: float = 16.0


def shade_sample(c_v, n, l, v, k_a, k_d, k_s, beta):
    """Blinn-Phong colour of one shaded sample (dvr.py:216-232), the formula
    K13 evaluates per sample: ambient + diffuse |n.l| + white specular
    |n.h|^beta (h = normalized v + l when |v + l| > 1e-12)."""
    h = np.asarray(v, np.float64) + np.asarray(l, np.float64)
    hn = float(np.sqrt(np.dot(h, h)))
    if hn > 1e-12:
        h = h / hn
    ndl = abs(float(np.dot(n, l)))
    ndh = abs(float(np.dot(n, h)))
    spec = k_s * ndh ** beta if (ndl > 0.0 and ndh > 0.0) else 0.0
    c = np.asarray(c_v, np.float64)
    return k_a * c + k_d * c * ndl + spec


def render_view_device(volume, tf, cam, light, material=None, step_scale=0.5, dev_values=None):
    """Ray-march one camera on the GPU; returns the (H, W, 4) float64 device
    tensor (premultiplied colour, resolved alpha)."""
    if isinstance(tf, (list, tuple)):
        tf = union_transfer_functions(list(tf))
    material = material or Material()
    vals = dev_values if dev_values is not None else D.to_dev(volume.values)
    d0, d1, d2 = volume.dims
    out = torch.empty((cam.height, cam.width, 4), dtype=torch.float64, device=vals.device)
    headlight = light.mode != "orbital"
    ld = np.zeros(3) if headlight else light_direction_from_angles(light.polar, light.azimuth)
    sp = np.ascontiguousarray(volume.spacing, np.float64)
    ldc = np.ascontiguousarray(ld, np.float64)
    mat = np.array([material.k_a, material.k_d, material.k_s, material.beta], np.float64)
    tv, tc, to = D.to_dev(tf.values), D.to_dev(tf.colors), D.to_dev(tf.opacities)
    cs = D.camera_struct(cam)
    dp = ctypes.POINTER(ctypes.c_double)
    L.check(L.lib().ivr_dvr_render(D.ptr(vals), d0, d1, d2, sp.ctypes.data_as(dp), D.ptr(tv),
                                   D.ptr(tc), D.ptr(to), tf.values.size, ctypes.byref(cs),
                                   1 if headlight else 0, ldc.ctypes.data_as(dp),
                                   mat.ctypes.data_as(dp), float(step_scale), D.ptr(out),
                                   D.stream_handle()), "ivr_dvr_render")
    torch.cuda.current_stream().synchronize()  # host arrays above must outlive the launch
    return out


def render_view(volume, tf, cam, light, material=None, step_scale=0.5):
    """Ray-march a full RGBA image for one camera (dvr.py:424-452)."""
    return render_view_device(volume, tf, cam, light, material, step_scale).cpu().numpy()


def raymarch_pixel(volume, tf, cam, light, pixel, material=None, step_scale=0.5):
    """RGBA of one pixel (dvr.py:388-407), from the device render."""
    px, py = pixel
    return render_view(volume, tf, cam, light, material, step_scale)[py, px]


VolumeDataset = ViewDataset  # cameras, images, light, manifest, bbox() (dvr.py:459-482)


def generate_dataset(volume, tf, cameras, light, out_dir, material=None, step_scale=0.5):
    """Render every camera on the GPU and write PNGs plus manifest.json
    (dvr.py:485-520)."""
    from PIL import Image
    material = material or Material()
    os.makedirs(out_dir, exist_ok=True)
    if isinstance(tf, (list, tuple)):
        tf = union_transfer_functions(list(tf))
    vals = D.to_dev(volume.values)
    images, entries = [], []
    for i, cam in enumerate(cameras):
        rgba = render_view_device(volume, tf, cam, light, material, step_scale, vals)
        img8 = torch.clamp(torch.round(rgba * 255.0), 0, 255).to(torch.uint8).cpu().numpy()
        fname = f"view_{i:04d}.png"
        Image.fromarray(img8, mode="RGBA").save(os.path.join(out_dir, fname))
        images.append(img8.astype(np.float64) / 255.0)
        entry = cam.to_dict()
        entry["file"] = fname
        entries.append(entry)
    manifest = {"version": MANIFEST_VERSION, "volume": volume.descriptor(),
                "transfer_function": tf.to_dict(),
                "light": {"mode": light.mode, "polar": light.polar, "azimuth": light.azimuth},
                "material": {"k_a": material.k_a, "k_d": material.k_d, "k_s": material.k_s,
                             "beta": material.beta},
                "cameras": entries}
    with open(os.path.join(out_dir, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
    return VolumeDataset(list(cameras), images, light.copy(), manifest)


def load_dataset(dataset_dir):
    """Load a dataset directory written by generate_dataset (dvr.py:523-533)."""
    from PIL import Image
    with open(os.path.join(dataset_dir, "manifest.json")) as f:
        manifest = json.load(f)
    cameras = [Camera.from_dict(e) for e in manifest["cameras"]]
    images = [np.asarray(Image.open(os.path.join(dataset_dir, e["file"]))).astype(np.float64) / 255.0
              for e in manifest["cameras"]]
    light = LightConfig(mode=manifest["light"]["mode"], polar=manifest["light"]["polar"],
                        azimuth=manifest["light"]["azimuth"])
    return VolumeDataset(cameras, images, light, manifest)
