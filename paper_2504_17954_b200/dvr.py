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


def _as_volume_array(values, spacing):
    """Validated float64 C-contiguous samples and a positive 3-vector spacing."""
    vals = np.ascontiguousarray(values, dtype=np.float64)
    if vals.ndim != 3 or min(vals.shape) < 2:
        raise ShapeMismatch(f"volume must be 3-d with dims >= 2, got {vals.shape}")
    if not np.isfinite(vals).all():
        raise OutOfRange("volume contains non-finite values")
    sp = np.asarray(spacing, dtype=np.float64).reshape(3)
    if (sp <= 0).any():
        raise OutOfRange("voxel spacing must be positive")
    return vals, sp


@dataclass
class VolumeGrid:
    """Regular-grid scalar field whose samples are centred on the origin
    (same fields and conventions as dvr.py:30-66: sample (i, j, k) sits at
    origin + (i, j, k) * spacing with origin = -(dims - 1) * spacing / 2)."""

    values: np.ndarray
    spacing: np.ndarray = field(default_factory=lambda: np.ones(3))
    kind: str = "custom"

    def __post_init__(self):
        self.values, self.spacing = _as_volume_array(self.values, self.spacing)

    @property
    def dims(self):
        return self.values.shape

    @property
    def extent(self):
        """Edge lengths of the sampled box."""
        return (np.asarray(self.dims, dtype=np.float64) - 1.0) * self.spacing

    @property
    def origin(self):
        return -0.5 * self.extent

    @property
    def bbox(self):
        return -0.5 * self.extent, 0.5 * self.extent

    def descriptor(self):
        return dict(kind=self.kind, dims=[int(d) for d in self.dims],
                    spacing=[float(x) for x in self.spacing])


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
    """Scalar -> (rgb, opacity) through linear interpolation between sorted
    control points, clamped outside them (dvr.py:111-170)."""

    values: np.ndarray
    colors: np.ndarray
    opacities: np.ndarray

    def __post_init__(self):
        x = np.asarray(self.values, dtype=np.float64).ravel()
        rgb = np.asarray(self.colors, dtype=np.float64).reshape(-1, 3)
        a = np.asarray(self.opacities, dtype=np.float64).ravel()
        if x.size < 2 or len(rgb) != x.size or a.size != x.size:
            raise ShapeMismatch("transfer function needs >= 2 aligned control points")
        if (x[1:] < x[:-1]).any():
            raise OutOfRange("transfer function control values must be sorted")
        if ((a < 0.0) | (a > 1.0)).any():
            raise OutOfRange("transfer function opacities must lie in [0, 1]")
        self.values, self.colors, self.opacities = x, rgb, a

    @classmethod
    def basic_bump(cls, v_lo, v_hi, color, max_opacity):
        """Triangle of opacity peaking at the midpoint, one colour throughout."""
        if not v_lo < v_hi:
            raise OutOfRange("bump needs v_lo < v_hi")
        rgb = np.tile(np.asarray(color, dtype=np.float64), (3, 1))
        return cls(np.array([v_lo, 0.5 * (v_lo + v_hi), v_hi]), rgb,
                   np.array([0.0, float(max_opacity), 0.0]))

    def support(self):
        """Interval outside which the opacity is zero (None if never opaque):
        the control points adjacent to the first and last opaque ones."""
        opaque = np.nonzero(self.opacities > 0.0)[0]
        if len(opaque) == 0:
            return None
        last = len(self.values) - 1
        return (self.values[max(int(opaque[0]) - 1, 0)],
                self.values[min(int(opaque[-1]) + 1, last)])

    def lookup(self, v):
        """(rgb, opacity) at value(s) v."""
        x = self.values
        v = np.clip(np.asarray(v, dtype=np.float64), x[0], x[-1])
        table = np.column_stack([self.colors, self.opacities])
        cols = [np.interp(v, x, table[:, c]) for c in range(4)]
        return np.stack(cols[:3], axis=-1), cols[3]

    def to_dict(self):
        return dict(values=self.values.tolist(), colors=self.colors.tolist(),
                    opacities=self.opacities.tolist())

    @classmethod
    def from_dict(cls, d):
        return cls(d["values"], d["colors"], d["opacities"])


def transfer_functions_disjoint(tfs):
    """No two opacity supports overlap (touching endpoints are allowed)."""
    spans = sorted(sp for sp in map(TransferFunction1D.support, tfs) if sp is not None)
    return all(prev[1] <= nxt[0] for prev, nxt in zip(spans, spans[1:]))


def union_transfer_functions(tfs):
    """One transfer function holding every control point of disjoint ones,
    ordered by their first control value (stable)."""
    if not transfer_functions_disjoint(tfs):
        raise OutOfRange("transfer function supports overlap; union is undefined")
    ordered = sorted(tfs, key=lambda tf: tf.values[0])
    return TransferFunction1D(np.hstack([tf.values for tf in ordered]),
                              np.vstack([tf.colors for tf in ordered]),
                              np.hstack([tf.opacities for tf in ordered]))


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
    return D.to_host(render_view_device(volume, tf, cam, light, material, step_scale))


def raymarch_pixel(volume, tf, cam, light, pixel, material=None, step_scale=0.5):
    """RGBA of one pixel (dvr.py:388-407), from the device render."""
    px, py = pixel
    return render_view(volume, tf, cam, light, material, step_scale)[py, px]


VolumeDataset = ViewDataset  # cameras, images, light, manifest, bbox() (dvr.py:459-482)


def _manifest(volume, tf, light, material, entries):
    """manifest.json contents (the reference's dataset layout, dvr.py:485-520)."""
    return {
        "version": MANIFEST_VERSION,
        "volume": volume.descriptor(),
        "transfer_function": tf.to_dict(),
        "light": dict(mode=light.mode, polar=light.polar, azimuth=light.azimuth),
        "material": dict(k_a=material.k_a, k_d=material.k_d, k_s=material.k_s, beta=material.beta),
        "cameras": entries,
    }


def generate_dataset(volume, tf, cameras, light, out_dir, material=None, step_scale=0.5):
    """Render every camera on the GPU, write view_NNNN.png (RGBA, rounded to
    8 bits) and manifest.json, and return the dataset (dvr.py:485-520)."""
    from PIL import Image
    material = material or Material()
    tf = union_transfer_functions(list(tf)) if isinstance(tf, (list, tuple)) else tf
    os.makedirs(out_dir, exist_ok=True)
    vals = D.to_dev(volume.values)
    images, entries = [], []
    for idx, cam in enumerate(cameras):
        rgba = render_view_device(volume, tf, cam, light, material, step_scale, vals)
        u8 = D.to_host((rgba * 255.0).round_().clamp_(0, 255).to(torch.uint8))
        name = "view_%04d.png" % idx
        Image.fromarray(u8, mode="RGBA").save(os.path.join(out_dir, name))
        images.append(u8 / 255.0)
        entries.append(dict(cam.to_dict(), file=name))
    manifest = _manifest(volume, tf, light, material, entries)
    with open(os.path.join(out_dir, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=2, sort_keys=True)
    return VolumeDataset(list(cameras), images, light.copy(), manifest)


def load_dataset(dataset_dir):
    """Read a directory written by generate_dataset (dvr.py:523-533)."""
    from PIL import Image
    with open(os.path.join(dataset_dir, "manifest.json")) as fh:
        manifest = json.load(fh)
    views = manifest["cameras"]
    cameras = [Camera.from_dict(v) for v in views]
    images = []
    for v in views:
        with Image.open(os.path.join(dataset_dir, v["file"])) as im:
            images.append(np.asarray(im, dtype=np.float64) / 255.0)
    lt = manifest["light"]
    return VolumeDataset(cameras, images, LightConfig(mode=lt["mode"], polar=lt["polar"],
                                                      azimuth=lt["azimuth"]), manifest)
