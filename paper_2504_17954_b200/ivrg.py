"""IVRG model files, loaded straight into HBM (drop-in for the save_model /
load_model pair of voxsplat/scene.py:242-436).

Format (unchanged, byte-compatible with the reference writer): ``IVRG`` magic,
u16 version, u16 flags, then tagged chunks ``tag(4) | u64 length | payload``
-- META (JSON), PALT (f32 palette per model), GEOM (per model: mu, n_raw),
RAWA (per model: q_raw, log_s, o_logit, then SH or the five shading
attributes) or QATT (per attribute: u32 K, f32 centroids, u8/u16 indices),
EDIT (JSON, composed scenes) -- and a trailing zlib CRC-32 of the body.

B200 path (``load_device``): one read of the file into pinned host memory,
one H2D copy of the whole body, the CRC-32 verified on the GPU (csrc/ivrg.cu,
all SMs), and every float32 chunk widened to float64 by a kernel directly into
the SoA tensors the renderer consumes (all models concatenated, scene ids
alongside) -- the reference's host f32 -> f64 -> device round trip does not
exist.  Codebook-quantized files are decoded with K6 on the device.  Only the
chunk table and the two JSON chunks are parsed on the host.
"""

from __future__ import annotations

import ctypes
import json
import os
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import device as D
from .errors import BadMagic, ChecksumMismatch, VersionUnsupported

MAGIC = b"IVRG"
FORMAT_VERSION = 1
FLAG_QUANTIZED = 1
FLAG_COMPOSED = 2

_GEOMETRY_ATTRS = ("q_raw", "log_s", "o_logit")
_SHADING_ATTRS = ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")
_ATTR_COMPONENTS = {"q_raw": 4, "log_s": 3, "o_logit": 1, "delta_c": 3, "k_a_raw": 1,
                    "k_d_raw": 1, "k_s_raw": 1, "log_beta": 1}
_UNPACK_F32, _UNPACK_U8, _UNPACK_U16 = 0, 1, 2


# ------------------------------------------------------------------ writer
def _f32_bytes(arr):
    return np.ascontiguousarray(arr, dtype="<f4").tobytes()


def _chunk(tag, payload):
    return tag + struct.pack("<Q", len(payload)) + payload


def _json_bytes(obj):
    return json.dumps(obj, sort_keys=True, separators=(",", ":")).encode("utf-8")


def _model_meta(model):
    from .scene import STAGE_BASE
    meta = {"stage": model.stage, "count": len(model), "metadata": model.metadata}
    if model.stage == STAGE_BASE:
        meta["sh_degree"] = int(model.sh.degree)
    meta["has_palette"] = model.palette is not None
    return meta


def _raw_attribute_payload(model):
    from .scene import STAGE_BASE
    parts = [_f32_bytes(getattr(model.geometry, a)) for a in _GEOMETRY_ATTRS]
    if model.stage == STAGE_BASE:
        parts.append(_f32_bytes(model.sh.coefficients))
    else:
        parts += [_f32_bytes(getattr(model.shading, a)) for a in _SHADING_ATTRS]
    return b"".join(parts)


def _quantized_payload(model):
    from .vq import QUANTIZED_ATTRIBUTES
    parts = []
    for name, _ in QUANTIZED_ATTRIBUTES:
        cb, idx = model.quantized[name]
        parts.append(struct.pack("<I", cb.k))
        parts.append(_f32_bytes(cb.centroids))
        parts.append(np.ascontiguousarray(idx, dtype="<u1" if cb.k <= 256 else "<u2").tobytes())
    return b"".join(parts)


def encode_model(obj):
    """The IVRG bytes of a basic model or composed scene (scene.py:286-329)."""
    from .scene import ComposedScene
    if isinstance(obj, ComposedScene):
        flags = FLAG_COMPOSED
        models = obj.models
        meta = {"kind": "composed", "models": [_model_meta(m) for m in models],
                "light": obj.light.to_dict()}
        edit_doc = [e.to_dict() for e in obj.edits]
        if obj.transform is not None:
            edit_doc = {"edits": edit_doc, "transform": obj.transform}
        edit_payload = _json_bytes(edit_doc)
    else:
        flags = FLAG_QUANTIZED if obj.is_quantized else 0
        models = [obj]
        meta = {"kind": "basic", "models": [_model_meta(obj)]}
        edit_payload = None
    geom = b"".join(_f32_bytes(m.geometry.mu) + _f32_bytes(m.geometry.n_raw) for m in models)
    palt = b"".join(_f32_bytes(m.palette.c_p if m.palette is not None else np.zeros(3))
                    for m in models)
    body = MAGIC + struct.pack("<HH", FORMAT_VERSION, flags)
    body += _chunk(b"META", _json_bytes(meta))
    body += _chunk(b"PALT", palt)
    body += _chunk(b"GEOM", geom)
    if flags & FLAG_QUANTIZED:
        body += _chunk(b"QATT", _quantized_payload(obj))
    else:
        body += _chunk(b"RAWA", b"".join(_raw_attribute_payload(m) for m in models))
    if edit_payload is not None:
        body += _chunk(b"EDIT", edit_payload)
    return body + struct.pack("<I", zlib.crc32(body))


def save_model(obj, path):
    """Serialize a basic model or composed scene to the IVRG format."""
    with open(path, "wb") as f:
        f.write(encode_model(obj))


# ------------------------------------------------------------------ reader
def parse_header(buf):
    """Validate magic and version on the host; returns the flags.  Raises
    BadMagic / VersionUnsupported like load_model (scene.py:354-358).  The CRC
    is checked on the device (``load_device``), then ``_chunk_table`` walks the
    chunks (ChecksumMismatch for one running past the body, scene.py:337-340)."""
    mv = memoryview(buf)
    if len(mv) < 12 or bytes(mv[:4]) != MAGIC:
        raise BadMagic("not an IVRG file")
    version, flags = struct.unpack_from("<HH", mv, 4)
    if version != FORMAT_VERSION:
        raise VersionUnsupported(f"IVRG version {version} not supported")
    return flags


def _chunk_table(mv):
    chunks = {}
    pos, end = 8, len(mv) - 4
    while pos < end:
        if pos + 12 > end:
            raise ChecksumMismatch("file truncated inside a chunk")
        tag = bytes(mv[pos:pos + 4])
        (length,) = struct.unpack_from("<Q", mv, pos + 4)
        pos += 12
        if pos + length > end:
            raise ChecksumMismatch("file truncated inside a chunk")
        chunks[tag] = (pos, length)
        pos += length
    return chunks


class _Cursor:
    """Sequential reader over one chunk (offsets into the device body)."""

    def __init__(self, off, length):
        self.pos, self.end = off, off + length

    def take(self, nbytes):
        if self.pos + nbytes > self.end:
            raise ChecksumMismatch("file truncated inside a chunk")
        p = self.pos
        self.pos += nbytes
        return p


@dataclass
class ResidentModel:
    """Per-model header of a device-resident file (the host keeps only the
    metadata and palette; the arrays live in ``DeviceModelFile``)."""

    stage: str
    count: int
    metadata: dict
    palette: object = None
    sh_degree: int = None
    rows: tuple = (0, 0)

    def __len__(self):
        return self.count


@dataclass
class DeviceModelFile:
    """An IVRG file resident in HBM: concatenated float64 SoA tensors of every
    model (``geometry``, ``shading`` or ``sh``), scene ids, and -- for
    quantized files -- the device codebooks and indices."""

    flags: int
    kind: str
    models: list
    geometry: dict
    shading: dict = None
    sh: torch.Tensor = None
    scene_id: torch.Tensor = None
    quantized: dict = None
    edits: list = None
    light: object = None
    transform: dict = None
    crc: int = 0
    nbytes: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def count(self):
        return sum(m.count for m in self.models)

    def device_scene(self):
        """A DeviceScene over the resident arrays (no host round trip)."""
        from .errors import MixedStage
        from .scene import STAGE_EDITABLE, ComposedScene, DeviceScene, EditState
        from .shading import LightConfig
        if any(m.stage != STAGE_EDITABLE for m in self.models):
            raise MixedStage("only editable-stage models compose")
        shading = self.shading if self.shading is not None else \
            self.extra.get("dequantized_shading")
        edits = self.edits if self.edits is not None else [EditState() for _ in self.models]
        sc = ComposedScene(list(self.models), edits, self.light or LightConfig(), self.transform)
        dg = D.DeviceGaussians(self.geometry, shading, None, self.geometry["mu"].device)
        dg.scene_id = self.scene_id
        return DeviceScene(sc, dg=dg)

    def to_host(self):
        """The BasicSceneModel / ComposedScene that load_model returns."""
        from .gaussians import GaussianGeometry, ShColor
        from .scene import STAGE_BASE, BasicSceneModel, ComposedScene
        from .shading import ShadingAttributes
        from .vq import Codebook
        host = lambda t, a, b: D.to_host(t[a:b])  # noqa: E731
        out = []
        for m in self.models:
            a, b = m.rows
            g = GaussianGeometry(*(host(self.geometry[k], a, b) for k in
                                   ("mu", "q_raw", "log_s", "o_logit", "n_raw")))
            if self.quantized is not None:
                quant = {name: (Codebook(name, c.cpu().numpy()), idx)
                         for name, (c, _, idx) in self.quantized.items()}
                out.append(BasicSceneModel(m.stage, g, palette=m.palette, quantized=quant,
                                           metadata=m.metadata))
            elif m.stage == STAGE_BASE:
                out.append(BasicSceneModel(m.stage, g, sh=ShColor(host(self.sh, a, b), m.sh_degree),
                                           metadata=m.metadata))
            else:
                sh_ = ShadingAttributes(*(host(self.shading[k], a, b) for k in _SHADING_ATTRS))
                out.append(BasicSceneModel(m.stage, g, shading=sh_, palette=m.palette,
                                           metadata=m.metadata))
        if self.flags & FLAG_COMPOSED:
            return ComposedScene(out, self.edits, self.light, self.transform)
        return out[0]


def _read_pinned(path):
    size = os.path.getsize(path)
    buf = torch.empty(max(size, 1), dtype=torch.uint8, pin_memory=True)
    with open(path, "rb") as f:
        got = f.readinto(memoryview(buf.numpy())[:size])
    return buf, got


def load_device(path, device=None):
    """Load an IVRG file into HBM; returns a DeviceModelFile.

    Error behaviour follows load_model (scene.py:349-436): BadMagic,
    VersionUnsupported, ChecksumMismatch (CRC over the body, checked on the
    GPU, or a chunk running past the end)."""
    from .gaussians import ShColor  # noqa: F401  (validates degrees below)
    from .scene import STAGE_BASE, EditState
    from .shading import LightConfig, Palette
    from .vq import QUANTIZED_ATTRIBUTES, decode_device
    dev = device or D.cuda_device()
    hbuf, size = _read_pinned(path)
    mv = memoryview(hbuf.numpy())[:size]
    flags = parse_header(mv)
    stream = D.stream_handle()
    body = hbuf[:size].to(dev, non_blocking=True)
    crc_dev = torch.empty(1, dtype=torch.int32, device=dev)
    L.check(L.lib().ivr_crc32(D.ptr(body), size - 4, D.ptr(crc_dev), stream), "ivr_crc32")
    stored = struct.unpack_from("<I", mv, size - 4)[0]
    got = int(crc_dev.item()) & 0xFFFFFFFF  # the one sync of the load
    if got != stored:
        raise ChecksumMismatch("CRC32 mismatch: file corrupt or truncated")
    chunks = _chunk_table(mv)

    def chunk(tag):
        if tag not in chunks:
            raise KeyError(tag)
        return _Cursor(*chunks[tag])

    def jload(tag):
        off, ln = chunks[tag]
        return json.loads(bytes(mv[off:off + ln]).decode("utf-8"))

    base_ptr = body.data_ptr()

    def unpack(pos, count, kind, dst):
        if count:
            L.check(L.lib().ivr_unpack(ctypes.c_void_p(base_ptr + pos), count, kind, D.ptr(dst),
                                       stream), "ivr_unpack")

    meta = jload(b"META")
    metas = meta["models"]
    counts = [int(mm["count"]) for mm in metas]
    N = sum(counts)
    palt, geo = chunk(b"PALT"), chunk(b"GEOM")
    f64 = lambda *shape: torch.empty(shape, dtype=torch.float64, device=dev)  # noqa: E731
    geometry = {"mu": f64(N, 3), "q_raw": f64(N, 4), "log_s": f64(N, 3), "o_logit": f64(N),
                "n_raw": f64(N, 3)}
    quant = None
    qshade = None
    shading = sh = None
    models = []
    raw = chunk(b"RAWA") if b"RAWA" in chunks else None
    row = 0
    for mm, n in zip(metas, counts):
        pal_off = palt.take(12)
        pal = np.frombuffer(bytes(mv[pal_off:pal_off + 12]), dtype="<f4").astype(np.float64)
        rm = ResidentModel(mm["stage"], n, mm["metadata"],
                           Palette(pal) if mm["has_palette"] else None,
                           mm.get("sh_degree"), (row, row + n))
        unpack(geo.take(12 * n), 3 * n, _UNPACK_F32, geometry["mu"][row:])
        unpack(geo.take(12 * n), 3 * n, _UNPACK_F32, geometry["n_raw"][row:])
        if flags & FLAG_QUANTIZED:
            q = chunk(b"QATT")
            quant = {}
            decoded = {}
            for name, _ in QUANTIZED_ATTRIBUTES:
                k = struct.unpack_from("<I", mv, q.take(4))[0]
                cent = f64(k)
                unpack(q.take(4 * k), k, _UNPACK_F32, cent)
                comp = _ATTR_COMPONENTS[name]
                wide = k > 256
                ipos = q.take((2 if wide else 1) * n * comp)
                idx_dev = torch.empty(n * comp, dtype=torch.int16, device=dev)
                unpack(ipos, n * comp, _UNPACK_U16 if wide else _UNPACK_U8, idx_dev)
                idx_host = np.frombuffer(bytes(mv[ipos:ipos + (2 if wide else 1) * n * comp]),
                                         dtype="<u2" if wide else "<u1")
                idx_host = idx_host.reshape((n, comp) if comp > 1 else (n,)).copy()
                quant[name] = (cent, idx_dev, idx_host)
                decoded[name] = decode_device(idx_dev, cent)  # K6 on the device
            for name, (vals, bad) in decoded.items():
                if int(bad.item()) >= 0:
                    from .errors import CorruptIndex
                    raise CorruptIndex(f"codebook {name!r}: index {int(bad.item())} >= K")
            for name in _GEOMETRY_ATTRS:
                geometry[name][row:row + n] = decoded[name][0].view(geometry[name][row:row + n].shape)
            # decoded shading stays on the device for rendering (the host model
            # keeps shading=None, as the reference's quantized load does)
            qshade = {name: decoded[name][0].view((n, 3) if name == "delta_c" else (n,))
                      for name in _SHADING_ATTRS}
            models.append(rm)
            row += n
            continue
        unpack(raw.take(16 * n), 4 * n, _UNPACK_F32, geometry["q_raw"][row:])
        unpack(raw.take(12 * n), 3 * n, _UNPACK_F32, geometry["log_s"][row:])
        unpack(raw.take(4 * n), n, _UNPACK_F32, geometry["o_logit"][row:])
        if mm["stage"] == STAGE_BASE:
            nb = (int(mm["sh_degree"]) + 1) ** 2
            if sh is None:
                sh = f64(N, nb, 3)
            if sh.shape[1] != nb:
                raise ValueError("models of one file with different SH degrees")
            unpack(raw.take(12 * nb * n), 3 * nb * n, _UNPACK_F32, sh[row:])
        else:
            if shading is None:
                shading = {"delta_c": f64(N, 3), "k_a_raw": f64(N), "k_d_raw": f64(N),
                           "k_s_raw": f64(N), "log_beta": f64(N)}
            for name in _SHADING_ATTRS:
                w = _ATTR_COMPONENTS[name]
                unpack(raw.take(4 * w * n), w * n, _UNPACK_F32, shading[name][row:])
        models.append(rm)
        row += n
    scene_id = torch.repeat_interleave(
        torch.arange(len(counts), dtype=torch.int32, device=dev),
        torch.tensor(counts, dtype=torch.int64, device=dev)) if counts else \
        torch.empty(0, dtype=torch.int32, device=dev)
    out = DeviceModelFile(flags, meta.get("kind", "basic"), models, geometry, shading, sh,
                          scene_id, quant, crc=got, nbytes=size)
    if flags & FLAG_COMPOSED:
        edit_doc = jload(b"EDIT")
        transform = None
        if isinstance(edit_doc, dict):
            transform = edit_doc.get("transform")
            edit_doc = edit_doc["edits"]
        out.edits = [EditState.from_dict(d) for d in edit_doc]
        out.light = LightConfig.from_dict(meta["light"])
        out.transform = transform
    if qshade is not None:
        out.extra["dequantized_shading"] = qshade
    out.extra["host_buffer"] = hbuf  # keep the pinned pages alive until the copies finish
    return out


def load_model(path):
    """Load an IVRG file into a BasicSceneModel or ComposedScene
    (scene.py:349-436) through the device path."""
    return load_device(path).to_host()


def crc32_device(data):
    """zlib.crc32 of a device uint8 tensor, computed on the GPU."""
    out = torch.empty(1, dtype=torch.int32, device=data.device)
    L.check(L.lib().ivr_crc32(D.ptr(data), data.numel(), D.ptr(out), D.stream_handle()),
            "ivr_crc32")
    return int(out.item()) & 0xFFFFFFFF
