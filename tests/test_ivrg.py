"""IVRG writer and header/chunk-table reader on the host, against files written
by the reference's save_model (tests/golden/ivrg/, make_golden.ivrg_case)."""

import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN

IVRG_DIR = os.path.join(GOLDEN, "ivrg")
GEOM = ("mu", "q_raw", "log_s", "o_logit", "n_raw")
SHADE = ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")


def _file(name):
    with open(os.path.join(IVRG_DIR, name + ".ivrg"), "rb") as f:
        return f.read()


def _arrays(name):
    with np.load(os.path.join(IVRG_DIR, name + ".npz")) as z:
        return {k: z[k] for k in z.files}


def _meta(buf):
    from paper_2504_17954_b200.ivrg import _chunk_table
    off, ln = _chunk_table(memoryview(buf))[b"META"]
    return json.loads(buf[off:off + ln].decode())


def _edits(buf):
    from paper_2504_17954_b200.ivrg import _chunk_table
    off, ln = _chunk_table(memoryview(buf))[b"EDIT"]
    return json.loads(buf[off:off + ln].decode())


def _host_models(name, buf):
    """Host model objects holding the values the reference's load_model
    returned (already float32-representable)."""
    from paper_2504_17954_b200 import (BasicSceneModel, Codebook, GaussianGeometry, Palette,
                                       ShadingAttributes, ShColor)
    a = _arrays(name)
    meta = _meta(buf)
    models = []
    for i, mm in enumerate(meta["models"]):
        g = GaussianGeometry(*(a[f"m{i}_{k}"] for k in GEOM))
        pal = Palette(a[f"m{i}_palette"]) if f"m{i}_palette" in a else None
        if f"m{i}_cb_q_raw" in a:
            from paper_2504_17954_b200.vq import QUANTIZED_ATTRIBUTES
            quant = {k: (Codebook(k, a[f"m{i}_cb_{k}"]), a[f"m{i}_idx_{k}"])
                     for k, _ in QUANTIZED_ATTRIBUTES}
            models.append(BasicSceneModel("editable", g, palette=pal, quantized=quant,
                                          metadata=mm["metadata"]))
        elif mm["stage"] == "base":
            models.append(BasicSceneModel("base", g, sh=ShColor(a[f"m{i}_sh"], mm["sh_degree"]),
                                          metadata=mm["metadata"]))
        else:
            models.append(BasicSceneModel("editable", g,
                                          shading=ShadingAttributes(*(a[f"m{i}_{k}"] for k in SHADE)),
                                          palette=pal, metadata=mm["metadata"]))
    return meta, models


@pytest.mark.parametrize("name", ["editable", "base", "quantized", "quantized_wide", "composed"])
def test_writer_byte_identical_to_reference(name):
    from paper_2504_17954_b200 import ComposedScene, EditState, LightConfig
    from paper_2504_17954_b200.ivrg import encode_model
    buf = _file(name)
    meta, models = _host_models(name, buf)
    if meta["kind"] == "composed":
        doc = _edits(buf)
        transform = doc.get("transform") if isinstance(doc, dict) else None
        edits = doc["edits"] if isinstance(doc, dict) else doc
        obj = ComposedScene(models, [EditState.from_dict(e) for e in edits],
                            LightConfig.from_dict(meta["light"]), transform)
    else:
        obj = models[0]
    assert encode_model(obj) == buf


def test_header_errors():
    from paper_2504_17954_b200 import BadMagic, ChecksumMismatch, VersionUnsupported
    from paper_2504_17954_b200.ivrg import _chunk_table, parse_header
    buf = bytearray(_file("editable"))
    assert parse_header(buf) == 0
    with pytest.raises(BadMagic):
        parse_header(b"IVRX" + bytes(buf[4:]))
    with pytest.raises(BadMagic):
        parse_header(buf[:11])
    bad = bytearray(buf)
    struct.pack_into("<H", bad, 4, 2)
    with pytest.raises(VersionUnsupported):
        parse_header(bad)
    # a chunk length running past the body
    short = bytes(buf[:40]) + bytes(buf[-4:])
    with pytest.raises(ChecksumMismatch):
        _chunk_table(memoryview(short))
    assert set(_chunk_table(memoryview(bytes(buf)))) == {b"META", b"PALT", b"GEOM", b"RAWA"}
    assert parse_header(_file("composed")) == 2 and parse_header(_file("quantized")) == 1
