"""IVRG load straight into HBM (device CRC-32 + unpack) vs the reference's
load_model outputs, and rendering from the resident arrays."""

import os
import zlib

import numpy as np
import pytest

from test_ivrg import GEOM, IVRG_DIR, SHADE, _arrays

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _path(name):
    return os.path.join(IVRG_DIR, name + ".ivrg")


@pytest.mark.parametrize("n", [0, 1, 3, 255, 256, 257, 4095, 65535, 65536, 65537, 200_003,
                               (1 << 24) + 13])
def test_device_crc32_matches_zlib(n):
    import torch
    from paper_2504_17954_b200.ivrg import crc32_device
    rng = np.random.default_rng(n)
    data = rng.integers(0, 256, n, dtype=np.uint8)
    dev = torch.from_numpy(data).cuda()
    assert crc32_device(dev) == zlib.crc32(data.tobytes())
    if n > 17:  # unaligned start
        assert crc32_device(dev[5:]) == zlib.crc32(data[5:].tobytes())


@pytest.mark.parametrize("name", ["editable", "base", "quantized", "quantized_wide", "composed"])
def test_load_matches_reference(name):
    from paper_2504_17954_b200 import ComposedScene
    from paper_2504_17954_b200.ivrg import load_model
    a = _arrays(name)
    obj = load_model(_path(name))
    models = obj.models if isinstance(obj, ComposedScene) else [obj]
    for i, m in enumerate(models):
        for k in GEOM:
            assert np.array_equal(getattr(m.geometry, k), a[f"m{i}_{k}"]), (i, k)
        if f"m{i}_sh" in a:
            assert np.array_equal(m.sh.coefficients, a[f"m{i}_sh"])
        if f"m{i}_delta_c" in a:
            for k in SHADE:
                assert np.array_equal(getattr(m.shading, k), a[f"m{i}_{k}"]), (i, k)
        if f"m{i}_cb_q_raw" in a:
            assert m.shading is None
            for k, (cb, idx) in m.quantized.items():
                assert np.array_equal(cb.centroids, a[f"m{i}_cb_{k}"])
                assert np.array_equal(idx, a[f"m{i}_idx_{k}"]) and idx.dtype == a[f"m{i}_idx_{k}"].dtype
        if f"m{i}_palette" in a:
            assert np.array_equal(m.palette.c_p, a[f"m{i}_palette"])
    if isinstance(obj, ComposedScene):
        assert obj.edits[1].opacity_scale == 0.5 and obj.transform["note"] == "fit"
        assert obj.light.mode == "orbital"


def test_corrupt_and_truncated_files(tmp_path):
    from paper_2504_17954_b200 import BadMagic, ChecksumMismatch
    from paper_2504_17954_b200.ivrg import load_model
    buf = bytearray(open(_path("composed"), "rb").read())
    bad = bytearray(buf)
    bad[len(bad) // 2] ^= 0x40
    p = tmp_path / "bad.ivrg"
    p.write_bytes(bytes(bad))
    with pytest.raises(ChecksumMismatch):
        load_model(str(p))
    p.write_bytes(bytes(buf[:len(buf) - 100]))
    with pytest.raises(ChecksumMismatch):
        load_model(str(p))
    p.write_bytes(b"JUNK" + bytes(buf[4:]))
    with pytest.raises(BadMagic):
        load_model(str(p))


def test_round_trip_save_load(tmp_path):
    from paper_2504_17954_b200.ivrg import load_model, save_model
    from paper_2504_17954_b200.synthetic import editable_model
    m = editable_model(9, 5000, f32=True)
    m.metadata = {"k": 1}
    p = str(tmp_path / "m.ivrg")
    save_model(m, p)
    back = load_model(p)
    for k in GEOM:
        assert np.array_equal(getattr(back.geometry, k), getattr(m.geometry, k))
    for k in SHADE:
        assert np.array_equal(getattr(back.shading, k), getattr(m.shading, k))
    assert back.metadata == {"k": 1}


@pytest.mark.parametrize("name", ["composed", "editable", "quantized"])
def test_render_from_resident_file_matches_host_scene(name):
    """DeviceScene over the device-loaded arrays == DeviceScene over the
    reference-loaded host scene (bit-identical images)."""
    from paper_2504_17954_b200 import ComposedScene, DeviceScene, orbit_camera
    from paper_2504_17954_b200.ivrg import load_device, load_model
    f = load_device(_path(name))
    ds_dev = f.device_scene()
    host = load_model(_path(name))
    if not isinstance(host, ComposedScene):
        host = ComposedScene.compose([host])
    ds_host = DeviceScene(host)
    cam = orbit_camera(np.zeros(3), 2.6, 0.3, 0.7, 0.9, 64, 48)
    a = ds_dev.render(cam, channels=("color", "alpha", "depth"))
    b = ds_host.render(cam, channels=("color", "alpha", "depth"))
    assert np.array_equal(a.color, b.color) and np.array_equal(a.alpha, b.alpha)
    assert np.array_equal(a.depth, b.depth)
    assert np.array_equal(a.per_pixel_contrib_count, b.per_pixel_contrib_count)
    assert a.alpha.max() > 0.1
