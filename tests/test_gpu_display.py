"""Display modes and the device frame path (render_modes.py, service frames)
vs the reference's render_mode_image (golden display.npz)."""

import io

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
MODES = ("shaded", "normal", "ambient", "diffuse", "specular", "depth", "alpha")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _scene():
    from paper_2504_17954_b200 import ComposedScene, EditState, LightConfig
    from paper_2504_17954_b200.synthetic import editable_model
    sc = ComposedScene.compose([editable_model(70 + i, 1500, spread=0.5, density=3000)
                                for i in range(2)],
                               LightConfig("orbital", 0.3, 0.7, np.array([1.1, 0.9, 1.0, 1.2])))
    sc.edits[1] = EditState(np.array([0.2, 0.7, 0.4]), 0.6)
    return sc


def _cam(d):
    from paper_2504_17954_b200 import Camera
    return Camera(d["cam_position"], d["cam_rotation"], float(d["cam_fov_y"]),
                  int(d["cam_width"]), int(d["cam_height"]))


@pytest.mark.parametrize("mode", MODES)
def test_render_mode_image_matches_reference(mode):
    from paper_2504_17954_b200.render_modes import render_mode_image
    d = golden("display")
    img = render_mode_image(_scene(), _cam(d), mode)
    ref = d["img_" + mode]
    assert img.shape == ref.shape
    assert np.abs(img - ref).max() <= 1e-4, mode


@pytest.mark.parametrize("mode", MODES)
def test_device_frame_u8_and_png(mode):
    from PIL import Image
    from paper_2504_17954_b200.render_modes import DisplayRenderer
    d = golden("display")
    R = DisplayRenderer(_scene())
    cam = _cam(d)
    u8 = R.frame_u8(cam, mode).cpu().numpy()
    ref = d["u8_" + mode]
    assert u8.shape == ref.shape and u8.dtype == np.uint8
    assert np.abs(u8.astype(int) - ref.astype(int)).max() <= 1  # float-image ulps at .5 steps
    assert (u8 == ref).mean() > 0.99
    png = R.frame_bytes(cam, mode, "png")
    dec = np.asarray(Image.open(io.BytesIO(png)))
    assert np.array_equal(dec, u8)
    assert R.frame_bytes(cam, mode, "raw") == u8.tobytes()


@pytest.mark.parametrize("mode", ("shaded", "alpha", "normal", "depth"))
def test_base_stage_modes(mode):
    from paper_2504_17954_b200 import BasicSceneModel, GaussianGeometry, ShColor
    from paper_2504_17954_b200.render_modes import render_mode_image
    from paper_2504_17954_b200.synthetic import GEOM_KEYS, editable_arrays
    d = golden("display")
    a = editable_arrays(75, 1200, spread=0.5, density=3000)
    sh = ShColor(np.random.default_rng(75).normal(0, 0.4, (1200, 4, 3)), 1)
    base = BasicSceneModel("base", GaussianGeometry(*(a[k] for k in GEOM_KEYS)), sh=sh)
    img = render_mode_image(base, _cam(d), mode)
    assert np.abs(img - d["base_" + mode]).max() <= 1e-4


def test_png_large_multi_block():
    """A frame larger than one stored deflate block (65535 bytes) round-trips."""
    import torch
    from PIL import Image
    from paper_2504_17954_b200 import _lib as L
    from paper_2504_17954_b200.device import ptr, stream_handle
    rng = np.random.default_rng(0)
    for H, W, C in ((300, 257, 4), (1, 1, 1), (123, 77, 3)):
        img = torch.from_numpy(rng.integers(0, 256, (H, W, C), dtype=np.uint8)).cuda()
        size = int(L.lib().ivr_png_size(H, W, C))
        out = torch.empty(size, dtype=torch.uint8, device="cuda")
        ws = torch.empty(64, dtype=torch.uint8, device="cuda")
        assert L.lib().ivr_png_encode(ptr(img), H, W, C, ptr(out), size, ptr(ws),
                                      stream_handle()) == 0
        dec = np.asarray(Image.open(io.BytesIO(out.cpu().numpy().tobytes())))
        ref = img.cpu().numpy()
        assert np.array_equal(dec.reshape(ref.shape), ref)
