"""GPU direct volume rendering (dataset generation) vs the reference's
dvr.render_view (golden dvr.npz): float64, same per-sample arithmetic."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _tf():
    from paper_2504_17954_b200.dvr import TransferFunction1D, union_transfer_functions
    return union_transfer_functions([TransferFunction1D.basic_bump(0.2, 0.45, (0.9, 0.3, 0.2), 0.8),
                                     TransferFunction1D.basic_bump(0.55, 0.8, (0.2, 0.5, 0.9), 0.6)])


@pytest.mark.parametrize("kind", ["shells", "lobes", "swirl"])
def test_render_view_matches_reference(kind):
    from paper_2504_17954_b200 import LightConfig, orbit_camera
    from paper_2504_17954_b200.dvr import Material, make_volume, render_view
    d = golden("dvr")
    cam = orbit_camera(np.zeros(3), 3.0 * 16.0, 0.4, 0.7, 0.8, 24, 20)
    vol = make_volume(kind, (24, 20, 28))
    head = render_view(vol, _tf(), cam, LightConfig())
    orb = render_view(vol, _tf(), cam, LightConfig("orbital", 0.3, -0.8), Material(0.3, 0.5, 0.4, 8.0),
                      step_scale=0.35)
    np.testing.assert_allclose(head, d[kind + "_head"], atol=1e-9)
    np.testing.assert_allclose(orb, d[kind + "_orb"], atol=1e-9)


def test_generate_and_load_dataset(tmp_path):
    from paper_2504_17954_b200 import LightConfig, orbit_camera
    from paper_2504_17954_b200.dvr import generate_dataset, load_dataset, make_volume, render_view
    vol = make_volume("shells", (20, 20, 20))
    cams = [orbit_camera(np.zeros(3), 40.0, 0.2, a, 0.8, 16, 12) for a in (0.0, 1.5)]
    ds = generate_dataset(vol, _tf(), cams, LightConfig(), str(tmp_path))
    back = load_dataset(str(tmp_path))
    assert len(back) == 2 and back.manifest["volume"]["dims"] == [20, 20, 20]
    for a, b, c in zip(ds.images, back.images, cams):
        assert np.array_equal(a, b)
        ref = np.clip(np.round(render_view(vol, _tf(), c, LightConfig()) * 255.0), 0, 255) / 255.0
        assert np.array_equal(a, ref)
    lo, hi = back.bbox()
    assert np.allclose(hi, 9.5)
