"""multigpu.render_views on the device (one process): every view equals the
uncaptured FAST render of the same camera, in the callers' order."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_17954_b200 import _lib
    _lib.lib()


def test_render_views_equals_per_view_renders():
    from paper_2504_17954_b200 import ComposedScene, DeviceScene, LightConfig
    from paper_2504_17954_b200.multigpu import render_views
    from paper_2504_17954_b200.synthetic import bench_camera, editable_model
    scene = ComposedScene.compose([editable_model(s, 20_000, density=40_000) for s in range(2)],
                                  LightConfig("orbital", 0.45, 0.9))
    cams = [bench_camera(160, 120, 0.3 * i) for i in range(4)] + [bench_camera(96, 64, 1.7)]
    imgs = render_views(scene, cams)
    ds = DeviceScene(scene)
    for cam, img in zip(cams, imgs):
        ds.render_frame(cam, fast=False)
        F = ds.render_frame(cam, fast=True, exact=False)
        assert img.shape == (cam.height, cam.width, 4)
        assert np.array_equal(img, F.out.cpu().numpy())
