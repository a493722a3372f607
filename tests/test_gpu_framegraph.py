"""CUDA-graph frames (FrameGraph) and the pipelined host path (FramePipeline):
identical images to the uncaptured renderer, edits picked up per frame, pair
capacity growth."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _scene():
    from paper_2504_17954_b200.synthetic import c2_scene
    return c2_scene(per_model=20_000, n_models=3, density=60_000)


def _cams(n, W=160, H=120):
    from paper_2504_17954_b200.synthetic import bench_camera
    return [bench_camera(W, H, 0.3 + 0.7 * i) for i in range(n)]


def test_graph_replay_matches_uncaptured_render():
    import torch
    from paper_2504_17954_b200 import DeviceScene, FrameGraph
    ds = DeviceScene(_scene())
    cams = _cams(4)
    fg = FrameGraph(ds, 160, 120, warm_cam=cams[0], slots=2)
    for cam in cams:
        F = fg.replay(cam)
        torch.cuda.synchronize()
        assert not fg.overflowed()
        got = F.out.cpu().numpy()
        ref = ds.render(cam, exact=False)
        assert np.array_equal(got[..., :3], ref.color) and np.array_equal(got[..., 3], ref.alpha)
        assert np.array_equal(F.contrib.cpu().numpy(), ref.per_pixel_contrib_count)


def test_pipeline_results_and_edits():
    from collections import deque
    from paper_2504_17954_b200 import DeviceScene, FrameGraph, FramePipeline
    sc = _scene()
    ds = DeviceScene(sc)
    cams = _cams(6)
    fg = FrameGraph(ds, 160, 120, warm_cam=cams[0], slots=2)
    pipe = FramePipeline(fg)
    pal = np.array([[0.9, 0.1, 0.1], [0.2, 0.8, 0.3], [0.1, 0.2, 0.9]])
    inflight, got = deque(), []
    for i, cam in enumerate(cams):
        kw = {"opacity_scales": np.array([1.0, 0.5, 1.0])} if i % 2 else {"palettes": pal}
        inflight.append((pipe.submit(cam, **kw), cam, kw))
        if len(inflight) >= 2:
            t, c, k = inflight.popleft()
            out = pipe.result(t)
            got.append((out.color.copy(), out.alpha.copy(), out.per_pixel_contrib_count.copy(), c, k))
    while inflight:
        t, c, k = inflight.popleft()
        out = pipe.result(t)
        got.append((out.color.copy(), out.alpha.copy(), out.per_pixel_contrib_count.copy(), c, k))
    for color, alpha, cnt, cam, kw in got:
        ref = ds.render(cam, exact=False, **kw)
        assert np.array_equal(color, ref.color) and np.array_equal(alpha, ref.alpha)
        assert np.array_equal(cnt, ref.per_pixel_contrib_count)
    assert pipe.d2h_bytes_per_frame() == 160 * 120 * 20 + 4


def test_pipeline_grows_pair_capacity():
    """A view needing more pairs than the captured capacity is re-rendered
    after the capacity grows (no silent truncation)."""
    from paper_2504_17954_b200 import DeviceScene, FrameGraph, FramePipeline
    from paper_2504_17954_b200.synthetic import bench_camera
    ds = DeviceScene(_scene())
    far = bench_camera(160, 120, 0.5)
    far.position = far.position * 3.0  # small footprint -> few pairs at capture
    fg = FrameGraph(ds, 160, 120, warm_cam=far, slots=2, headroom=1.0)
    fg.capacity = 4096
    fg._capture(far)
    near = _cams(1)[0]
    pipe = FramePipeline(fg)
    out = pipe.result(pipe.submit(near))
    ref = ds.render(near, exact=False)
    assert np.array_equal(out.color, ref.color)
    assert fg.capacity > 4096


def test_static_cache_is_bit_identical():
    """K1 / K4b with the per-Gaussian static cache == without it (records,
    depth keys, float64 parity outputs, images, inverse gradients)."""
    import torch
    from paper_2504_17954_b200 import DeviceScene
    from paper_2504_17954_b200.synthetic import bench_camera
    ds = DeviceScene(_scene())
    assert ds.dg.cache is not None and ds.dg.cache_ok
    cam = bench_camera(96, 80, 1.3)
    kw = dict(debug=True, want_state=True, palettes=np.array([[0.9, 0.1, 0.1], [0.2, 0.8, 0.3],
                                                               [0.1, 0.2, 0.9]]),
              opacity_scales=np.array([1.0, 0.5, 1.7]))
    a = ds.render_frame(cam, exact=True, **kw)
    torch.cuda.synchronize()
    got = {k: v.clone() for k, v in a.dbg.items()}
    rec, keys, out = a.rec.clone(), a.depth_key.clone(), a.out.clone()
    ds.dg.drop_cache()
    b = ds.render_frame(cam, exact=True, **kw)
    torch.cuda.synchronize()
    for k, v in b.dbg.items():
        assert torch.equal(got[k], v), k
    assert torch.equal(rec, b.rec) and torch.equal(keys, b.depth_key) and torch.equal(out, b.out)


def test_compose_device_matches_host_compose():
    """compose_device (ivr_concat of resident models) renders bit-identically
    to DeviceScene(ComposedScene.compose(host models)) with edits."""
    from paper_2504_17954_b200 import ComposedScene, DeviceScene, LightConfig, compose_device
    from paper_2504_17954_b200.device import DeviceGaussians
    from paper_2504_17954_b200.synthetic import bench_camera, editable_model
    models = [editable_model(20 + i, 3000 + 500 * i, density=20_000) for i in range(3)]
    light = LightConfig("orbital", 0.4, 1.0, np.array([1.1, 0.9, 1.0, 1.0]))
    host = DeviceScene(ComposedScene.compose(models, light))
    dev = compose_device([DeviceGaussians(m.geometry, m.shading) for m in models],
                         [m.palette.c_p for m in models], light)
    assert int(dev.dg.scene_id[-1]) == 2 and dev.n == host.n
    cam = bench_camera(96, 72, 0.6)
    kw = dict(palettes=np.array([[0.9, 0.1, 0.1], [0.2, 0.8, 0.3], [0.1, 0.2, 0.9]]),
              opacity_scales=np.array([1.0, 0.5, 1.0]))
    a, b = dev.render(cam, **kw), host.render(cam, **kw)
    assert np.array_equal(a.color, b.color) and np.array_equal(a.alpha, b.alpha)
