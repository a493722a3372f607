"""GPU parity: K1 preprocess, K2 bin/sort and K3 blend vs the reference.

Golden fixtures (tests/golden, produced from the real reference) pin exact
values; the CPU oracle (oracle/) is used for sizes without fixtures.
Contract (BASELINE.json north_star): sort keys, tile ranges and per-tile
lists bit-exact; images within 1e-4 max abs (we also report how many pixels
are bit-identical); contributor counts exact.
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

IMG_TOL = 1e-4  # north_star: max abs pixel error <= 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_17954_b200 import _lib
    _lib.lib()  # fail loudly if the native library is missing


def _geom(d):
    from paper_2504_17954_b200 import GaussianGeometry
    return GaussianGeometry(d["mu"], d["q_raw"], d["log_s"], d["o_logit"], d["n_raw"])


def _cam(d):
    from paper_2504_17954_b200 import Camera
    return Camera(d["cam_position"], d["cam_rotation"], float(d["cam_fov_y"]),
                  int(d["cam_width"]), int(d["cam_height"]))


def _light(d):
    from paper_2504_17954_b200 import LightConfig
    return LightConfig(str(d["light_mode"]), float(d["light_polar"]), float(d["light_azimuth"]),
                       d["light_ts"])


CASES = ["render_c1", "render_fixture", "render_ragged"]


@pytest.mark.parametrize("case", CASES)
def test_preprocess_matches_reference(case):
    from paper_2504_17954_b200 import project_gaussians
    d = golden(case)
    p = project_gaussians(_geom(d), _cam(d))
    # no transcendental on these paths: bit-exact
    assert np.array_equal(p["depth"], d["depth"])
    assert np.array_equal(p["mean2d"], d["mean2d"])
    assert np.array_equal(p["valid"], d["valid"])
    # exp(log_s) differs from numpy's SIMD exp by <= 1 ulp on some inputs
    for k in ("cov2d", "conic"):
        ref = d[k].reshape(p[k].shape)
        rel = np.abs(p[k] - ref) / np.maximum(np.abs(ref), 1e-300)
        assert np.nanmax(rel[d["valid"]]) < 1e-12, k


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("case", CASES)
def test_sort_and_image_match_reference(case, exact):
    from paper_2504_17954_b200 import rasterize_forward
    d = golden(case)
    out, st = rasterize_forward(_geom(d), d["rgb"], _cam(d), dtype=np.float32, exact=exact)
    F = st["frame"]
    P = int(F.n_pairs.item())
    assert P == d["pair_splat"].size
    assert np.array_equal(F.pairs(), d["pair_splat"])
    assert np.array_equal(F.tile_ranges.cpu().numpy(), d["tile_ranges"])
    rec = F.rec.cpu().numpy().reshape(-1, 8)
    vis = np.zeros(len(d["depth"]), bool)
    vis[np.unique(d["pair_splat"])] = True
    assert np.array_equal(rec[vis, 0:2], d["kmean2d"][vis])
    assert np.array_equal(rec[vis, 2], d["kopacity"][vis])
    conic = np.stack([2 * rec[:, 4], rec[:, 5], 2 * rec[:, 6]], axis=1)
    assert (conic[vis] != d["kconic"][vis]).sum() <= 2
    assert np.abs(out.color - d["color"]).max() <= IMG_TOL
    assert np.abs(out.alpha - d["alpha"]).max() <= IMG_TOL
    assert np.array_equal(out.per_pixel_contrib_count, d["contrib"])
    assert np.array_equal(F.last_pos.cpu().numpy(), d["last_pos"])
    if exact:  # bit-faithful mode: every pixel identical to the reference
        same = np.mean(out.color == d["color"])
        assert same > 0.999, same
    assert np.abs(F.t_final.cpu().numpy() - d["t_final"]).max() <= 1e-5


@pytest.mark.parametrize("fast", [False, True])
@pytest.mark.parametrize("case", CASES)
def test_fused_shading_render(case, fast):
    """K1 with fused Blinn-Phong shading vs reference render_composed."""
    from paper_2504_17954_b200 import (BasicSceneModel, ComposedScene, DeviceScene, Palette,
                                       ShadingAttributes)
    d = golden(case)
    attrs = ShadingAttributes(d["delta_c"], d["k_a_raw"], d["k_d_raw"], d["k_s_raw"], d["log_beta"])
    m = BasicSceneModel("editable", _geom(d), shading=attrs, palette=Palette(d["palette"]))
    ds = DeviceScene(ComposedScene.compose([m], _light(d)))
    F = ds.render_frame(_cam(d), debug=True)
    rgb = F.dbg["rgb"].cpu().numpy().reshape(-1, 3)
    rel = np.abs(rgb - d["rgb"]) / np.maximum(np.abs(d["rgb"]), 1e-300)
    assert rel.max() < 1e-12
    for _ in range(2):  # second fast frame reuses the learned pair capacity
        out = ds.render(_cam(d), fast=fast)
        assert np.abs(out.color - d["color"]).max() <= IMG_TOL
        assert np.abs(out.alpha - d["alpha"]).max() <= IMG_TOL
        assert np.array_equal(out.per_pixel_contrib_count, d["contrib"])


def _composed_scene(d):
    from paper_2504_17954_b200 import (BasicSceneModel, ComposedScene, EditState, GaussianGeometry,
                                       LightConfig, Palette, ShadingAttributes)
    models = []
    for i in range(3):
        g = GaussianGeometry(*(d[f"m{i}_{k}"] for k in ("mu", "q_raw", "log_s", "o_logit", "n_raw")))
        a = ShadingAttributes(*(d[f"m{i}_{k}"] for k in ("delta_c", "k_a_raw", "k_d_raw",
                                                          "k_s_raw", "log_beta")))
        models.append(BasicSceneModel("editable", g, shading=a, palette=Palette(d[f"m{i}_palette"])))
    sc = ComposedScene.compose(models, LightConfig("orbital", 0.45, 0.9,
                                                   np.array([1.2, 0.8, 1.0, 1.0])))
    sc.edits[1] = EditState(palette_override=np.array([0.2, 0.6, 0.9]))
    sc.edits[2] = EditState(opacity_scale=0.5)
    return sc


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_composed_edit_render(dtype):
    from paper_2504_17954_b200 import render_composed
    d = golden("composed_edit")
    sc = _composed_scene(d)
    out = render_composed(sc, _cam(d), dtype=dtype)
    tag = "32" if dtype == np.float32 else "64"
    assert np.abs(out.color - d["color" + tag]).max() <= IMG_TOL
    assert np.abs(out.alpha - d["alpha" + tag]).max() <= IMG_TOL
    assert np.array_equal(out.per_pixel_contrib_count, d["contrib" + tag])


def test_empty_and_offscreen():
    from paper_2504_17954_b200 import Camera, GaussianGeometry, rasterize_forward
    cam = Camera.look_at((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), np.pi / 3, 32, 32)
    g0 = GaussianGeometry(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                          np.zeros((0, 3)))
    out, _ = rasterize_forward(g0, np.zeros((0, 3)), cam)
    assert out.color.shape == (32, 32, 3) and float(np.abs(out.color).max()) == 0.0
    # everything behind the camera -> no pairs, background only
    g1 = GaussianGeometry.from_natural([(0, 0, -10.0)], [(1, 0, 0, 0)], [(0.1, 0.1, 0.1)], [0.9],
                                       [(0, 0, 1.0)])
    out, st = rasterize_forward(g1, np.ones((1, 3)), cam)
    assert int(st["frame"].n_pairs.item()) == 0
    assert float(out.alpha.max()) == 0.0


def test_random_scenes_vs_oracle():
    """Seeded scenes without fixtures: GPU vs the CPU oracle (oracle/)."""
    import oracle as O
    from paper_2504_17954_b200 import GaussianGeometry, rasterize_forward
    from paper_2504_17954_b200.synthetic import editable_arrays, bench_camera
    for seed, n, W, H in ((5, 20000, 200, 144), (6, 5000, 33, 47)):
        a = editable_arrays(seed, n, density=n)
        cam = bench_camera(W, H, azimuth=0.3 * seed)
        rng = np.random.default_rng(seed)
        colors = rng.uniform(0, 1, (n, 3))
        geom = GaussianGeometry(a["mu"], a["q_raw"], a["log_s"], a["o_logit"], a["n_raw"])
        for dtype, exact in ((np.float32, True), (np.float64, True), (np.float32, False),
                             (np.float64, False)):
            out, st = rasterize_forward(geom, colors, cam, dtype=dtype, exact=exact)
            ref = O.rasterize(a["mu"], a["q_raw"], a["log_s"], a["o_logit"], a["n_raw"], colors,
                              cam, dtype=dtype)
            F = st["frame"]
            assert np.array_equal(F.pairs(), ref["pair_splat"])
            assert np.array_equal(F.tile_ranges.cpu().numpy(), ref["tile_ranges"])
            m = O.maps(ref)
            assert np.abs(out.color - m["color"]).max() <= IMG_TOL
            assert np.array_equal(out.per_pixel_contrib_count, ref["contrib"])


def test_depth_sort_fallback_long_runs():
    """Thousands of depths within ~100 ulps plus one far outlier collapse into
    one 31-bit coarse bucket: the 64-bit fallback sort must keep lexsort order."""
    import oracle as O
    from paper_2504_17954_b200 import Camera, GaussianGeometry, rasterize_forward
    rng = np.random.default_rng(3)
    n = 3000
    mu = np.column_stack([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), 1e-13 * rng.normal(size=n)])
    mu[0] = (0.0, 0.0, 1e4)
    geom = GaussianGeometry(mu, rng.normal(size=(n, 4)), np.full((n, 3), np.log(0.05)),
                            rng.normal(size=n), rng.normal(size=(n, 3)))
    cam = Camera.look_at((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), np.pi / 3, 96, 64)
    colors = rng.uniform(0, 1, (n, 3))
    out, st = rasterize_forward(geom, colors, cam)
    ref = O.rasterize(geom.mu, geom.q_raw, geom.log_s, geom.o_logit, geom.n_raw, colors, cam)
    assert np.array_equal(st["frame"].pairs(), ref["pair_splat"])
    assert np.array_equal(st["frame"].tile_ranges.cpu().numpy(), ref["tile_ranges"])
    assert np.array_equal(out.per_pixel_contrib_count, ref["contrib"])


@pytest.mark.parametrize("exact", [True, False])
@pytest.mark.parametrize("W,H", [(1920, 1080), (3840, 2160)])
def test_large_frames_banded_placement(W, H, exact):
    """Tile grids too large for the shared-memory placement tables (1080p: 2
    bands, 4K: 6 bands) give the reference's lists and image, with the EXACT
    and the FAST (certified float32) blend."""
    import oracle as O
    from paper_2504_17954_b200 import GaussianGeometry, rasterize_forward
    from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays
    n = 30000
    a = editable_arrays(11, n, density=n)
    cam = bench_camera(W, H, azimuth=0.7)
    colors = np.random.default_rng(11).uniform(0, 1, (n, 3))
    geom = GaussianGeometry(a["mu"], a["q_raw"], a["log_s"], a["o_logit"], a["n_raw"])
    out, st = rasterize_forward(geom, colors, cam, exact=exact)
    ref = O.rasterize(a["mu"], a["q_raw"], a["log_s"], a["o_logit"], a["n_raw"], colors, cam)
    F = st["frame"]
    assert np.array_equal(F.pairs(), ref["pair_splat"])
    assert np.array_equal(F.tile_ranges.cpu().numpy(), ref["tile_ranges"])
    assert np.array_equal(out.per_pixel_contrib_count, ref["contrib"])
    assert np.array_equal(F.last_pos.cpu().numpy(), ref["last_pos"])
    assert np.abs(out.color - O.maps(ref)["color"]).max() <= IMG_TOL


@pytest.mark.parametrize("counts", [(50,), (60, 45, 30)])
def test_composed_render_equals_union_rasterization(counts):
    """The reference's compose contract (tests/test_scene.py:41-78): rendering
    a composed scene equals shading the concatenated primitives and
    rasterizing the union list, bit for bit (float64)."""
    from paper_2504_17954_b200 import (ComposedScene, GaussianGeometry, ShadingAttributes,
                                       rasterize_forward, render_composed, shade_gaussians)
    from paper_2504_17954_b200.synthetic import bench_camera, editable_model
    models = [editable_model(30 + i, c, spread=0.5, density=400) for i, c in enumerate(counts)]
    sc = ComposedScene.compose(models)
    cam = bench_camera(64, 48, 0.5)
    img = render_composed(sc, cam, dtype=np.float64)
    geom = GaussianGeometry.concat([m.geometry for m in sc.models])
    attrs = ShadingAttributes.concat([m.shading for m in sc.models])
    palette = np.concatenate([np.broadcast_to(m.palette.c_p, (len(m), 3)) for m in sc.models])
    rgb, _, _ = shade_gaussians(geom, attrs, palette, sc.light, cam)
    union, _ = rasterize_forward(geom, rgb, cam, dtype=np.float64)
    assert np.array_equal(img.color, union.color)
    assert np.array_equal(img.alpha, union.alpha)
