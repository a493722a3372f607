"""Edge cases of the render / backward path vs the oracle: odd frame sizes,
equal depths (lexsort ties), near-plane and behind-camera splats, opaque
stacks (early termination + FAST-mode ambiguity replays), many channels
(KMAX = 32 kernels)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
IMG_TOL = 1e-4


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _check(geom, colors, cam, attrs=None, channels=("color", "alpha"), dtypes=(np.float32,)):
    import oracle as O
    from paper_2504_17954_b200 import rasterize_forward
    for dtype in dtypes:
        for exact in (True, False):
            out, st = rasterize_forward(geom, colors, cam, channels=channels, attrs=attrs,
                                        dtype=dtype, exact=exact)
            ref = O.rasterize(geom.mu, geom.q_raw, geom.log_s, geom.o_logit, geom.n_raw, colors,
                              cam, channels=channels, attrs=attrs, dtype=dtype)
            if not st.get("empty"):
                assert np.array_equal(st["frame"].pairs(), ref["pair_splat"])
                assert np.array_equal(st["frame"].tile_ranges.cpu().numpy(), ref["tile_ranges"])
            m = O.maps(ref)
            assert np.array_equal(out.per_pixel_contrib_count, ref["contrib"]), (dtype, exact)
            if "color" in channels:
                assert np.abs(out.color - m["color"]).max() <= IMG_TOL
            assert np.abs(out.alpha - m["alpha"]).max() <= IMG_TOL
            for k in (attrs or {}):
                assert np.abs(out.attr[k] - m[k]).max() <= IMG_TOL, k
    return out, st


@pytest.mark.parametrize("W,H", [(1, 1), (16, 16), (17, 15), (300, 7), (5, 130)])
def test_odd_frame_sizes(W, H):
    from paper_2504_17954_b200 import GaussianGeometry
    from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays
    a = editable_arrays(W * 7 + H, 4000, density=4000)
    geom = GaussianGeometry(a["mu"], a["q_raw"], a["log_s"], a["o_logit"], a["n_raw"])
    colors = np.random.default_rng(1).uniform(0, 1, (4000, 3))
    _check(geom, colors, bench_camera(W, H, 0.4), dtypes=(np.float32, np.float64))


def test_equal_depth_ties_and_near_plane():
    """Many splats at exactly equal depth (order by index), splats behind the
    camera and straddling the near plane."""
    from paper_2504_17954_b200 import Camera, GaussianGeometry
    rng = np.random.default_rng(4)
    n = 3000
    mu = np.column_stack([rng.uniform(-0.8, 0.8, n), rng.uniform(-0.8, 0.8, n), np.zeros(n)])
    mu[:1000, 2] = 0.25                  # a plane of exactly equal depths
    mu[1000:1100, 2] = -3.995           # around the near plane (camera at z = -4)
    mu[1100:1200, 2] = -10.0            # behind the camera
    geom = GaussianGeometry(mu, rng.normal(size=(n, 4)), np.log(rng.uniform(0.01, 0.08, (n, 3))),
                            rng.normal(size=n), rng.normal(size=(n, 3)))
    cam = Camera.look_at((0.0, 0.0, -4.0), (0.0, 0.0, 0.0), np.pi / 3, 80, 64)
    _check(geom, rng.uniform(0, 1, (n, 3)), cam)


def test_opaque_stack_early_termination():
    """Dense opaque layers: every pixel stops at T < 1e-4 (and some land in
    FAST mode's ambiguity band and are re-walked exactly)."""
    from paper_2504_17954_b200 import GaussianGeometry
    from paper_2504_17954_b200.synthetic import bench_camera
    rng = np.random.default_rng(9)
    n = 20000
    mu = rng.uniform(-0.5, 0.5, (n, 3))
    logit = np.full(n, 6.0) + rng.normal(0, 0.5, n)   # opacity ~ 0.99+
    geom = GaussianGeometry(mu, rng.normal(size=(n, 4)), np.log(rng.uniform(0.05, 0.2, (n, 3))),
                            logit, rng.normal(size=(n, 3)))
    out, st = _check(geom, rng.uniform(0, 1, (n, 3)), bench_camera(64, 48, 1.0),
                     dtypes=(np.float32, np.float64))
    assert (st["frame"].t_final.cpu().numpy() < 1e-4).mean() > 0.1  # covered pixels stop


def test_many_channels_kmax32_forward_backward():
    """K = 3 + 1 + 1 + 3 + 20 attribute channels: the KMAX = 32 forward and
    backward kernels vs the oracle."""
    import oracle as O
    from paper_2504_17954_b200 import GaussianGeometry, rasterize_backward, rasterize_forward
    from paper_2504_17954_b200.synthetic import bench_camera, editable_arrays
    n = 3000
    a = editable_arrays(33, n, density=n)
    geom = GaussianGeometry(a["mu"], a["q_raw"], a["log_s"], a["o_logit"], a["n_raw"])
    rng = np.random.default_rng(2)
    colors = rng.uniform(0, 1, (n, 3))
    attrs = {"f0": rng.normal(size=(n, 3)), "f1": rng.normal(size=n), "f2": rng.normal(size=(n, 2)),
             "f3": rng.normal(size=(n, 3)), "f4": rng.normal(size=(n, 3)), "f5": rng.normal(size=(n, 3)),
             "f6": rng.normal(size=(n, 3)), "f7": rng.normal(size=(n, 2))}
    channels = ("color", "alpha", "depth", "normal")
    cam = bench_camera(48, 40, 0.9)
    _check(geom, colors, cam, attrs=attrs, channels=channels)
    out, st = rasterize_forward(geom, colors, cam, channels=channels, attrs=attrs)
    H, W = 40, 48
    d_maps = {"color": rng.normal(size=(H, W, 3)), "alpha": rng.normal(size=(H, W)),
              "f0": rng.normal(size=(H, W, 3)), "f7": rng.normal(size=(H, W, 2))}
    g = rasterize_backward(st, d_maps)
    ref = O.rasterize(geom.mu, geom.q_raw, geom.log_s, geom.o_logit, geom.n_raw, colors, cam,
                      channels=channels, attrs=attrs)
    rg = O.rasterize_backward(ref, d_maps)
    for k in ("d_mu", "d_colors", "d_o_logit"):
        err = np.linalg.norm(g[k] - rg[k])
        assert err <= 1e-3 * max(np.linalg.norm(rg[k]), 1e-12), (k, err)
    for k in ("f0", "f7"):
        err = np.linalg.norm(g["d_attrs"][k] - rg["d_attrs"][k])
        assert err <= 1e-3 * max(np.linalg.norm(rg["d_attrs"][k]), 1e-12), k
