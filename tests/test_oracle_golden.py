"""Pin the CPU oracle (oracle/) against golden vectors from the real reference.

The fixtures were produced by tests/golden/make_golden.py calling voxsplat's
own public functions; these tests need neither a GPU nor /root/reference.
"""

import numpy as np
import pytest

import oracle as O
from conftest import golden


class Cam:
    def __init__(self, d):
        self.position = d["cam_position"]
        self.rotation = d["cam_rotation"]
        self.fov_y = float(d["cam_fov_y"])
        self.width = int(d["cam_width"])
        self.height = int(d["cam_height"])


GEOM = ("mu", "q_raw", "log_s", "o_logit", "n_raw")
SHADE = ("delta_c", "k_a_raw", "k_d_raw", "k_s_raw", "log_beta")


def _light(d):
    return (str(d["light_mode"]), float(d["light_polar"]), float(d["light_azimuth"]), d["light_ts"])


@pytest.mark.parametrize("case", ["render_c1", "render_fixture", "render_ragged"])
def test_render_pipeline_bit_exact(case):
    d = golden(case)
    cam = Cam(d)
    assert O.ocam(cam).focal == float(d["cam_focal"])
    rgb, _ = O.shade(*(d[k] for k in ("mu", "n_raw")), *(d[k] for k in SHADE), d["palette"],
                     _light(d), cam)
    assert np.array_equal(rgb, d["rgb"])
    st = O.rasterize(*(d[k] for k in GEOM), rgb, cam, dtype=np.float32)
    p = st["proj"]
    for k in ("depth", "mean2d", "conic", "cov2d", "valid"):
        assert np.array_equal(p[k], d[k]), k
    assert np.array_equal(st["pair_splat"], d["pair_splat"])
    assert np.array_equal(st["tile_ranges"], d["tile_ranges"])
    for k in ("kmean2d", "kconic", "kopacity", "values"):
        assert np.array_equal(st[k], d[k]), k
    m = O.maps(st)
    assert np.array_equal(m["color"], d["color"])
    assert np.array_equal(m["alpha"], d["alpha"])
    assert np.array_equal(st["contrib"], d["contrib"])
    assert np.array_equal(st["last_pos"], d["last_pos"])
    assert np.array_equal(st["t_final"], d["t_final"])


def _composed(d):
    parts = [{k: d[f"m{i}_{k}"] for k in GEOM + SHADE + ("palette",)} for i in range(3)]
    cat = {k: np.concatenate([p[k] for p in parts]) for k in GEOM + SHADE}
    sizes = [p["mu"].shape[0] for p in parts]
    ids = np.repeat(np.arange(3), sizes)
    pal = np.stack([parts[0]["palette"], np.array([0.2, 0.6, 0.9]), parts[2]["palette"]])
    scale = np.array([1.0, 1.0, 0.5])[ids]
    return cat, pal[ids], scale


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_composed_edit_render(dtype):
    d = golden("composed_edit")
    cat, pal, scale = _composed(d)
    cam = Cam(d)
    o_eff = O.effective_o_logit(cat["o_logit"], scale)
    assert np.array_equal(o_eff, d["eff_o_logit"])
    light = ("orbital", 0.45, 0.9, np.array([1.2, 0.8, 1.0, 1.0]))
    rgb, _ = O.shade(cat["mu"], cat["n_raw"], *(cat[k] for k in SHADE), pal, light, cam)
    assert np.array_equal(rgb, d["rgb"])
    st = O.rasterize(cat["mu"], cat["q_raw"], cat["log_s"], o_eff, cat["n_raw"], rgb, cam, dtype=dtype)
    m = O.maps(st)
    tag = "32" if dtype == np.float32 else "64"
    assert np.array_equal(m["color"], d["color" + tag])
    assert np.array_equal(m["alpha"], d["alpha" + tag])
    assert np.array_equal(st["contrib"], d["contrib" + tag])


def test_rasterize_backward_matches_reference():
    d = golden("backward_small")
    cam = Cam(d)
    attrs = {"ka": d["attr_ka"]}
    st = O.rasterize(*(d[k] for k in GEOM), d["colors"], cam,
                     channels=("color", "alpha", "depth", "normal"), attrs=attrs, dtype=np.float64)
    m = O.maps(st)
    assert np.array_equal(m["color"], d["color"]) and np.array_equal(m["depth"], d["depth_map"])
    w = {k: d["w_" + k] for k in ("color", "alpha", "depth", "normal", "ka")}
    g = O.rasterize_backward(st, w)
    for k in ("d_mu", "d_q_raw", "d_log_s", "d_o_logit", "d_n_raw", "d_colors", "d_mean2d"):
        np.testing.assert_array_equal(g[k], d[k], err_msg=k)
    np.testing.assert_array_equal(g["d_attrs"]["ka"], d["d_attr_ka"])


@pytest.mark.parametrize("tag", ["head", "orb"])
def test_shade_forward_backward(tag):
    d = golden("shade")
    cam = Cam(d)
    if tag == "head":
        light, ct, pal = ("headlight", 0.0, 0.0, np.ones(4)), None, d["palette"]
    else:
        light = ("orbital", 0.45, 0.9, np.array([1.2, 0.8, 1.0, 1.1]))
        ct = (np.array([1.2, 0.8, 1.1, 0.9]), np.array([0.01, -0.02, 0.03, 0.2]))
        pal = d["palette_ps"]
    rgb, cache = O.shade(d["mu"], d["n_raw"], *(d[k] for k in SHADE), pal, light, cam,
                         coeff_transform=ct)
    assert np.array_equal(rgb, d[tag + "_rgb"])
    g = O.shade_backward(cache, d["d_rgb"])
    for k, v in g.items():
        np.testing.assert_array_equal(np.asarray(v), d[f"{tag}_{k}"], err_msg=k)


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_sh_colour_forward_backward(deg):
    d = golden("sh")
    rgb, cache = O.sh_colors(d["mu"], d[f"coeffs{deg}"], deg, d["pos"])
    assert np.array_equal(rgb, d[f"rgb{deg}"])
    d_c, d_mu = O.sh_colors_backward(cache, d[f"drgb{deg}"])
    assert np.array_equal(d_c, d[f"dcoeffs{deg}"])
    assert np.array_equal(d_mu, d[f"dmu{deg}"])


def test_vq_assign_and_kmeans():
    d = golden("vq")
    idx = O.vq_assign(d["values"], d["centroids"])
    assert np.array_equal(idx, d["indices"])
    assert np.array_equal(O.kmeans(d["samples"], 16, seed=1), d["kmeans16"])
    assert np.array_equal(O.vq_decode(idx, d["centroids"])[100:200], d["centroids"][d["indices"][100:200]])


def test_photometric_loss():
    d = golden("loss")
    loss, g = O.photometric_loss(d["pred"], d["gt"])
    assert loss == float(d["loss"])
    assert np.array_equal(g, d["d"])


def test_inverse_step_and_fit():
    d = golden("inverse")
    parts = [{k: d[f"m{i}_{k}"] for k in GEOM + SHADE + ("palette",)} for i in range(2)]
    geom = tuple(np.concatenate([p[k] for p in parts]) for k in GEOM)
    shading = tuple(np.concatenate([p[k] for p in parts]) for k in SHADE)
    ids = np.repeat(np.arange(2), [p["mu"].shape[0] for p in parts])
    c_p = np.stack([p["palette"] for p in parts])
    cam = Cam(d)
    light = ("headlight", 0.0, 0.0, np.ones(4))
    o_raw = O.inv_softplus(np.ones(2))
    loss, g, _ = O.inverse_step(geom, shading, ids, light, c_p, o_raw, np.ones(4), np.zeros(4),
                                0.0, 0.0, cam, d["reference"])
    assert loss == float(d["loss0"])
    for k, v in g.items():
        np.testing.assert_array_equal(v, d["g_" + k], err_msg=k)


def test_blinn_phong_worked_example():
    """The reference's scalar worked example (n.l = 0.5, n.h = 0.9)."""
    from paper_2504_17954_b200.dvr import shade_sample
    from paper_2504_17954_b200.shading import blinn_phong
    n = np.array([0.0, 0.0, 1.0])
    l = np.array([np.sqrt(3) / 2, 0.0, 0.5])
    h = np.array([np.sqrt(0.19), 0.0, 0.9])
    v = 2.0 * np.dot(h, l) * h - l
    c_v = np.array([0.6, 0.0, 0.0])
    rgb, amb, dif, spec = blinn_phong(c_v, n, l, v, np.array(0.2), np.array(0.5), np.array(0.3),
                                      np.array(8.0))
    expected = 0.2 * c_v + 0.5 * c_v * 0.5 + 0.3 * np.ones(3) * 0.9 ** 8
    np.testing.assert_allclose(rgb, expected, atol=1e-12)
    np.testing.assert_allclose(amb, [0.12, 0.0, 0.0])
    np.testing.assert_allclose(shade_sample(c_v, n, l, v, 0.2, 0.5, 0.3, 8.0), expected, atol=1e-12)


def test_mathutil_helpers():
    from paper_2504_17954_b200 import _mathutil as M
    x = np.array([-800.0, -3.0, 0.0, 2.5, 800.0])
    s = M.sigmoid(x)
    assert np.all(np.isfinite(s)) and s[2] == 0.5
    np.testing.assert_allclose(M.inv_sigmoid(M.sigmoid(x[1:4])), x[1:4], atol=1e-12)
    np.testing.assert_allclose(M.inv_softplus(M.softplus(x[1:4])), x[1:4], atol=1e-12)
    v = np.array([[3.0, 4.0, 0.0]])
    np.testing.assert_allclose(M.normalize_rows(v), [[0.6, 0.8, 0.0]])
    d = M.normalize_rows_backward(v, np.array([[1.0, 0.0, 0.0]]))
    np.testing.assert_allclose(d @ M.normalize_rows(v).T, [[0.0]], atol=1e-15)


def test_stage2_step():
    """oracle.stage2_step (the C3 parity checker) vs the reference's
    trainer._stage2_step (trainer.py:397-444) with all regularizers."""
    d = golden("stage2")
    light = ("orbital", 0.3, -0.7, np.array([1.0, 1.1, 0.9, 1.0]))
    loss, g, stat = O.stage2_step({k: d[k] for k in GEOM + SHADE}, d["palette"], light, Cam(d),
                                  d["gt"])
    assert loss == float(d["loss"])
    for k, v in g.items():
        np.testing.assert_array_equal(v, d["g_" + k], err_msg=k)
    np.testing.assert_array_equal(stat, d["stat"])
