"""Stage-1 SH colour kernels and the stage-1 training step on the GPU vs the
reference (golden fixtures from voxsplat.gaussians.eval_sh / trainer._stage1_step)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

GEOM = ("mu", "q_raw", "log_s", "o_logit", "n_raw")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _cam(d):
    from paper_2504_17954_b200 import Camera
    return Camera(d["cam_position"], d["cam_rotation"], float(d["cam_fov_y"]),
                  int(d["cam_width"]), int(d["cam_height"]))


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_sh_kernels_match_reference(deg):
    """Forward and backward at 1e-12 relative (float64; einsum summation
    order is the only difference)."""
    import torch
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.sh import sh_backward_device, sh_eval_device
    d = golden("sh")
    mu, c = to_dev(d["mu"]), to_dev(d[f"coeffs{deg}"])
    rgb = sh_eval_device(mu, c, deg, d["pos"]).cpu().numpy()
    np.testing.assert_allclose(rgb, d[f"rgb{deg}"], rtol=1e-12, atol=1e-14)
    assert np.array_equal(rgb == 0.0, d[f"rgb{deg}"] == 0.0)  # same clamped channels
    d_mu = torch.zeros_like(mu)
    d_c = sh_backward_device(mu, c, deg, d["pos"], to_dev(d[f"drgb{deg}"]), d_mu).cpu().numpy()
    np.testing.assert_allclose(d_c, d[f"dcoeffs{deg}"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(d_mu.cpu().numpy(), d[f"dmu{deg}"], rtol=1e-9, atol=1e-12)


def test_sh_vs_oracle_random():
    import oracle as O
    from paper_2504_17954_b200 import Camera, GaussianGeometry, ShColor, orbit_camera
    from paper_2504_17954_b200.sh import sh_colors, sh_colors_backward
    rng = np.random.default_rng(5)
    n = 5000
    mu = rng.normal(size=(n, 3))
    geom = GaussianGeometry(mu, rng.normal(size=(n, 4)), rng.normal(size=(n, 3)) - 3,
                            rng.normal(size=n), rng.normal(size=(n, 3)))
    cam = orbit_camera(np.zeros(3), 4.0, 0.2, 1.1, 0.8, 64, 64)
    assert isinstance(cam, Camera)
    sh = ShColor(rng.normal(0, 0.4, (n, 16, 3)), 3)
    rgb = sh_colors(geom, sh, cam)
    ref, cache = O.sh_colors(mu, sh.coefficients, 3, cam.position)
    np.testing.assert_allclose(rgb, ref, rtol=1e-12, atol=1e-14)
    d_rgb = rng.normal(size=(n, 3))
    d_c, d_mu = sh_colors_backward(geom, sh, cam, d_rgb)
    rc, rmu = O.sh_colors_backward(cache, d_rgb)
    np.testing.assert_allclose(d_c, rc, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(d_mu, rmu, rtol=1e-9, atol=1e-12)


def test_sh_bad_degree():
    import torch
    from paper_2504_17954_b200._lib import NativeLibraryMissing  # noqa: F401
    from paper_2504_17954_b200.errors import VoxSplatError
    from paper_2504_17954_b200.sh import sh_eval_device
    mu = torch.zeros((4, 3), dtype=torch.float64, device="cuda")
    with pytest.raises(Exception) as e:
        sh_eval_device(mu, torch.zeros((4, 25, 3), dtype=torch.float64, device="cuda"), 4,
                       np.ones(3))
    assert isinstance(e.value, (VoxSplatError, RuntimeError, ValueError))


def test_stage1_step_matches_reference():
    from paper_2504_17954_b200.device import to_dev
    from paper_2504_17954_b200.trainer import BaseTrainer
    d = golden("stage1")
    params = {k: d[k] for k in GEOM}
    params["sh"] = d["sh"]
    tr = BaseTrainer(params, 2)
    loss, grads, stat = tr.step(_cam(d), to_dev(d["gt"]))
    assert abs(float(loss) - float(d["loss"])) <= 1e-5 * float(d["loss"])
    for k in GEOM + ("sh",):
        got = grads[k].cpu().numpy().reshape(d["g_" + k].shape)
        ref = d["g_" + k]
        err = np.linalg.norm(got - ref)
        assert err <= 1e-3 * max(np.linalg.norm(ref), 1e-12), (k, err, np.linalg.norm(ref))
    s = stat.cpu().numpy()
    assert np.linalg.norm(s - d["stat"]) <= 1e-3 * np.linalg.norm(d["stat"])


def test_render_model_base_stage_matches_rasterize():
    """render_model on a base-stage model = rasterize_forward of the SH colours."""
    import oracle as O
    from paper_2504_17954_b200 import BasicSceneModel, ShColor, orbit_camera, render_model
    from paper_2504_17954_b200.synthetic import editable_model
    m = editable_model(7, 1500, spread=0.5, density=1500)
    rng = np.random.default_rng(3)
    sh = ShColor(rng.normal(0, 0.3, (1500, 4, 3)), 1)
    base = BasicSceneModel("base", m.geometry, sh=sh)
    cam = orbit_camera(np.zeros(3), 2.5, 0.3, 0.4, 0.9, 48, 40)
    img = render_model(base, cam, dtype=np.float64)
    rgb, _ = O.sh_colors(m.geometry.mu, sh.coefficients, 1, cam.position)
    g = m.geometry
    st = O.rasterize(g.mu, g.q_raw, g.log_s, g.o_logit, g.n_raw, rgb, cam,
                     dtype=np.float64)
    ref = O.maps(st)
    np.testing.assert_allclose(img[..., :3], ref["color"], atol=1e-4)
    np.testing.assert_allclose(img[..., 3], ref["alpha"], atol=1e-4)


def test_train_base_short_run_improves():
    """train_base on renders of a known base model: holdout PSNR improves and
    the densify schedule runs (stage-1 loop, trainer.py:532-560)."""
    from paper_2504_17954_b200 import (BasicSceneModel, LightConfig, ShColor, TrainConfig,
                                       ViewDataset, orbit_camera, render_model, train_base)
    from paper_2504_17954_b200.synthetic import editable_model
    m = editable_model(11, 1500, spread=0.5, density=1500)
    rng = np.random.default_rng(4)
    gt_model = BasicSceneModel("base", m.geometry, sh=ShColor(rng.normal(0, 0.3, (1500, 4, 3)), 1))
    cams = [orbit_camera(np.zeros(3), 2.5, 0.3, az, 0.9, 48, 48) for az in (0.2, 1.4, 2.6, 3.8)]
    ds = ViewDataset(cams, [render_model(gt_model, c, dtype=np.float64) for c in cams],
                     LightConfig(), {})
    cfg = TrainConfig(stage1_iters=150, log_interval=25, densify_interval=50,
                      densify_start_iter=50, init_count=800, sh_degree=1)
    model, log = train_base(ds, cfg)
    assert len(log) == 6 and all(np.isfinite(r["loss"]) for r in log)
    assert log[-1]["psnr"] > log[0]["psnr"]
    assert model.stage == "base" and model.sh.degree == 1 and len(model) == log[-1]["count"]
